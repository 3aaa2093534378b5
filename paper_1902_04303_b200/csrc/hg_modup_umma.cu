// hg_modup_umma.cu -- ModUp (radix-2^32 words -> residues) on tcgen05 (UTCIMMA, TMEM).
//
// r_j(a) = sum_{w,q} a_{w,q} * 2^(32w+8q) mod p_j (a_{w,q} = byte q of word w).  Splitting the
// constants into bytes, D[n][(j,r)] = sum_{(w,q)} a_{w,q} * byte_r(2^(32w+8q) mod p_j) is one
// u8 x u8 -> s32 GEMM with rows = coefficients (M = 128), K = (word, byte) -- the A tile is
// the input words verbatim -- and columns = (prime, byte r): 4 TMEM columns per prime.  Each
// epilogue thread owns a TMEM lane = one coefficient, folds its 4 column digits into a < 2^49
// integer, reduces it mod p_j, applies the two's-complement / automorphism-negation
// corrections and stores a coalesced residue row.
//
// Persistent and warp-specialised (one CTA per SM walks 128-coefficient tiles of every
// operand); roles are linked by mbarrier rings:
//   warp 0      B producer: per 64-prime chunk the first 4*W8 K bytes of the constant image
//   warp 1      MMA issuer: W8/8 k-steps of 128x256x32 per chunk into one of 2 TMEM stages
//   warps 2-5   A loaders: gather the words of 128 coefficients (automorphism permutation),
//               write the K-major core layout, record sign / negation flags
//   warps 6-21  epilogue: four warps per TMEM lane quarter split a chunk's 64 primes
// TMEM is double-buffered per prime chunk, so the epilogue of chunk c overlaps the MMAs of c+1
// and the A / B rings keep the loads of the next tile in flight.
#include <type_traits>

#include "hg_internal.cuh"

namespace {

constexpr int kRows = 128;        // coefficients per tile (UMMA M)
constexpr int kPrimesChunk = 64;  // primes per accumulation (N = 256)
constexpr int kWMax = 64;         // widest operand handled here (words)
constexpr int kBChunkBytes = 256 * 4 * kWMax;   // 64 KB: 256 rows x 256 K bytes
constexpr int kAStage = kRows * 4 * kWMax;      // 32 KB
constexpr int kEpiGroups = 4;    // epilogue warps per TMEM lane quarter
#ifndef HG_MODUP_LOADERS
#define HG_MODUP_LOADERS 8   // A-loader warps: 4 (one coefficient per thread) or 8 (two threads per coefficient, each gathering every other 32-word batch: both batches of a level-1550 operand in flight at once; 72 registers, no spills; ModUp 23.96 -> 22.0 ms per batch step, profiles/r2_modup_loader_ab.txt)
#endif
constexpr int kLoaders = HG_MODUP_LOADERS;
constexpr int kEpiWarp0 = 2 + kLoaders;
constexpr int kWarps = kEpiWarp0 + 4 * kEpiGroups;
constexpr int kEpiPrimes = kPrimesChunk / kEpiGroups;   // primes per epilogue warp and chunk
constexpr size_t kSmem = 2 * (size_t)kBChunkBytes + 2 * (size_t)kAStage;   // 192 KB

struct MOps {
    const uint32_t* words[4];
    int bits[4];
    int is_signed[4];
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            "selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(bar), "r"(parity));
    }
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
// HG_MODUP_PROF (diagnostic builds only): per-CTA, per-warp cycles spent in each barrier wait
// (and in the loaders' gather / the epilogue's column loop), read back with hg_modup_prof_read:
// [cta][warp][0..3 waits / work by role, 5 = elapsed]
#ifdef HG_MODUP_PROF
__device__ unsigned long long g_modup_prof[160][32][8];
#define MWAIT(cat, bar, par)                                  \
    do {                                                      \
        const long long _t = clock64();                       \
        mbar_wait(bar, par);                                  \
        prof[cat] += (unsigned long long)(clock64() - _t);    \
    } while (0)
#else
#define MWAIT(cat, bar, par) mbar_wait(bar, par)
#endif
__device__ __forceinline__ void umma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(bar) : "memory");
}
#ifdef HG_MODUP_FOLD30
// a * b + c, 32 x 32 -> 64-bit multiply-add (one IMAD.WIDE)
__device__ __forceinline__ uint64_t madw(uint32_t a, uint32_t b, uint64_t c) {
    uint64_t d;
    asm("mad.wide.u32 %0, %1, %2, %3;\n" : "=l"(d) : "r"(a), "r"(b), "l"(c));
    return d;
}
#endif
template <typename T>
__device__ __forceinline__ T pick(const T (&a)[4], int k) {
    return k == 0 ? a[0] : k == 1 ? a[1] : k == 2 ? a[2] : a[3];
}

// SIGNED: some operand is two's complement (else the sign correction is compiled out);
// AUTOMORPH: the gather runs through x -> x^k (else the negation correction is compiled out)
// LOGN: log2 N as a compile-time constant (row strides of the loaders' word gathers and of the
// epilogue's residue stores become address immediates), 0 = N at run time
template <bool SIGNED, bool AUTOMORPH, int LOGN>
__global__ void __launch_bounds__(kWarps * 32, 1) modup_umma_kernel(
    MOps ops, int nops, int N_rt, const PrimeInfo* __restrict__ pinfo,
    const uint32_t* __restrict__ modup_tab, const uint8_t* __restrict__ Bimg, int P,
    uint32_t* __restrict__ out, int64_t automorph_kinv) {
    const int N = LOGN ? (1 << LOGN) : N_rt;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* s_b = smem;                           // 2 x 64 KB
    uint8_t* s_a = smem + 2 * kBChunkBytes;        // 2 x 32 KB
    __shared__ uint32_t tmem_base;
    __shared__ __align__(8) uint64_t bar_b_full[2], bar_b_empty[2], bar_a_full[2], bar_a_empty[2];
    __shared__ __align__(8) uint64_t bar_tm_full[2], bar_tm_empty[2], bar_fl_full[2], bar_fl_empty[2];
    __shared__ uint32_t s_fl[2][kRows];            // bit0 sign, bit1 negate, bit2 any-nonzero
    __shared__ uint32_t s_flp[kLoaders == 8 ? 2 : 1][2][kLoaders == 8 ? kRows : 1];   // per loader part
    // per prime: p, 2^30 mod p (+ Shoup); per operand and prime: the sign correction
    // p - 2^bits mod p and the negation base (p for signed, p + 2^bits mod p for unsigned)
    // padded by a prime chunk so the epilogue indexes base + constant without clamping
    __shared__ uint4 s_pc[HG_MAX_PRIMES + kPrimesChunk];
    __shared__ uint2 s_corr[4][HG_MAX_PRIMES + kPrimesChunk];

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
#ifdef HG_MODUP_PROF
    unsigned long long prof[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const long long t_start = clock64();
#endif
    for (int j = tid; j < P + kPrimesChunk; j += blockDim.x) {
        if (j >= P) {
            s_pc[j] = make_uint4(1u, 2u, 0u, 0xffffffffu);
            for (int k = 0; k < 4; ++k) s_corr[k][j] = make_uint2(0u, 0u);
            continue;
        }
        const PrimeInfo pi = pinfo[j];
#ifdef HG_MODUP_FOLD30
        s_pc[j] = make_uint4(pi.p, pi.c30, pi.c30_sh, 0u);
#else
        // (p, 2p, floor(2^48 / p) = the Shoup companion of 2^16 mod p = 2^16, -p)
        s_pc[j] = make_uint4(pi.p, 2u * pi.p, (uint32_t)((1ull << 48) / pi.p), 0u - pi.p);
#endif
        for (int k = 0; k < nops; ++k) {
            const int bits = pick(ops.bits, k);
            const uint32_t pw = reduce_u64((uint64_t)modup_tab[(size_t)j * HG_MODUP_WMAX + (bits >> 5)] << (bits & 31), pi);
            // sign correction (- 2^bits mod p) and the negation base for a value in [0, 3p):
            // 3p (signed: -x) or 3p + (2^bits mod p) (unsigned: 2^bits - x)
            s_corr[k][j] = make_uint2(pw ? pi.p - pw : 0u, pick(ops.is_signed, k) ? 3u * pi.p : 3u * pi.p + pw);
        }
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base)), "n"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (tid == 0) {
        auto init = [](uint64_t* b, int cnt) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(cnt));
        };
        for (int s = 0; s < 2; ++s) {
            init(&bar_b_full[s], 1);
            init(&bar_b_empty[s], 1);
            init(&bar_a_full[s], kLoaders);
            init(&bar_a_empty[s], 1);
            init(&bar_tm_full[s], 1);
            init(&bar_tm_empty[s], 4 * kEpiGroups);
            init(&bar_fl_full[s], kLoaders);
            init(&bar_fl_empty[s], 4 * kEpiGroups);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t tmem = tmem_base;
    const int tpo = N / kRows;
    const int ntiles = nops * tpo;
    const int nch = (P + kPrimesChunk - 1) / kPrimesChunk;

    if (warp == 0) {
        // ---------------- B producer ----------------
        if (lane == 0) {
            int ib = 0;
            for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
                const int op = tile / tpo;
                const int W8 = (((pick(ops.bits, op) + 31) >> 5) + 7) & ~7;
                const uint32_t bytes = (uint32_t)(W8 / 4) * 4096u;   // K chunks 0 .. W8/4-1
                for (int ch = 0; ch < nch; ++ch, ++ib) {
                    const int s = ib & 1;
                    MWAIT(0, smem_u32(&bar_b_empty[s]), ((ib >> 1) & 1) ^ 1);
                    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(&bar_b_full[s])), "r"(bytes) : "memory");
                    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                                 ::"r"(smem_u32(s_b + s * kBChunkBytes)), "l"(Bimg + (size_t)ch * kBChunkBytes),
                                 "r"(bytes), "r"(smem_u32(&bar_b_full[s]))
                                 : "memory");
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer ----------------
        if (lane == 0) {
            const uint32_t idesc = (2u << 4) | ((uint32_t)(256 >> 3) << 17) | ((uint32_t)(kRows >> 4) << 24);
            const uint32_t a_base = smem_u32(s_a), b_base = smem_u32(s_b);
            int ia = 0, ib = 0, ic = 0;
            for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++ia) {
                const int op = tile / tpo;
                const int W8 = (((pick(ops.bits, op) + 31) >> 5) + 7) & ~7;
                const int sa_ = ia & 1;
                MWAIT(0, smem_u32(&bar_a_full[sa_]), (ia >> 1) & 1);
                for (int ch = 0; ch < nch; ++ch, ++ib, ++ic) {
                    const int sb_ = ib & 1, ts = ic & 1;
                    MWAIT(1, smem_u32(&bar_b_full[sb_]), (ib >> 1) & 1);
                    MWAIT(2, smem_u32(&bar_tm_empty[ts]), ((ic >> 1) & 1) ^ 1);
                    asm volatile("tcgen05.fence::after_thread_sync;\n");
                    for (int k = 0; k < W8 / 8; ++k) {
                        // A: core (row group g, K chunk c) at (16g + c) * 128; B: at (32c + g) * 128
                        const uint64_t da = umma_desc(a_base + (uint32_t)(sa_ * kAStage + 2 * k * 128), 128, 16 * 128);
                        const uint64_t db = umma_desc(b_base + (uint32_t)(sb_ * kBChunkBytes + 2 * k * 4096), 4096, 128);
                        const uint32_t acc = k > 0 ? 1u : 0u;
                        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                                     "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                                     ::"r"(tmem + (uint32_t)(ts * 256)), "l"(da), "l"(db), "r"(idesc), "r"(acc));
                    }
                    umma_commit(smem_u32(&bar_b_empty[sb_]));
                    umma_commit(smem_u32(&bar_tm_full[ts]));
                }
                umma_commit(smem_u32(&bar_a_empty[sa_]));
            }
        }
    } else if (warp < kEpiWarp0) {
        // ---------------- A loaders ----------------
        // kLoaders = 8: warps (c, c + 4) share coefficients 32c .. 32c+31, each loading half of
        // the 32-word batches (more loads in flight per coefficient); flags merge in s_fl2
        const int lw = warp - 2;
        const int n = (lw & 3) * 32 + lane;
        const int part = kLoaders == 8 ? lw >> 2 : 0;
        const int g = n >> 3, rr = n & 7;
        int ia = 0;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++ia) {
            const int op = tile / tpo, cb = (tile - op * tpo) * kRows;
            const uint32_t* in = pick(ops.words, op);
            const int bits = pick(ops.bits, op);
            const int is_signed = pick(ops.is_signed, op);
            const int W = (bits + 31) >> 5;
            const int W8 = (W + 7) & ~7;
            const uint32_t top_mask = (bits & 31) ? ((1u << (bits & 31)) - 1u) : 0xffffffffu;
            const int i = cb + n;
            int src = i;
            bool neg = false;
            if (automorph_kinv != 0) {
                int64_t j = ((int64_t)i * automorph_kinv) & ((2ll * N) - 1);
                if (j >= N) { neg = true; j -= N; }
                src = (int)j;
            }
            const int sa_ = ia & 1;
            MWAIT(0, smem_u32(&bar_a_empty[sa_]), ((ia >> 1) & 1) ^ 1);
            MWAIT(1, smem_u32(&bar_fl_empty[sa_]), ((ia >> 1) & 1) ^ 1);
#ifdef HG_MODUP_PROF
            const long long t_ld = clock64();
#endif
            // WAR across proxies: the tensor core's reads of this stage precede our stores
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            uint8_t* dst = s_a + sa_ * kAStage + (g * 16) * 128 + rr * 16;
            uint32_t any = 0, sign = 0;
            // batches of 32 words: part p of kLoaders/4 parts takes batches p, p + parts, ...
            constexpr int kParts = kLoaders / 4;
            for (int w0 = 32 * part; w0 < W8; w0 += 32 * kParts) {
                uint32_t wv[32];
                if (w0 + 32 < W) {
                    // interior batch (all 32 words below the top word): no predicates, no masks
                    const uint32_t* pw = in + (size_t)w0 * N + src;
#pragma unroll
                    for (int e = 0; e < 32; ++e) wv[e] = __ldg(pw + (size_t)e * N);
#pragma unroll
                    for (int e = 0; e < 32; ++e) any |= wv[e];
#pragma unroll
                    for (int c = 0; c < 8; ++c)
                        *reinterpret_cast<uint4*>(dst + ((w0 >> 2) + c) * 128) =
                            make_uint4(wv[4 * c], wv[4 * c + 1], wv[4 * c + 2], wv[4 * c + 3]);
                    continue;
                }
#pragma unroll
                for (int e = 0; e < 32; ++e) {
                    const int w = w0 + e;
                    wv[e] = w < W ? __ldg(in + (size_t)w * N + src) : 0u;
                }
#pragma unroll
                for (int e = 0; e < 32; ++e) {
                    const int w = w0 + e;
                    if (w == W - 1) {
                        wv[e] &= top_mask;
                        sign = is_signed ? (wv[e] >> ((bits - 1) & 31)) & 1u : 0u;
                    }
                    any |= wv[e];
                }
#pragma unroll
                for (int c = 0; c < 8; ++c)
                    if (w0 + 4 * c < W8)
                        *reinterpret_cast<uint4*>(dst + ((w0 >> 2) + c) * 128) =
                            make_uint4(wv[4 * c], wv[4 * c + 1], wv[4 * c + 2], wv[4 * c + 3]);
            }
            const uint32_t fl = (sign ? 1u : 0u) | (neg ? 2u : 0u) | (any ? 4u : 0u);
            if (kParts == 1) s_fl[sa_][n] = fl;
            else s_flp[part][sa_][n] = fl;
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(smem_u32(&bar_a_full[sa_]));
                mbar_arrive(smem_u32(&bar_fl_full[sa_]));
            }
#ifdef HG_MODUP_PROF
            prof[2] += (unsigned long long)(clock64() - t_ld);
#endif
        }
    } else {
        // ---------------- epilogue ----------------
        const int q = warp & 3, h = (warp - kEpiWarp0) >> 2;   // lane quarter, prime group
        const int n = q * 32 + lane;
        int ia = 0, ic = 0;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++ia) {
            const int op = tile / tpo, cb = (tile - op * tpo) * kRows;
            const uint2* corr = s_corr[op];
            uint32_t* outp = out + (size_t)op * P * N + cb + n;
            const int sa_ = ia & 1;
            MWAIT(0, smem_u32(&bar_fl_full[sa_]), (ia >> 1) & 1);
            const uint32_t fl = kLoaders == 8 ? (s_flp[0][sa_][n] | s_flp[1][sa_][n]) : s_fl[sa_][n];
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&bar_fl_empty[sa_]));
            const uint32_t sgn01 = fl & 1u;
            const bool ng = (fl & 2u) && (fl & 4u);
            for (int ch = 0; ch < nch; ++ch, ++ic) {
                const int ts = ic & 1;
                MWAIT(1, smem_u32(&bar_tm_full[ts]), (ic >> 1) & 1);
#ifdef HG_MODUP_PROF
                const long long t_col = clock64();
#endif
                asm volatile("tcgen05.fence::after_thread_sync;\n");
                const int jbase = ch * kPrimesChunk + h * kEpiPrimes;
                const uint32_t lane_addr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(ts * 256) +
                                           (uint32_t)(h * kEpiPrimes * 4);
                // outputs are left lazily reduced in [0, 4p): every ModUp result feeds the forward
                // NTT, whose butterflies take [0, 4p) inputs (fwd_bfly)
                uint32_t* orow = outp + (size_t)jbase * N;
                const uint4* pcb = s_pc + jbase;
                const uint2* crb = corr + jbase;
#pragma unroll 1
                for (int jj = 0; jj < kEpiPrimes && jbase + jj < P; jj += 8) {
                    uint32_t d[32];
                    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                                 "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
                                 : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]),
                                   "=r"(d[6]), "=r"(d[7]), "=r"(d[8]), "=r"(d[9]), "=r"(d[10]), "=r"(d[11]),
                                   "=r"(d[12]), "=r"(d[13]), "=r"(d[14]), "=r"(d[15]), "=r"(d[16]), "=r"(d[17]),
                                   "=r"(d[18]), "=r"(d[19]), "=r"(d[20]), "=r"(d[21]), "=r"(d[22]), "=r"(d[23]),
                                   "=r"(d[24]), "=r"(d[25]), "=r"(d[26]), "=r"(d[27]), "=r"(d[28]), "=r"(d[29]),
                                   "=r"(d[30]), "=r"(d[31])
                                 : "r"(lane_addr + (uint32_t)(jj * 4)));
                    asm volatile("tcgen05.wait::ld.sync.aligned;\n");
                    const int nv = P - (jbase + jj);   // primes of this group that exist (warp-uniform)
                    uint32_t* og = orow + (size_t)jj * N;
                    // FULL: all 8 primes exist (every group but a basis' last): unpredicated stores
                    auto group = [&](auto full) {
                        constexpr bool FULL = decltype(full)::value;
#pragma unroll
                        for (int e = 0; e < 8; ++e) {
                            // branch-free: the 8 primes are independent chains the scheduler interleaves
                            const uint4 pc = pcb[jj + e];
#ifdef HG_MODUP_FOLD30
                            // digits < 2^24 (K <= 256 bytes): v < 2^49, one 2^30 fold reaches [0, 4p)
                            const uint32_t p = pc.x;
                            const uint32_t t = d[4 * e + 3] * 256u + d[4 * e + 2];   // < 2^31 (byte 3 < 64)
                            const uint64_t v = madw(t, 1u << 16, madw(d[4 * e + 1], 256u, (uint64_t)d[4 * e]));
                            uint32_t r = mul_shoup_lazy((uint32_t)(v >> 30), pc.y, pc.z, p) +
                                         ((uint32_t)v & 0x3fffffffu);
#else
                            // v = D0 + D1 2^8 + D2 2^16 + D3 2^24 (digits <= 256 * 255^2 < 2^24, D3 < 2^22)
                            //   = T' 2^16 + (U mod 2^16),  U = D1 2^8 + D0 < 2^32,  T' = D3 2^8 + D2 + (U >> 16) < 2^31
                            // so one Shoup product by 2^16 (one multiply-high; T' 2^16 + (U mod 2^16) mod 2^32 is a
                            // byte permute) lands in [0, 2p + 2^16) within [0, 3p), all in 32-bit arithmetic:
                            // r = (T' 2^16 | U mod 2^16) - q p, as one multiply-add by -p
                            const uint32_t u = (d[4 * e + 1] << 8) + d[4 * e];
                            const uint32_t tt = (d[4 * e + 3] << 8) + d[4 * e + 2] + (u >> 16);
                            const uint32_t q = __umulhi(tt, pc.z);
                            uint32_t r = q * pc.w + __byte_perm(u, tt, 0x5410);
#endif
                            if (SIGNED || AUTOMORPH) {
                                const uint2 cr = crb[jj + e];
#ifdef HG_MODUP_FOLD30
                                r = min(r, r - 2u * pc.x);          // [0, 2p)
#else
                                r = min(r, r - pc.y);               // [0, 2p)
#endif
                                if (SIGNED) r += sgn01 * cr.x;      // two's-complement sign: -2^bits, [0, 3p)
                                if (AUTOMORPH) r = ng ? cr.y - r : r;   // automorphism sign, (0, 4p)
                            }
                            if (FULL || e < nv) og[(size_t)e * N] = r;
                        }
                    };
                    if (nv >= 8) group(std::true_type{});
                    else group(std::false_type{});
                }
                asm volatile("tcgen05.fence::before_thread_sync;\n");
                __syncwarp();
                if (lane == 0) mbar_arrive(smem_u32(&bar_tm_empty[ts]));
#ifdef HG_MODUP_PROF
                prof[2] += (unsigned long long)(clock64() - t_col);
#endif
            }
        }
    }
#ifdef HG_MODUP_PROF
    if (lane == 0 && blockIdx.x < 160 && warp < 32) {
        prof[5] = (unsigned long long)(clock64() - t_start);
        for (int k = 0; k < 8; ++k) g_modup_prof[blockIdx.x][warp][k] = prof[k];
    }
#endif
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(512));
}

}  // namespace

#ifdef HG_MODUP_PROF
// copies the wait-cycle table of the last tcgen05 ModUp launch: [160][32][8] u64
extern "C" int hg_modup_prof_read(unsigned long long* out) {
    return cudaMemcpyFromSymbol(out, g_modup_prof, sizeof(g_modup_prof)) == cudaSuccess ? 0 : 1;
}
#endif

// B images, K-chunk-major so that a W-word operand copies only its first W8/4 K chunks:
// chunk ch = primes 64ch..64ch+63 -> 256 rows (j, r) x K = 256 bytes (64 words x 4 bytes);
// core (row group g, K chunk c) at (32c + g) * 128, row s at +16s; byte 4e+q of K chunk c
// (word w = 4c+e) = byte r of 2^(32w+8q) mod p_j.
int hg_modup_build_umma(hg_ctx* ctx) {
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (ctx->d_modup_umma) return HG_OK;
    const int P = ctx->nprimes, nch = (P + kPrimesChunk - 1) / kPrimesChunk;
    std::vector<uint8_t> img((size_t)nch * kBChunkBytes, 0);
    for (int j = 0; j < P; ++j) {
        const uint64_t p = ctx->primes[j];
        const int ch = j / kPrimesChunk, jl = j % kPrimesChunk;
        for (int w = 0; w < kWMax; ++w)
            for (int q = 0; q < 4; ++q) {
                uint64_t v = 1, base = 2, e = 32ull * w + 8ull * q;
                while (e) {
                    if (e & 1) v = v * base % p;
                    base = base * base % p;
                    e >>= 1;
                }
                for (int rb = 0; rb < 4; ++rb) {
                    const int row = jl * 4 + rb, g = row >> 3, s = row & 7;
                    const int c = w >> 2, byte = (w & 3) * 4 + q;
                    img[(size_t)ch * kBChunkBytes + ((size_t)(c * 32 + g) * 8 + s) * 16 + byte] =
                        (uint8_t)(v >> (8 * rb));
                }
            }
    }
    if (cudaMalloc(&ctx->d_modup_umma, img.size()) != cudaSuccess) return hg_fail(HG_ENOMEM, "modup umma table");
    cudaMemcpy(ctx->d_modup_umma, img.data(), img.size(), cudaMemcpyHostToDevice);
    return HG_OK;
}

// 1 if handled, 0 to fall back, <0 on error
int hg_modup_umma_launch(hg_ctx* ctx, const uint32_t* const* words, const int* bits,
                         const int* is_signed, int nops, int P, uint32_t* out, int64_t kinv,
                         cudaStream_t st) {
    int maxw = 0;
    for (int k = 0; k < nops; ++k) maxw = std::max(maxw, (bits[k] + 31) >> 5);
    if (ctx->N < kRows || maxw > kWMax || maxw < 1 || nops > 4) return 0;
    int rc = hg_modup_build_umma(ctx);
    if (rc) return -rc;
    static std::atomic<uint64_t> attr_set{0};
    const int nsm = ctx->nsm;
    using Kern = void (*)(MOps, int, int, const PrimeInfo*, const uint32_t*, const uint8_t*, int, uint32_t*, int64_t);
    // [log_n class: run-time N, 2^16, 2^17][signed][automorphism]
    static const Kern kerns[3][2][2] = {
        {{modup_umma_kernel<false, false, 0>, modup_umma_kernel<false, true, 0>},
         {modup_umma_kernel<true, false, 0>, modup_umma_kernel<true, true, 0>}},
        {{modup_umma_kernel<false, false, 16>, modup_umma_kernel<false, true, 16>},
         {modup_umma_kernel<true, false, 16>, modup_umma_kernel<true, true, 16>}},
        {{modup_umma_kernel<false, false, 17>, modup_umma_kernel<false, true, 17>},
         {modup_umma_kernel<true, false, 17>, modup_umma_kernel<true, true, 17>}}};
    if (hg_first_on_device(attr_set, ctx->device)) {
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 2; ++b)
                for (int c = 0; c < 2; ++c)
                    if (cudaFuncSetAttribute(kerns[a][b][c], cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem) != cudaSuccess)
                        return -hg_fail(HG_ECUDA, "modup_umma smem attribute");
    }
    MOps o{};
    for (int k = 0; k < nops; ++k) {
        o.words[k] = words[k];
        o.bits[k] = bits[k];
        o.is_signed[k] = is_signed[k];
    }
    const int ntiles = nops * (ctx->N / kRows);
    const int grid = ntiles < nsm ? ntiles : nsm;
    bool any_signed = false;
    for (int k = 0; k < nops; ++k) any_signed |= is_signed[k] != 0;
    const int lc = ctx->log_n == 17 ? 2 : (ctx->log_n == 16 ? 1 : 0);
    kerns[lc][any_signed ? 1 : 0][kinv ? 1 : 0]<<<grid, kWarps * 32, kSmem, st>>>(
        o, nops, ctx->N, ctx->d_pinfo, ctx->d_modup, ctx->d_modup_umma, P, out, kinv);
    ctx->launches.fetch_add(1, std::memory_order_relaxed);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return -hg_fail(HG_ECUDA, std::string("modup_umma launch: ") + cudaGetErrorString(e));
    return 1;
}
