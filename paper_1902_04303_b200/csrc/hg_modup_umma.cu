// hg_modup_umma.cu -- ModUp (radix-2^32 words -> residues) on tcgen05 (UTCIMMA, TMEM).
//
// r_j(a) = sum_{w,q} a_{w,q} * 2^(32w+8q) mod p_j (a_{w,q} = byte q of word w).  Splitting the
// constants into bytes, D[n][(j,r)] = sum_{(w,q)} a_{w,q} * byte_r(2^(32w+8q) mod p_j) is one
// u8 x u8 -> s32 GEMM with rows = coefficients (M = 128), K = (word, byte) -- the A tile is
// the input words verbatim -- and columns = (prime, byte r): 4 TMEM columns per prime.  Each
// thread owns a TMEM lane = one coefficient, folds its 4 column digits into a < 2^49 integer,
// reduces it mod p_j, applies the two's-complement / automorphism-negation corrections and
// stores a coalesced residue row.  Primes are processed 64 at a time (N = 256) with the B
// images streamed by the bulk-copy engine; warps 0-3 and 4-7 split each chunk's primes.
#include "hg_internal.cuh"

namespace {

constexpr int kRows = 128;        // coefficients per CTA (UMMA M)
constexpr int kPrimesChunk = 64;  // primes per accumulation pass (N = 256)
constexpr int kWMax = 64;         // widest operand handled here (words)
constexpr int kBChunkBytes = 256 * 4 * kWMax;   // 64 KB: 256 rows x 256 K bytes

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

__global__ void __launch_bounds__(256) modup_umma_kernel(
    MOps ops, int N, const PrimeInfo* __restrict__ pinfo, const uint32_t* __restrict__ modup_tab,
    const uint8_t* __restrict__ Bimg, int P, uint32_t* __restrict__ out, int64_t automorph_kinv) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t tmem_base;
    __shared__ __align__(8) uint64_t mbar_b[2], mbar_mma[2];
    __shared__ uint32_t flags[kRows];   // bit0 sign, bit1 negate, bit2 any-nonzero
    __shared__ uint32_t spw[HG_MAX_PRIMES];
    const int op = blockIdx.y;
    const uint32_t* in = op == 0 ? ops.words[0] : op == 1 ? ops.words[1] : op == 2 ? ops.words[2] : ops.words[3];
    const int bits = op == 0 ? ops.bits[0] : op == 1 ? ops.bits[1] : op == 2 ? ops.bits[2] : ops.bits[3];
    const int is_signed = op == 0 ? ops.is_signed[0] : op == 1 ? ops.is_signed[1]
                        : op == 2 ? ops.is_signed[2] : ops.is_signed[3];
    const int W = (bits + 31) >> 5;
    const int W8 = (W + 7) & ~7;            // K = 4 * W8 bytes, W8/8 k-steps of 32 bytes
    const int tid = threadIdx.x, warp = tid >> 5;
    const int cb = blockIdx.x * kRows;
    uint8_t* sa = smem;                              // A: 128 rows x 4*kWMax bytes (core layout)
    uint8_t* sb = smem + (size_t)kRows * 4 * kWMax;  // B: 2 stages x 64 KB
    const int kc16 = kWMax / 4;                      // 16-byte K chunks per A/B row (16)

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base)), "n"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (tid == 0) {
        for (int s = 0; s < 2; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&mbar_b[s])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&mbar_mma[s])));
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n");
    }
    // ---- A tile: thread pair (n, half) loads words of coefficient n (automorphism gather) ------
    {
        const int n = tid & (kRows - 1), half = tid >> 7;
        const int i = cb + n;
        int src = i;
        bool neg = false;
        if (automorph_kinv != 0) {
            int64_t j = ((int64_t)i * automorph_kinv) & ((2ll * N) - 1);
            if (j >= N) { neg = true; j -= N; }
            src = (int)j;
        }
        const uint32_t top_mask = (bits & 31) ? ((1u << (bits & 31)) - 1u) : 0xffffffffu;
        const int g = n >> 3, rr = n & 7;
        uint32_t any = 0, sign = 0;
        // all of this half's loads are issued before any is consumed (32 in flight per thread)
        uint32_t wv[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) {
            const int w = 4 * (half + 2 * (e >> 2)) + (e & 3);
            wv[e] = w < W ? __ldg(in + (size_t)w * N + src) : 0u;
        }
#pragma unroll
        for (int cc = 0; cc < 8; ++cc) {
            const int c = half + 2 * cc;              // 16-byte chunk = words 4c .. 4c+3
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int w = 4 * c + e;
                if (w == W - 1) {
                    wv[4 * cc + e] &= top_mask;
                    sign = is_signed ? (wv[4 * cc + e] >> ((bits - 1) & 31)) & 1u : 0u;
                }
                any |= wv[4 * cc + e];
            }
            if (4 * c < W8)
                *reinterpret_cast<uint4*>(sa + ((size_t)(g * kc16 + c) * 8 + rr) * 16) =
                    make_uint4(wv[4 * cc], wv[4 * cc + 1], wv[4 * cc + 2], wv[4 * cc + 3]);
        }
        // both halves contribute flags
        if (half == 0) flags[n] = 0;
        __syncthreads();
        atomicOr(&flags[n], (sign ? 1u : 0u) | (neg ? 2u : 0u) | (any ? 4u : 0u));
    }
    // 2^bits mod p_j for the sign / negation corrections, once per CTA
    for (int j = tid; j < P; j += blockDim.x)
        spw[j] = reduce_u64((uint64_t)modup_tab[(size_t)j * HG_MODUP_WMAX + (bits >> 5)] << (bits & 31), pinfo[j]);
    asm volatile("fence.proxy.async.shared::cta;\n");
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t tmem = tmem_base;
    const int n = tid & (kRows - 1);
    const uint32_t fl = flags[n];
    const bool sgn = fl & 1u, ng = (fl & 2u) && (fl & 4u);
    const uint32_t a_base = smem_u32(sa), b_base = smem_u32(sb);
    const int nchunks = (P + kPrimesChunk - 1) / kPrimesChunk;
    const uint32_t idesc = (2u << 4) | ((uint32_t)(256 >> 3) << 17) | ((uint32_t)(kRows >> 4) << 24);
    uint32_t bphase[2] = {0u, 0u}, mphase[2] = {0u, 0u};
    uint32_t* outp = out + (size_t)op * P * N;
    // pipeline (B stages and TMEM both double buffered): MMA(ch+1) is issued before the epilogue of
    // ch and the B image of ch+2 is copied while both run
    auto copy_b = [&](int ch) {
        const int s2 = ch & 1;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(&mbar_b[s2])), "r"(kBChunkBytes));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                     ::"r"(b_base + (uint32_t)(s2 * kBChunkBytes)),
                     "l"(Bimg + (size_t)ch * kBChunkBytes), "r"(kBChunkBytes),
                     "r"(smem_u32(&mbar_b[s2])) : "memory");
    };
    auto mma_chunk = [&](int ch) {
        const int s2 = ch & 1;
        mbar_wait(smem_u32(&mbar_b[s2]), bphase[s2]);
        bphase[s2] ^= 1u;
        asm volatile("tcgen05.fence::after_thread_sync;\n");
        for (int k = 0; k < W8 / 8; ++k) {
            const uint64_t da = umma_desc(a_base + (uint32_t)(2 * k * 128), 128, kc16 * 128);
            const uint64_t db = umma_desc(b_base + (uint32_t)(s2 * kBChunkBytes + 2 * k * 128), 128, kc16 * 128);
            const uint32_t acc = k > 0 ? 1u : 0u;
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                         "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                         ::"r"(tmem + (uint32_t)(s2 * 256)), "l"(da), "l"(db), "r"(idesc), "r"(acc));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n"
                     ::"r"(smem_u32(&mbar_mma[s2])));
    };
    if (tid == 0) {
        copy_b(0);
        if (nchunks > 1) copy_b(1);
        mma_chunk(0);
    }
    for (int ch = 0; ch < nchunks; ++ch) {
        const int s = ch & 1;
        // everyone: wait for this chunk's accumulators
        mbar_wait(smem_u32(&mbar_mma[s]), mphase[s]);
        mphase[s] ^= 1u;
        asm volatile("tcgen05.fence::after_thread_sync;\n");
        if (tid == 0) {
            if (ch + 1 < nchunks) mma_chunk(ch + 1);   // TMEM stage s^1: its readers (ch-1) are done
            if (ch + 2 < nchunks) copy_b(ch + 2);      // B stage s: MMA(ch) has retired
        }
        // epilogue: warps w and w+4 share TMEM lane quarter w%4; split the chunk's primes
        const int jbase = ch * kPrimesChunk + (warp >> 2) * (kPrimesChunk / 2);
        const uint32_t lane_addr = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(s * 256) +
                                   (uint32_t)((warp >> 2) * (kPrimesChunk / 2) * 4);
#pragma unroll 1
        for (int jj = 0; jj < kPrimesChunk / 2; jj += 4) {
            uint32_t d[16];
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
                         : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]),
                           "=r"(d[6]), "=r"(d[7]), "=r"(d[8]), "=r"(d[9]), "=r"(d[10]), "=r"(d[11]),
                           "=r"(d[12]), "=r"(d[13]), "=r"(d[14]), "=r"(d[15])
                         : "r"(lane_addr + (uint32_t)(jj * 4)));
            asm volatile("tcgen05.wait::ld.sync.aligned;\n");
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int j = jbase + jj + e;
                if (j >= P) break;
                const PrimeInfo pi = pinfo[j];
                const uint64_t v = (uint64_t)d[4 * e] + ((uint64_t)d[4 * e + 1] << 8) +
                                   ((uint64_t)d[4 * e + 2] << 16) + ((uint64_t)d[4 * e + 3] << 24);
                uint32_t r = reduce_u64(v, pi);
                if (sgn || ng) {
                    const uint32_t pw = spw[j];
                    if (sgn) r = r >= pw ? r - pw : r + pi.p - pw;
                    if (ng) {
                        if (is_signed) r = r ? pi.p - r : 0;
                        else r = pw >= r ? pw - r : pw + pi.p - r;
                    }
                }
                outp[(size_t)j * N + cb + n] = r;
            }
        }
        // TMEM stage s is reused by chunk ch+2: its readers must be done before that MMA
        asm volatile("tcgen05.fence::before_thread_sync;\n");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;\n");
    }
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(512));
}

}  // namespace

// B images: chunk ch = primes 64ch..64ch+63 -> 256 rows (j, r) x K = 256 bytes (64 words x 4
// bytes), K-major core layout: core (row group g, k chunk c) at (g * 16 + c) * 128, row s at
// +16s; byte 4e+q of chunk c (word w = 4c+e) = byte r of 2^(32w+8q) mod p_j.
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
                    img[(size_t)ch * kBChunkBytes + ((size_t)(g * (kWMax / 4) + c) * 8 + s) * 16 + byte] =
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
    // narrow operands (compact plaintexts, low levels) stay on the mma.sync path: the full-K
    // B images (64 KB per 64 primes) would dominate their cost
    if (ctx->N < kRows || maxw > kWMax || maxw < 24) return 0;
    int rc = hg_modup_build_umma(ctx);
    if (rc) return -rc;
    static bool attr = false;
    const size_t smem = (size_t)kRows * 4 * kWMax + 2 * (size_t)kBChunkBytes;   // 160 KB
    if (!attr) {
        if (cudaFuncSetAttribute(modup_umma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
            return -hg_fail(HG_ECUDA, "modup_umma smem attribute");
        attr = true;
    }
    MOps o{};
    for (int k = 0; k < nops; ++k) {
        o.words[k] = words[k];
        o.bits[k] = bits[k];
        o.is_signed[k] = is_signed[k];
    }
    dim3 grid(ctx->N / kRows, nops);
    modup_umma_kernel<<<grid, 256, smem, st>>>(o, ctx->N, ctx->d_pinfo, ctx->d_modup,
                                               ctx->d_modup_umma, P, out, kinv);
    ctx->launches.fetch_add(1, std::memory_order_relaxed);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return -hg_fail(HG_ECUDA, std::string("modup_umma launch: ") + cudaGetErrorString(e));
    return 1;
}
