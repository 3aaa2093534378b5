// hg_crt_umma.cu -- CRT reconstruction on the 5th-gen tensor cores (tcgen05.mma kind::i8,
// SASS UTCIMMA), accumulators in TMEM.
//
// "Digit" layout: with y_j = sum_q yb_{j,q} 2^(8q) and the 32-bit words of Q/p_j split into
// bytes, column t of the exact product is
//     col_t = sum_{s=0..6} E_s(t) 2^(8s),   E_s(t) = sum_j sum_q yb_{j,q} * byte_{s-q}(M[j][t]),
// i.e. one u8 x u8 -> s32 GEMM with rows = coefficients (M = 128 per CTA), K = (prime, byte of y)
// and columns = (output word t, digit s) -- 8 TMEM columns per output word (s = 7 is zero).
// Every TMEM lane (= thread) therefore holds all digits of its own coefficient: the epilogue is
// a per-thread radix-2^8 -> radix-2^32 fold plus the exact carry chain, with no shuffles.
// A (the y bytes) is computed from the residues straight into shared memory in the UMMA
// K-major core-matrix layout; B (constant per prime basis) is streamed in 32-prime K chunks.
#include "hg_internal.cuh"

namespace {

constexpr int kRows = 128;      // coefficients per CTA = UMMA M
constexpr int kColChunk = 32;   // output words per accumulation pass (N = 256)
constexpr int kKChunk = 128;    // bytes of K per pipeline stage (32 primes, 4 UMMA k-steps)
constexpr int kBStage = kColChunk * 8 * kKChunk;   // 32 KB

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);  // SWIZZLE_NONE, v1
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

// HG_CRT_PROF (diagnostic builds only): per-CTA, per-warp cycles spent in each barrier wait of
// the pipelined kernel, read back with hg_crt_prof_read
#ifdef HG_CRT_PROF
__device__ unsigned long long g_crt_prof[160][20][8];
#define PWAIT(cat, bar, par)                                  \
    do {                                                      \
        const long long _t = clock64();                       \
        mbar_wait(bar, par);                                  \
        prof[cat] += (unsigned long long)(clock64() - _t);    \
    } while (0)
#else
#define PWAIT(cat, bar, par) mbar_wait(bar, par)
#endif

constexpr int kMaxOuts = 8;   // outputs per launch (the pipelined kernel; older kernels take 4)
struct UOuts {
    uint32_t* out[kMaxOuts];
};
// select, not index: a dynamic index into the parameter struct would copy it to the stack
__device__ __forceinline__ uint32_t* pick_out(const UOuts& o, int k) {
    return k == 0 ? o.out[0] : k == 1 ? o.out[1] : k == 2 ? o.out[2] : k == 3 ? o.out[3]
         : k == 4 ? o.out[4] : k == 5 ? o.out[5] : k == 6 ? o.out[6] : o.out[7];
}

// exact column scan for one coefficient (rare fallback when the truncated carry window is
// ambiguous); y_j read back from the A tile (row n, byte 4j)
__device__ void umma_rescan_exact(const uint8_t* sa, int kc16, int n, int P, int W,
                                  const uint32_t* __restrict__ Mtab,
                                  const uint32_t* __restrict__ negQ, uint32_t v, int shift,
                                  int out_bits, uint32_t* __restrict__ out, int N, int i) {
    const int sw = shift >> 5, sb = shift & 31;
    const int out_w = (out_bits + 31) >> 5;
    const uint32_t top_mask = (out_bits & 31) ? ((1u << (out_bits & 31)) - 1u) : 0xffffffffu;
    const int T = sw + out_w + (sb ? 1 : 0);
    const int round_col = shift > 0 ? ((shift - 1) >> 5) : -1;
    const uint32_t round_bit = shift > 0 ? (1u << ((shift - 1) & 31)) : 0u;
    const int g = n >> 3, rr = n & 7;
    uint64_t carry = 0;
    uint32_t prev = 0;
    for (int t = 0; t < T; ++t) {
        uint64_t x = (uint64_t)v * negQ[t] + (t == round_col ? round_bit : 0u) + (uint32_t)carry;
        uint64_t top = (carry >> 32) + (x >> 32);
        uint64_t acc = (uint32_t)x;
        for (int j = 0; j < P; ++j) {
            const int c = j >> 2;
            const uint32_t y = *reinterpret_cast<const uint32_t*>(sa + ((size_t)(g * kc16 + c) * 8 + rr) * 16 + (j & 3) * 4);
            acc += (uint64_t)y * Mtab[(size_t)j * W + t];
            top += acc >> 32;
            acc &= 0xffffffffull;
        }
        const uint32_t word = (uint32_t)acc;
        carry = top;
        if (t >= sw) {
            if (sb == 0) {
                const int u = t - sw;
                out[(size_t)u * N + i] = (u == out_w - 1) ? (word & top_mask) : word;
            } else if (t > sw) {
                const int u = t - sw - 1;
                const uint32_t o = (prev >> sb) | (word << (32 - sb));
                out[(size_t)u * N + i] = (u == out_w - 1) ? (o & top_mask) : o;
            }
        }
        prev = word;
    }
}

__global__ void __launch_bounds__(2 * kRows) crt_umma_kernel(
    const uint32_t* __restrict__ res, int P, int P32, int N, const PrimeInfo* __restrict__ pinfo,
    const uint8_t* __restrict__ Bconv, const uint32_t* __restrict__ Mtab, int W,
    const uint32_t* __restrict__ negQ, const uint32_t* __restrict__ cinv,
    const uint32_t* __restrict__ cinv_sh, const double* __restrict__ invp, int shift,
    int out_bits, int tb0, UOuts outs) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t tmem_base;
    __shared__ __align__(8) uint64_t mbar[2];
    const int K = 4 * P32;                 // bytes of K
    const int kc16 = K / 16;               // 16-byte K chunks per row
    uint8_t* sa = smem;                    // A: 128 rows x K bytes (core-matrix layout)
    uint8_t* sb = smem + (size_t)kRows * K;  // B: 2 stages x 32 KB
    const int tid = threadIdx.x, warp = tid >> 5;
    const int cb = blockIdx.x * kRows;
    const int oy = blockIdx.y;
    const uint32_t* r = res + (size_t)oy * P * N;
    uint32_t* out = oy == 0 ? outs.out[0] : oy == 1 ? outs.out[1] : oy == 2 ? outs.out[2] : outs.out[3];

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base)), "n"(256));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    __shared__ __align__(8) uint64_t mbar_b[2];   // B stage landed (bulk copy tx count)
    __shared__ __align__(8) uint64_t mbar_ld;     // residue chunk landed
    __shared__ __align__(8) uint64_t mbar_done;   // all MMAs of a column chunk retired
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&mbar[0])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&mbar[1])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&mbar_b[0])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&mbar_b[1])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&mbar_ld)));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&mbar_done)));
        asm volatile("fence.mbarrier_init.release.cluster;\n");
    }
    __syncthreads();

    // ---- phase 1: residues of 128 primes at a time land in the (still idle) B stages through
    // bulk copies (one 512-byte row per prime); two threads per coefficient (alternating
    // 16-prime groups) turn them into y_j -> A (K-major core layout) and S = sum y_j / p_j -> v --
    __shared__ double ssum[2 * kRows];
    {
        double S = 0.0;
        const int n = tid & (kRows - 1), half = tid >> 7, g = n >> 3, rr = n & 7;
        const uint32_t* stage = reinterpret_cast<const uint32_t*>(sb);
        uint32_t ld_phase = 0;
        for (int jc = 0; jc < P32; jc += 128) {
            const int cnt = P - jc < 128 ? P - jc : 128;
            if (cnt > 0) {
                if (tid == 0) {
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n"
                                 ::"r"(smem_u32(&mbar_ld)), "r"(cnt * kRows * 4));
                    for (int jj = 0; jj < cnt; ++jj)
                        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                                     ::"r"(smem_u32(sb) + jj * kRows * 4),
                                     "l"(r + (size_t)(jc + jj) * N + cb), "n"(kRows * 4),
                                     "r"(smem_u32(&mbar_ld))
                                     : "memory");
                }
                mbar_wait(smem_u32(&mbar_ld), ld_phase);
                ld_phase ^= 1u;
            }
            const int jend = jc + 128 < P32 ? jc + 128 : P32;
        for (int j0 = jc + 16 * half; j0 < jend; j0 += 32) {
            uint32_t x[16];
#pragma unroll
            for (int u = 0; u < 16; ++u) {
                const int j = j0 + u;
                x[u] = j < P ? stage[(j - jc) * kRows + n] : 0u;
            }
#pragma unroll
            for (int c4 = 0; c4 < 4; ++c4) {
                uint32_t y[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int j = j0 + 4 * c4 + u;
                    y[u] = 0;
                    if (j < P) {
                        const uint32_t p = pinfo[j].p;
                        y[u] = reduce_2p(mul_shoup_lazy(x[4 * c4 + u], cinv[j], cinv_sh[j], p), p);
                        S += (double)y[u] * invp[j];
                    }
                }
                const int c = (j0 >> 2) + c4;
                *reinterpret_cast<uint4*>(sa + ((size_t)(g * kc16 + c) * 8 + rr) * 16) =
                    make_uint4(y[0], y[1], y[2], y[3]);
            }
        }
            // the staging rows are rewritten by the async proxy next: order our reads first
            asm volatile("fence.proxy.async.shared::cta;\n");
            __syncthreads();
        }
        ssum[tid] = S;
    }
    asm volatile("fence.proxy.async.shared::cta;\n");
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const int nn = tid & (kRows - 1);
    const uint32_t v = (uint32_t)floor(ssum[nn] + ssum[kRows + nn] + 0.5);
    const bool epi = tid < kRows;   // warps 0-3 own TMEM lanes 0-127
    const uint32_t tmem = tmem_base;

    // ---- phase 2/3: column chunks: K-pipelined UMMA into TMEM, then the per-thread chain ------
    const int sw = shift >> 5, sbit = shift & 31;
    const int out_w = (out_bits + 31) >> 5;
    const uint32_t top_mask = (out_bits & 31) ? ((1u << (out_bits & 31)) - 1u) : 0xffffffffu;
    const int T = sw + out_w + (sbit ? 1 : 0);
    const int round_col = shift > 0 ? ((shift - 1) >> 5) : -1;
    const uint32_t round_bit = shift > 0 ? (1u << ((shift - 1) & 31)) : 0u;
    const int nkc = P32 / 32;
    const uint32_t a_base = smem_u32(sa);
    const uint32_t b_base = smem_u32(sb);
    const int i = cb + nn;
    uint64_t carry = 0;
    uint32_t prev = 0;
    bool amb = false;
    uint32_t phase[2] = {0u, 0u};     // MMA-commit barriers (tid 0's bookkeeping)
    uint32_t bphase[2] = {0u, 0u};    // B-landed barriers (tid 0)
    uint32_t done_phase = 0u;         // chunk-done barrier (everyone)
    bool used[2] = {false, false};
    int stage_ctr = 0;
    for (int t0 = tb0; t0 < T; t0 += kColChunk) {
        int ncols = T - t0;
        if (ncols > kColChunk) ncols = kColChunk;
        ncols = (ncols + 1) & ~1;                      // N = 8 * ncols, a multiple of 16
        const uint32_t Nn = 8u * ncols;
        const uint32_t idesc = (2u << 4) | ((Nn >> 3) << 17) | ((uint32_t)(kRows >> 4) << 24);
        const int tg0 = t0 >> 3;                       // first 8-column group in the B table
        // one thread drives the pipeline: bulk-copy B stage kc+1 while the MMAs of stage kc run
        if (tid == 0) {
            const int ngroups = (ncols + 7) >> 3;
            auto issue_b = [&](int kc) {
                const int s = (stage_ctr + kc) & 1;
                if (used[s]) {                         // the MMAs that read this stage retired
                    mbar_wait(smem_u32(&mbar[s]), phase[s]);
                    phase[s] ^= 1u;
                    used[s] = false;
                }
                const uint32_t bytes = (uint32_t)ngroups * 8192u;
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n"
                             ::"r"(smem_u32(&mbar_b[s])), "r"(bytes));
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                             ::"r"(b_base + (uint32_t)(s * kBStage)),
                             "l"(Bconv + ((size_t)kc * (W >> 3) + tg0) * 8192), "r"(bytes),
                             "r"(smem_u32(&mbar_b[s]))
                             : "memory");
            };
            issue_b(0);
            for (int kc = 0; kc < nkc; ++kc) {
                const int s = (stage_ctr + kc) & 1;
                mbar_wait(smem_u32(&mbar_b[s]), bphase[s]);
                bphase[s] ^= 1u;
                asm volatile("tcgen05.fence::after_thread_sync;\n");
#pragma unroll
                for (int k = 0; k < kKChunk / 32; ++k) {
                    const uint64_t da = umma_desc(a_base + (uint32_t)((kc * (kKChunk / 16) + 2 * k) * 128), 128, kc16 * 128);
                    const uint64_t db = umma_desc(b_base + (uint32_t)(s * kBStage + 2 * k * 128), 128, 8 * 128);
                    const uint32_t acc = (kc > 0 || k > 0) ? 1u : 0u;
                    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                                 "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                                 ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(acc));
                }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n"
                             ::"r"(smem_u32(&mbar[s])));
                used[s] = true;
                if (kc + 1 < nkc) issue_b(kc + 1);
            }
            // one more commit tracking every MMA issued so far: the chunk is complete when it fires
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n"
                         ::"r"(smem_u32(&mbar_done)));
        }
        stage_ctr += nkc;
        mbar_wait(smem_u32(&mbar_done), done_phase);
        done_phase ^= 1u;
        asm volatile("tcgen05.fence::after_thread_sync;\n");
        // epilogue: this thread's TMEM lane = its coefficient
        const uint32_t lane_addr = tmem + ((uint32_t)((warp & 3) * 32) << 16);
        for (int tl = 0; epi && tl < ncols; tl += 2) {   // warp-uniform: warps 4-7 skip
            uint32_t e[16];
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
                         : "=r"(e[0]), "=r"(e[1]), "=r"(e[2]), "=r"(e[3]), "=r"(e[4]), "=r"(e[5]),
                           "=r"(e[6]), "=r"(e[7]), "=r"(e[8]), "=r"(e[9]), "=r"(e[10]), "=r"(e[11]),
                           "=r"(e[12]), "=r"(e[13]), "=r"(e[14]), "=r"(e[15])
                         : "r"(lane_addr + (uint32_t)(tl * 8)));
            asm volatile("tcgen05.wait::ld.sync.aligned;\n");
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int t = t0 + tl + h;
                if (t >= T) break;
                const uint32_t* E = e + 8 * h;
                const uint64_t lo = (uint64_t)E[0] + ((uint64_t)E[1] << 8) + ((uint64_t)E[2] << 16) + ((uint64_t)E[3] << 24);
                const uint64_t hi = (uint64_t)E[4] + ((uint64_t)E[5] << 8) + ((uint64_t)E[6] << 16) + ((uint64_t)E[7] << 24);
                const uint64_t extra = (uint64_t)v * negQ[t] + (t == round_col ? round_bit : 0u);
                const uint64_t sum = (lo & 0xffffffffull) + (carry & 0xffffffffull) + (extra & 0xffffffffull);
                const uint32_t word = (uint32_t)sum;
                carry = (sum >> 32) + (lo >> 32) + hi + (carry >> 32) + (extra >> 32);
                if (t < sw) {
                    if (t == tb0 + 1) amb = word >= 0xFFFFFF00u;
                    else if (t > tb0 + 1) amb = amb && (word == 0xffffffffu);
                } else if (sbit == 0) {
                    const int u = t - sw;
                    out[(size_t)u * N + i] = (u == out_w - 1) ? (word & top_mask) : word;
                } else if (t > sw) {
                    const int u = t - sw - 1;
                    const uint32_t o = (prev >> sbit) | (word << (32 - sbit));
                    out[(size_t)u * N + i] = (u == out_w - 1) ? (o & top_mask) : o;
                }
                prev = word;
            }
        }
        // all lanes must finish reading TMEM before the next chunk's MMAs overwrite it
        asm volatile("tcgen05.fence::before_thread_sync;\n");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;\n");
    }
    if (epi && tb0 > 0 && amb)
        umma_rescan_exact(sa, kc16, nn, P, W, Mtab, negQ, v, shift, out_bits, out, N, i);
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(256));
}

// ==========================================================================================
// Persistent, warp-specialised variant (the production path).  One CTA per SM walks jobs =
// (tile of 128 coefficients of one output polynomial, block of <= 32 output words): N <= 256 per
// job, so TMEM holds two job accumulators and the epilogue of job i overlaps the MMAs of job
// i+1.  The y bytes (A) are streamed per K chunk through a ring (recomputed for each column
// block of a tile: the residues come back from L2).  The reduction term v * (-Q) is one more K
// row (slot P: A = v, B = the digits of -Q mod 2^(32W)), so the epilogue only folds digits and
// runs the carry chain.  Roles, linked by mbarrier rings:
//   warp 0      residue producer: cp.async.bulk of 32 prime rows (16 KB) per K chunk
//   warp 1      MMA issuer (lane 0): 4 k-steps of 128 x N x 32 per K chunk; commits free the
//               A / B stages, the job's last commit hands its TMEM buffer to the epilogue
//   warp 2      B producer: the job's digit-layout B slice of the K chunk (<= 32 KB) per stage
//   warps 3-10  converters: residues -> y_j = x_j (Q/p_j)^{-1} -> A stage; v = round(sum y_j/p_j)
//   warps 11-18 epilogue, two groups of 4 taking alternate jobs: TMEM lane = coefficient:
//               digit fold, carry chain (handed between the groups), window emission
//   warp 19     (fused finish only) addend producer: the job's 32 addend words of its 128
//               coefficients as one 2-D TMA box into a 2-stage ring
constexpr int kConvWarp0 = 3, kEpiWarp0 = 11, kAddWarp = 19;
template <bool FUSED> struct PipeCfg {
    static constexpr int kWarps = FUSED ? 20 : 19;
#ifndef HG_CRT_RR_FUSED
#define HG_CRT_RR_FUSED 3
#endif
#ifndef HG_CRT_RR_PLAIN
#define HG_CRT_RR_PLAIN 4
#endif
    static constexpr int kRR = FUSED ? HG_CRT_RR_FUSED : HG_CRT_RR_PLAIN;
#ifndef HG_CRT_RA_FUSED
#define HG_CRT_RA_FUSED 3
#endif
#ifndef HG_CRT_RA_PLAIN
#define HG_CRT_RA_PLAIN 4
#endif
    static constexpr int kRA = FUSED ? HG_CRT_RA_FUSED : HG_CRT_RA_PLAIN;
    static constexpr int kRB = FUSED ? 2 : 3;
};
#ifndef HG_CRT_JOBCOLS
#define HG_CRT_JOBCOLS 56   // 49-52-word windows are one job; 56 frees smem for a third / fourth residue stage
#endif
constexpr int kJobCols = HG_CRT_JOBCOLS;          // output words per job (4 columns each: N <= 256)
constexpr int kResStage = 32 * kRows * 4;        // 16 KB: 32 prime rows of 128 residues
constexpr int kAStage = kRows * kKChunk;         // 16 KB
constexpr int kBStagePipe = kJobCols * 4 * kKChunk;   // 32 KB
constexpr int kBGran = 4096;                     // B image bytes per (K chunk, 8-word group)
constexpr int kAddStage = kJobCols * kRows * 4;  // 32 KB: 64 addend words of 128 coefficients
template <bool FUSED>
constexpr size_t pipe_smem() {
    return (size_t)PipeCfg<FUSED>::kRR * kResStage + (size_t)PipeCfg<FUSED>::kRA * kAStage + (size_t)PipeCfg<FUSED>::kRB * kBStagePipe +
           (FUSED ? 2 * (size_t)kAddStage : 0);
}

// a * b + c, 32 x 32 -> 64-bit multiply-add (one IMAD.WIDE)
__device__ __forceinline__ uint64_t madw(uint32_t a, uint32_t b, uint64_t c) {
    uint64_t d;
    asm("mad.wide.u32 %0, %1, %2, %3;\n" : "=l"(d) : "r"(a), "r"(b), "l"(c));
    return d;
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                 ::"r"(dst), "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(bar) : "memory");
}

// Output stage of the pipelined kernel.  Plain: word u of the CRT window goes to out[u].
// Fused finish (CrtFinish): the window value e (out_bits = l bits) is streamed through
//     s = (e + addend + 2^(post-1)) mod 2^l,   out = bits [post, l) of s
// -- the add of ckks.mult / _apply_automorphism followed by the rescale's divide_round
// (ckks.py:166-184, 247-253, 310-313) -- with the addend optionally read through the ring
// automorphism (out[i] = +/- add[i * kinv mod 2N], the negation as ~a + 1).
struct Emitter {
    uint32_t* out;
    const uint32_t* add;
    int N, i, src, out_w, post, rw, rb, out2_w, rw2;
    uint32_t top_l, top2, rbit2, c2, prev2;
    bool plain, negate;
    __device__ __forceinline__ void init(uint32_t* o, int n, int ii, int out_bits, const CrtFinish& f,
                                         const uint32_t* addp) {
        out = o;
        N = n;
        i = ii;
        out_w = (out_bits + 31) >> 5;
        top_l = (out_bits & 31) ? ((1u << (out_bits & 31)) - 1u) : 0xffffffffu;
        add = addp;
        post = f.post;
        plain = addp == nullptr && post == 0;
        src = ii;
        bool neg = false;
        if (addp && f.kinv != 0) {
            int64_t j = ((int64_t)ii * f.kinv) & (2ll * n - 1);
            neg = j >= n;
            src = (int)(neg ? j - n : j);
        }
        c2 = neg ? 1u : 0u;   // -a = ~a + 1
        prev2 = 0u;
        negate = neg;
        rw = post >> 5;
        rb = post & 31;
        const int bits2 = out_bits - post;
        out2_w = (bits2 + 31) >> 5;
        top2 = (bits2 & 31) ? ((1u << (bits2 & 31)) - 1u) : 0xffffffffu;
        rw2 = post > 0 ? (post - 1) >> 5 : -1;
        rbit2 = post > 0 ? 1u << ((post - 1) & 31) : 0u;
    }
    // addend word u (0 when there is none); callers prefetch it off the carry chain
    __device__ __forceinline__ uint32_t load_add(int u) const {
        return (add && u >= 0 && u < out_w) ? __ldg(add + (size_t)u * N + src) : 0u;
    }
    __device__ __forceinline__ void put(int u, uint32_t e, uint32_t a) {
        if (u == out_w - 1) e &= top_l;
        if (plain) {
            out[(size_t)u * N + i] = e;
            return;
        }
        if (negate) a = ~a;
        const uint64_t sum = (uint64_t)e + a + c2 + (u == rw2 ? rbit2 : 0u);
        uint32_t w = (uint32_t)sum;
        c2 = (uint32_t)(sum >> 32);
        if (u == out_w - 1) w &= top_l;
        if (rb == 0) {
            const int v = u - rw;
            if (v >= 0 && v < out2_w) out[(size_t)v * N + i] = v == out2_w - 1 ? (w & top2) : w;
        } else {
            const int v = u - rw - 1;
            if (v >= 0 && v < out2_w)
                out[(size_t)v * N + i] = __funnelshift_r(prev2, w, rb) & (v == out2_w - 1 ? top2 : 0xffffffffu);
            prev2 = w;
        }
    }
    __device__ __forceinline__ void flush() {
        if (plain || rb == 0) return;
        const int v = out_w - 1 - rw;
        if (v >= 0 && v < out2_w) out[(size_t)v * N + i] = (prev2 >> rb) & (v == out2_w - 1 ? top2 : 0xffffffffu);
    }
};

// exact column scan for one coefficient with y_j and v recomputed from the residues (rare)
__device__ void pipe_rescan_exact(const uint32_t* __restrict__ r, int P, int N, int W,
                                  const PrimeInfo* __restrict__ pinfo,
                                  const uint32_t* __restrict__ cinv,
                                  const uint32_t* __restrict__ cinv_sh,
                                  const double* __restrict__ invp,
                                  const uint32_t* __restrict__ Mtab,
                                  const uint32_t* __restrict__ negQ, int shift, int out_bits,
                                  bool prescaled, Emitter em) {
    const int i = em.i;
    // prescaled residues already carry the factor (Q/p_j)^-1 N^-1 2^32 and sit in [0, 2p)
    auto yj = [&](int j) {
        const uint32_t p = pinfo[j].p, x = r[(size_t)j * N + i];
        return reduce_2p(prescaled ? x : mul_shoup_lazy(x, cinv[j], cinv_sh[j], p), p);
    };
    double S = 0.0;
    for (int j = 0; j < P; ++j) S += (double)yj(j) * invp[j];
    const uint32_t v = (uint32_t)floor(S + 0.5);
    const int sw = shift >> 5, sb = shift & 31;
    const int out_w = (out_bits + 31) >> 5;
    const uint32_t top_mask = (out_bits & 31) ? ((1u << (out_bits & 31)) - 1u) : 0xffffffffu;
    const int T = sw + out_w + (sb ? 1 : 0);
    const int round_col = shift > 0 ? ((shift - 1) >> 5) : -1;
    const uint32_t round_bit = shift > 0 ? (1u << ((shift - 1) & 31)) : 0u;
    uint64_t carry = 0;
    uint32_t prev = 0;
    for (int t = 0; t < T; ++t) {
        uint64_t x = (uint64_t)v * negQ[t] + (t == round_col ? round_bit : 0u) + (uint32_t)carry;
        uint64_t top = (carry >> 32) + (x >> 32);
        uint64_t acc = (uint32_t)x;
        for (int j = 0; j < P; ++j) {
            acc += (uint64_t)yj(j) * Mtab[(size_t)j * W + t];
            top += acc >> 32;
            acc &= 0xffffffffull;
        }
        const uint32_t word = (uint32_t)acc;
        carry = top;
        if (t >= sw) {
            if (sb == 0) em.put(t - sw, word, em.load_add(t - sw));
            else if (t > sw) em.put(t - sw - 1, (prev >> sb) | (word << (32 - sb)), em.load_add(t - sw - 1));
        }
        prev = word;
    }
    em.flush();
    (void)top_mask;
}

// PRESCALED: the residues were produced from operands pre-multiplied by the per-prime CRT
// constant (hg_key / hg_ctprep prepared for this window), so y_j = x_j mod p_j is one
// conditional subtraction instead of a Shoup product
// LOGN: log2 N as a compile-time constant (the epilogue's word-row strides become address
// immediates), 0 = N at run time
template <bool FUSED, bool PRESCALED, int LOGN>
__global__ void __launch_bounds__(PipeCfg<FUSED>::kWarps * 32, 1) crt_umma_pipe_kernel(
    const __grid_constant__ CUtensorMap res_map, const __grid_constant__ CUtensorMap add_map,
    const uint32_t* __restrict__ res, int P, int P32p, int N_rt, int nouts,
    const PrimeInfo* __restrict__ pinfo, const uint8_t* __restrict__ Bpipe,
    const uint32_t* __restrict__ Mtab, int W, const uint32_t* __restrict__ negQ,
    const uint32_t* __restrict__ cinv, const uint32_t* __restrict__ cinv_sh,
    const double* __restrict__ invp, int shift, int out_bits, int tb0, UOuts outs, CrtFinish fin) {
    constexpr int kRR = PipeCfg<FUSED>::kRR;
    constexpr int kRA = PipeCfg<FUSED>::kRA;
    constexpr int kRB = PipeCfg<FUSED>::kRB;
    const int N = LOGN ? (1 << LOGN) : N_rt;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* s_res = smem;
    uint8_t* s_a = smem + kRR * kResStage;
    uint8_t* s_b = s_a + kRA * kAStage;
    const uint32_t* s_add = reinterpret_cast<const uint32_t*>(s_b + kRB * kBStagePipe);
    __shared__ __align__(8) uint64_t bar_add_full[2], bar_add_empty[2];
    __shared__ __align__(8) uint64_t bar_res_full[kRR], bar_res_empty[kRR];
    __shared__ __align__(8) uint64_t bar_a_full[kRA], bar_a_empty[kRA];
    __shared__ __align__(8) uint64_t bar_b_full[kRB], bar_b_empty[kRB];
    __shared__ __align__(8) uint64_t bar_tm_full[2], bar_tm_empty[2];
    __shared__ __align__(8) uint64_t bar_hand_full[2], bar_hand_empty[2];
    __shared__ uint4 s_hand[2][kRows];             // carry lo/hi, previous word, ambiguity
    __shared__ uint2 s_hand2[2][kRows];            // emitter state: carry, previous word
    __shared__ uint32_t tmem_base;
    // p, cinv, cinv_sh, floor(2^55/p) (1,0,0,0 padding); PRESCALED: p, ~0, 0, floor(2^55/p)
    __shared__ uint4 s_pc[HG_MAX_PRIMES + 32];
    __shared__ uint32_t s_acc[2][kRows];

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int j = tid; j < P32p; j += blockDim.x) {
        const bool ok = j < P;
        const uint32_t p = ok ? pinfo[j].p : 1u;
        s_pc[j] = !ok ? make_uint4(1u, 0u, 0u, 0u)
              : PRESCALED ? make_uint4(p, 0xffffffffu, 0u, (uint32_t)((1ull << 55) / p))
                          : make_uint4(p, cinv[j], cinv_sh[j], (uint32_t)((1ull << 55) / p));
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base)), "n"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (tid == 0) {
        auto init = [](uint64_t* b, int cnt) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(cnt));
        };
        for (int s = 0; s < kRR; ++s) { init(&bar_res_full[s], 1); init(&bar_res_empty[s], 8); }
        for (int s = 0; s < kRA; ++s) { init(&bar_a_full[s], 8); init(&bar_a_empty[s], 1); }
        for (int s = 0; s < kRB; ++s) { init(&bar_b_full[s], 1); init(&bar_b_empty[s], 1); }
        for (int s = 0; s < 2; ++s) { init(&bar_tm_full[s], 1); init(&bar_tm_empty[s], 4); }
        for (int s = 0; s < 2; ++s) { init(&bar_hand_full[s], 4); init(&bar_hand_empty[s], 4); }
        for (int s = 0; s < 2; ++s) { init(&bar_add_full[s], 1); init(&bar_add_empty[s], 4); }
        asm volatile("fence.mbarrier_init.release.cluster;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t tmem = tmem_base;
#ifdef HG_CRT_PROF
    unsigned long long prof[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const long long t_start = clock64();
#endif

    const int tpo = N / kRows;
    const int sw = shift >> 5, sbit = shift & 31;
    const int out_w = (out_bits + 31) >> 5;
    const int T = sw + out_w + (sbit ? 1 : 0);
    const int jpt = (T - tb0 + kJobCols - 1) / kJobCols;   // jobs (column blocks) per tile
    // job width: the tile's columns split evenly over its jobs, in multiples of 8 words (the B
    // image granule), the last job taking the remainder (<= 32).  The two epilogue groups take
    // alternate jobs and the carry chain runs through them in order, so an even split keeps
    // one group from waiting on a 32-column job while the other has a short tail.
    const int jc = [&] {
        const int total = T - tb0;
        int w = (((total + jpt - 1) / jpt) / 8) * 8;
        if (w < 8) w = 8;
        if (total - (jpt - 1) * w > kJobCols) w += 8;
        return w > kJobCols ? kJobCols : w;
    }();
    const int ntiles = nouts * tpo;
    const int nkc = P32p / 32;
    // columns of job block h: [tb0 + jc h, min(T, tb0 + jc (h + 1))), padded to a multiple of
    // 4 words (UMMA N = 4 x words must be a multiple of 16)
    auto job_cols = [&](int h) {
        const int c0 = tb0 + h * jc;
        const int c = h == jpt - 1 ? T - c0 : (T - c0 < jc ? T - c0 : jc);
        return (c + 3) & ~3;
    };

    if (warp == 0) {
        // ---------------- residue producer ----------------
        // one 2-D TMA box (128 coefficients x 32 prime rows) per K chunk; rows past P belong to
        // the next output (or are zero-filled past the end) and meet cinv = 0 in the converters
        if (lane == 0) {
            int it = 0;
            for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x)
                for (int h = 0; h < jpt; ++h) {
                    const int oy = tile / tpo, cb = (tile - oy * tpo) * kRows;
                    for (int kc = 0; kc < nkc; ++kc, ++it) {
                        const int s = it % kRR;
                        PWAIT(0, smem_u32(&bar_res_empty[s]), ((it / kRR) & 1) ^ 1);
                        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                        mbar_expect_tx(smem_u32(&bar_res_full[s]), (uint32_t)kResStage);
                        asm volatile(
                            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                            " [%0], [%1, {%2, %3}], [%4];\n"
                            ::"r"(smem_u32(s_res + s * kResStage)), "l"(reinterpret_cast<uint64_t>(&res_map)),
                            "r"(cb), "r"(oy * P + kc * 32), "r"(smem_u32(&bar_res_full[s]))
                            : "memory");
                    }
                }
        }
    } else if (warp == 2) {
        // ---------------- B producer ----------------
        if (lane == 0) {
            int it = 0;
            for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x)
              for (int h = 0; h < jpt; ++h) {
                const uint32_t bytes = (uint32_t)((job_cols(h) + 7) >> 3) * kBGran;
                const uint8_t* bsrc = Bpipe + (size_t)((tb0 >> 3) + h * (jc / 8)) * kBGran;
                for (int kc = 0; kc < nkc; ++kc, ++it) {
                    const int s = it % kRB;
                    PWAIT(0, smem_u32(&bar_b_empty[s]), ((it / kRB) & 1) ^ 1);
                    mbar_expect_tx(smem_u32(&bar_b_full[s]), bytes);
                    bulk_g2s(smem_u32(s_b + s * kBStagePipe), bsrc + (size_t)kc * (W >> 3) * kBGran, bytes,
                             smem_u32(&bar_b_full[s]));
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer ----------------
        if (lane == 0) {
            const uint32_t a_base = smem_u32(s_a), b_base = smem_u32(s_b);
            int ia = 0, ib = 0, ij = 0;
            for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x)
              for (int h = 0; h < jpt; ++h, ++ij) {
                const uint32_t Nn = 4u * (uint32_t)job_cols(h);
                const uint32_t idesc = (2u << 4) | ((Nn >> 3) << 17) | ((uint32_t)(kRows >> 4) << 24);
                const int tb = ij & 1;
                PWAIT(0, smem_u32(&bar_tm_empty[tb]), ((ij >> 1) & 1) ^ 1);
                asm volatile("tcgen05.fence::after_thread_sync;\n");
                for (int kc = 0; kc < nkc; ++kc, ++ia, ++ib) {
                    const int sa_ = ia % kRA, sb_ = ib % kRB;
                    PWAIT(1, smem_u32(&bar_a_full[sa_]), (ia / kRA) & 1);
                    PWAIT(2, smem_u32(&bar_b_full[sb_]), (ib / kRB) & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;\n");
#pragma unroll
                    for (int k = 0; k < kKChunk / 32; ++k) {
                        const uint64_t da = umma_desc(a_base + (uint32_t)(sa_ * kAStage + 2 * k * 128), 128, 1024);
                        const uint64_t db = umma_desc(b_base + (uint32_t)(sb_ * kBStagePipe + 2 * k * 128), 128, 1024);
                        const uint32_t acc = (kc > 0 || k > 0) ? 1u : 0u;
                        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                                     "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                                     ::"r"(tmem + (uint32_t)(tb * 256)), "l"(da), "l"(db), "r"(idesc), "r"(acc));
                    }
                    umma_commit(smem_u32(&bar_a_empty[sa_]));
                    umma_commit(smem_u32(&bar_b_empty[sb_]));
                }
                umma_commit(smem_u32(&bar_tm_full[tb]));
            }
        }
    } else if (warp == kAddWarp) {
        // ---------------- addend producer (fused finish) ----------------
        if (FUSED && lane == 0) {
            int ij = 0;
            for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x)
                for (int h = 0; h < jpt; ++h, ++ij) {
                    const int oy = tile / tpo, cb = (tile - oy * tpo) * kRows;
                    const int ubase = tb0 + h * jc - sw - (sbit ? 1 : 0);
                    const int s = ij & 1;
                    PWAIT(0, smem_u32(&bar_add_empty[s]), ((ij >> 1) & 1) ^ 1);
                    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                    mbar_expect_tx(smem_u32(&bar_add_full[s]), (uint32_t)kAddStage);
                    asm volatile(
                        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                        " [%0], [%1, {%2, %3}], [%4];\n"
                        ::"r"(smem_u32(s_add + s * (kAddStage / 4))), "l"(reinterpret_cast<uint64_t>(&add_map)),
                        "r"(cb), "r"(oy * out_w + ubase), "r"(smem_u32(&bar_add_full[s]))
                        : "memory");
                }
        }
    } else if (warp < kEpiWarp0) {
        // ---------------- converters ----------------
        // warp pair (c, c + 4) owns coefficients 32c .. 32c+31; each takes 16 of a chunk's 32 primes
        const int cw = warp - kConvWarp0, q = cw & 3, half = cw >> 2;
        const int n = q * 32 + lane;
        const int g = n >> 3, rr = n & 7;
        int ir = 0, ia = 0;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x)
          for (int h = 0; h < jpt; ++h) {
            // v = round(sum y_j / p_j) in 32-bit fixed point with 23 fraction bits: each term
            // umulhi(y_j, floor(2^55 / p_j)) is y_j / p_j 2^23 less at most 2 units, so the sum
            // (< 321 2^23 < 2^32) is within 2^-13.6 below the true value, and the true value lies
            // within 1/8 of an integer (|c| < Q/8): rounding is exact.  One multiply-high and a
            // 32-bit add per residue instead of a 64-bit multiply-accumulate.
            uint32_t acc = 0;
            for (int kc = 0; kc < nkc; ++kc, ++ir, ++ia) {
                const int s = ir % kRR, sa_ = ia % kRA;
                PWAIT(0, smem_u32(&bar_res_full[s]), (ir / kRR) & 1);
                const uint32_t* stg = reinterpret_cast<const uint32_t*>(s_res + s * kResStage) + half * 16 * kRows;
                const int j0 = kc * 32 + half * 16;
                uint32_t y[16];
#pragma unroll
                for (int u = 0; u < 16; ++u) y[u] = stg[u * kRows + n];
                // the residue stage is free as soon as it sits in registers
                __syncwarp();
                if (lane == 0) mbar_arrive(smem_u32(&bar_res_empty[s]));
#pragma unroll
                for (int u = 0; u < 16; ++u) {
                    // padding primes: x is stale but cinv = 0 (PRESCALED: mask 0) gives y = 0
                    // (PRESCALED: a padding slot keeps a stale value -- its B rows are zero and its
                    // floor(2^55/p) is 0, so neither the GEMM nor v sees it)
                    const uint4 pc = s_pc[j0 + u];
                    const uint32_t yy = PRESCALED ? y[u] : mul_shoup_lazy(y[u], pc.y, pc.z, pc.x);
                    y[u] = min(yy, yy - pc.x);   // [0, 2p) -> [0, p)
                    acc += __umulhi(y[u], pc.w);
                }
                if (kc == nkc - 1) {
#ifdef HG_CRT_PROF
                    const long long t_bs = clock64();
#endif
                    // slot P of the last chunk carries v (its B row holds -Q): combine the halves
                    s_acc[half][n] = acc;
                    asm volatile("bar.sync 1, %0;\n" ::"n"(8 * 32) : "memory");
                    const uint32_t tot = s_acc[0][n] + s_acc[1][n];
                    asm volatile("bar.sync 1, %0;\n" ::"n"(8 * 32) : "memory");
                    const uint32_t v = (tot + (1u << 22)) >> 23;
#pragma unroll
                    for (int u = 0; u < 16; ++u)
                        if (j0 + u == P) y[u] = v;
#ifdef HG_CRT_PROF
                    prof[3] += (unsigned long long)(clock64() - t_bs);
#endif
                }
                PWAIT(1, smem_u32(&bar_a_empty[sa_]), ((ia / kRA) & 1) ^ 1);
#ifdef HG_CRT_PROF
                const long long t_st = clock64();
#endif
                // WAR across proxies: the tensor core's (async-proxy) reads of this stage must be
                // ordered before our generic stores
#ifndef HG_EXP_NO_WAR_FENCE
                asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
#endif
                uint8_t* dst = s_a + sa_ * kAStage + (g * 8 + 4 * half) * 128 + rr * 16;
#pragma unroll
                for (int c = 0; c < 4; ++c)
                    *reinterpret_cast<uint4*>(dst + c * 128) =
                        make_uint4(y[4 * c], y[4 * c + 1], y[4 * c + 2], y[4 * c + 3]);
                asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive(smem_u32(&bar_a_full[sa_]));
#ifdef HG_CRT_PROF
                prof[2] += (unsigned long long)(clock64() - t_st);
#endif
            }
        }
    } else {
        // ---------------- epilogue ----------------
        const int q = warp & 3;
        const int n = q * 32 + lane;
        const int round_col = shift > 0 ? ((shift - 1) >> 5) : -1;
        const uint32_t round_bit = shift > 0 ? (1u << ((shift - 1) & 31)) : 0u;
        const uint32_t top_l = (out_bits & 31) ? ((1u << (out_bits & 31)) - 1u) : 0xffffffffu;
        // two groups take alternate jobs (job parity = TMEM buffer); within a tile the carry
        // state moves from the group that finished column block h to the one taking h+1
        const int grp = (warp - kEpiWarp0) >> 2;
        // fused finish (see Emitter): window word u -> s = u + addend + c2 (+ the rescale's
        // rounding bit), output word v = bits [post, l) of s; the pipelined launcher takes no
        // automorphism on the addend
        const int post = FUSED ? fin.post : 0;
        const int rw = post >> 5, rb = post & 31, vsh = rb ? 1 : 0, ush = sbit ? 1 : 0;
        const int bits2 = out_bits - post;
        const int out2_w = (bits2 + 31) >> 5;
        const uint32_t top2 = (bits2 & 31) ? ((1u << (bits2 & 31)) - 1u) : 0xffffffffu;
        const int rw2 = post > 0 ? (post - 1) >> 5 : -1;
        const uint32_t rbit2 = post > 0 ? 1u << ((post - 1) & 31) : 0u;
        uint64_t carry = 0;
        uint32_t prev = 0, c2 = 0, prev2 = 0;
        bool amb = false;
        int nwr = 0, nrd = 0;   // handoffs written to slot grp / read from slot 1 - grp
        int ij = 0;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x)
          for (int h = 0; h < jpt; ++h, ++ij) {
            if ((ij & 1) != grp) continue;
            const int oy = tile / tpo, cb = (tile - oy * tpo) * kRows;
            uint32_t* out = pick_out(outs, oy);
            // the launcher requires the addends to be consecutive out_bits-wide polynomials
            const uint32_t* addp = fin.add[0] ? fin.add[0] + (size_t)oy * ((out_bits + 31) >> 5) * N : nullptr;
            const int i = cb + n;
            uint32_t* const outi = out + i;
            if (h == 0) {
                carry = 0;
                prev = 0;
                amb = false;
                c2 = 0;
                prev2 = 0;
            } else {
                const int sl = 1 - grp;
                PWAIT(0, smem_u32(&bar_hand_full[sl]), nrd & 1);
                const uint4 hv = s_hand[sl][n];
                const uint2 hv2 = s_hand2[sl][n];
                __syncwarp();
                if (lane == 0) mbar_arrive(smem_u32(&bar_hand_empty[sl]));
                ++nrd;
                carry = ((uint64_t)hv.y << 32) | hv.x;
                prev = hv.z;
                amb = hv.w != 0;
                c2 = hv2.x;
                prev2 = hv2.y;
            }
            const int tb = ij & 1;
            const int c0 = tb0 + h * jc;
            const int ncols = job_cols(h);
            // the job's addend words (output word u = c0 + k - sw - (sbit != 0)), loaded before
            // the accumulator wait so their latency is off the carry chain
            const uint32_t* av = s_add + tb * (kAddStage / 4) + n;   // addend word k at av[k * 128]
            if (FUSED) PWAIT(1, smem_u32(&bar_add_full[tb]), (ij >> 1) & 1);
            PWAIT(2, smem_u32(&bar_tm_full[tb]), (ij >> 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;\n");
            const uint32_t lane_addr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(tb * 256);
            // steps [fast_lo, fast_hi] (first column of an 8-word step) take the interior path:
            // window words u = t - sw - ush in [max(0, rw2 + 1), out_w - 2] (no top-word mask, no
            // rescale rounding bit), past the key switch's rounding column, and fused output
            // words v = u - rw - vsh in [0, out2_w - 2]
            int fast_lo = sw + ush + (rw2 + 1 > 0 ? rw2 + 1 : 0);
            if (shift > 0 && fast_lo <= round_col) fast_lo = round_col + 1;
            int fast_hi = out_w - 2 + sw + ush - 7;
            if (FUSED) {
                if (fast_lo < sw + ush + rw + vsh) fast_lo = sw + ush + rw + vsh;
                const int hi2 = out2_w - 2 + rw + vsh + sw + ush - 7;
                if (fast_hi > hi2) fast_hi = hi2;
            }
            const int fast_v0 = sw + ush + rw + vsh;   // column of output word v = 0 (fused)
#ifdef HG_CRT_WIDE_FOLD
            // digit weights the compiler cannot see through: one IMAD.WIDE per digit instead of
            // the shift / high-shift / add-with-carry sequence (N < 2^31, so the term is 0)
            const uint32_t kz = (uint32_t)(N >> 31);
            const uint32_t k8 = 256u + kz, k16 = (1u << 16) + kz, k24 = (1u << 24) + kz;
#else
            constexpr uint32_t k8 = 256u, k16 = 1u << 16, k24 = 1u << 24;
#endif
#ifdef HG_CRT_PROF
            const long long t_loop = clock64();
#endif
            for (int tl = 0; tl < ncols; tl += 8) {
                uint32_t e[32];
#ifdef HG_CRT_PROF
                const long long t_ld = clock64();
#endif
                asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                             "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
                             : "=r"(e[0]), "=r"(e[1]), "=r"(e[2]), "=r"(e[3]), "=r"(e[4]), "=r"(e[5]),
                               "=r"(e[6]), "=r"(e[7]), "=r"(e[8]), "=r"(e[9]), "=r"(e[10]), "=r"(e[11]),
                               "=r"(e[12]), "=r"(e[13]), "=r"(e[14]), "=r"(e[15]), "=r"(e[16]), "=r"(e[17]),
                               "=r"(e[18]), "=r"(e[19]), "=r"(e[20]), "=r"(e[21]), "=r"(e[22]), "=r"(e[23]),
                               "=r"(e[24]), "=r"(e[25]), "=r"(e[26]), "=r"(e[27]), "=r"(e[28]), "=r"(e[29]),
                               "=r"(e[30]), "=r"(e[31])
                             : "r"(lane_addr + (uint32_t)(tl * 4)));
                asm volatile("tcgen05.wait::ld.sync.aligned;\n");
#ifdef HG_CRT_PROF
                prof[4] += (unsigned long long)(clock64() - t_ld);
#endif
                // the eight words' digit sums first (independent of the carry), then the short
                // carry chain, then emission: word value = D0 + D1 2^8 + D2 2^16 + D3 2^24 < 2^51
                // (the packed layout already carries the previous word's high digits);
                // columns past T (padding of the last job) only disturb the dead carry
                uint64_t val[8];
#pragma unroll
                for (int hh = 0; hh < 8; ++hh) {
                    const uint32_t* E = e + 4 * hh;
                    val[hh] = madw(E[3], k24, madw(E[2], k16, madw(E[1], k8, (uint64_t)E[0])));
                }
                uint32_t wv[8];
                const int t0 = c0 + tl;
                if (t0 >= fast_lo && t0 <= fast_hi) {
                    // interior step: every word is a full (unmasked) window word past the rounding
                    // column and, fused, a full output word past the rescale's rounding bit --
                    // no per-word predicates, pointer-stepped stores
#pragma unroll
                    for (int hh = 0; hh < 8; ++hh) {
                        const uint64_t x = val[hh] + carry;
                        wv[hh] = (uint32_t)x;
                        carry = x >> 32;
                    }
                    if (FUSED) {
                        uint32_t* op = outi + (size_t)(t0 - fast_v0) * N;
                        const uint32_t* ap = av + tl * kRows;
#pragma unroll
                        for (int hh = 0; hh < 8; ++hh) {
                            const uint32_t o = sbit ? __funnelshift_r(prev, wv[hh], sbit) : wv[hh];
                            prev = wv[hh];
                            const uint64_t sum = (uint64_t)o + ap[hh * kRows] + c2;
                            const uint32_t w = (uint32_t)sum;
                            c2 = (uint32_t)(sum >> 32);
                            op[(size_t)hh * N] = rb ? __funnelshift_r(prev2, w, rb) : w;
                            prev2 = w;
                        }
                    } else {
                        uint32_t* op = outi + (size_t)(t0 - sw - ush) * N;
                        if (sbit) {
#pragma unroll
                            for (int hh = 0; hh < 8; ++hh) {
                                op[(size_t)hh * N] = __funnelshift_r(prev, wv[hh], sbit);
                                prev = wv[hh];
                            }
                        } else {
#pragma unroll
                            for (int hh = 0; hh < 8; ++hh) op[(size_t)hh * N] = wv[hh];
                            prev = wv[7];
                        }
                    }
                    continue;
                }
#pragma unroll
                for (int hh = 0; hh < 8; ++hh) {
                    const uint64_t x = val[hh] + carry + (c0 + tl + hh == round_col ? round_bit : 0u);
                    wv[hh] = (uint32_t)x;
                    carry = x >> 32;
                }
                // emission, predicated rather than branched (every condition is warp-uniform):
                // window word u = t - sw - (sbit != 0) is valid for 0 <= u < out_w (so t < T)
#pragma unroll
                for (int hh = 0; hh < 8; ++hh) {
                    const int t = c0 + tl + hh;
                    const uint32_t word = wv[hh];
                    if (t < sw) {   // below the window: the truncated-column ambiguity flag
                        if (t == tb0 + 1) amb = word >= 0xFFFFFF00u;
                        else if (t > tb0 + 1) amb = amb && (word == 0xffffffffu);
                    }
                    const int u = t - sw - ush;
                    const uint32_t o = sbit ? __funnelshift_r(prev, word, sbit) : word;
                    prev = word;
                    if (u >= 0 && u < out_w) {
                        const uint32_t mu = u == out_w - 1 ? top_l : 0xffffffffu;
                        if (FUSED) {
                            const uint64_t sum = (uint64_t)(o & mu) + av[(tl + hh) * kRows] + c2 +
                                                 (u == rw2 ? rbit2 : 0u);
                            const uint32_t w = (uint32_t)sum & mu;
                            c2 = (uint32_t)(sum >> 32);
                            const int v = u - rw - vsh;
                            const uint32_t ov = rb ? __funnelshift_r(prev2, w, rb) : w;
                            prev2 = w;
                            if (v >= 0 && v < out2_w) outi[(size_t)v * N] = ov & (v == out2_w - 1 ? top2 : 0xffffffffu);
                        } else {
                            outi[(size_t)u * N] = o & mu;
                        }
                    }
                }
            }
            if (FUSED) {
                __syncwarp();
                if (lane == 0) mbar_arrive(smem_u32(&bar_add_empty[tb]));
            }
#ifdef HG_CRT_PROF
            const long long t_post = clock64();
            prof[6] += (unsigned long long)(t_post - t_loop);
#endif
            if (FUSED && h == jpt - 1 && rb) {   // the last output word: the top bits of prev2
                const int v = out_w - 1 - rw;
                if (v >= 0 && v < out2_w) outi[(size_t)v * N] = (prev2 >> rb) & (v == out2_w - 1 ? top2 : 0xffffffffu);
            }
            asm volatile("tcgen05.fence::before_thread_sync;\n");
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&bar_tm_empty[tb]));
            if (h < jpt - 1) {
                PWAIT(3, smem_u32(&bar_hand_empty[grp]), (nwr & 1) ^ 1);
                s_hand[grp][n] = make_uint4((uint32_t)carry, (uint32_t)(carry >> 32), prev, amb ? 1u : 0u);
                if (FUSED) s_hand2[grp][n] = make_uint2(c2, prev2);
                __syncwarp();
                if (lane == 0) mbar_arrive(smem_u32(&bar_hand_full[grp]));
                ++nwr;
            }
#ifdef HG_CRT_PROF
            prof[7] += (unsigned long long)(clock64() - t_post);
#endif
            if (h == jpt - 1 && tb0 > 0 && amb) {
                Emitter fresh;
                fresh.init(out, N, i, out_bits, fin, FUSED ? addp : nullptr);
                pipe_rescan_exact(res + (size_t)oy * P * N, P, N, W, pinfo, cinv, cinv_sh, invp, Mtab,
                                  negQ, shift, out_bits, PRESCALED, fresh);
            }
        }
    }
#ifdef HG_CRT_PROF
    prof[5] = (unsigned long long)(clock64() - t_start);
    if (lane == 0 && blockIdx.x < 160)
        for (int c = 0; c < 8; ++c) g_crt_prof[blockIdx.x][warp][c] = prof[c];
#endif
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(512));
}

}  // namespace

// true when the pipelined kernel covers this window
bool hg_crt_umma_pipe_ok(const CrtTable* tab, int N, int shift, int out_bits, int tb0) {
    const int sw = shift >> 5, sbit = shift & 31;
    const int T = sw + (out_bits + 31) / 32 + (sbit ? 1 : 0);
    const int ncols = ((T - tb0) + 1) & ~1;
    return tab->d_Bpipe && N % kRows == 0 && ncols >= 2 && (tb0 & 7) == 0 &&
           tb0 + 8 * ((ncols + 7) >> 3) <= tab->W && tab->P32p + 32 <= HG_MAX_PRIMES + 32;
}

int hg_crt_umma_pipe_launch(hg_ctx* ctx, const CrtTable* tab, const uint32_t* res, int nouts, int P,
                            int shift, int out_bits, int tb0, uint32_t* const* outs_in,
                            cudaStream_t st, const CrtFinish* finish, bool prescaled) {
    static std::atomic<uint64_t> attr_set{0};
    const int nsm = ctx->nsm;
    using Kern = void (*)(const CUtensorMap, const CUtensorMap, const uint32_t*, int, int, int, int, const PrimeInfo*,
                          const uint8_t*, const uint32_t*, int, const uint32_t*, const uint32_t*, const uint32_t*,
                          const double*, int, int, int, UOuts, CrtFinish);
    // [log_n class: run-time N, 2^16, 2^17][fused finish][prescaled]
    static const Kern kerns[3][2][2] = {
        {{crt_umma_pipe_kernel<false, false, 0>, crt_umma_pipe_kernel<false, true, 0>},
         {crt_umma_pipe_kernel<true, false, 0>, crt_umma_pipe_kernel<true, true, 0>}},
        {{crt_umma_pipe_kernel<false, false, 16>, crt_umma_pipe_kernel<false, true, 16>},
         {crt_umma_pipe_kernel<true, false, 16>, crt_umma_pipe_kernel<true, true, 16>}},
        {{crt_umma_pipe_kernel<false, false, 17>, crt_umma_pipe_kernel<false, true, 17>},
         {crt_umma_pipe_kernel<true, false, 17>, crt_umma_pipe_kernel<true, true, 17>}}};
    if (hg_first_on_device(attr_set, ctx->device)) {
        for (int a = 0; a < 3; ++a)
            for (int c = 0; c < 2; ++c) {
                HG_CUDA_TRY(cudaFuncSetAttribute(kerns[a][0][c], cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)pipe_smem<false>()));
                HG_CUDA_TRY(cudaFuncSetAttribute(kerns[a][1][c], cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)pipe_smem<true>()));
            }
    }
    const int lc = ctx->log_n == 17 ? 2 : (ctx->log_n == 16 ? 1 : 0);
    UOuts o{};
    for (int k = 0; k < nouts; ++k) o.out[k] = outs_in[k];
    const int ntiles = nouts * (ctx->N / kRows);
    const int grid = ntiles < nsm ? ntiles : nsm;
    CUtensorMap res_map, add_map;
    if (int rc = hg_tmap_2d_u32(&res_map, res, (uint64_t)ctx->N, (uint64_t)nouts * P, kRows, 32)) return rc;
    const CrtFinish fin = finish ? *finish : CrtFinish{};
    const bool fused = finish != nullptr;
    if (fused) {
        // the addends are nouts consecutive out_bits-wide polynomials starting at add[0]
        const int out_w = (out_bits + 31) / 32;
        for (int k = 0; k < nouts; ++k)
            if (fin.kinv != 0 || fin.add[k] != fin.add[0] + (size_t)k * out_w * ctx->N)
                return hg_fail(HG_EINVAL, "fused CRT finish: addends must be consecutive, no automorphism");
        if (int rc = hg_tmap_2d_u32(&add_map, fin.add[0], (uint64_t)ctx->N, (uint64_t)nouts * out_w, kRows,
                                    kJobCols))
            return rc;
        const Kern kern = kerns[lc][1][prescaled ? 1 : 0];
        kern<<<grid, PipeCfg<true>::kWarps * 32, pipe_smem<true>(), st>>>(
            res_map, add_map, res, P, tab->P32p, ctx->N, nouts, ctx->d_pinfo, tab->d_Bpipe, tab->d_M, tab->W,
            tab->d_negQ, tab->d_cinv, tab->d_cinv_sh, tab->d_invp, shift, out_bits, tb0, o, fin);
    } else {
        const Kern kern = kerns[lc][0][prescaled ? 1 : 0];
        kern<<<grid, PipeCfg<false>::kWarps * 32, pipe_smem<false>(), st>>>(
            res_map, res_map, res, P, tab->P32p, ctx->N, nouts, ctx->d_pinfo, tab->d_Bpipe, tab->d_M, tab->W,
            tab->d_negQ, tab->d_cinv, tab->d_cinv_sh, tab->d_invp, shift, out_bits, tb0, o, fin);
    }
    HG_LAUNCH_CHECK(ctx);
    return HG_OK;
}

// B in the digit layout, pre-arranged as the exact shared-memory image the kernel copies:
// [K chunk kc (32 primes)][8-column group tg][row group t (8 rows: digits s)][16-byte K chunk c]
// [row s][16 bytes]; byte 4jj+q of row (t,s) = byte (s-q) of M[32kc+4c+jj][t] (0 if out of 0..3).
int hg_crt_build_conv(const CrtTable& t, int P, int P32, std::vector<uint8_t>& out,
                      const std::vector<uint32_t>& M) {
    const int W = t.W, nkc = P32 / 32, ntg = W / 8;
    out.assign((size_t)nkc * ntg * 8192, 0);
    for (int kc = 0; kc < nkc; ++kc)
        for (int tg = 0; tg < ntg; ++tg)
            for (int tl = 0; tl < 8; ++tl) {
                const int col = tg * 8 + tl;
                for (int c = 0; c < 8; ++c)
                    for (int s = 0; s < 8; ++s)
                        for (int jj = 0; jj < 4; ++jj)
                            for (int q = 0; q < 4; ++q) {
                                const int j = kc * 32 + c * 4 + jj;
                                const int rbyte = s - q;
                                uint8_t val = 0;
                                if (j < P && rbyte >= 0 && rbyte < 4)
                                    val = (uint8_t)(M[(size_t)j * W + col] >> (8 * rbyte));
                                const size_t off = ((size_t)kc * ntg + tg) * 8192 +
                                                   ((size_t)(tl * 8 + c) * 8 + s) * 16 + jj * 4 + q;
                                out[off] = val;
                            }
            }
    return HG_OK;
}

// B in the PACKED digit layout of the pipelined kernel: 4 TMEM columns per output word.  Byte
// q of y_j times byte r of word t of M_j lands at bit 32t + 8(q + r): digit q + r of word t when
// q + r < 4, else digit q + r - 4 of word t + 1.  So column (word T, digit s) gathers
//     B[(j, q), (T, s)] = byte (s - q) of M[j][T]          (s >= q)
//                         byte (s - q + 4) of M[j][T - 1]  (s <  q)
// -- every (K row, column) entry is live (the 8-column layout above is half zeros), and the
// epilogue folds 4 digits (< 2^27 each) per word instead of 7.  Image: [K chunk kc][8-word group
// tg][row group rg (8 N-rows = words 2rg, 2rg+1 x digits 0-3)][16-byte K chunk c][row][16 bytes];
// 4096 bytes per (kc, tg).
int hg_crt_build_pack4(const CrtTable& t, int P, int P32, std::vector<uint8_t>& out,
                       const std::vector<uint32_t>& M) {
    const int W = t.W, nkc = P32 / 32, ntg = W / 8;
    out.assign((size_t)nkc * ntg * 4096, 0);
    for (int kc = 0; kc < nkc; ++kc)
        for (int tg = 0; tg < ntg; ++tg)
            for (int rg = 0; rg < 4; ++rg)
                for (int c = 0; c < 8; ++c)
                    for (int rr = 0; rr < 8; ++rr) {
                        const int T = tg * 8 + rg * 2 + (rr >> 2), sd = rr & 3;
                        for (int jj = 0; jj < 4; ++jj)
                            for (int q = 0; q < 4; ++q) {
                                const int j = kc * 32 + c * 4 + jj;
                                const int word = sd >= q ? T : T - 1;
                                const int byte = sd >= q ? sd - q : sd - q + 4;
                                uint8_t val = 0;
                                if (j < P && word >= 0)
                                    val = (uint8_t)(M[(size_t)j * W + word] >> (8 * byte));
                                const size_t off = ((size_t)kc * ntg + tg) * 4096 +
                                                   ((size_t)(rg * 8 + c) * 8 + rr) * 16 + jj * 4 + q;
                                out[off] = val;
                            }
                    }
    return HG_OK;
}

size_t hg_crt_umma_smem(int P32) { return (size_t)kRows * 4 * P32 + 2 * (size_t)kBStage; }

int hg_crt_umma_launch(hg_ctx* ctx, const CrtTable* tab, const uint32_t* res, int nouts, int P,
                       int shift, int out_bits, int tb0, uint32_t* const* outs_in, cudaStream_t st) {
    const size_t smem = hg_crt_umma_smem(tab->P32);
    static std::atomic<uint64_t> attr_set{0};
    if (hg_first_on_device(attr_set, ctx->device)) {
        // 227 KB per block includes the kernel's static shared variables
        HG_CUDA_TRY(cudaFuncSetAttribute(crt_umma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         220 * 1024));
    }
    UOuts o{};
    for (int k = 0; k < nouts; ++k) o.out[k] = outs_in[k];
    dim3 grid(ctx->N / kRows, nouts);
    if (int rc = hg_crt_ensure_fallback(ctx, tab)) return rc;
    crt_umma_kernel<<<grid, 2 * kRows, smem, st>>>(res, P, tab->P32, ctx->N, ctx->d_pinfo, tab->d_Bconv,
                                               tab->d_M, tab->W, tab->d_negQ, tab->d_cinv,
                                               tab->d_cinv_sh, tab->d_invp, shift, out_bits, tb0, o);
    HG_LAUNCH_CHECK(ctx);
    return HG_OK;
}

#ifdef HG_CRT_PROF
// copies the wait-cycle table of the last pipelined CRT launch: [160][20][6] u64
extern "C" int hg_crt_prof_read(unsigned long long* out) {
    return cudaMemcpyFromSymbol(out, g_crt_prof, sizeof(g_crt_prof)) == cudaSuccess ? 0 : 1;
}
#endif
