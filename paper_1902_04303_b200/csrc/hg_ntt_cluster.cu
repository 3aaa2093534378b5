// hg_ntt_cluster.cu -- length-2^17 negacyclic NTT / inverse NTT in ONE HBM round trip: a
// thread-block cluster of 8 CTAs owns one transform (512 KB), exchanging it once through
// distributed shared memory (DSMEM) instead of a second pass through HBM.
//
// N = 2^17 = 64 rows x 2048 columns (row r = words [2048 r, 2048 r + 2048)).  The 6 strided
// ("hi") stages act on columns, the 11 contiguous ("lo") stages on rows (same merged
// Cooley-Tukey / Gentleman-Sande butterflies, twiddle indices and lazy ranges as hg_ntt.cu,
// so the outputs are the same residues).
//   forward:  CTA k loads columns [256k, 256k+256) (thread t = one column, its 64 words in
//             registers, coalesced row by row) and runs the 6 hi stages in registers; the
//             column values are stored straight into the shared memory of the CTA that owns
//             their row (rows [8c, 8c+8) belong to CTA c; st.shared::cluster); after one
//             cluster barrier every warp owns one row: 6 lo stages with lane l holding words
//             l + 32m, one warp-private shared-memory exchange, 5 stages with lane l holding
//             words [64l, 64l+64), then the row goes back to HBM coalesced.
//   inverse:  the mirror image (rows first, one DSMEM exchange, columns last).  The NTT-domain
//             products of hg_ntt.cu's fused inverse (key switch, tensor, plain, shared factor)
//             are computed as the rows are loaded; with several outputs the CTA computes
//             every product once, stashes outputs 1.. as raw rows of the output (the same
//             thread reads them back), and transforms the outputs one after another.  Inputs
//             may alias outputs row for row (in-place use), as in hg_ntt.cu.
// Shared memory: 64 KB per CTA (8 rows x 2048 words, XOR-swizzled so both lane layouts are
// conflict-free; the inverse exchange reuses it as 64 rows x 256 columns), 2 CTAs per SM.
// Round-B twiddles (lane-dependent) come from a transposed per-prime table (d_twc_*) so each
// warp load is one coalesced 256-byte line; every other twiddle is warp- or CTA-uniform.
//
// Measured (tools/ntt_bench.py, 656 rows = 4 x 164 primes, same box): forward 0.789 us/row vs
// 0.557 for the two passes, inverse 0.649 vs 0.525 -- HBM bytes halve (ncu: 516 MB read / 311 MB
// written vs 860 / 580), instructions per butterfly drop (8.3 vs 10.3), but 128 registers per
// thread leave 16 warps per SM (33 clusters resident) and the load -> compute -> exchange ->
// compute -> store phases of a CTA do not overlap: warps active 22%, FMA pipe 34%, long-
// scoreboard stalls on the lo-phase twiddles 53% of samples.  With no twiddle loads at all
// (HG_FAKE_TW timing build) it still runs 0.615 us/row.  So the two-pass kernels stay the
// default (hg_set_ntt_variant / HG_NTT_CLUSTER=1 select this path; tests keep it bit-exact).
#include "hg_ntt_common.cuh"

#include <chrono>

namespace {

constexpr int kCS = 8;                 // CTAs per cluster
constexpr int kRowW = 2048;            // words per row
constexpr int kNRows = 64;             // rows per transform
constexpr int kN = kRowW * kNRows;     // 2^17
constexpr int kTwcRow = 1984;          // transposed round-B twiddles per row: 32 (2+4+8+16+32)
constexpr size_t kSmemBytes = (size_t)kNRows * (kRowW / kCS) * 4;   // 64 KB

using hgntt::fwd_bfly;
using hgntt::inv_bfly;
using hgntt::stage64;
using hgntt::hi_stages;

// position of word q of a row inside its 2048-word shared-memory row: bits 0-4 ^= bits 6-10
__device__ __forceinline__ int swz(int q) { return q ^ ((q >> 6) & 31); }

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint32_t map_rank(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_cluster(uint32_t addr, uint32_t v) {
    asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void cluster_arrive_relaxed() {
    asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_arrive() {
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// round A: lo stages ls = 0..5 of row G - 64 with lane l holding words q = l + 32 m (x[m]);
// twiddle psi_rev[G 2^ls + (m >> (6 - ls))] is warp-uniform
template <bool FWD>
__device__ __forceinline__ void lo_round_a(uint32_t (&x)[64], const uint2* __restrict__ twp,
                                           int G, uint32_t p) {
    if (FWD) {
        stage64<true, 32, 1>(x, twp + G, p);
        stage64<true, 16, 1>(x, twp + (G << 1), p);
        stage64<true, 8, 1>(x, twp + (G << 2), p);
        stage64<true, 4, 1>(x, twp + (G << 3), p);
        stage64<true, 2, 1>(x, twp + (G << 4), p);
        stage64<true, 1, 1>(x, twp + (G << 5), p);
    } else {
        stage64<false, 1, 1>(x, twp + (G << 5), p);
        stage64<false, 2, 1>(x, twp + (G << 4), p);
        stage64<false, 4, 1>(x, twp + (G << 3), p);
        stage64<false, 8, 1>(x, twp + (G << 2), p);
        stage64<false, 16, 1>(x, twp + (G << 1), p);
        stage64<false, 32, 1>(x, twp + G, p);
    }
}

// round B: lo stages ls = 6..10 with lane l holding words q = 64 l + m (x[m]); twiddle
// psi_rev[G 2^ls + l 2^(ls-5) + (m >> (11 - ls))] = twc[32 (2^(ls-5) - 2) + 32 kk + l] of the
// transposed table (twc already points at lane l of the row)
template <bool FWD>
__device__ __forceinline__ void lo_round_b(uint32_t (&x)[64], const uint2* __restrict__ twc,
                                           uint32_t p) {
    if (FWD) {
        stage64<true, 16, 32>(x, twc, p);
        stage64<true, 8, 32>(x, twc + 64, p);
        stage64<true, 4, 32>(x, twc + 192, p);
        stage64<true, 2, 32>(x, twc + 448, p);
        stage64<true, 1, 32>(x, twc + 960, p);
    } else {
        stage64<false, 1, 32>(x, twc + 960, p);
        stage64<false, 2, 32>(x, twc + 448, p);
        stage64<false, 4, 32>(x, twc + 192, p);
        stage64<false, 8, 32>(x, twc + 64, p);
        stage64<false, 16, 32>(x, twc, p);
    }
}

// rows [B][P][N]; grid (8, B, P); row (bb, jp) uses prime prime_offset + jp
__global__ void __cluster_dims__(kCS, 1, 1) __launch_bounds__(256, 2)
ntt_fwd_c8_kernel(uint32_t* __restrict__ data, int P, int prime_offset,
                  const PrimeInfo* __restrict__ pinfo, const uint2* __restrict__ tw,
                  const uint2* __restrict__ twc) {
    extern __shared__ __align__(16) uint32_t sm[];
    cluster_arrive_relaxed();   // matched by the wait before the first remote store
    const int k = blockIdx.x;
    const int jp = blockIdx.z, bb = blockIdx.y;
    const int prime = prime_offset + jp;
    const uint32_t p = pinfo[prime].p;
    const uint2* twp = tw + (size_t)prime * kN;
    uint32_t* rowp = data + ((size_t)bb * P + jp) * kN;
    const int t = threadIdx.x;
    uint32_t x[64];

    // hi: column c = 256 k + t
    const int c = (k << 8) + t;
#pragma unroll
    for (int r = 0; r < 64; ++r) x[r] = rowp[r * kRowW + c];
    hi_stages<true>(x, twp, p);
    cluster_wait();
    {
        const uint32_t base = smem_u32(sm) + 4u * (uint32_t)swz(c);
#pragma unroll
        for (int dst = 0; dst < kCS; ++dst) {
            const uint32_t rb = map_rank(base, dst);
#pragma unroll
            for (int lr = 0; lr < 8; ++lr) st_cluster(rb + 4u * (uint32_t)(lr * kRowW), x[dst * 8 + lr]);
        }
    }
    cluster_arrive();
    cluster_wait();

    // lo: warp w owns row 8k + w
    const int w = t >> 5, l = t & 31;
    uint32_t* srow = sm + w * kRowW;
    const int r = 8 * k + w;
    const int G = kNRows + r;
#pragma unroll
    for (int m = 0; m < 64; ++m) x[m] = srow[swz(l + 32 * m)];
    lo_round_a<true>(x, twp, G, p);
#pragma unroll
    for (int m = 0; m < 64; ++m) srow[swz(l + 32 * m)] = x[m];
    __syncwarp();
#pragma unroll
    for (int m = 0; m < 64; ++m) x[m] = srow[swz(64 * l + m)];
    lo_round_b<true>(x, twc + (size_t)prime * (kNRows * kTwcRow) + (size_t)r * kTwcRow + l, p);
#pragma unroll
    for (int m = 0; m < 64; ++m) srow[swz(64 * l + m)] = x[m];
    __syncwarp();
    uint32_t* orow = rowp + (size_t)r * kRowW;
#pragma unroll
    for (int m = 0; m < 64; ++m) orow[hgntt::ntt_pos(l + 32 * m)] = srow[swz(l + 32 * m)];
}

// Inverse.  PRE 0: plain, rows [B][P][N] in place (grid (8, B, P), prime prime_offset + jp).
// PRE 1 (key switch): outs (x kb, x ka); PRE 2 (tensor): (a0b0, a0b1 + a1b0, a1b1);
// PRE 3: a b; PRE 5: x b -- as intt_lo8_fused_kernel (hg_ntt.cu), grid (8, batch, P),
// prime jp, in0 / out advanced by blockIdx.y * bstride_in / bstride_out.
template <int PRE>
struct InvOuts { static constexpr int value = PRE == 1 ? 2 : (PRE == 2 ? 3 : 1); };

template <int PRE>
__global__ void __cluster_dims__(kCS, 1, 1) __launch_bounds__(256, 2)
ntt_inv_c8_kernel(uint32_t* out, const uint32_t* in0, const uint32_t* in1, const uint32_t* in2,
                  const uint32_t* in3, int P, int prime_offset, const PrimeInfo* __restrict__ pinfo,
                  const uint2* __restrict__ tw, const uint2* __restrict__ twc, size_t bstride_in,
                  size_t bstride_out) {
    extern __shared__ __align__(16) uint32_t sm[];
    constexpr int RB = InvOuts<PRE>::value;
    const int k = blockIdx.x;
    const int jp = blockIdx.z;
    int prime;
    size_t plane;   // words between output rows
    if (PRE == 0) {
        prime = prime_offset + jp;
        out += ((size_t)blockIdx.y * P + jp) * kN;
        plane = 0;
    } else {
        prime = jp;
        out += blockIdx.y * bstride_out + (size_t)jp * kN;
        in0 += blockIdx.y * bstride_in + (size_t)jp * kN;
        in1 += (size_t)jp * kN;
        if (PRE == 1 || PRE == 2) in2 += (size_t)jp * kN;
        if (PRE == 2) in3 += (size_t)jp * kN;
        plane = (size_t)P * kN;
    }
    const PrimeInfo pi = pinfo[prime];
    const uint32_t p = pi.p, p2 = p << 1;
    const uint2* twp = tw + (size_t)prime * kN;
    const int t = threadIdx.x;
    const int w = t >> 5, l = t & 31;
    const int r = 8 * k + w;
    const int G = kNRows + r;
    const uint2* twc_row = twc + (size_t)prime * (kNRows * kTwcRow) + (size_t)r * kTwcRow + l;
    uint32_t* srow = sm + w * kRowW;
    // NTT-domain words in the transposed storage order (ntt_pos): word l + 32 m of row r
    const size_t roff = (size_t)r * kRowW;
    auto qi = [&](int m) { return roff + (size_t)hgntt::ntt_pos(l + 32 * m); };
    uint32_t x[64];

#pragma unroll 1
    for (int o = 0; o < RB; ++o) {
        uint32_t* orow = out + o * plane;
        // ---- load the row in lane layout q = l + 32 m (products computed here) --------------
        if (o == 0) {
            if (PRE == 0) {
#pragma unroll
                for (int m = 0; m < 64; ++m) x[m] = orow[qi(m)];
            } else {
#pragma unroll
                for (int m = 0; m < 64; ++m) {
                    const size_t q = qi(m);
                    const uint32_t u0 = in0[q];
                    const uint32_t a = min(u0, u0 - p2);
                    if (PRE == 1) {
                        x[m] = mont_mul(a, in1[q], p, pi.pinv_neg);
                        out[plane + q] = mont_mul(a, in2[q], p, pi.pinv_neg);   // raw, output 1
                    } else if (PRE == 2) {
                        const uint32_t u1 = in1[q], u2 = in2[q], u3 = in3[q];
                        const uint32_t a1 = min(u1, u1 - p2);
                        const uint32_t b0 = min(u2, u2 - p2);
                        const uint32_t b1 = min(u3, u3 - p2);
                        x[m] = mont_mul(a, b0, p, pi.pinv_neg);
                        const uint32_t d1 = mont_mul(a, b1, p, pi.pinv_neg) + mont_mul(a1, b0, p, pi.pinv_neg);
                        out[plane + q] = min(d1, d1 - p2);
                        out[2 * plane + q] = mont_mul(a1, b1, p, pi.pinv_neg);
                    } else if (PRE == 5) {
                        x[m] = mont_mul(a, in1[q], p, pi.pinv_neg);
                    } else {
                        const uint32_t u1 = in1[q];
                        x[m] = mont_mul(a, min(u1, u1 - p2), p, pi.pinv_neg);
                    }
                }
            }
        } else {
            // raw product rows stashed by this same thread in pass 0
#pragma unroll
            for (int m = 0; m < 64; ++m) x[m] = orow[qi(m)];
            __syncthreads();   // the previous output's column reads of sm are done
        }
        // ---- rows: round B (distances 1..16) then round A (32..1024) ------------------------
#pragma unroll
        for (int m = 0; m < 64; ++m) srow[swz(l + 32 * m)] = x[m];
        __syncwarp();
#pragma unroll
        for (int m = 0; m < 64; ++m) x[m] = srow[swz(64 * l + m)];
        lo_round_b<false>(x, twc_row, p);
#pragma unroll
        for (int m = 0; m < 64; ++m) srow[swz(64 * l + m)] = x[m];
        __syncwarp();
#pragma unroll
        for (int m = 0; m < 64; ++m) x[m] = srow[swz(l + 32 * m)];
        lo_round_a<false>(x, twp, G, p);
        // ---- exchange: word q = l + 32 m of row r -> CTA q >> 8, column q & 255 -------------
        cluster_arrive();   // this CTA's row reads of sm are done (all in registers)
        cluster_wait();     // ... and every other CTA's
        {
            const uint32_t base = smem_u32(sm) + 4u * (uint32_t)(r * 256 + l);
#pragma unroll
            for (int dst = 0; dst < kCS; ++dst) {
                const uint32_t rb = map_rank(base, dst);
#pragma unroll
                for (int mm = 0; mm < 8; ++mm) st_cluster(rb + 4u * (uint32_t)(32 * mm), x[dst * 8 + mm]);
            }
        }
        cluster_arrive();
        cluster_wait();
        // ---- columns: thread t = column 256 k + t ----------------------------------------------
#pragma unroll
        for (int rr = 0; rr < 64; ++rr) x[rr] = sm[rr * 256 + t];
        hi_stages<false>(x, twp, p);
        uint32_t* col = orow + (k << 8) + t;
#pragma unroll
        for (int rr = 0; rr < 64; ++rr) col[(size_t)rr * kRowW] = x[rr];
    }
}

// transposed round-B twiddles: twc[j][r][32 (2^(ls-5) - 2) + 32 kk + l] = tw[j][(64 + r) 2^ls
// + l 2^(ls-5) + kk], ls = 6..10
__global__ void twc_kernel(uint2* __restrict__ dst, const uint2* __restrict__ src) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;   // 0 .. 64 * 1984
    if (e >= kNRows * kTwcRow) return;
    const int j = blockIdx.y;
    const int r = e / kTwcRow, f = e % kTwcRow;
    int ls = 6;
    while (ls < 10 && f >= 32 * ((1 << (ls - 4)) - 2)) ++ls;
    const int g = f - 32 * ((1 << (ls - 5)) - 2);
    const int kk = g >> 5, l = g & 31;
    dst[(size_t)j * kNRows * kTwcRow + e] =
        src[(size_t)j * kN + ((size_t)(kNRows + r) << ls) + ((size_t)l << (ls - 5)) + kk];
}

std::atomic<uint64_t> g_attr_seen{0};

int ensure_attrs(hg_ctx* ctx) {
    if (!hg_first_on_device(g_attr_seen, ctx->device)) return HG_OK;
    HG_CUDA_TRY(cudaFuncSetAttribute(ntt_fwd_c8_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes));
    HG_CUDA_TRY(cudaFuncSetAttribute(ntt_inv_c8_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes));
    HG_CUDA_TRY(cudaFuncSetAttribute(ntt_inv_c8_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes));
    HG_CUDA_TRY(cudaFuncSetAttribute(ntt_inv_c8_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes));
    HG_CUDA_TRY(cudaFuncSetAttribute(ntt_inv_c8_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes));
    HG_CUDA_TRY(cudaFuncSetAttribute(ntt_inv_c8_kernel<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes));
    return HG_OK;
}

// the transposed tables for every prime (both directions), built once from d_tw_*
int ensure_twc(hg_ctx* ctx) {
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (ctx->d_twc_fwd) return HG_OK;
    const size_t per = (size_t)kNRows * kTwcRow;
    const size_t bytes = per * ctx->nprimes * sizeof(uint2);
    uint2 *f = nullptr, *i = nullptr;
    if (cudaMalloc(&f, bytes) != cudaSuccess) {
        cudaGetLastError();
        return hg_fail(HG_ENOMEM, "cluster NTT twiddle table");
    }
    if (cudaMalloc(&i, bytes) != cudaSuccess) {
        cudaGetLastError();
        cudaFree(f);
        return hg_fail(HG_ENOMEM, "cluster NTT twiddle table");
    }
    const dim3 g((unsigned)((per + 255) / 256), ctx->nprimes);
    twc_kernel<<<g, 256>>>(f, ctx->d_tw_fwd);
    twc_kernel<<<g, 256>>>(i, ctx->d_tw_inv);
    HG_CUDA_TRY(cudaGetLastError());
    HG_CUDA_TRY(cudaDeviceSynchronize());
    ctx->d_twc_fwd = f;
    ctx->d_twc_inv = i;
    return HG_OK;
}

}  // namespace

bool hg_ntt_cluster_ok(const hg_ctx* ctx, int P) {
    return ctx->log_n == 17 && P <= 65535 && ctx->ntt_cluster == 1;
}

// NTT variant: 0 = the two-pass kernels of hg_ntt.cu, 1 = this file's DSMEM cluster kernels
// (log_n = 17), 2 = hg_ntt.cu's one-launch cluster kernels with the intermediate through L2
// (log_n = 17).  All give the same words (same butterflies, same order, same lazy ranges).
extern "C" int hg_set_ntt_variant(hg_ctx* ctx, int variant) {
    if (!ctx) return hg_fail(HG_EINVAL, "hg_set_ntt_variant: null context");
    if (variant < 0 || variant > 2) return hg_fail(HG_EINVAL, "hg_set_ntt_variant: variant must be 0, 1 or 2");
    ctx->ntt_cluster = variant;
    if (variant != 1 && ctx->d_twc_fwd) {
        // the DSMEM variant's transposed twiddles (~650 MB at log_n 17) go with it; cudaFree
        // waits for queued work that may still read them
        std::lock_guard<std::mutex> lk(ctx->mu);
        cudaFree(ctx->d_twc_fwd);
        cudaFree(ctx->d_twc_inv);
        ctx->d_twc_fwd = ctx->d_twc_inv = nullptr;
    }
    return HG_OK;
}

// forward or plain inverse over rows [B][P][N] (rows = B P), in place
int hg_ntt_cluster(hg_ctx* ctx, uint32_t* data, int rows, int P, int prime_offset, bool forward,
                   cudaStream_t st) {
    int rc;
    if ((rc = hg_ensure_twiddles(ctx, ctx->nprimes)) || (rc = ensure_twc(ctx)) || (rc = ensure_attrs(ctx)))
        return rc;
    const int B = rows / P;
    if (B > 65535) return hg_fail(HG_EINVAL, "cluster NTT: too many rows");
    HgTimed tm(ctx, st, HG_K_NTT, (double)rows * (kN / 2) * 17);
    const dim3 g(kCS, B, P);
    if (forward)
        ntt_fwd_c8_kernel<<<g, 256, kSmemBytes, st>>>(data, P, prime_offset, ctx->d_pinfo, ctx->d_tw_fwd,
                                                      ctx->d_twc_fwd);
    else
        ntt_inv_c8_kernel<0><<<g, 256, kSmemBytes, st>>>(data, nullptr, nullptr, nullptr, nullptr, P,
                                                         prime_offset, ctx->d_pinfo, ctx->d_tw_inv,
                                                         ctx->d_twc_inv, 0, 0);
    HG_LAUNCH_CHECK(ctx);
    return HG_OK;
}

// fused product + inverse NTT (hg_intt_fused's contract)
int hg_intt_fused_cluster(hg_ctx* ctx, int pre, uint32_t* out, const uint32_t* i0, const uint32_t* i1,
                          const uint32_t* i2, const uint32_t* i3, int P, cudaStream_t st, int batch) {
    int rc;
    if ((rc = hg_ensure_twiddles(ctx, ctx->nprimes)) || (rc = ensure_twc(ctx)) || (rc = ensure_attrs(ctx)))
        return rc;
    const int rb = pre == 1 ? 2 : (pre == 2 ? 3 : 1);
    HgTimed tm(ctx, st, HG_K_NTT, (double)batch * rb * P * (kN / 2) * 17);
    const dim3 g(kCS, batch, P);
    const size_t bsi = (size_t)P * kN, bso = (size_t)rb * P * kN;
#define HG_INVC(PR)                                                                                  \
    ntt_inv_c8_kernel<PR><<<g, 256, kSmemBytes, st>>>(out, i0, i1, i2, i3, P, 0, ctx->d_pinfo,      \
                                                      ctx->d_tw_inv, ctx->d_twc_inv, bsi, bso)
    switch (pre) {
        case 1: HG_INVC(1); break;
        case 2: HG_INVC(2); break;
        case 3: HG_INVC(3); break;
        case 5: HG_INVC(5); break;
        default: return -1;
    }
#undef HG_INVC
    HG_LAUNCH_CHECK(ctx);
    return HG_OK;
}
