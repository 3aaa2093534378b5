// hg_ntt.cu -- batched negacyclic NTT / inverse NTT over 30-bit primes.
//
// Forward: merged Cooley-Tukey with psi powers in bit-reversed order (natural input,
// bit-reversed output), Harvey lazy butterflies keeping values in [0, 4p).
// Inverse: Gentleman-Sande (bit-reversed input, natural output), values in [0, 2p); the
// N^{-1} scaling is folded into the CRT constants (hg_context.cu, cinv).
//
// N = 2^log_n is split as 2^k1 (strided "hi" stages) x 2^k2 (contiguous "lo" stages,
// k2 = min(log_n, 11)); each pass stages one 2048-word tile in shared memory, so a
// length-2^17 transform is one HBM round trip per pass.  Rows are laid out [row][N],
// row r uses prime prime_offset + (r % P).
#include "hg_internal.cuh"

namespace {

constexpr int kTile = 2048;  // words per shared-memory tile

__device__ __forceinline__ void fwd_bfly(uint32_t& x, uint32_t& y, uint32_t w, uint32_t wsh,
                                         uint32_t p) {
    uint32_t p2 = p << 1;
    uint32_t a = x >= p2 ? x - p2 : x;
    uint32_t t = mul_shoup_lazy(y, w, wsh, p);
    x = a + t;
    y = a - t + p2;
}
__device__ __forceinline__ void inv_bfly(uint32_t& x, uint32_t& y, uint32_t w, uint32_t wsh,
                                         uint32_t p) {
    uint32_t p2 = p << 1;
    uint32_t s = x + y;
    s = s >= p2 ? s - p2 : s;
    uint32_t d = x - y + p2;
    x = s;
    y = mul_shoup_lazy(d, w, wsh, p);
}

// ---- "lo" pass: contiguous chunks of 2^k2 words, stages [s_begin, s_end) ----------------
template <bool FWD>
__global__ void __launch_bounds__(256) ntt_lo_kernel(uint32_t* __restrict__ data, int log_n,
                                                     int k2, int s_begin, int s_end, int P,
                                                     int prime_offset,
                                                     const PrimeInfo* __restrict__ pinfo,
                                                     const uint32_t* __restrict__ tw,
                                                     const uint32_t* __restrict__ tw_sh) {
    __shared__ uint32_t sm[kTile];
    const int N = 1 << log_n;
    const int chunk = 1 << k2;
    const int row = blockIdx.y;
    const int prime = prime_offset + row % P;
    const uint32_t p = pinfo[prime].p;
    const uint32_t* twp = tw + (size_t)prime * N;
    const uint32_t* twsp = tw_sh + (size_t)prime * N;
    uint32_t* rowp = data + (size_t)row * N;
    const int base = blockIdx.x * chunk;
    for (int i = threadIdx.x; i < chunk; i += blockDim.x) sm[i] = rowp[base + i];
    __syncthreads();
    const int half = chunk >> 1;
    if (FWD) {
        for (int s = s_begin; s < s_end; ++s) {
            const int lt = log_n - s - 1;  // log2 t
            const int t = 1 << lt;
            for (int b = threadIdx.x; b < half; b += blockDim.x) {
                int q0 = ((b >> lt) << (lt + 1)) | (b & (t - 1));
                int idx = (1 << s) + ((base + q0) >> (log_n - s));
                uint32_t x = sm[q0], y = sm[q0 + t];
                fwd_bfly(x, y, twp[idx], twsp[idx], p);
                sm[q0] = x;
                sm[q0 + t] = y;
            }
            __syncthreads();
        }
    } else {
        for (int s = s_end - 1; s >= s_begin; --s) {
            const int lt = log_n - s - 1;
            const int t = 1 << lt;
            for (int b = threadIdx.x; b < half; b += blockDim.x) {
                int q0 = ((b >> lt) << (lt + 1)) | (b & (t - 1));
                int idx = (1 << s) + ((base + q0) >> (log_n - s));
                uint32_t x = sm[q0], y = sm[q0 + t];
                inv_bfly(x, y, twp[idx], twsp[idx], p);
                sm[q0] = x;
                sm[q0 + t] = y;
            }
            __syncthreads();
        }
    }
    for (int i = threadIdx.x; i < chunk; i += blockDim.x) rowp[base + i] = sm[i];
}

// ---- "hi" pass: 2^k1 rows (stride 2^k2) x TC consecutive columns, stages [0, k1) ---------
template <bool FWD>
__global__ void __launch_bounds__(256) ntt_hi_kernel(uint32_t* __restrict__ data, int log_n,
                                                     int k1, int P, int prime_offset,
                                                     const PrimeInfo* __restrict__ pinfo,
                                                     const uint32_t* __restrict__ tw,
                                                     const uint32_t* __restrict__ tw_sh) {
    __shared__ uint32_t sm[kTile];
    const int N = 1 << log_n;
    const int k2 = log_n - k1;
    const int R = 1 << k1;
    const int TC = kTile >> k1;  // columns per tile
    const int row = blockIdx.y;
    const int prime = prime_offset + row % P;
    const uint32_t p = pinfo[prime].p;
    const uint32_t* twp = tw + (size_t)prime * N;
    const uint32_t* twsp = tw_sh + (size_t)prime * N;
    uint32_t* rowp = data + (size_t)row * N;
    const int cb = blockIdx.x * TC;
    for (int i = threadIdx.x; i < kTile; i += blockDim.x) {
        int c = i % TC, r = i / TC;
        sm[i] = rowp[((size_t)r << k2) + cb + c];
    }
    __syncthreads();
    const int nb = kTile >> 1;
    if (FWD) {
        for (int s = 0; s < k1; ++s) {
            const int ltr = k1 - 1 - s;  // log2 of the row distance
            for (int b = threadIdx.x; b < nb; b += blockDim.x) {
                int c = b % TC, rr = b / TC;
                int gi = rr >> ltr;
                int r0 = (gi << (ltr + 1)) | (rr & ((1 << ltr) - 1));
                int idx = (1 << s) + gi;
                uint32_t x = sm[r0 * TC + c], y = sm[(r0 + (1 << ltr)) * TC + c];
                fwd_bfly(x, y, twp[idx], twsp[idx], p);
                sm[r0 * TC + c] = x;
                sm[(r0 + (1 << ltr)) * TC + c] = y;
            }
            __syncthreads();
        }
    } else {
        for (int s = k1 - 1; s >= 0; --s) {
            const int ltr = k1 - 1 - s;
            for (int b = threadIdx.x; b < nb; b += blockDim.x) {
                int c = b % TC, rr = b / TC;
                int gi = rr >> ltr;
                int r0 = (gi << (ltr + 1)) | (rr & ((1 << ltr) - 1));
                int idx = (1 << s) + gi;
                uint32_t x = sm[r0 * TC + c], y = sm[(r0 + (1 << ltr)) * TC + c];
                inv_bfly(x, y, twp[idx], twsp[idx], p);
                sm[r0 * TC + c] = x;
                sm[(r0 + (1 << ltr)) * TC + c] = y;
            }
            __syncthreads();
        }
    }
    (void)R;
    for (int i = threadIdx.x; i < kTile; i += blockDim.x) {
        int c = i % TC, r = i / TC;
        rowp[((size_t)r << k2) + cb + c] = sm[i];
    }
}

}  // namespace

// rows = number of length-N rows, P = period of the prime index.
int hg_ntt_launch(hg_ctx* ctx, uint32_t* data, int rows, int P, int prime_offset, bool forward,
                  cudaStream_t stream) {
    if (rows <= 0) return HG_OK;
    int rc = hg_ensure_twiddles(ctx, prime_offset + P);
    if (rc) return rc;
    const int log_n = ctx->log_n, N = ctx->N;
    const int k2 = log_n < 11 ? log_n : 11;
    const int k1 = log_n - k2;
    const int chunk = 1 << k2;
    const int lo_threads = chunk / 2 < 256 ? (chunk / 2 < 32 ? 32 : chunk / 2) : 256;
    dim3 glo(N / chunk, rows);
    dim3 ghi(k1 > 0 ? N / kTile : 1, rows);  // 2^k2 columns / (kTile >> k1) per tile
    const uint32_t* tw = forward ? ctx->d_psi : ctx->d_ipsi;
    const uint32_t* twsh = forward ? ctx->d_psi_sh : ctx->d_ipsi_sh;
    HgTimed tm(ctx, stream, HG_K_NTT, (double)rows * (N / 2) * log_n);
    if (forward) {
        if (k1 > 0) {
            ntt_hi_kernel<true><<<ghi, 256, 0, stream>>>(data, log_n, k1, P, prime_offset,
                                                          ctx->d_pinfo, tw, twsh);
            HG_LAUNCH_CHECK(ctx);
        }
        ntt_lo_kernel<true><<<glo, lo_threads, 0, stream>>>(data, log_n, k2, k1, log_n, P,
                                                            prime_offset, ctx->d_pinfo, tw, twsh);
        HG_LAUNCH_CHECK(ctx);
    } else {
        ntt_lo_kernel<false><<<glo, lo_threads, 0, stream>>>(data, log_n, k2, k1, log_n, P,
                                                             prime_offset, ctx->d_pinfo, tw, twsh);
        HG_LAUNCH_CHECK(ctx);
        if (k1 > 0) {
            ntt_hi_kernel<false><<<ghi, 256, 0, stream>>>(data, log_n, k1, P, prime_offset,
                                                           ctx->d_pinfo, tw, twsh);
            HG_LAUNCH_CHECK(ctx);
        }
    }
    return HG_OK;
}

extern "C" int hg_ntt_forward(hg_ctx* ctx, uint32_t* data, int count, int prime_offset,
                              void* stream) {
    if (!ctx || !data || count < 0 || prime_offset < 0 || prime_offset >= ctx->nprimes)
        return hg_fail(HG_EINVAL, "bad NTT arguments");
    int P = ctx->nprimes - prime_offset;
    if (count < P) P = count;
    return hg_ntt_launch(ctx, data, count, P, prime_offset, true, (cudaStream_t)stream);
}

extern "C" int hg_ntt_inverse(hg_ctx* ctx, uint32_t* data, int count, int prime_offset,
                              void* stream) {
    if (!ctx || !data || count < 0 || prime_offset < 0 || prime_offset >= ctx->nprimes)
        return hg_fail(HG_EINVAL, "bad NTT arguments");
    int P = ctx->nprimes - prime_offset;
    if (count < P) P = count;
    return hg_ntt_launch(ctx, data, count, P, prime_offset, false, (cudaStream_t)stream);
}
