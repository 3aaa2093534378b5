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

// ======================= radix-8 register-round kernels (v2) ===============================
// A round applies R <= 3 consecutive stages to 8 elements a thread holds in registers:
// element m sits at position pos_base + m * 2^b (pos_base has zero bits [b, b+3)), the
// stage distances are 2^(b+R-1) ... 2^b.  For stage s = s0 + k the butterfly group of the
// pair starting at element m is (pos_base >> (b+R-k)) + (m >> (R-k)), so the twiddle is
// psi_rev[2^s + group] (the same rule as the merged negacyclic transform).
template <bool FWD, int R>
__device__ __forceinline__ void round8(uint32_t (&x)[8], int s0, int pos_base, int b,
                                       const uint32_t* __restrict__ twp,
                                       const uint32_t* __restrict__ twsp, uint32_t p) {
    if (FWD) {
#pragma unroll
        for (int k = 0; k < R; ++k) {
            const int d = 1 << (R - 1 - k);
            const int gbase = (1 << (s0 + k)) + (pos_base >> (b + R - k));
#pragma unroll
            for (int m = 0; m < 8; ++m) {
                if (m & d) continue;
                const int idx = gbase + (m >> (R - k));
                fwd_bfly(x[m], x[m + d], __ldg(twp + idx), __ldg(twsp + idx), p);
            }
        }
    } else {
#pragma unroll
        for (int k = R - 1; k >= 0; --k) {
            const int d = 1 << (R - 1 - k);
            const int gbase = (1 << (s0 + k)) + (pos_base >> (b + R - k));
#pragma unroll
            for (int m = 0; m < 8; ++m) {
                if (m & d) continue;
                const int idx = gbase + (m >> (R - k));
                inv_bfly(x[m], x[m + d], __ldg(twp + idx), __ldg(twsp + idx), p);
            }
        }
    }
}

template <bool FWD>
__device__ __forceinline__ void round8_dispatch(uint32_t (&x)[8], int R, int s0, int pos_base,
                                                int b, const uint32_t* twp, const uint32_t* twsp,
                                                uint32_t p) {
    if (R == 3) round8<FWD, 3>(x, s0, pos_base, b, twp, twsp, p);
    else if (R == 2) round8<FWD, 2>(x, s0, pos_base, b, twp, twsp, p);
    else round8<FWD, 1>(x, s0, pos_base, b, twp, twsp, p);
}

// smem swizzle (a bijection on [0, 2048)): bits 2-4 ^= bits 5-7, so the stride-32 groups of
// the b = 2 round and the stride-1 warps of the b = 5 round both hit 32 distinct banks
__device__ __forceinline__ int swz(int i) { return i ^ (((i >> 5) & 7) << 2); }

// Grid: x = chunk index, y = prime-major row (rows sharing a prime are adjacent so their
// twiddles are re-read from L2).  Block = chunk/8 threads, 8 elements each.
template <bool FWD>
__global__ void __launch_bounds__(256) ntt_lo8_kernel(uint32_t* __restrict__ data, int log_n,
                                                      int k2, int P, int B, int prime_offset,
                                                      const PrimeInfo* __restrict__ pinfo,
                                                      const uint32_t* __restrict__ tw,
                                                      const uint32_t* __restrict__ tw_sh) {
    __shared__ uint32_t sm[2][kTile + 64];
    const int N = 1 << log_n;
    const int k1 = log_n - k2;
    const int jp = blockIdx.y / B, bb = blockIdx.y - jp * B;
    const int prime = prime_offset + jp;
    const uint32_t p = pinfo[prime].p;
    const uint32_t* twp = tw + (size_t)prime * N;
    const uint32_t* twsp = tw_sh + (size_t)prime * N;
    uint32_t* rowp = data + ((size_t)bb * P + jp) * N;
    const int cbase = blockIdx.x << k2;
    const int t = threadIdx.x;
    const int nrounds = (k2 + 2) / 3;
    uint32_t x[8];
    for (int ri = 0; ri < nrounds; ++ri) {
        const int r = FWD ? ri : nrounds - 1 - ri;
        const int s0 = k1 + 3 * r;
        const int R = (log_n - s0) < 3 ? (log_n - s0) : 3;
        const int b = log_n - s0 - R;
        const int base = ((t >> b) << (b + 3)) | (t & ((1 << b) - 1));
        if (ri == 0) {
#pragma unroll
            for (int m = 0; m < 8; ++m) x[m] = rowp[cbase + base + (m << b)];
        } else {
            const uint32_t* s = sm[(ri - 1) & 1];
#pragma unroll
            for (int m = 0; m < 8; ++m) x[m] = s[swz(base + (m << b))];
        }
        round8_dispatch<FWD>(x, R, s0, cbase + base, b, twp, twsp, p);
        if (ri == nrounds - 1) {
#pragma unroll
            for (int m = 0; m < 8; ++m) rowp[cbase + base + (m << b)] = x[m];
        } else {
            uint32_t* s = sm[ri & 1];
#pragma unroll
            for (int m = 0; m < 8; ++m) s[swz(base + (m << b))] = x[m];
            __syncthreads();
        }
    }
}

// Strided stages [0, k1) with k1 in {3, 6}: tile of 2^k1 rows (stride 2^k2) x TC columns;
// thread = (column c, row group g) holding 8 rows.  k1 = 3 needs no shared memory.
template <bool FWD>
__global__ void __launch_bounds__(256) ntt_hi8_kernel(uint32_t* __restrict__ data, int log_n,
                                                      int k1, int P, int B, int prime_offset,
                                                      const PrimeInfo* __restrict__ pinfo,
                                                      const uint32_t* __restrict__ tw,
                                                      const uint32_t* __restrict__ tw_sh) {
    __shared__ uint32_t sm[kTile];
    const int N = 1 << log_n;
    const int k2 = log_n - k1;
    const int TC = kTile >> k1;
    const int jp = blockIdx.y / B, bb = blockIdx.y - jp * B;
    const int prime = prime_offset + jp;
    const uint32_t p = pinfo[prime].p;
    const uint32_t* twp = tw + (size_t)prime * N;
    const uint32_t* twsp = tw_sh + (size_t)prime * N;
    uint32_t* rowp = data + ((size_t)bb * P + jp) * N;
    const int c = threadIdx.x % TC, g = threadIdx.x / TC;
    const int cb = blockIdx.x * TC;
    const int nrounds = k1 / 3;
    uint32_t x[8];
    for (int ri = 0; ri < nrounds; ++ri) {
        const int r = FWD ? ri : nrounds - 1 - ri;
        const int s0 = 3 * r;
        const int b = k1 - s0 - 3;
        const int rbase = ((g >> b) << (b + 3)) | (g & ((1 << b) - 1));
        if (ri == 0) {
#pragma unroll
            for (int m = 0; m < 8; ++m) x[m] = rowp[((size_t)(rbase + (m << b)) << k2) + cb + c];
        } else {
#pragma unroll
            for (int m = 0; m < 8; ++m) x[m] = sm[(rbase + (m << b)) * TC + c];
        }
        round8<FWD, 3>(x, s0, rbase, b, twp, twsp, p);
        if (ri == nrounds - 1) {
#pragma unroll
            for (int m = 0; m < 8; ++m) rowp[((size_t)(rbase + (m << b)) << k2) + cb + c] = x[m];
        } else {
#pragma unroll
            for (int m = 0; m < 8; ++m) sm[(rbase + (m << b)) * TC + c] = x[m];
            __syncthreads();
        }
    }
}

}  // namespace

// rows = number of length-N rows laid out [B][P][N]; row r uses prime prime_offset + r % P.
int hg_ntt_launch(hg_ctx* ctx, uint32_t* data, int rows, int P, int prime_offset, bool forward,
                  cudaStream_t stream) {
    if (rows <= 0) return HG_OK;
    int rc = hg_ensure_twiddles(ctx, prime_offset + P);
    if (rc) return rc;
    const int log_n = ctx->log_n, N = ctx->N;
    const uint32_t* tw = forward ? ctx->d_psi : ctx->d_ipsi;
    const uint32_t* twsh = forward ? ctx->d_psi_sh : ctx->d_ipsi_sh;
    HgTimed tm(ctx, stream, HG_K_NTT, (double)rows * (N / 2) * log_n);
    if (log_n >= 3 && rows % P == 0) {
        // v2: radix-8 register rounds; split log_n = k1 (0, 3 or 6 strided stages) + k2 (<= 11)
        const int k1 = log_n <= 11 ? 0 : (log_n <= 14 ? 3 : 6);
        const int k2 = log_n - k1;
        const int B = rows / P;
        dim3 glo(N >> k2, rows);
        dim3 ghi(N / kTile, rows);
        const int lo_threads = (1 << k2) / 8;
        if (forward) {
            if (k1) {
                ntt_hi8_kernel<true><<<ghi, 256, 0, stream>>>(data, log_n, k1, P, B, prime_offset,
                                                              ctx->d_pinfo, tw, twsh);
                HG_LAUNCH_CHECK(ctx);
            }
            ntt_lo8_kernel<true><<<glo, lo_threads, 0, stream>>>(data, log_n, k2, P, B, prime_offset,
                                                                 ctx->d_pinfo, tw, twsh);
            HG_LAUNCH_CHECK(ctx);
        } else {
            ntt_lo8_kernel<false><<<glo, lo_threads, 0, stream>>>(data, log_n, k2, P, B, prime_offset,
                                                                  ctx->d_pinfo, tw, twsh);
            HG_LAUNCH_CHECK(ctx);
            if (k1) {
                ntt_hi8_kernel<false><<<ghi, 256, 0, stream>>>(data, log_n, k1, P, B, prime_offset,
                                                               ctx->d_pinfo, tw, twsh);
                HG_LAUNCH_CHECK(ctx);
            }
        }
        return HG_OK;
    }
    // v1 fallback (tiny rings / ragged row counts): radix-2 stages in shared memory
    const int k2 = log_n < 11 ? log_n : 11;
    const int k1 = log_n - k2;
    const int chunk = 1 << k2;
    const int lo_threads = chunk / 2 < 256 ? (chunk / 2 < 32 ? 32 : chunk / 2) : 256;
    dim3 glo(N / chunk, rows);
    dim3 ghi(k1 > 0 ? N / kTile : 1, rows);  // 2^k2 columns / (kTile >> k1) per tile
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
