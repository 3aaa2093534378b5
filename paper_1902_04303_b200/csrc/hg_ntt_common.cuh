// hg_ntt_common.cuh -- butterflies and register-resident 64-point stage sequences shared by the
// NTT kernels (hg_ntt.cu) and the DSMEM cluster variant (hg_ntt_cluster.cu).
//
// Forward: merged Cooley-Tukey, Harvey lazy butterflies keeping values in [0, 4p); inverse:
// Gentleman-Sande, values in [0, 2p).  Twiddles are (w, floor(w 2^32 / p)) pairs.
#pragma once

#include "hg_internal.cuh"

namespace hgntt {

__device__ __forceinline__ void fwd_bfly(uint32_t& x, uint32_t& y, uint2 w, uint32_t p) {
    const uint32_t p2 = p << 1;
    const uint32_t a = min(x, x - p2);   // [0, 4p) -> [0, 2p)
    const uint32_t t = mul_shoup_lazy(y, w.x, w.y, p);
    x = a + t;
    y = a - t + p2;
}
__device__ __forceinline__ void inv_bfly(uint32_t& x, uint32_t& y, uint2 w, uint32_t p) {
    const uint32_t p2 = p << 1;
    uint32_t s = x + y;
    s = min(s, s - p2);
    const uint32_t d = x - y + p2;
    x = s;
    y = mul_shoup_lazy(d, w.x, w.y, p);
}

// NTT-domain storage order.  The forward transform's bit-reversed output (and the inverse's
// input) is stored with every 512-word block transposed as a 32 x 4 matrix of 16-byte vectors:
// word q = 512 b + 16 a + 4 v + j (a < 32, v < 4, j < 4) sits at 512 b + 128 v + 4 a + j.  A
// contiguous-pass thread holds E consecutive words in its unit-stride round, so in natural
// order a warp's 16-byte accesses stride 4E bytes (16 cache lines and twice the ideal sectors
// per STG.128 at E = 16); in this order every 16-byte access of a warp lands in 128-byte runs.
// Every NTT-domain consumer is elementwise (products, sums, prepared operands), so the order is
// invisible outside the transforms; rows of 2^k >= 512 words use it (chunks of the contiguous
// pass are >= 512 words exactly then), shorter rows keep natural order.
__host__ __device__ __forceinline__ int ntt_pos(int q) {
    return (q & ~511) | (((q >> 2) & 3) << 7) | (((q >> 4) & 31) << 2) | (q & 3);
}

// One stage on x[64]: butterflies (2 D g + i, 2 D g + i + D) for the 32 / D groups g, group g
// taking twiddle tw[g * TS] (TS = the twiddle stride of the caller's table).  Template
// parameters keep every index compile-time, so x stays in registers.
template <bool FWD, int D, int TS>
__device__ __forceinline__ void stage64(uint32_t (&x)[64], const uint2* __restrict__ tw, uint32_t p) {
#pragma unroll
    for (int g = 0; g < 32 / D; ++g) {
#ifdef HG_FAKE_TW   // timing experiment only: twiddles without loads (wrong results)
        const uint2 w = make_uint2(0x1234567u + g * 977u + (uint32_t)(size_t)tw, 0x2345678u + g);
#else
        const uint2 w = __ldg(tw + g * TS);
#endif
#pragma unroll
        for (int i = 0; i < D; ++i) {
            if (FWD) fwd_bfly(x[2 * D * g + i], x[2 * D * g + i + D], w, p);
            else inv_bfly(x[2 * D * g + i], x[2 * D * g + i + D], w, p);
        }
    }
}

// the 6 strided stages of a 64-row column x[r] = word (r 2^K2 + c): stage s uses
// psi_rev[2^s + (r >> (6 - s))] (twp = the prime's table), warp-uniform
template <bool FWD>
__device__ __forceinline__ void hi_stages(uint32_t (&x)[64], const uint2* __restrict__ twp, uint32_t p) {
    if (FWD) {
        stage64<true, 32, 1>(x, twp + 1, p);
        stage64<true, 16, 1>(x, twp + 2, p);
        stage64<true, 8, 1>(x, twp + 4, p);
        stage64<true, 4, 1>(x, twp + 8, p);
        stage64<true, 2, 1>(x, twp + 16, p);
        stage64<true, 1, 1>(x, twp + 32, p);
    } else {
        stage64<false, 1, 1>(x, twp + 32, p);
        stage64<false, 2, 1>(x, twp + 16, p);
        stage64<false, 4, 1>(x, twp + 8, p);
        stage64<false, 8, 1>(x, twp + 4, p);
        stage64<false, 16, 1>(x, twp + 2, p);
        stage64<false, 32, 1>(x, twp + 1, p);
    }
}

}  // namespace hgntt
