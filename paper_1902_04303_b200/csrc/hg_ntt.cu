// hg_ntt.cu -- batched negacyclic NTT / inverse NTT over 30-bit primes.
//
// Forward: merged Cooley-Tukey with psi powers in bit-reversed order (natural input,
// bit-reversed output), Harvey lazy butterflies keeping values in [0, 4p).
// Inverse: Gentleman-Sande (bit-reversed input, natural output), values in [0, 2p); the
// N^{-1} scaling is folded into the CRT constants (hg_context.cu, cinv).
// Twiddles are stored interleaved, (w, floor(w 2^32 / p)) per uint2, so each butterfly
// issues one 8-byte load.
//
// N = 2^log_n = 2^k1 (strided "hi" stages, k1 in {0, 3, 6}) x 2^k2 (contiguous "lo" stages,
// k2 <= 11).  Each pass keeps a 2048-word tile in registers + shared memory: every thread
// holds 8 elements and applies up to 3 stages per register round (radix-8), so a length-2^17
// transform is 2 HBM round trips with 3 + 1 shared-memory exchanges.  The round structure is
// a template on (k2, k1), so all index and address arithmetic is compile-time.  Rows are laid
// out [B][P][N]; the grid walks rows prime-major so polys sharing a prime reuse its twiddles
// from L2.
#include "hg_ntt_common.cuh"

namespace {

constexpr int kTile = 2048;  // words per shared-memory tile
// occupancy bounds (minimum resident blocks per SM), measured on the config-3 batch step:
#ifndef HG_FUSED_MINB
#define HG_FUSED_MINB 4   // fused inverse pass, 72 -> 64 registers, 3 -> 4 blocks: -2.7 ms of NTT
#endif
#ifndef HG_FUSED16_MINB
#define HG_FUSED16_MINB 6  // radix-16 fused inverse pass (128-thread blocks): 4 -> 6 blocks per SM: -3 ms of NTT per step
#endif
#ifndef HG_LO_MINB
#define HG_LO_MINB 3      // contiguous pass (radix 16, 128-thread blocks): >= 6 blocks per SM, 80 registers
#endif
#ifndef HG_HI_MINB
#define HG_HI_MINB 5      // strided pass (3-row variant 64 -> 48 registers): -15 ms of NTT
#endif

using hgntt::fwd_bfly;
using hgntt::inv_bfly;

// ---- v1 fallback (tiny rings / ragged row counts): radix-2 stages in shared memory -------
template <bool FWD>
__global__ void __launch_bounds__(256) ntt_lo_kernel(uint32_t* __restrict__ data, int log_n,
                                                     int k2, int s_begin, int s_end, int P,
                                                     int prime_offset,
                                                     const PrimeInfo* __restrict__ pinfo,
                                                     const uint2* __restrict__ tw) {
    __shared__ uint32_t sm[kTile];
    const int N = 1 << log_n;
    const int chunk = 1 << k2;
    const int row = blockIdx.y;
    const int prime = prime_offset + row % P;
    const uint32_t p = pinfo[prime].p;
    const uint2* twp = tw + (size_t)prime * N;
    uint32_t* rowp = data + (size_t)row * N;
    const int base = blockIdx.x * chunk;
    const bool perm = k2 >= 9;   // NTT-domain side in the transposed order (ntt_pos)
    for (int i = threadIdx.x; i < chunk; i += blockDim.x)
        sm[i] = rowp[!FWD && perm ? hgntt::ntt_pos(base + i) : base + i];
    __syncthreads();
    const int half = chunk >> 1;
    for (int si = s_begin; si < s_end; ++si) {
        const int s = FWD ? si : (s_end - 1 - (si - s_begin));
        const int lt = log_n - s - 1;
        const int t = 1 << lt;
        for (int b = threadIdx.x; b < half; b += blockDim.x) {
            const int q0 = ((b >> lt) << (lt + 1)) | (b & (t - 1));
            const int idx = (1 << s) + ((base + q0) >> (log_n - s));
            uint32_t x = sm[q0], y = sm[q0 + t];
            if (FWD) fwd_bfly(x, y, twp[idx], p);
            else inv_bfly(x, y, twp[idx], p);
            sm[q0] = x;
            sm[q0 + t] = y;
        }
        __syncthreads();
    }
    for (int i = threadIdx.x; i < chunk; i += blockDim.x)
        rowp[FWD && perm ? hgntt::ntt_pos(base + i) : base + i] = sm[i];
}

template <bool FWD>
__global__ void __launch_bounds__(256) ntt_hi_kernel(uint32_t* __restrict__ data, int log_n,
                                                     int k1, int P, int prime_offset,
                                                     const PrimeInfo* __restrict__ pinfo,
                                                     const uint2* __restrict__ tw) {
    __shared__ uint32_t sm[kTile];
    const int N = 1 << log_n;
    const int k2 = log_n - k1;
    const int TC = kTile >> k1;
    const int row = blockIdx.y;
    const int prime = prime_offset + row % P;
    const uint32_t p = pinfo[prime].p;
    const uint2* twp = tw + (size_t)prime * N;
    uint32_t* rowp = data + (size_t)row * N;
    const int cb = blockIdx.x * TC;
    for (int i = threadIdx.x; i < kTile; i += blockDim.x)
        sm[i] = rowp[((size_t)(i / TC) << k2) + cb + i % TC];
    __syncthreads();
    const int nb = kTile >> 1;
    for (int si = 0; si < k1; ++si) {
        const int s = FWD ? si : k1 - 1 - si;
        const int ltr = k1 - 1 - s;
        for (int b = threadIdx.x; b < nb; b += blockDim.x) {
            const int c = b % TC, rr = b / TC;
            const int gi = rr >> ltr;
            const int r0 = (gi << (ltr + 1)) | (rr & ((1 << ltr) - 1));
            const int idx = (1 << s) + gi;
            uint32_t x = sm[r0 * TC + c], y = sm[(r0 + (1 << ltr)) * TC + c];
            if (FWD) fwd_bfly(x, y, twp[idx], p);
            else inv_bfly(x, y, twp[idx], p);
            sm[r0 * TC + c] = x;
            sm[(r0 + (1 << ltr)) * TC + c] = y;
        }
        __syncthreads();
    }
    for (int i = threadIdx.x; i < kTile; i += blockDim.x)
        rowp[((size_t)(i / TC) << k2) + cb + i % TC] = sm[i];
}

// ---- v2: compile-time radix-8 register rounds ------------------------------------------------
// A round applies R <= 3 consecutive stages to 8 elements a thread holds: element m sits at
// local position base + m*2^B (base has zero bits [B, B+3)); the stage distances are
// 2^(B+R-1) ... 2^B.  For local stage LS0 + k the butterfly group of the pair starting at
// element m is G*2^(LS0+k) + (base >> (B+R-k)) + (m >> (R-k)), twiddle psi_rev[group]
// (G = 2^k1 + chunk index for the contiguous pass, 1 for the strided pass).  A block carries
// RB rows of the same prime (batch rows of one [B][P][N] launch): the twiddles of a stage are
// loaded once and applied to every row, and the rows' butterflies interleave.
template <bool FWD, int R, int B, int LS0, int RB, int E = 8>
__device__ __forceinline__ void round8(uint32_t (&x)[RB][E], int G, int base,
                                       const uint2* __restrict__ twp, uint32_t p) {
#pragma unroll
    for (int kk = 0; kk < R; ++kk) {
        const int k = FWD ? kk : R - 1 - kk;
        const int d = 1 << (R - 1 - k);
        // the E >> (R-k) twiddles of this stage are contiguous and aligned to their count:
        // 16-byte loads.  Unsigned 32-bit index: one shift-add into the block's table pointer
        const uint2* tg = twp + (((uint32_t)G << (LS0 + k)) + ((uint32_t)base >> (B + R - k)));
        constexpr int kMaxT = E / 2;
        uint2 w[kMaxT];
        const int nt = E >> (R - k);
        if (nt == 1) {
            w[0] = __ldg(tg);
        } else {
#pragma unroll
            for (int v = 0; v < nt / 2; ++v) {
                const uint4 q = __ldg(reinterpret_cast<const uint4*>(tg) + v);
                w[2 * v] = make_uint2(q.x, q.y);
                w[2 * v + 1] = make_uint2(q.z, q.w);
            }
        }
#pragma unroll
        for (int m = 0; m < E; ++m) {
            if (m & d) continue;
#pragma unroll
            for (int r = 0; r < RB; ++r) {
                if (FWD) fwd_bfly(x[r][m], x[r][m + d], w[m >> (R - k)], p);
                else inv_bfly(x[r][m], x[r][m + d], w[m >> (R - k)], p);
            }
        }
    }
}

// PERM: the words are NTT-domain data in the transposed storage order (ntt_pos; B == 0 only)
template <int B, int E = 8, bool PERM = false>
__device__ __forceinline__ void load8(uint32_t (&x)[E], const uint32_t* src, int base) {
    if (B == 0) {   // contiguous: 16-byte accesses
#pragma unroll
        for (int v = 0; v < E / 4; ++v) {
            const uint4 a = *reinterpret_cast<const uint4*>(src + (PERM ? hgntt::ntt_pos(base + 4 * v) : base + 4 * v));
            x[4 * v] = a.x; x[4 * v + 1] = a.y; x[4 * v + 2] = a.z; x[4 * v + 3] = a.w;
        }
    } else {
#pragma unroll
        for (int m = 0; m < E; ++m) x[m] = src[base + (m << B)];
    }
}
template <int B, int E = 8, bool PERM = false>
__device__ __forceinline__ void store8(const uint32_t (&x)[E], uint32_t* dst, int base) {
    if (B == 0) {
#pragma unroll
        for (int v = 0; v < E / 4; ++v)
            *reinterpret_cast<uint4*>(dst + (PERM ? hgntt::ntt_pos(base + 4 * v) : base + 4 * v)) = make_uint4(x[4 * v], x[4 * v + 1], x[4 * v + 2], x[4 * v + 3]);
    } else {
#pragma unroll
        for (int m = 0; m < E; ++m) dst[base + (m << B)] = x[m];
    }
}

// Shared-memory rows are padded: word i of a 2048-word row sits at
//     pad(i) = i + 4 (i >> 5) + 8 (i >> 7)
// (four spare words after every 32, eight more after every 128), which keeps every round's
// access pattern -- radix-8 and radix-16, every stride 2^B -- free of bank conflicts and, unlike
// an XOR swizzle, makes a thread's words one base address plus compile-time offsets: a thread's
// base has zero bits [B, B + log2 E) and its words add m 2^B, so (base mod 128) + (m 2^B mod 128)
// never carries past bit 6 and pad(base + m 2^B) = pad(base) + pad(m 2^B).
__device__ __forceinline__ int pad(int i) { return i + ((i >> 5) << 2) + ((i >> 7) << 3); }
template <int B>
__device__ __forceinline__ constexpr int pad_c(int m) {
    return (m << B) + (((m << B) >> 5) << 2) + (((m << B) >> 7) << 3);
}
template <int B, int E = 8>
__device__ __forceinline__ void sload8(uint32_t (&x)[E], const uint32_t* s, int base) {
    const uint32_t* sb = s + pad(base);
    if (B == 0) {   // E words inside one 32-word block: 16-byte accesses
#pragma unroll
        for (int v = 0; v < E / 4; ++v) {
            const uint4 a = *reinterpret_cast<const uint4*>(sb + 4 * v);
            x[4 * v] = a.x; x[4 * v + 1] = a.y; x[4 * v + 2] = a.z; x[4 * v + 3] = a.w;
        }
    } else {
#pragma unroll
        for (int m = 0; m < E; ++m) x[m] = sb[pad_c<B>(m)];
    }
}
template <int B, int E = 8>
__device__ __forceinline__ void sstore8(const uint32_t (&x)[E], uint32_t* s, int base) {
    uint32_t* sb = s + pad(base);
    if (B == 0) {
#pragma unroll
        for (int v = 0; v < E / 4; ++v)
            *reinterpret_cast<uint4*>(sb + 4 * v) = make_uint4(x[4 * v], x[4 * v + 1], x[4 * v + 2], x[4 * v + 3]);
    } else {
#pragma unroll
        for (int m = 0; m < E; ++m) sb[pad_c<B>(m)] = x[m];
    }
}

constexpr int kSmRow = kTile + kTile / 8 + kTile / 16;   // padded row (2432 words)

// Words per thread of the contiguous passes: radix-16 rounds (4 stages per shared-memory
// exchange, 2^K2 / 16 threads per chunk) from K2 = 8 up, radix 8 below (HG_NTT_E=8 forces 8)
#ifndef HG_NTT_E
#define HG_NTT_E 16
#endif
template <int K2>
struct LoE { static constexpr int value = (HG_NTT_E == 16 && K2 >= 10) ? 16 : 8; };
template <int K2>
struct LoThreads { static constexpr int value = (1 << K2) / LoE<K2>::value; };

template <bool FWD, int K2, int ROUND, int RB, bool PRELOADED = false, int E = LoE<K2>::value>
__device__ __forceinline__ void lo_round(uint32_t (&x)[RB][E], uint32_t* __restrict__ rowp,
                                         size_t rstride, uint32_t* __restrict__ sm, int G, int t,
                                         const uint2* __restrict__ twp, uint32_t p) {
    constexpr int LE = E == 16 ? 4 : 3;                    // stages per full round
    constexpr int NR = (K2 + LE - 1) / LE;
    constexpr int R_IDX = FWD ? ROUND : NR - 1 - ROUND;   // which stage group
    constexpr int LS0 = LE * R_IDX;
    constexpr int R = (K2 - LS0) < LE ? (K2 - LS0) : LE;  // a short round is the last (B = 0)
    constexpr int B = K2 - LS0 - R;
    const int base = ((t >> B) << (B + LE)) | (t & ((1 << B) - 1));
#pragma unroll
    for (int r = 0; r < RB; ++r) {
        if (ROUND == 0) {
            if (!PRELOADED) load8<B, E, (K2 >= 9)>(x[r], rowp + r * rstride, base);
        } else {
            sload8<B, E>(x[r], sm + r * kSmRow, base);
        }
    }
    // one buffer, updated in place: a round reads and writes the same words of each row (its
    // thread -> word map partitions the row), so one barrier per round orders it after the
    // previous round's writes
    round8<FWD, R, B, LS0, RB, E>(x, G, base, twp, p);
    if (ROUND == NR - 1) {
#pragma unroll
        for (int r = 0; r < RB; ++r) store8<B, E, (K2 >= 9)>(x[r], rowp + r * rstride, base);
    } else {
#pragma unroll
        for (int r = 0; r < RB; ++r) sstore8<B, E>(x[r], sm + r * kSmRow, base);
        __syncthreads();
    }
}

// Contiguous stages on chunk `chunk` (2^K2 words) of RB rows of one prime; K2/3 rounds, 2^K2 / 8
// threads.  Leaves sm free (its last shared-memory round is followed by a barrier).
template <bool FWD, int K2, int RB, int E = LoE<K2>::value>
__device__ __forceinline__ void lo_chunk(uint32_t* __restrict__ rowp0, size_t rstride, int chunk,
                                         int k1, uint32_t* __restrict__ sm,
                                         const uint2* __restrict__ twp, uint32_t p) {
    uint32_t* rowp = rowp0 + ((size_t)chunk << K2);
    const int G = (1 << k1) + chunk;
    const int t = threadIdx.x;
    uint32_t x[RB][E];
    constexpr int NR = (K2 + (E == 16 ? 3 : 2)) / (E == 16 ? 4 : 3);
    lo_round<FWD, K2, 0, RB, false, E>(x, rowp, rstride, sm, G, t, twp, p);
    if (NR > 1) lo_round<FWD, K2, (NR > 1 ? 1 : 0), RB, false, E>(x, rowp, rstride, sm, G, t, twp, p);
    if (NR > 2) lo_round<FWD, K2, (NR > 2 ? 2 : 0), RB, false, E>(x, rowp, rstride, sm, G, t, twp, p);
    if (NR > 3) lo_round<FWD, K2, (NR > 3 ? 3 : 0), RB, false, E>(x, rowp, rstride, sm, G, t, twp, p);
}

// Contiguous stages: chunk of 2^K2 words, K2/3 rounds; block = 2^K2 / 8 threads.
// grid = (N >> K2 chunks, batch-row groups of RB, primes): prime-major scheduling keeps the
// prime's twiddles in L2 while its batch rows pass.
template <bool FWD, int K2, int RB>
__global__ void __launch_bounds__(LoThreads<K2>::value, HG_LO_MINB * (LoE<K2>::value / 8)) ntt_lo8_kernel(uint32_t* __restrict__ data, int log_n,
                                                      int P, int bb0, int prime_offset,
                                                      const PrimeInfo* __restrict__ pinfo,
                                                      const uint2* __restrict__ tw) {
    __shared__ __align__(16) uint32_t sm[RB * kSmRow];
    const int N = 1 << log_n;
    const int jp = blockIdx.z, bb = bb0 + blockIdx.y * RB;
    const int prime = prime_offset + jp;
    lo_chunk<FWD, K2, RB>(data + ((size_t)bb * P + jp) * N, (size_t)P * N, blockIdx.x, log_n - K2, sm,
                          tw + (size_t)prime * N, pinfo[prime].p);
}

// Strided stages [0, K1), K1 in {3, 6}: tile `tile` of 2^K1 rows (stride 2^k2) x (2048 >> K1)
// columns of RB rows (rows rowp0 + r rstride); thread = (column c, row group g) holding 8 rows.
// K1 = 3 needs no shared memory.  K2 = log_n - K1 as a template parameter: every row / column
// offset is a compile-time immediate (fewer address instructions per butterfly in this
// memory-heavy pass).  Ends with a barrier when it used sm (K1 = 6).
template <bool FWD, int K1, int RB, int K2>
__device__ __forceinline__ void hi_tile(uint32_t* __restrict__ rowp0, size_t rstride, int tile,
                                        uint32_t* __restrict__ sm, const uint2* __restrict__ twp,
                                        uint32_t p) {
    constexpr int TC = kTile >> K1;
    constexpr int k2 = K2;
    const int c = threadIdx.x % TC, g = threadIdx.x / TC;
    uint32_t* colp = rowp0 + tile * TC + c;
    uint32_t x[RB][8];
    if (K1 == 3) {
#pragma unroll
        for (int r = 0; r < RB; ++r)
#pragma unroll
            for (int m = 0; m < 8; ++m) x[r][m] = colp[r * rstride + ((size_t)m << k2)];
        round8<FWD, 3, 0, 0, RB>(x, 1, 0, twp, p);
#pragma unroll
        for (int r = 0; r < RB; ++r)
#pragma unroll
            for (int m = 0; m < 8; ++m) colp[r * rstride + ((size_t)m << k2)] = x[r][m];
    } else {
        // forward: stages 0-2 on rows g + 8m, then 3-5 on rows 8g + m; inverse reversed
        constexpr int BA = FWD ? 3 : 0;   // first round's row stride exponent
        constexpr int BB = FWD ? 0 : 3;
        const int ra = BA ? g : 8 * g;
        const int rb = BB ? g : 8 * g;
        uint32_t* pa[RB];
        uint32_t* pb[RB];
#pragma unroll
        for (int r = 0; r < RB; ++r) {
            pa[r] = colp + r * rstride + ((size_t)ra << k2);
            pb[r] = colp + r * rstride + ((size_t)rb << k2);
        }
#pragma unroll
        for (int r = 0; r < RB; ++r)
#pragma unroll
            for (int m = 0; m < 8; ++m) x[r][m] = pa[r][(m << BA) << k2];
        round8<FWD, 3, BA, (FWD ? 0 : 3), RB>(x, 1, ra, twp, p);
#pragma unroll
        for (int r = 0; r < RB; ++r)
#pragma unroll
            for (int m = 0; m < 8; ++m) sm[r * kTile + (ra + (m << BA)) * TC + c] = x[r][m];
        __syncthreads();
#pragma unroll
        for (int r = 0; r < RB; ++r)
#pragma unroll
            for (int m = 0; m < 8; ++m) x[r][m] = sm[r * kTile + (rb + (m << BB)) * TC + c];
        round8<FWD, 3, BB, (FWD ? 3 : 0), RB>(x, 1, rb, twp, p);
#pragma unroll
        for (int r = 0; r < RB; ++r)
#pragma unroll
            for (int m = 0; m < 8; ++m) pb[r][(m << BB) << k2] = x[r][m];
        __syncthreads();
    }
}

template <bool FWD, int K1, int RB, int K2>
__global__ void __launch_bounds__(256, HG_HI_MINB) ntt_hi8_kernel(uint32_t* __restrict__ data, int log_n,
                                                      int P, int bb0, int prime_offset,
                                                      const PrimeInfo* __restrict__ pinfo,
                                                      const uint2* __restrict__ tw) {
    __shared__ uint32_t sm[K1 > 3 ? RB * kTile : 1];
    constexpr int N = 1 << (K1 + K2);
    (void)log_n;
    const int jp = blockIdx.z, bb = bb0 + blockIdx.y * RB;
    const int prime = prime_offset + jp;
    hi_tile<FWD, K1, RB, K2>(data + ((size_t)bb * P + jp) * N, (size_t)P * N, blockIdx.x, sm,
                             tw + (size_t)prime * N, pinfo[prime].p);
}

// Strided stages [0, 6), register-resident: thread = one column (64 words, rows 2^K2 apart,
// loaded / stored coalesced across the warp), all 6 stages in registers -- no shared-memory
// exchange, no barrier, every twiddle warp-uniform (so no batch-row grouping is needed).
#ifndef HG_HI64
#define HG_HI64 0   // measured slower than the tiled pass (16 warps per SM at 128 registers): 152.3 vs 147.5 ms of NTT per step
#endif
#ifndef HG_HI64_MINB
#define HG_HI64_MINB 2
#endif
template <bool FWD, int K2>
__global__ void __launch_bounds__(256, HG_HI64_MINB) ntt_hi64_kernel(uint32_t* __restrict__ data, int P,
                                                                  int prime_offset,
                                                                  const PrimeInfo* __restrict__ pinfo,
                                                                  const uint2* __restrict__ tw) {
    constexpr int N = 1 << (6 + K2);
    const int jp = blockIdx.z, bb = blockIdx.y;
    const int prime = prime_offset + jp;
    const uint32_t p = pinfo[prime].p;
    const uint2* twp = tw + (size_t)prime * N;
    uint32_t* col = data + ((size_t)bb * P + jp) * N + blockIdx.x * 256 + threadIdx.x;
    uint32_t x[64];
#pragma unroll
    for (int r = 0; r < 64; ++r) x[r] = col[(size_t)r << K2];
    hgntt::hi_stages<FWD>(x, twp, p);
#pragma unroll
    for (int r = 0; r < 64; ++r) col[(size_t)r << K2] = x[r];
}

template <bool FWD>
int launch_hi64(int log_n, int B, int P, cudaStream_t st, uint32_t* data, int off, const PrimeInfo* pinfo,
                const uint2* tw) {
    switch (log_n) {
        case 15: ntt_hi64_kernel<FWD, 9><<<dim3(2, B, P), 256, 0, st>>>(data, P, off, pinfo, tw); return 0;
        case 16: ntt_hi64_kernel<FWD, 10><<<dim3(4, B, P), 256, 0, st>>>(data, P, off, pinfo, tw); return 0;
        case 17: ntt_hi64_kernel<FWD, 11><<<dim3(8, B, P), 256, 0, st>>>(data, P, off, pinfo, tw); return 0;
    }
    return -1;
}

// Inverse contiguous pass with the NTT-domain product fused into its first round (which is
// unit-stride: each thread's 8 words are contiguous).  The products are Montgomery products of
// lazily reduced inputs, left in [0, 2p) (the inverse butterflies accept < 2p; the CRT reduces).
//   PRE 1 (key switch):  out rows (x*kb, x*ka)           in0 = x [0,4p), in1 = kb, in2 = ka [0,p)
//   PRE 2 (tensor):      out rows (a0b0, a0b1+a1b0, a1b1) in0..in3 = a0, a1, b0, b1 [0,4p)
//   PRE 3 (product):     out row  a*b                    in0, in1 [0,4p)
//   PRE 5 (shared factor): out row x*b                   in0 = x [0,4p), in1 = b [0,p)
// Inputs and outputs are [rows][P][N]; a block reads its chunk of every input row before its
// last round writes, so the outputs may alias the inputs chunk-for-chunk (in-place use).
template <int PRE>
struct PreRows { static constexpr int value = PRE == 1 ? 2 : (PRE == 2 ? 3 : 1); };   // PRE 3, 5: 1

// blockIdx.y selects one of a batch of independent products sharing in1..in3 (PRE 1: several
// key switches with one key, or one ciphertext times several plaintexts; PRE 5: several
// polynomials times one plaintext): in0 advances by bstride_in words, out by bstride_out
template <int K2, int PRE, int E = LoE<K2>::value>
__device__ __forceinline__ void lo_fused_chunk(uint32_t* out, const uint32_t* in0, const uint32_t* in1,
                                               const uint32_t* in2, const uint32_t* in3, size_t rstride,
                                               size_t roff0, int chunk, int k1, const PrimeInfo& pi,
                                               uint32_t* __restrict__ sm, const uint2* __restrict__ twp) {
    constexpr int RB = PreRows<PRE>::value;
    const uint32_t p = pi.p, p2 = p << 1;
    const size_t roff = roff0 + ((size_t)chunk << K2);
    const int G = (1 << k1) + chunk;
    const int t = threadIdx.x;
    const int base = t * E;     // round 0 of the inverse pass has B = 0
    uint32_t x[RB][E];
    {
        uint32_t u0[E], u1[E], u2[E], u3[E];
        constexpr bool PERM = K2 >= 9;
        load8<0, E, PERM>(u0, in0 + roff, base);
        load8<0, E, PERM>(u1, in1 + roff, base);
        if (PRE != 3 && PRE != 5) load8<0, E, PERM>(u2, in2 + roff, base);
        if (PRE == 2) load8<0, E, PERM>(u3, in3 + roff, base);
#pragma unroll
        for (int m = 0; m < E; ++m) {
            const uint32_t a = min(u0[m], u0[m] - p2);
            if (PRE == 1) {
                x[0][m] = mont_mul(a, u1[m], p, pi.pinv_neg);
                x[RB - 1][m] = mont_mul(a, u2[m], p, pi.pinv_neg);
            } else if (PRE == 2) {
                const uint32_t a1 = min(u1[m], u1[m] - p2);
                const uint32_t b0 = min(u2[m], u2[m] - p2);
                const uint32_t b1 = min(u3[m], u3[m] - p2);
                x[0][m] = mont_mul(a, b0, p, pi.pinv_neg);
                const uint32_t d1 = mont_mul(a, b1, p, pi.pinv_neg) + mont_mul(a1, b0, p, pi.pinv_neg);
                x[RB > 1 ? 1 : 0][m] = min(d1, d1 - p2);
                x[RB - 1][m] = mont_mul(a1, b1, p, pi.pinv_neg);
            } else if (PRE == 5) {
                x[0][m] = mont_mul(a, u1[m], p, pi.pinv_neg);
            } else {
                x[0][m] = mont_mul(a, min(u1[m], u1[m] - p2), p, pi.pinv_neg);
            }
        }
    }
    uint32_t* rowp = out + roff;
    constexpr int NR = (K2 + (E == 16 ? 3 : 2)) / (E == 16 ? 4 : 3);
    lo_round<false, K2, 0, RB, true, E>(x, rowp, rstride, sm, G, t, twp, p);
    if (NR > 1) lo_round<false, K2, (NR > 1 ? 1 : 0), RB, false, E>(x, rowp, rstride, sm, G, t, twp, p);
    if (NR > 2) lo_round<false, K2, (NR > 2 ? 2 : 0), RB, false, E>(x, rowp, rstride, sm, G, t, twp, p);
    if (NR > 3) lo_round<false, K2, (NR > 3 ? 3 : 0), RB, false, E>(x, rowp, rstride, sm, G, t, twp, p);
}

template <int K2, int PRE>
__global__ void __launch_bounds__(LoThreads<K2>::value, LoE<K2>::value == 16 ? HG_FUSED16_MINB : HG_FUSED_MINB) intt_lo8_fused_kernel(
    uint32_t* out, const uint32_t* in0, const uint32_t* in1, const uint32_t* in2,
    const uint32_t* in3, int log_n, int P, const PrimeInfo* __restrict__ pinfo,
    const uint2* __restrict__ tw, size_t bstride_in, size_t bstride_out) {
    out += blockIdx.y * bstride_out;
    in0 += blockIdx.y * bstride_in;
    constexpr int RB = PreRows<PRE>::value;
    __shared__ __align__(16) uint32_t sm[RB * kSmRow];
    const int N = 1 << log_n;
    const int jp = blockIdx.z;
    const PrimeInfo pi = pinfo[jp];
    lo_fused_chunk<K2, PRE>(out, in0, in1, in2, in3, (size_t)P * N, (size_t)jp * N, blockIdx.x,
                            log_n - K2, pi, sm, tw + (size_t)jp * N);
}

// ---- one-launch transforms on 8-CTA clusters, the intermediate through L2 ----------------------
// The two passes of a transform (strided tiles, contiguous chunks) run in ONE launch: the 8 CTAs
// of a cluster own RB transforms of one prime; CTA k runs the strided stages of tiles
// [k T/8, (k+1) T/8) (forward) with the code of the two-pass kernels, one cluster barrier
// (release / acquire: every CTA's stores are visible to the others, L1 invalidated), then the
// contiguous stages of chunks [8k, 8k+8) -- the inverse in the opposite order, with the NTT-domain
// product fused into its first phase.  The intermediate is written and re-read within a few
// microseconds, so it stays in L2: one HBM round trip per transform instead of two, while every
// CTA keeps the low register count (and 3 CTAs per SM) of the tile kernels.  Measured slower than
// the two passes (tools/ntt_bench.py, 656 rows: forward 0.584 vs 0.511 us per row, inverse 0.548
// vs 0.490; batch step 244 vs 223 ms): the barrier holds each CTA until its cluster's slowest
// member has finished the first phase.  Opt-in (hg_set_ntt_variant(ctx, 2)), log_n = 17 only
// (256 threads per 2048-word chunk).
#ifndef HG_CL_MINB
#define HG_CL_MINB 3
#endif
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

template <bool FWD, int RB, int K2>
__global__ void __cluster_dims__(8, 1, 1) __launch_bounds__(256, HG_CL_MINB)
ntt_c8l2_kernel(uint32_t* __restrict__ data, int P, int bb0, int prime_offset,
                const PrimeInfo* __restrict__ pinfo, const uint2* __restrict__ tw) {
    __shared__ __align__(16) uint32_t sm[RB * kSmRow];
    constexpr int K1 = 6, N = 1 << (K1 + K2);
    constexpr int TPC = (N / kTile) / 8;   // strided tiles per CTA
    constexpr int CPC = (1 << K1) / 8;     // contiguous chunks per CTA
    const int k = blockIdx.x;
    const int jp = blockIdx.z, bb = bb0 + blockIdx.y * RB;
    const int prime = prime_offset + jp;
    const uint32_t p = pinfo[prime].p;
    const uint2* twp = tw + (size_t)prime * N;
    uint32_t* rowp0 = data + ((size_t)bb * P + jp) * N;
    const size_t rs = (size_t)P * N;
    if (FWD) {
#pragma unroll 1
        for (int i = 0; i < TPC; ++i) hi_tile<true, K1, RB, K2>(rowp0, rs, k * TPC + i, sm, twp, p);
        cluster_sync_all();
#pragma unroll 1
        for (int i = 0; i < CPC; ++i) {
            lo_chunk<true, K2, RB, 8>(rowp0, rs, k * CPC + i, K1, sm, twp, p);
            __syncthreads();
        }
    } else {
#pragma unroll 1
        for (int i = 0; i < CPC; ++i) {
            lo_chunk<false, K2, RB, 8>(rowp0, rs, k * CPC + i, K1, sm, twp, p);
            __syncthreads();
        }
        cluster_sync_all();
#pragma unroll 1
        for (int i = 0; i < TPC; ++i) hi_tile<false, K1, RB, K2>(rowp0, rs, k * TPC + i, sm, twp, p);
    }
}

template <int K2, int PRE>
__global__ void __cluster_dims__(8, 1, 1) __launch_bounds__(256, HG_CL_MINB)
intt_fused_c8l2_kernel(uint32_t* out, const uint32_t* in0, const uint32_t* in1, const uint32_t* in2,
                       const uint32_t* in3, int P, const PrimeInfo* __restrict__ pinfo,
                       const uint2* __restrict__ tw, size_t bstride_in, size_t bstride_out) {
    constexpr int RB = PreRows<PRE>::value;
    __shared__ __align__(16) uint32_t sm[RB * kSmRow];
    constexpr int K1 = 6, N = 1 << (K1 + K2);
    constexpr int TPC = (N / kTile) / 8;
    constexpr int CPC = (1 << K1) / 8;
    out += blockIdx.y * bstride_out;
    in0 += blockIdx.y * bstride_in;
    const int k = blockIdx.x, jp = blockIdx.z;
    const PrimeInfo pi = pinfo[jp];
    const uint2* twp = tw + (size_t)jp * N;
    const size_t rs = (size_t)P * N;
#pragma unroll 1
    for (int i = 0; i < CPC; ++i) {
        lo_fused_chunk<K2, PRE, 8>(out, in0, in1, in2, in3, rs, (size_t)jp * N, k * CPC + i, K1, pi, sm, twp);
        __syncthreads();
    }
    cluster_sync_all();
#pragma unroll 1
    for (int i = 0; i < TPC; ++i) hi_tile<false, K1, RB, K2>(out + (size_t)jp * N, rs, k * TPC + i, sm, twp, pi.p);
}

template <bool FWD, int RB>
int launch_c8l2(int log_n, dim3 grid, cudaStream_t st, uint32_t* data, int P, int bb0, int off,
                const PrimeInfo* pinfo, const uint2* tw) {
    switch (log_n) {
        case 15: ntt_c8l2_kernel<FWD, RB, 9><<<grid, 256, 0, st>>>(data, P, bb0, off, pinfo, tw); return 0;
        case 16: ntt_c8l2_kernel<FWD, RB, 10><<<grid, 256, 0, st>>>(data, P, bb0, off, pinfo, tw); return 0;
        case 17: ntt_c8l2_kernel<FWD, RB, 11><<<grid, 256, 0, st>>>(data, P, bb0, off, pinfo, tw); return 0;
    }
    return -1;
}

template <int PRE>
int launch_fused_c8l2(int log_n, dim3 grid, cudaStream_t st, uint32_t* out, const uint32_t* i0,
                      const uint32_t* i1, const uint32_t* i2, const uint32_t* i3, int P,
                      const PrimeInfo* pinfo, const uint2* tw, size_t bsi, size_t bso) {
    switch (log_n) {
        case 15: intt_fused_c8l2_kernel<9, PRE><<<grid, 256, 0, st>>>(out, i0, i1, i2, i3, P, pinfo, tw, bsi, bso); return 0;
        case 16: intt_fused_c8l2_kernel<10, PRE><<<grid, 256, 0, st>>>(out, i0, i1, i2, i3, P, pinfo, tw, bsi, bso); return 0;
        case 17: intt_fused_c8l2_kernel<11, PRE><<<grid, 256, 0, st>>>(out, i0, i1, i2, i3, P, pinfo, tw, bsi, bso); return 0;
    }
    return -1;
}

// both passes of a transform over all rows in one cluster launch (groups of 2 batch rows, 3 for an
// odd count, 1 if B == 1), as ntt_pass groups them
template <bool FWD>
int ntt_c8l2(hg_ctx* ctx, uint32_t* data, int B, int P, int off, const uint2* tw, cudaStream_t st) {
    auto run = [&](int rb, int groups, int bb0) {
        const dim3 g(8, groups, P);
        int rc = rb == 1 ? launch_c8l2<FWD, 1>(ctx->log_n, g, st, data, P, bb0, off, ctx->d_pinfo, tw)
               : rb == 2 ? launch_c8l2<FWD, 2>(ctx->log_n, g, st, data, P, bb0, off, ctx->d_pinfo, tw)
                         : launch_c8l2<FWD, 3>(ctx->log_n, g, st, data, P, bb0, off, ctx->d_pinfo, tw);
        if (rc) return hg_fail(HG_EINVAL, "cluster NTT: unsupported size");
        HG_LAUNCH_CHECK(ctx);
        return HG_OK;
    };
    int rc;
    if (B == 1) return run(1, 1, 0);
    const int odd = B & 1;
    const int pairs = (B - 3 * odd) / 2;
    if (pairs > 0 && (rc = run(2, pairs, 0))) return rc;
    if (odd && (rc = run(3, 1, 2 * pairs))) return rc;
    return HG_OK;
}

template <int PRE>
int launch_fused_lo8(int k2, dim3 grid, cudaStream_t st, uint32_t* out, const uint32_t* i0,
                     const uint32_t* i1, const uint32_t* i2, const uint32_t* i3, int log_n, int P,
                     const PrimeInfo* pinfo, const uint2* tw, size_t bsi = 0, size_t bso = 0) {
    switch (k2) {
#define HG_LOF(K)                                                                               \
    case K:                                                                                     \
        intt_lo8_fused_kernel<K, PRE><<<grid, LoThreads<K>::value, 0, st>>>(out, i0, i1, i2, i3, log_n, P, \
                                                                pinfo, tw, bsi, bso);           \
        return 0;
        HG_LOF(3) HG_LOF(4) HG_LOF(5) HG_LOF(6) HG_LOF(7) HG_LOF(8) HG_LOF(9) HG_LOF(10) HG_LOF(11)
#undef HG_LOF
    }
    return -1;
}

template <bool FWD, int RB>
int launch_lo8(int k2, dim3 grid, cudaStream_t st, uint32_t* data, int log_n, int P, int bb0,
               int off, const PrimeInfo* pinfo, const uint2* tw) {
    switch (k2) {
#define HG_LO(K)                                                                                     \
    case K:                                                                                          \
        ntt_lo8_kernel<FWD, K, RB><<<grid, LoThreads<K>::value, 0, st>>>(data, log_n, P, bb0, off, pinfo, tw); \
        return 0;
        HG_LO(3) HG_LO(4) HG_LO(5) HG_LO(6) HG_LO(7) HG_LO(8) HG_LO(9) HG_LO(10) HG_LO(11)
#undef HG_LO
    }
    return -1;
}

template <bool FWD, int RB>
int launch_hi8(int k1, dim3 grid, cudaStream_t st, uint32_t* data, int log_n, int P, int bb0,
               int off, const PrimeInfo* pinfo, const uint2* tw) {
    // k1 = 3 for log_n 12..14, 6 for 15..17 (hg_ntt_launch)
    switch (log_n) {
#define HG_HI(LN, K1)                                                                              \
    case LN:                                                                                       \
        ntt_hi8_kernel<FWD, K1, RB, LN - K1><<<grid, 256, 0, st>>>(data, log_n, P, bb0, off, pinfo, tw); \
        return 0;
        HG_HI(12, 3) HG_HI(13, 3) HG_HI(14, 3) HG_HI(15, 6) HG_HI(16, 6) HG_HI(17, 6)
#undef HG_HI
    }
    (void)k1;
    return -1;
}

// one pass over all rows: groups of 2 batch rows per block (3 for an odd count), 1 if B == 1
// [j0, j0 + pz) of the P primes (pz < 0: all): the row stride stays P
template <bool FWD>
int ntt_pass(hg_ctx* ctx, bool hi, int k1, int k2, uint32_t* data, int B, int P, int off,
             const uint2* tw, cudaStream_t st, int j0 = 0, int pz = -1) {
    const int log_n = ctx->log_n, N = ctx->N;
    if (pz < 0) pz = P;
    data += (size_t)j0 * N;
    off += j0;
    if (HG_HI64 && hi && k1 == 6 && B <= 65535) {
        if (pz != P || (FWD ? launch_hi64<true>(log_n, B, P, st, data, off, ctx->d_pinfo, tw)
                            : launch_hi64<false>(log_n, B, P, st, data, off, ctx->d_pinfo, tw)))
            return hg_fail(HG_EINVAL, "strided NTT pass: unsupported size");
        HG_LAUNCH_CHECK(ctx);
        return HG_OK;
    }
    const int gx = hi ? N / kTile : N >> k2;
    auto run = [&](int rb, int groups, int bb0) {
        const dim3 g(gx, groups, pz);
        if (rb == 1) {
            if (hi) launch_hi8<FWD, 1>(k1, g, st, data, log_n, P, bb0, off, ctx->d_pinfo, tw);
            else launch_lo8<FWD, 1>(k2, g, st, data, log_n, P, bb0, off, ctx->d_pinfo, tw);
        } else if (rb == 2) {
            if (hi) launch_hi8<FWD, 2>(k1, g, st, data, log_n, P, bb0, off, ctx->d_pinfo, tw);
            else launch_lo8<FWD, 2>(k2, g, st, data, log_n, P, bb0, off, ctx->d_pinfo, tw);
        } else {
            if (hi) launch_hi8<FWD, 3>(k1, g, st, data, log_n, P, bb0, off, ctx->d_pinfo, tw);
            else launch_lo8<FWD, 3>(k2, g, st, data, log_n, P, bb0, off, ctx->d_pinfo, tw);
        }
        HG_LAUNCH_CHECK(ctx);
        return HG_OK;
    };
    int rc;
    if (B == 1) return run(1, 1, 0);
    const int odd = B & 1;                  // an odd count ends with one 3-row group
    const int pairs = (B - 3 * odd) / 2;
    if (pairs > 0 && (rc = run(2, pairs, 0))) return rc;
    if (odd && (rc = run(3, 1, 2 * pairs))) return rc;
    return HG_OK;
}

// Primes per group of launches when a transform's two passes run prime range by prime range, so
// that a range's rows (`rows_per_prime` rows of N words per prime) stay in L2 between the passes
// (HG_NTT_L2_MB: the budget in MB, 0 = one launch per pass over all primes).
int prime_chunk(const hg_ctx* ctx, int rows_per_prime, int P) {
    static const int mb = [] { const char* e = getenv("HG_NTT_L2_MB"); return e ? atoi(e) : 0; }();
    if (mb <= 0) return P;
    const size_t per_prime = (size_t)rows_per_prime * ctx->N * sizeof(uint32_t);
    int pc = (int)(((size_t)mb << 20) / per_prime);
    if (pc < 1) pc = 1;
    if (pc >= P) return P;
    const int chunks = (P + pc - 1) / pc;   // even ranges
    return (P + chunks - 1) / chunks;
}

}  // namespace

// rows = number of length-N rows laid out [B][P][N]; row r uses prime prime_offset + r % P.
int hg_ntt_launch(hg_ctx* ctx, uint32_t* data, int rows, int P, int prime_offset, bool forward,
                  cudaStream_t stream) {
    if (rows <= 0) return HG_OK;
    int rc = hg_ensure_twiddles(ctx, prime_offset + P);
    if (rc) return rc;
    const int log_n = ctx->log_n, N = ctx->N;
    const uint2* tw = forward ? ctx->d_tw_fwd : ctx->d_tw_inv;
    if (rows % P == 0 && rows / P <= 65535 && hg_ntt_cluster_ok(ctx, P))
        return hg_ntt_cluster(ctx, data, rows, P, prime_offset, forward, stream);
    HgTimed tm(ctx, stream, HG_K_NTT, (double)rows * (N / 2) * log_n);
    if (log_n >= 3 && rows % P == 0 && P <= 65535) {
        const int k1 = log_n <= 11 ? 0 : (log_n <= 14 ? 3 : 6);
        const int k2 = log_n - k1;
        const int B = rows / P;
        if (ctx->ntt_cluster == 2 && log_n == 17)   // 256 threads per 2048-word chunk and per tile
            return forward ? ntt_c8l2<true>(ctx, data, B, P, prime_offset, tw, stream)
                           : ntt_c8l2<false>(ctx, data, B, P, prime_offset, tw, stream);
        const int pc = k1 ? prime_chunk(ctx, B, P) : P;
        for (int j0 = 0; j0 < P; j0 += pc) {
            const int pz = P - j0 < pc ? P - j0 : pc;
            if (forward) {
                if (k1 && (rc = ntt_pass<true>(ctx, true, k1, k2, data, B, P, prime_offset, tw, stream, j0, pz))) return rc;
                if ((rc = ntt_pass<true>(ctx, false, k1, k2, data, B, P, prime_offset, tw, stream, j0, pz))) return rc;
            } else {
                if ((rc = ntt_pass<false>(ctx, false, k1, k2, data, B, P, prime_offset, tw, stream, j0, pz))) return rc;
                if (k1 && (rc = ntt_pass<false>(ctx, true, k1, k2, data, B, P, prime_offset, tw, stream, j0, pz))) return rc;
            }
        }
        return HG_OK;
    }
    // v1 fallback
    const int k2 = log_n < 11 ? log_n : 11;
    const int k1 = log_n - k2;
    const int chunk = 1 << k2;
    const int lo_threads = chunk / 2 < 256 ? (chunk / 2 < 32 ? 32 : chunk / 2) : 256;
    dim3 glo(N / chunk, rows);
    dim3 ghi(k1 > 0 ? N / kTile : 1, rows);
    if (forward) {
        if (k1 > 0) {
            ntt_hi_kernel<true><<<ghi, 256, 0, stream>>>(data, log_n, k1, P, prime_offset, ctx->d_pinfo, tw);
            HG_LAUNCH_CHECK(ctx);
        }
        ntt_lo_kernel<true><<<glo, lo_threads, 0, stream>>>(data, log_n, k2, k1, log_n, P, prime_offset,
                                                            ctx->d_pinfo, tw);
        HG_LAUNCH_CHECK(ctx);
    } else {
        ntt_lo_kernel<false><<<glo, lo_threads, 0, stream>>>(data, log_n, k2, k1, log_n, P, prime_offset,
                                                             ctx->d_pinfo, tw);
        HG_LAUNCH_CHECK(ctx);
        if (k1 > 0) {
            ntt_hi_kernel<false><<<ghi, 256, 0, stream>>>(data, log_n, k1, P, prime_offset, ctx->d_pinfo, tw);
            HG_LAUNCH_CHECK(ctx);
        }
    }
    return HG_OK;
}

// Inverse NTT with the pointwise product fused in (see intt_lo8_fused_kernel): `out` receives
// RB = 2 / 3 / 1 rows [RB][P][N] for pre = 1 / 2 / 3.  Returns -1 if the shape is not covered
// (the caller then runs the separate pointwise kernel + hg_ntt_launch).
int hg_intt_fused(hg_ctx* ctx, int pre, uint32_t* out, const uint32_t* i0, const uint32_t* i1,
                  const uint32_t* i2, const uint32_t* i3, int P, cudaStream_t st, int batch) {
    const int log_n = ctx->log_n, N = ctx->N;
    if (log_n < 3 || P > 65535) return -1;
    int rc = hg_ensure_twiddles(ctx, P);
    if (rc) return rc;
    const int k1 = log_n <= 11 ? 0 : (log_n <= 14 ? 3 : 6);
    const int k2 = log_n - k1;
    const int rb = pre == 1 ? 2 : (pre == 2 ? 3 : 1);
    if (batch < 1 || (batch > 1 && pre != 1 && pre != 5) || batch > 65535) return -1;
    if (hg_ntt_cluster_ok(ctx, P)) return hg_intt_fused_cluster(ctx, pre, out, i0, i1, i2, i3, P, st, batch);
    HgTimed tm(ctx, st, HG_K_NTT, (double)batch * rb * P * (N / 2) * log_n);
    // batch > 1 (key switch only): input g's x rows at i0 + g P N, its two outputs at out + g 2 P N
    const size_t bsi = (size_t)P * N, bso = (size_t)rb * P * N;
    if (ctx->ntt_cluster == 2 && log_n == 17) {
        const dim3 gc(8, batch, P);
        if (pre == 1) launch_fused_c8l2<1>(log_n, gc, st, out, i0, i1, i2, i3, P, ctx->d_pinfo, ctx->d_tw_inv, bsi, bso);
        else if (pre == 2) launch_fused_c8l2<2>(log_n, gc, st, out, i0, i1, i2, i3, P, ctx->d_pinfo, ctx->d_tw_inv, bsi, bso);
        else if (pre == 5) launch_fused_c8l2<5>(log_n, gc, st, out, i0, i1, i2, i3, P, ctx->d_pinfo, ctx->d_tw_inv, bsi, bso);
        else launch_fused_c8l2<3>(log_n, gc, st, out, i0, i1, i2, i3, P, ctx->d_pinfo, ctx->d_tw_inv, bsi, bso);
        HG_LAUNCH_CHECK(ctx);
        return HG_OK;
    }
    const int pc = k1 ? prime_chunk(ctx, batch * rb, P) : P;
    for (int j0 = 0; j0 < P; j0 += pc) {
        const int pz = P - j0 < pc ? P - j0 : pc;
        const dim3 g(N >> k2, batch, pz);
        const size_t o = (size_t)j0 * N;
        const PrimeInfo* pin = ctx->d_pinfo + j0;
        const uint2* twj = ctx->d_tw_inv + o;
        const uint32_t* j2 = i2 ? i2 + o : i2;
        const uint32_t* j3 = i3 ? i3 + o : i3;
        if (pre == 1) launch_fused_lo8<1>(k2, g, st, out + o, i0 + o, i1 + o, j2, j3, log_n, P, pin, twj, bsi, bso);
        else if (pre == 2) launch_fused_lo8<2>(k2, g, st, out + o, i0 + o, i1 + o, j2, j3, log_n, P, pin, twj);
        else if (pre == 5) launch_fused_lo8<5>(k2, g, st, out + o, i0 + o, i1 + o, j2, j3, log_n, P, pin, twj, bsi, bso);
        else launch_fused_lo8<3>(k2, g, st, out + o, i0 + o, i1 + o, j2, j3, log_n, P, pin, twj);
        HG_LAUNCH_CHECK(ctx);
        if (k1 && (rc = ntt_pass<false>(ctx, true, k1, k2, out, batch * rb, P, 0, ctx->d_tw_inv, st, j0, pz))) return rc;
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
