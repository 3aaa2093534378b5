// hg_elementwise.cu -- HBM-bound limb-major ring kernels (ring.py:114-196).
//
// One thread per coefficient walks the W words of that coefficient (word w of all
// coefficients is contiguous, so every word access is coalesced across the warp) and
// carries between words in registers.  Values are canonical residues mod 2^bits.
#include "hg_internal.cuh"

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ uint32_t mask_for(int bits) {
    return (bits & 31) ? ((1u << (bits & 31)) - 1u) : 0xffffffffu;
}

// out = a + b (or a - b) mod 2^bits           RingElement.add / sub  ring.py:114-130
template <bool SUB>
__global__ void __launch_bounds__(kThreads) add_kernel(uint32_t* __restrict__ out,
                                                       const uint32_t* __restrict__ a,
                                                       const uint32_t* __restrict__ b, int W,
                                                       int bits, int N) {
    const int i = blockIdx.x * kThreads + threadIdx.x;
    if (i >= N) return;
    uint32_t carry = SUB ? 1u : 0u;  // a - b = a + ~b + 1
    for (int w = 0; w < W; ++w) {
        uint32_t x = a[(size_t)w * N + i];
        uint32_t y = b[(size_t)w * N + i];
        if (SUB) y = ~y;
        uint64_t s = (uint64_t)x + y + carry;
        uint32_t r = (uint32_t)s;
        carry = (uint32_t)(s >> 32);
        if (w == W - 1) r &= mask_for(bits);
        out[(size_t)w * N + i] = r;
    }
}

// out = -a mod 2^bits                          RingElement.neg  ring.py:132-134
__global__ void __launch_bounds__(kThreads) neg_kernel(uint32_t* __restrict__ out,
                                                       const uint32_t* __restrict__ a, int W,
                                                       int bits, int N) {
    const int i = blockIdx.x * kThreads + threadIdx.x;
    if (i >= N) return;
    uint32_t carry = 1u;
    for (int w = 0; w < W; ++w) {
        uint64_t s = (uint64_t)(~a[(size_t)w * N + i]) + carry;
        uint32_t r = (uint32_t)s;
        carry = (uint32_t)(s >> 32);
        if (w == W - 1) r &= mask_for(bits);
        out[(size_t)w * N + i] = r;
    }
}

struct ScalarWords {
    uint32_t k[HG_MODUP_WMAX];
};

// out = a * k mod 2^bits, k given mod 2^bits as kw words (truncated schoolbook, column
// order so every output word is written once)   RingElement.scalar_mul  ring.py:136-138
__global__ void __launch_bounds__(kThreads) scalar_mul_kernel(uint32_t* __restrict__ out,
                                                              const uint32_t* __restrict__ a,
                                                              int W, int bits, int N,
                                                              ScalarWords ks, int kw) {
    const int i = blockIdx.x * kThreads + threadIdx.x;
    if (i >= N) return;
    uint64_t carry_lo = 0;  // running column carry (< 2^(32+log2 W+1))
    uint32_t carry_hi = 0;
    for (int w = 0; w < W; ++w) {
        uint64_t acc = carry_lo;
        uint32_t hi = carry_hi;
        int jmax = w < kw - 1 ? w : kw - 1;
        for (int j = 0; j <= jmax; ++j) {
            uint64_t prod = (uint64_t)a[(size_t)(w - j) * N + i] * ks.k[j];
            uint64_t s = acc + prod;
            hi += (s < acc);
            acc = s;
        }
        uint32_t r = (uint32_t)acc;
        if (w == W - 1) r &= mask_for(bits);
        out[(size_t)w * N + i] = r;
        carry_lo = (acc >> 32) | ((uint64_t)hi << 32);
        carry_hi = 0;
    }
}

// out (out_bits) = a mod 2^out_bits              RingElement.reduce_to  ring.py:168-175
// out (out_bits) = sign-extended a (in_bits)     RingElement.lift_centered_to  ring.py:177-182
template <bool LIFT>
__global__ void __launch_bounds__(kThreads) resize_kernel(uint32_t* __restrict__ out, int out_bits,
                                                          const uint32_t* __restrict__ a,
                                                          int in_bits, int N) {
    const int i = blockIdx.x * kThreads + threadIdx.x;
    if (i >= N) return;
    const int Wo = (out_bits + 31) >> 5, Wi = (in_bits + 31) >> 5;
    uint32_t fill = 0;
    if (LIFT) {
        // centered(): c > 2^(in_bits-1) is negative; c == 2^(in_bits-1) stays positive
        // (ring.py:106-110).  Negative <=> top bit set and lower bits not all zero.
        uint32_t topw = a[(size_t)(Wi - 1) * N + i] & mask_for(in_bits);
        bool topbit = (topw >> ((in_bits - 1) & 31)) & 1u;
        bool rest = (topw & ~(1u << ((in_bits - 1) & 31))) != 0;
        for (int w = 0; w < Wi - 1 && !rest; ++w) rest = a[(size_t)w * N + i] != 0;
        if (topbit && rest) fill = 0xffffffffu;
    }
    for (int w = 0; w < Wo; ++w) {
        uint32_t r;
        if (w < Wi) {
            r = a[(size_t)w * N + i];
            if (w == Wi - 1) {
                uint32_t m = mask_for(in_bits);
                r = (r & m) | (fill & ~m);
            }
        } else {
            r = fill;
        }
        if (w == Wo - 1) r &= mask_for(out_bits);
        out[(size_t)w * N + i] = r;
    }
}

// out (out_bits) = ((a + 2^(shift-1)) >> shift) mod 2^out_bits   divide_round  ring.py:184-196
__global__ void __launch_bounds__(kThreads) divide_round_kernel(uint32_t* __restrict__ out,
                                                                int out_bits,
                                                                const uint32_t* __restrict__ a,
                                                                int in_bits, int shift, int N) {
    const int i = blockIdx.x * kThreads + threadIdx.x;
    if (i >= N) return;
    const int Wi = (in_bits + 31) >> 5, Wo = (out_bits + 31) >> 5;
    const int sw = shift >> 5, sb = shift & 31;
    const int rc = shift > 0 ? (shift - 1) >> 5 : -1;
    const uint32_t rbit = shift > 0 ? 1u << ((shift - 1) & 31) : 0u;
    // value words v[t] = (a + round)[t] for t in [0, Wi]; word Wi holds the final carry
    uint32_t carry = 0;
    uint32_t prev = 0;
    const int T = sw + Wo + 1;
    for (int t = 0; t < T; ++t) {
        uint32_t x = 0;
        if (t < Wi) {
            x = a[(size_t)t * N + i];
            if (t == Wi - 1) x &= mask_for(in_bits);
        }
        uint64_t s = (uint64_t)x + carry + (t == rc ? rbit : 0u);
        uint32_t word = (uint32_t)s;
        carry = (uint32_t)(s >> 32);
        if (sb == 0) {
            if (t >= sw && t - sw < Wo) {
                int u = t - sw;
                uint32_t o = word;
                if (u == Wo - 1) o &= mask_for(out_bits);
                out[(size_t)u * N + i] = o;
            }
        } else if (t > sw && t - sw - 1 < Wo) {
            int u = t - sw - 1;
            uint32_t o = (prev >> sb) | (word << (32 - sb));
            if (u == Wo - 1) o &= mask_for(out_bits);
            out[(size_t)u * N + i] = o;
        }
        prev = word;
    }
}

// out[i] = (+/-) a[i * kinv mod 2N]  for x -> x^k            automorphism  ring.py:152-166
__global__ void __launch_bounds__(kThreads) automorphism_kernel(uint32_t* __restrict__ out,
                                                                const uint32_t* __restrict__ a,
                                                                int W, int bits, int N,
                                                                int64_t kinv) {
    const int i = blockIdx.x * kThreads + threadIdx.x;
    if (i >= N) return;
    int64_t j = ((int64_t)i * kinv) & (2ll * N - 1);
    bool neg = j >= N;
    int src = (int)(neg ? j - N : j);
    uint32_t carry = 1u;
    for (int w = 0; w < W; ++w) {
        uint32_t x = a[(size_t)w * N + src];
        uint32_t r;
        if (neg) {
            uint64_t s = (uint64_t)(~x) + carry;
            r = (uint32_t)s;
            carry = (uint32_t)(s >> 32);
        } else {
            r = x;
        }
        if (w == W - 1) r &= mask_for(bits);
        out[(size_t)w * N + i] = r;
    }
}

// The CRT-finish addends of a batched rotation (hg_rns.cu automorph_batch_impl), item g =
// blockIdx.y: dst[2g] = phi(c0_g) (+ c0_g with acc), dst[2g+1] = c1_g with acc, else 0 -- so the
// key switch's epilogue writes phi(c0) + e0 (+ c0) and e1 (+ c1) straight to the outputs
struct AutoItems {
    const uint32_t* c0[4];
    const uint32_t* c1[4];
};
__global__ void __launch_bounds__(kThreads) automorph_addend_kernel(uint32_t* __restrict__ dst, AutoItems it,
                                                                    int acc, int W, int bits, int N,
                                                                    int64_t kinv) {
    const int i = blockIdx.x * kThreads + threadIdx.x;
    if (i >= N) return;
    const int g = blockIdx.y;
    const uint32_t* __restrict__ a = it.c0[g];
    const uint32_t* __restrict__ c1 = it.c1[g];
    uint32_t* __restrict__ d0 = dst + (size_t)(2 * g) * W * N;
    uint32_t* __restrict__ d1 = d0 + (size_t)W * N;
    int64_t j = ((int64_t)i * kinv) & (2ll * N - 1);
    const bool neg = j >= N;
    const int src = (int)(neg ? j - N : j);
    uint32_t ncarry = 1u;   // -x = ~x + 1
    uint64_t carry = 0;
    for (int w = 0; w < W; ++w) {
        const size_t o = (size_t)w * N;
        uint32_t x = a[o + src];
        if (neg) {
            uint64_t s = (uint64_t)(~x) + ncarry;
            x = (uint32_t)s;
            ncarry = (uint32_t)(s >> 32);
        }
        uint64_t s = carry + x + (acc ? a[o + i] : 0u);
        uint32_t r = (uint32_t)s;
        carry = s >> 32;
        uint32_t r1 = acc ? c1[o + i] : 0u;
        if (w == W - 1) {
            r &= mask_for(bits);
            r1 &= mask_for(bits);
        }
        d0[o + i] = r;
        d1[o + i] = r1;
    }
}

// out (+)= sum of up to kSumTerms polys: one thread per coefficient, 64-bit column sums with
// the carry taken word to word; the loads of one word over all terms are independent
constexpr int kSumTerms = 64;
struct SumTerms {
    const uint32_t* p[kSumTerms];
};
__global__ void __launch_bounds__(kThreads) sum_kernel(uint32_t* __restrict__ out, SumTerms t,
                                                       int count, int accumulate, int W, int bits,
                                                       int N) {
    const int i = blockIdx.x * kThreads + threadIdx.x;
    if (i >= N) return;
    uint64_t carry = 0;
    for (int w = 0; w < W; ++w) {
        const size_t o = (size_t)w * N + i;
        uint64_t acc = carry + (accumulate ? out[o] : 0u);
#pragma unroll 8
        for (int k = 0; k < count; ++k) acc += __ldg(t.p[k] + o);
        uint32_t r = (uint32_t)acc;
        if (w == W - 1) r &= mask_for(bits);
        out[o] = r;
        carry = acc >> 32;
    }
}

inline dim3 grid_for(int N) { return dim3((N + kThreads - 1) / kThreads); }

int64_t inv_mod_pow2(int64_t k, int64_t n2) {
    uint64_t x = (uint64_t)k, inv = x;
    for (int it = 0; it < 6; ++it) inv *= 2 - x * inv;
    return (int64_t)(inv & (uint64_t)(n2 - 1));
}

// ---- batched ciphertext-level kernels: grid.y walks up to kPolys polys per launch -------------
constexpr int kPolys = 16;
struct PolyPtrs {
    const uint32_t* a[kPolys];
    const uint32_t* b[kPolys];
    uint32_t* out[kPolys];
};
template <typename T>
__device__ __forceinline__ T sel16(const T (&v)[kPolys], int k) {
    T r = v[0];
#pragma unroll
    for (int q = 1; q < kPolys; ++q) r = k == q ? v[q] : r;   // select, not a dynamic index
    return r;
}

// divide_round over a batch of polys                 rescale  ckks.py:197-224
__device__ __forceinline__ void divide_round_one(uint32_t* __restrict__ out, int out_bits,
                                                 const uint32_t* __restrict__ a, int in_bits,
                                                 int shift, int N, int i) {
    const int Wi = (in_bits + 31) >> 5, Wo = (out_bits + 31) >> 5;
    const int sw = shift >> 5, sb = shift & 31;
    const int rc = shift > 0 ? (shift - 1) >> 5 : -1;
    const uint32_t rbit = shift > 0 ? 1u << ((shift - 1) & 31) : 0u;
    uint32_t carry = 0, prev = 0;
    const int T = sw + Wo + 1;
    for (int t = 0; t < T; ++t) {
        uint32_t x = 0;
        if (t < Wi) {
            x = a[(size_t)t * N + i];
            if (t == Wi - 1) x &= mask_for(in_bits);
        }
        const uint64_t s = (uint64_t)x + carry + (t == rc ? rbit : 0u);
        const uint32_t word = (uint32_t)s;
        carry = (uint32_t)(s >> 32);
        const int u = sb ? t - sw - 1 : t - sw;
        if (u >= 0 && u < Wo) {
            uint32_t o = sb ? __funnelshift_r(prev, word, sb) : word;
            if (u == Wo - 1) o &= mask_for(out_bits);
            out[(size_t)u * N + i] = o;
        }
        prev = word;
    }
}

__global__ void __launch_bounds__(kThreads) rescale_batch_kernel(PolyPtrs p, int out_bits, int in_bits,
                                                                 int shift, int N) {
    const int i = blockIdx.x * kThreads + threadIdx.x;
    if (i >= N) return;
    divide_round_one(sel16(p.out, blockIdx.y), out_bits, sel16(p.a, blockIdx.y), in_bits, shift, N, i);
}

// a +/- b over a batch of poly pairs                  add / sub  ckks.py:108-125
template <bool SUB>
__global__ void __launch_bounds__(kThreads) add_batch_kernel(PolyPtrs p, int W, int bits, int N) {
    const int i = blockIdx.x * kThreads + threadIdx.x;
    if (i >= N) return;
    const uint32_t* a = sel16(p.a, blockIdx.y);
    const uint32_t* b = sel16(p.b, blockIdx.y);
    uint32_t* out = sel16(p.out, blockIdx.y);
    uint32_t carry = SUB ? 1u : 0u;
    for (int w = 0; w < W; ++w) {
        uint32_t y = b[(size_t)w * N + i];
        if (SUB) y = ~y;
        const uint64_t s = (uint64_t)a[(size_t)w * N + i] + y + carry;
        uint32_t r = (uint32_t)s;
        carry = (uint32_t)(s >> 32);
        if (w == W - 1) r &= mask_for(bits);
        out[(size_t)w * N + i] = r;
    }
}

// HeEngine.mult_const (an encode_constant plaintext: a single coefficient k, ckks.py:351-356
// with encoding.py:82-90) followed by its rescale, in one pass: the words of (c * k mod 2^level)
// -- |k| < 2^32, negatives as the two's-complement negation of c * |k| -- stream straight into
// divide_round by `shift`
__global__ void __launch_bounds__(kThreads) mult_const_rescale_kernel(PolyPtrs p, int level, int shift,
                                                                      uint32_t kabs, int negative, int N) {
    const int i = blockIdx.x * kThreads + threadIdx.x;
    if (i >= N) return;
    const uint32_t* a = sel16(p.a, blockIdx.y);
    uint32_t* out = sel16(p.out, blockIdx.y);
    const int out_bits = level - shift;
    const int Wi = (level + 31) >> 5, Wo = (out_bits + 31) >> 5;
    const int sw = shift >> 5, sb = shift & 31;
    const int rc = shift > 0 ? (shift - 1) >> 5 : -1;
    const uint32_t rbit = shift > 0 ? 1u << ((shift - 1) & 31) : 0u;
    uint64_t pc = 0;                      // product column carry (< 2^32)
    uint32_t nc = negative ? 1u : 0u;     // negation carry: -x = ~x + 1
    uint32_t carry = 0, prev = 0;
    const int T = sw + Wo + 1;
    for (int t = 0; t < T; ++t) {
        uint32_t x = 0;
        if (t < Wi) {
            const uint64_t pr = (uint64_t)a[(size_t)t * N + i] * kabs + pc;
            pc = pr >> 32;
            x = (uint32_t)pr;
            if (negative) {
                const uint64_t ns = (uint64_t)(~x) + nc;
                x = (uint32_t)ns;
                nc = (uint32_t)(ns >> 32);
            }
            if (t == Wi - 1) x &= mask_for(level);
        }
        const uint64_t s = (uint64_t)x + carry + (t == rc ? rbit : 0u);
        const uint32_t word = (uint32_t)s;
        carry = (uint32_t)(s >> 32);
        const int u = sb ? t - sw - 1 : t - sw;
        if (u >= 0 && u < Wo) {
            uint32_t o = sb ? __funnelshift_r(prev, word, sb) : word;
            if (u == Wo - 1) o &= mask_for(out_bits);
            out[(size_t)u * N + i] = o;
        }
        prev = word;
    }
}

// ---- decode: centered coefficients -> float64 (encoding.py:93-105) -------------------------
// The reference converts each centered coefficient c to float with Python's float(int) --
// round to nearest, ties to even -- after shifting every coefficient right (floor) by
// s = bitlen(max |c|) - 500 when that bit length exceeds 960.  These kernels reproduce that
// bit for bit: magnitudes are read word by word from the two's-complement canonical words,
// s comes from a device-wide max of the bit lengths, and the quotient is rounded from a
// 64-bit window plus sticky / all-ones flags of the bits below it.

// Word w of |centered(c)| for a coefficient whose canonical words are a[w*N + i].
struct CenteredMag {
    const uint32_t* a;
    int N, i, W, bits, z;  // z: lowest nonzero word (negation carry stops there)
    bool neg;
    __device__ uint32_t word(int w) const {
        if (w < 0 || w >= W) return 0u;
        uint32_t x = a[(size_t)w * N + i];
        if (neg) x = w < z ? 0u : (w == z ? 0u - x : ~x);
        if (w == W - 1) x &= mask_for(bits);
        return x;
    }
};

__device__ __forceinline__ CenteredMag centered_mag(const uint32_t* a, int W, int bits, int N, int i) {
    CenteredMag m{a, N, i, W, bits, W, false};
    // centered: c > 2^(bits-1) -> c - 2^bits (ring.py:106-110); c == 2^(bits-1) stays positive
    const int tb = (bits - 1) & 31;
    const bool top = (a[(size_t)(W - 1) * N + i] >> tb) & 1u;
    int z = W;
    for (int w = 0; w < W; ++w) {
        uint32_t x = a[(size_t)w * N + i];
        if (w == W - 1) x &= mask_for(bits);
        if (x) { z = w; break; }
    }
    bool above_half = false;
    if (top) {  // any bit below bit bits-1 set?
        const uint32_t topw = a[(size_t)(W - 1) * N + i] & mask_for(bits) & ((1u << tb) - 1u);
        above_half = topw != 0u || z < W - 1;
    }
    m.neg = above_half;
    m.z = z;
    return m;
}

// bit length of the magnitude (0 for zero)
__device__ __forceinline__ int mag_bitlen(const CenteredMag& m) {
    for (int w = m.W - 1; w >= 0; --w) {
        uint32_t x = m.word(w);
        if (x) return 32 * w + 32 - __clz(x);
    }
    return 0;
}

// 64 bits of the magnitude starting at bit `lo` (bits past the top read as 0)
__device__ __forceinline__ uint64_t mag_bits64(const CenteredMag& m, int lo) {
    const int w0 = lo >> 5, sh = lo & 31;
    uint64_t v = (uint64_t)m.word(w0) | ((uint64_t)m.word(w0 + 1) << 32);
    if (sh) v = (v >> sh) | ((uint64_t)m.word(w0 + 2) << (64 - sh));
    return v;
}

// any / all bits of the magnitude in [lo, hi)
__device__ __forceinline__ void mag_range_flags(const CenteredMag& m, int lo, int hi, bool& any,
                                                bool& all) {
    any = false;
    all = true;
    for (int w = lo >> 5; w << 5 < hi; ++w) {
        const int b0 = max(lo, w << 5) - (w << 5), b1 = min(hi, (w << 5) + 32) - (w << 5);
        const uint32_t mask = (b1 - b0 == 32) ? 0xffffffffu : (((1u << (b1 - b0)) - 1u) << b0);
        const uint32_t x = m.word(w) & mask;
        any |= x != 0u;
        all &= x == mask;
    }
}

__global__ void __launch_bounds__(kThreads) decode_bitlen_kernel(const uint32_t* __restrict__ a, int W,
                                                                 int bits, int N, int* __restrict__ maxlen) {
    const int i = blockIdx.x * kThreads + threadIdx.x;
    int bl = 0;
    if (i < N) bl = mag_bitlen(centered_mag(a, W, bits, N, i));
    for (int o = 16; o; o >>= 1) bl = max(bl, __shfl_xor_sync(0xffffffffu, bl, o));
    if ((threadIdx.x & 31) == 0 && bl) atomicMax(maxlen, bl);
}

// out[i] = float(centered(c_i) >> s), s = bitlen - 500 if bitlen > 960 else 0 (maxlen[0] holds
// the bit length on entry; maxlen[1] receives s)
__global__ void __launch_bounds__(kThreads) decode_double_kernel(const uint32_t* __restrict__ a, int W,
                                                                 int bits, int N, int* __restrict__ maxlen,
                                                                 double* __restrict__ out) {
    const int i = blockIdx.x * kThreads + threadIdx.x;
    const int top = maxlen[0];
    const int s = top > 960 ? top - 500 : 0;
    if (i == 0) maxlen[1] = s;
    if (i >= N) return;
    const CenteredMag m = centered_mag(a, W, bits, N, i);
    const int bl = mag_bitlen(m);
    // floor(c / 2^s): q = mag >> s for c >= 0, -(mag >> s) - (low s bits nonzero) for c < 0
    bool low_any = false, low_all = true;
    if (s > 0) mag_range_flags(m, 0, min(s, bl), low_any, low_all);
    const bool add1 = m.neg && low_any;
    const int hq = bl - s;  // bit length of q
    double r;
    if (hq <= 64) {
        const uint64_t q = hq > 0 ? mag_bits64(m, s) & (hq == 64 ? ~0ull : ((1ull << hq) - 1ull)) : 0ull;
        if (add1 && q == ~0ull)
            r = 18446744073709551616.0;  // 2^64
        else
            r = __ull2double_rn(q + (add1 ? 1ull : 0ull));
    } else {
        const int lo = s + hq - 64;  // window = bits [lo, lo + 64) of mag, top bit set
        uint64_t win = mag_bits64(m, lo);
        bool any, all;
        mag_range_flags(m, s, lo, any, all);
        bool sticky = any;
        int e = lo - s;
        if (add1) {
            if (all) {
                sticky = false;
                if (++win == 0ull) {  // 2^64 * 2^e exactly
                    win = 1ull << 63;
                    e += 1;
                }
            } else {
                sticky = true;
            }
        }
        uint64_t mant = win >> 11;
        const uint32_t rem = (uint32_t)(win & 0x7ffu);
        if (rem > 0x400u || (rem == 0x400u && (sticky || (mant & 1ull)))) mant += 1ull;
        r = ldexp((double)mant, e + 11);
    }
    out[i] = m.neg ? -r : r;
}

}  // namespace

int hg_ew_to_double(hg_ctx* ctx, double* out, int* aux, const uint32_t* a, int bits, cudaStream_t st) {
    const int W = words_for_bits(bits);
    HgTimed tm(ctx, st, HG_K_ELEMENTWISE, (double)ctx->N);
    if (cudaMemsetAsync(aux, 0, 2 * sizeof(int), st) != cudaSuccess)
        return hg_fail(HG_ECUDA, "hg_poly_to_double: memset failed");
    decode_bitlen_kernel<<<grid_for(ctx->N), kThreads, 0, st>>>(a, W, bits, ctx->N, aux);
    HG_LAUNCH_CHECK(ctx);
    decode_double_kernel<<<grid_for(ctx->N), kThreads, 0, st>>>(a, W, bits, ctx->N, aux, out);
    HG_LAUNCH_CHECK(ctx);
    return HG_OK;
}

// ---- internal entry points (used by the fused drivers in hg_rns.cu) --------------------------
int hg_ew_add(hg_ctx* ctx, uint32_t* out, const uint32_t* a, const uint32_t* b, int bits,
              bool subtract, cudaStream_t st) {
    int W = words_for_bits(bits);
    HgTimed tm(ctx, st, HG_K_ELEMENTWISE, (double)ctx->N);
    if (subtract)
        add_kernel<true><<<grid_for(ctx->N), kThreads, 0, st>>>(out, a, b, W, bits, ctx->N);
    else
        add_kernel<false><<<grid_for(ctx->N), kThreads, 0, st>>>(out, a, b, W, bits, ctx->N);
    HG_LAUNCH_CHECK(ctx);
    return HG_OK;
}

int hg_ew_divide_round(hg_ctx* ctx, uint32_t* out, int out_bits, const uint32_t* a, int in_bits,
                       int shift, cudaStream_t st) {
    HgTimed tm(ctx, st, HG_K_ELEMENTWISE, (double)ctx->N);
    divide_round_kernel<<<grid_for(ctx->N), kThreads, 0, st>>>(out, out_bits, a, in_bits, shift,
                                                               ctx->N);
    HG_LAUNCH_CHECK(ctx);
    return HG_OK;
}

int hg_ew_automorphism(hg_ctx* ctx, uint32_t* out, const uint32_t* a, int bits, int64_t k,
                       cudaStream_t st) {
    int64_t n2 = 2ll * ctx->N;
    int64_t kk = ((k % n2) + n2) % n2;
    if ((kk & 1) == 0) return hg_fail(HG_EINVAL, "automorphism exponent must be odd");
    HgTimed tm(ctx, st, HG_K_ELEMENTWISE, (double)ctx->N);
    automorphism_kernel<<<grid_for(ctx->N), kThreads, 0, st>>>(out, a, words_for_bits(bits), bits,
                                                               ctx->N, inv_mod_pow2(kk, n2));
    HG_LAUNCH_CHECK(ctx);
    return HG_OK;
}

int hg_ew_automorph_addends(hg_ctx* ctx, uint32_t* dst, const uint32_t* const* c0s,
                            const uint32_t* const* c1s, int G, int bits, int64_t k, bool acc,
                            cudaStream_t st) {
    int64_t n2 = 2ll * ctx->N;
    int64_t kk = ((k % n2) + n2) % n2;
    if ((kk & 1) == 0 || G < 1 || G > 4) return hg_fail(HG_EINVAL, "automorph addends: bad arguments");
    AutoItems it{};
    for (int g = 0; g < G; ++g) {
        it.c0[g] = c0s[g];
        it.c1[g] = c1s[g];
    }
    HgTimed tm(ctx, st, HG_K_ELEMENTWISE, (double)ctx->N * G);
    dim3 grid = grid_for(ctx->N);
    grid.y = G;
    automorph_addend_kernel<<<grid, kThreads, 0, st>>>(dst, it, acc ? 1 : 0, words_for_bits(bits), bits,
                                                       ctx->N, inv_mod_pow2(kk, n2));
    HG_LAUNCH_CHECK(ctx);
    return HG_OK;
}

// ---- C-ABI -------------------------------------------------------------------------------------
#define HG_CHECK_ARGS(cond, msg) \
    do {                          \
        if (!(cond)) return hg_fail(HG_EINVAL, msg); \
    } while (0)

extern "C" int hg_poly_add(hg_ctx* ctx, uint32_t* out, const uint32_t* a, const uint32_t* b,
                           int bits, void* stream) {
    HG_CHECK_ARGS(ctx && out && a && b && bits >= 1, "hg_poly_add: bad arguments");
    return hg_ew_add(ctx, out, a, b, bits, false, (cudaStream_t)stream);
}

extern "C" int hg_poly_sub(hg_ctx* ctx, uint32_t* out, const uint32_t* a, const uint32_t* b,
                           int bits, void* stream) {
    HG_CHECK_ARGS(ctx && out && a && b && bits >= 1, "hg_poly_sub: bad arguments");
    return hg_ew_add(ctx, out, a, b, bits, true, (cudaStream_t)stream);
}

extern "C" int hg_poly_sum(hg_ctx* ctx, uint32_t* out, const uint32_t* const* terms, int count,
                           int bits, void* stream) {
    HG_CHECK_ARGS(ctx && out && terms && count >= 1 && bits >= 1, "hg_poly_sum: bad arguments");
    const int W = words_for_bits(bits);
    HgTimed tm(ctx, (cudaStream_t)stream, HG_K_ELEMENTWISE, (double)ctx->N);
    for (int k0 = 0; k0 < count; k0 += kSumTerms) {
        SumTerms t{};
        const int c = count - k0 < kSumTerms ? count - k0 : kSumTerms;
        for (int k = 0; k < c; ++k) {
            HG_CHECK_ARGS(terms[k0 + k] != nullptr, "hg_poly_sum: null term");
            // a later chunk reads `out` as its running sum, so no term may alias it
            HG_CHECK_ARGS(terms[k0 + k] != out || k0 == 0, "hg_poly_sum: term aliases the output");
            t.p[k] = terms[k0 + k];
        }
        sum_kernel<<<grid_for(ctx->N), kThreads, 0, (cudaStream_t)stream>>>(out, t, c, k0 > 0, W, bits,
                                                                              ctx->N);
        HG_LAUNCH_CHECK(ctx);
    }
    return HG_OK;
}

extern "C" int hg_poly_neg(hg_ctx* ctx, uint32_t* out, const uint32_t* a, int bits,
                           void* stream) {
    HG_CHECK_ARGS(ctx && out && a && bits >= 1, "hg_poly_neg: bad arguments");
    HgTimed tm(ctx, (cudaStream_t)stream, HG_K_ELEMENTWISE, (double)ctx->N);
    neg_kernel<<<grid_for(ctx->N), kThreads, 0, (cudaStream_t)stream>>>(out, a, words_for_bits(bits),
                                                                        bits, ctx->N);
    HG_LAUNCH_CHECK(ctx);
    return HG_OK;
}

extern "C" int hg_poly_scalar_mul(hg_ctx* ctx, uint32_t* out, const uint32_t* a, int bits,
                                  const uint32_t* k_words_host, int kw, void* stream) {
    HG_CHECK_ARGS(ctx && out && a && bits >= 1 && k_words_host && kw >= 1,
                  "hg_poly_scalar_mul: bad arguments");
    int W = words_for_bits(bits);
    HG_CHECK_ARGS(kw <= W && W <= HG_MODUP_WMAX, "hg_poly_scalar_mul: scalar wider than the ring");
    ScalarWords ks{};
    for (int j = 0; j < kw; ++j) ks.k[j] = k_words_host[j];
    // an out-of-place product: `out` must not alias `a` (columns read lower words)
    HG_CHECK_ARGS(out != a || kw == 1, "hg_poly_scalar_mul: in-place needs a one-word scalar");
    HgTimed tm(ctx, (cudaStream_t)stream, HG_K_ELEMENTWISE, (double)ctx->N);
    scalar_mul_kernel<<<grid_for(ctx->N), kThreads, 0, (cudaStream_t)stream>>>(out, a, W, bits,
                                                                               ctx->N, ks, kw);
    HG_LAUNCH_CHECK(ctx);
    return HG_OK;
}

extern "C" int hg_poly_reduce_to(hg_ctx* ctx, uint32_t* out, int out_bits, const uint32_t* a,
                                 int in_bits, void* stream) {
    HG_CHECK_ARGS(ctx && out && a && out_bits >= 1 && out_bits <= in_bits,
                  "hg_poly_reduce_to: bad arguments");
    HgTimed tm(ctx, (cudaStream_t)stream, HG_K_ELEMENTWISE, (double)ctx->N);
    resize_kernel<false><<<grid_for(ctx->N), kThreads, 0, (cudaStream_t)stream>>>(out, out_bits, a,
                                                                                  in_bits, ctx->N);
    HG_LAUNCH_CHECK(ctx);
    return HG_OK;
}

extern "C" int hg_poly_lift_centered(hg_ctx* ctx, uint32_t* out, int out_bits, const uint32_t* a,
                                     int in_bits, void* stream) {
    HG_CHECK_ARGS(ctx && out && a && in_bits >= 1 && out_bits >= in_bits,
                  "hg_poly_lift_centered: bad arguments");
    HgTimed tm(ctx, (cudaStream_t)stream, HG_K_ELEMENTWISE, (double)ctx->N);
    resize_kernel<true><<<grid_for(ctx->N), kThreads, 0, (cudaStream_t)stream>>>(out, out_bits, a,
                                                                                 in_bits, ctx->N);
    HG_LAUNCH_CHECK(ctx);
    return HG_OK;
}

extern "C" int hg_poly_divide_round(hg_ctx* ctx, uint32_t* out, int out_bits, const uint32_t* a,
                                    int in_bits, int shift, void* stream) {
    HG_CHECK_ARGS(ctx && out && a && out_bits >= 1 && in_bits >= 1 && shift >= 0,
                  "hg_poly_divide_round: bad arguments");
    HG_CHECK_ARGS(out != a, "hg_poly_divide_round: out must not alias the input");
    return hg_ew_divide_round(ctx, out, out_bits, a, in_bits, shift, (cudaStream_t)stream);
}

extern "C" int hg_poly_to_double(hg_ctx* ctx, double* out, int* aux, const uint32_t* a, int bits,
                                 void* stream) {
    HG_CHECK_ARGS(ctx && out && aux && a && bits >= 1, "hg_poly_to_double: bad arguments");
    return hg_ew_to_double(ctx, out, aux, a, bits, (cudaStream_t)stream);
}

extern "C" int hg_poly_automorphism(hg_ctx* ctx, uint32_t* out, const uint32_t* a, int bits,
                                    int64_t k, void* stream) {
    HG_CHECK_ARGS(ctx && out && a && bits >= 1 && out != a, "hg_poly_automorphism: bad arguments");
    return hg_ew_automorphism(ctx, out, a, bits, k, (cudaStream_t)stream);
}

// ---- batched ciphertext-level entry points (arrays of device pointers, host arrays) ---------------
// Each takes `count` ciphertexts as (c0, c1) pointer arrays and writes (out0, out1); polys go
// kPolys per launch.  Outputs may not alias inputs.
namespace {
template <typename Launch>
int over_polys(int count, const uint32_t* const* a0, const uint32_t* const* a1, const uint32_t* const* b0,
               const uint32_t* const* b1, uint32_t* const* o0, uint32_t* const* o1, Launch launch) {
    const int polys = 2 * count;
    for (int k0 = 0; k0 < polys; k0 += kPolys) {
        PolyPtrs p{};
        const int c = polys - k0 < kPolys ? polys - k0 : kPolys;
        for (int k = 0; k < c; ++k) {
            const int q = (k0 + k) >> 1, h = (k0 + k) & 1;
            p.a[k] = h ? a1[q] : a0[q];
            p.b[k] = b0 ? (h ? b1[q] : b0[q]) : nullptr;
            p.out[k] = h ? o1[q] : o0[q];
            if (!p.a[k] || !p.out[k] || (b0 && !p.b[k])) return hg_fail(HG_EINVAL, "null ciphertext pointer");
        }
        if (int rc = launch(p, c)) return rc;
    }
    return HG_OK;
}
}  // namespace

/* rescale (ckks.py:197-224) of `count` ciphertexts at `level` by `bits`. */
extern "C" int hg_ct_rescale_batch(hg_ctx* ctx, int count, const uint32_t* const* c0s,
                                   const uint32_t* const* c1s, int level, int bits,
                                   uint32_t* const* out0s, uint32_t* const* out1s, void* stream) {
    HG_CHECK_ARGS(ctx && count >= 0 && (!count || (c0s && c1s && out0s && out1s)) && bits >= 1 &&
                  bits < level, "hg_ct_rescale_batch: bad arguments");
    cudaStream_t st = (cudaStream_t)stream;
    HgTimed tm(ctx, st, HG_K_ELEMENTWISE, (double)ctx->N * 2 * count);
    return over_polys(count, c0s, c1s, nullptr, nullptr, out0s, out1s, [&](const PolyPtrs& p, int c) {
        dim3 grid = grid_for(ctx->N);
        grid.y = c;
        rescale_batch_kernel<<<grid, kThreads, 0, st>>>(p, level - bits, level, bits, ctx->N);
        HG_LAUNCH_CHECK(ctx);
        return HG_OK;
    });
}

/* add / sub (ckks.py:108-125) of `count` aligned ciphertext pairs at `bits`. */
extern "C" int hg_ct_add_batch(hg_ctx* ctx, int count, const uint32_t* const* a0s, const uint32_t* const* a1s,
                               const uint32_t* const* b0s, const uint32_t* const* b1s, int bits, int subtract,
                               uint32_t* const* out0s, uint32_t* const* out1s, void* stream) {
    HG_CHECK_ARGS(ctx && count >= 0 && (!count || (a0s && a1s && b0s && b1s && out0s && out1s)) && bits >= 1,
                  "hg_ct_add_batch: bad arguments");
    cudaStream_t st = (cudaStream_t)stream;
    const int W = words_for_bits(bits);
    HgTimed tm(ctx, st, HG_K_ELEMENTWISE, (double)ctx->N * 2 * count);
    return over_polys(count, a0s, a1s, b0s, b1s, out0s, out1s, [&](const PolyPtrs& p, int c) {
        dim3 grid = grid_for(ctx->N);
        grid.y = c;
        if (subtract) add_batch_kernel<true><<<grid, kThreads, 0, st>>>(p, W, bits, ctx->N);
        else add_batch_kernel<false><<<grid, kThreads, 0, st>>>(p, W, bits, ctx->N);
        HG_LAUNCH_CHECK(ctx);
        return HG_OK;
    });
}

/* HeEngine.mult_const: product with the integer constant k (|k| < 2^32), then rescale by
   `shift` (the constant's scale), for `count` ciphertexts at `level`; one pass per poly. */
extern "C" int hg_ct_mult_const_rescale_batch(hg_ctx* ctx, int count, const uint32_t* const* c0s,
                                              const uint32_t* const* c1s, int level, int64_t k,
                                              int shift, uint32_t* const* out0s, uint32_t* const* out1s,
                                              void* stream) {
    HG_CHECK_ARGS(ctx && count >= 0 && (!count || (c0s && c1s && out0s && out1s)) && shift >= 1 &&
                  shift < level && k > -(1ll << 32) && k < (1ll << 32),
                  "hg_ct_mult_const_rescale_batch: bad arguments");
    cudaStream_t st = (cudaStream_t)stream;
    const uint32_t kabs = (uint32_t)(k < 0 ? -k : k);
    HgTimed tm(ctx, st, HG_K_ELEMENTWISE, (double)ctx->N * 2 * count);
    return over_polys(count, c0s, c1s, nullptr, nullptr, out0s, out1s, [&](const PolyPtrs& p, int c) {
        dim3 grid = grid_for(ctx->N);
        grid.y = c;
        mult_const_rescale_kernel<<<grid, kThreads, 0, st>>>(p, level, shift, kabs, k < 0 ? 1 : 0, ctx->N);
        HG_LAUNCH_CHECK(ctx);
        return HG_OK;
    });
}
