// hg_rns.cu -- the exact product engine: ModUp (radix 2^32 -> RNS residues), pointwise
// Montgomery products in the NTT domain, and the CRT reconstruction that emits a bit window
// of the exact negacyclic convolution.  Also the key-switch / ciphertext-multiply drivers.
//
// Reference semantics replaced here:
//   ring.negacyclic_mul / RingElement.mul / mul_mod     ring.py:46-65, 140-150
//   ckks._keyswitch                                     ckks.py:187-194
//   ckks.mult (tensor + relinearise) + rescale          ckks.py:166-184, 197-224, 310-313
//   ckks._apply_automorphism                            ckks.py:247-253
#include "hg_internal.cuh"

#include <chrono>
#include <cmath>
#include <cstdio>

int hg_ntt_launch(hg_ctx* ctx, uint32_t* data, int rows, int P, int prime_offset, bool forward,
                  cudaStream_t stream);
int hg_ew_add(hg_ctx* ctx, uint32_t* out, const uint32_t* a, const uint32_t* b, int bits,
              bool subtract, cudaStream_t stream);
int hg_ew_divide_round(hg_ctx* ctx, uint32_t* out, int out_bits, const uint32_t* a,
                       int in_bits, int shift, cudaStream_t stream);
int hg_ew_automorph_addends(hg_ctx* ctx, uint32_t* dst, const uint32_t* const* c0s,
                            const uint32_t* const* c1s, int G, int bits, int64_t k, bool acc,
                            cudaStream_t st);
int hg_ew_automorphism(hg_ctx* ctx, uint32_t* out, const uint32_t* a, int bits, int64_t k,
                       cudaStream_t stream);
int hg_intt_fused(hg_ctx* ctx, int pre, uint32_t* out, const uint32_t* i0, const uint32_t* i1,
                  const uint32_t* i2, const uint32_t* i3, int P, cudaStream_t st, int batch = 1);
// pointwise product fused into the inverse NTT unless HG_NO_FUSE is set (A/B checks)
static bool fuse_pointwise() {
    static const bool on = getenv("HG_NO_FUSE") == nullptr;
    return on;
}

namespace {

constexpr int kModupThreads = 128;
constexpr int kCrtThreads = 64;

struct OperandSet {
    const uint32_t* words[4];
    int bits[4];
    int is_signed[4];
};
struct OutSet {
    uint32_t* out[8];   // up to 8 through the pipelined CRT; the older kernels take 4 per launch
};

// ---- ModUp ---------------------------------------------------------------------------------
// One thread per coefficient; the coefficient's W words are staged in shared memory
// ([W][threads], conflict-free), then reduced mod each prime with a 64-bit multiply-
// accumulate against 2^(32w) mod p (folded every 2 products to stay below 2^64).
// gridDim.y selects the operand; output rows [y][P][N].  If automorph_kinv != 0 the
// coefficient order is permuted on load: out[i] = (+/-) in[i * kinv mod 2N] (x -> x^k).
__global__ void __launch_bounds__(kModupThreads) modup_kernel(
    OperandSet ops, int N, int log_n, const PrimeInfo* __restrict__ pinfo,
    const uint32_t* __restrict__ modup_tab, int P, uint32_t* __restrict__ out,
    int64_t automorph_kinv) {
    extern __shared__ uint32_t ws[];
    const int op = blockIdx.y;
    // select, not index: a dynamic index into the parameter struct spills it to the stack
    const uint32_t* in = op == 0 ? ops.words[0] : op == 1 ? ops.words[1] : op == 2 ? ops.words[2] : ops.words[3];
    const int bits = op == 0 ? ops.bits[0] : op == 1 ? ops.bits[1] : op == 2 ? ops.bits[2] : ops.bits[3];
    const int is_signed = op == 0 ? ops.is_signed[0] : op == 1 ? ops.is_signed[1]
                        : op == 2 ? ops.is_signed[2] : ops.is_signed[3];
    const int W = (bits + 31) >> 5;
    const int TB = blockDim.x;
    const int i = blockIdx.x * TB + threadIdx.x;
    const uint32_t top_mask = (bits & 31) ? ((1u << (bits & 31)) - 1u) : 0xffffffffu;
    int src = i;
    bool negate = false;
    if (automorph_kinv != 0) {
        int64_t j = ((int64_t)i * automorph_kinv) & ((2ll * N) - 1);
        if (j >= N) { negate = true; j -= N; }
        src = (int)j;
    }
    uint32_t any = 0;
    for (int w = 0; w < W; ++w) {
        uint32_t v = in[(size_t)w * N + src];
        if (w == W - 1) v &= top_mask;
        any |= v;
        ws[w * TB + threadIdx.x] = v;
    }
    const bool sign = is_signed && ((ws[(W - 1) * TB + threadIdx.x] >> ((bits - 1) & 31)) & 1u);
    uint32_t* outp = out + (size_t)op * P * N;
    for (int j = 0; j < P; ++j) {
        const PrimeInfo pi = pinfo[j];
        const uint32_t* C = modup_tab + (size_t)j * HG_MODUP_WMAX;
        uint64_t acc = 0;
        int w = 0;
        for (; w + 1 < W; w += 2) {
            acc += (uint64_t)ws[w * TB + threadIdx.x] * C[w];
            acc += (uint64_t)ws[(w + 1) * TB + threadIdx.x] * C[w + 1];
            acc = (uint64_t)(uint32_t)(acc >> 32) * pi.c32 + (uint32_t)acc;
        }
        if (w < W) acc += (uint64_t)ws[w * TB + threadIdx.x] * C[w];
        uint32_t r = reduce_u64(acc, pi);
        // 2^bits mod p for the two's complement / negation corrections
        uint32_t pw = 0;
        if (sign || negate) {
            uint64_t t = (uint64_t)C[bits >> 5] << (bits & 31);  // < 2^61
            pw = reduce_u64(t, pi);
        }
        if (sign) r = r >= pw ? r - pw : r + pi.p - pw;           // value - 2^bits
        if (negate && any) {                                       // (2^bits - x) mod 2^bits
            // for signed operands negation is plain -x; for unsigned it is 2^bits - x
            if (is_signed) r = r ? pi.p - r : 0;
            else r = pw >= r ? pw - r : pw + pi.p - r;
        }
        outp[(size_t)j * N + i] = r;
    }
}

// Register-resident ModUp for operands of at most WB words: the W words of one coefficient
// stay in registers (zero padded to WB, so no per-word predicate), every prime's constants
// 2^(32w) mod p are read as warp-uniform 16-byte loads, and the 64-bit accumulator is folded
// through 2^32 mod p every two products after the first four.
template <int WB>
__global__ void __launch_bounds__(128) modup_reg_kernel(
    OperandSet ops, int N, const PrimeInfo* __restrict__ pinfo,
    const uint32_t* __restrict__ modup_tab, int P, uint32_t* __restrict__ out,
    int64_t automorph_kinv) {
    const int op = blockIdx.y;
    // select, not index: a dynamic index into the parameter struct spills it to the stack
    const uint32_t* in = op == 0 ? ops.words[0] : op == 1 ? ops.words[1] : op == 2 ? ops.words[2] : ops.words[3];
    const int bits = op == 0 ? ops.bits[0] : op == 1 ? ops.bits[1] : op == 2 ? ops.bits[2] : ops.bits[3];
    const int is_signed = op == 0 ? ops.is_signed[0] : op == 1 ? ops.is_signed[1]
                        : op == 2 ? ops.is_signed[2] : ops.is_signed[3];
    const int W = (bits + 31) >> 5;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t top_mask = (bits & 31) ? ((1u << (bits & 31)) - 1u) : 0xffffffffu;
    int src = i;
    bool negate = false;
    if (automorph_kinv != 0) {
        int64_t j = ((int64_t)i * automorph_kinv) & ((2ll * N) - 1);
        if (j >= N) { negate = true; j -= N; }
        src = (int)j;
    }
    uint32_t a[WB];
    uint32_t any = 0;
#pragma unroll
    for (int w = 0; w < WB; ++w) {
        uint32_t v = 0;
        if (w < W) {
            v = in[(size_t)w * N + src];
            if (w == W - 1) v &= top_mask;
        }
        any |= v;
        a[w] = v;
    }
    bool sign = false;
#pragma unroll
    for (int w = 0; w < WB; ++w)
        if (w == W - 1) sign = is_signed && ((a[w] >> ((bits - 1) & 31)) & 1u);
    uint32_t* outp = out + (size_t)op * P * N;
    for (int j = 0; j < P; ++j) {
        const PrimeInfo pi = pinfo[j];
        const uint4* C4 = reinterpret_cast<const uint4*>(modup_tab + (size_t)j * HG_MODUP_WMAX);
        uint64_t acc = 0;
#pragma unroll
        for (int w4 = 0; w4 < WB / 4; ++w4) {
            const uint4 c = C4[w4];
            acc += (uint64_t)a[4 * w4] * c.x;
            acc += (uint64_t)a[4 * w4 + 1] * c.y;
            if (w4) acc = (uint64_t)(uint32_t)(acc >> 32) * pi.c32 + (uint32_t)acc;
            acc += (uint64_t)a[4 * w4 + 2] * c.z;
            acc += (uint64_t)a[4 * w4 + 3] * c.w;
            acc = (uint64_t)(uint32_t)(acc >> 32) * pi.c32 + (uint32_t)acc;
        }
        uint32_t r = reduce_u64(acc, pi);
        if (sign || negate) {
            uint32_t pw = reduce_u64((uint64_t)modup_tab[(size_t)j * HG_MODUP_WMAX + (bits >> 5)]
                                         << (bits & 31), pi);
            if (sign) r = r >= pw ? r - pw : r + pi.p - pw;
            if (negate && any) {
                if (is_signed) r = r ? pi.p - r : 0;
                else r = pw >= r ? pw - r : pw + pi.p - r;
            }
        }
        outp[(size_t)j * N + i] = r;
    }
}

// ---- pointwise products ------------------------------------------------------------------
// a, b: forward-NTT outputs in [0, 4p) (or keys in [0, p)); result mont(a,b) in [0, 2p).
__global__ void pw_mul_kernel(uint32_t* __restrict__ a, const uint32_t* __restrict__ b,
                              int P, int N, const PrimeInfo* __restrict__ pinfo) {
    const int j = blockIdx.y;
    const PrimeInfo pi = pinfo[j];
    const size_t off = (size_t)j * N;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) {
        uint32_t x = a[off + i], y = b[off + i];
        uint32_t p2 = pi.p << 1;
        x = x >= p2 ? x - p2 : x;
        y = y >= p2 ? y - p2 : y;
        uint32_t r = mont_mul(x, y, pi.p, pi.pinv_neg);
        a[off + i] = r >= pi.p ? r - pi.p : r;
    }
}

// buf = [A0 | A1 | B0 | B1] each [P][N] -> [D0 | D1 | D2] in place (rows 0..2).
__global__ void pw_tensor_kernel(uint32_t* __restrict__ buf, int P, int N,
                                 const PrimeInfo* __restrict__ pinfo) {
    const int j = blockIdx.y;
    const PrimeInfo pi = pinfo[j];
    const size_t stride = (size_t)P * N;
    const size_t off = (size_t)j * N;
    const uint32_t p2 = pi.p << 1;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) {
        size_t o = off + i;
        uint32_t a0 = buf[o], a1 = buf[o + stride], b0 = buf[o + 2 * stride], b1 = buf[o + 3 * stride];
        a0 = a0 >= p2 ? a0 - p2 : a0;
        a1 = a1 >= p2 ? a1 - p2 : a1;
        b0 = b0 >= p2 ? b0 - p2 : b0;
        b1 = b1 >= p2 ? b1 - p2 : b1;
        uint32_t d0 = mont_mul(a0, b0, pi.p, pi.pinv_neg);
        uint32_t d1 = mont_mul(a0, b1, pi.p, pi.pinv_neg) + mont_mul(a1, b0, pi.p, pi.pinv_neg);
        uint32_t d2 = mont_mul(a1, b1, pi.p, pi.pinv_neg);
        d0 = d0 >= pi.p ? d0 - pi.p : d0;
        d1 = d1 >= p2 ? d1 - p2 : d1;
        d1 = d1 >= pi.p ? d1 - pi.p : d1;
        d2 = d2 >= pi.p ? d2 - pi.p : d2;
        buf[o] = d0;
        buf[o + stride] = d1;
        buf[o + 2 * stride] = d2;
    }
}

// buf = [X | T0 | T1] each [P][N]: T0 = X*KB, T1 = X*KA (Montgomery), keys in [0, p).
__global__ void pw_key2_kernel(uint32_t* __restrict__ buf, const uint32_t* __restrict__ kb,
                               const uint32_t* __restrict__ ka, int P, int N,
                               const PrimeInfo* __restrict__ pinfo) {
    const int j = blockIdx.y;
    const PrimeInfo pi = pinfo[j];
    const size_t stride = (size_t)P * N;
    const size_t off = (size_t)j * N;
    const uint32_t p2 = pi.p << 1;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) {
        size_t o = off + i;
        uint32_t x = buf[o];
        x = x >= p2 ? x - p2 : x;
        uint32_t t0 = mont_mul(x, kb[o], pi.p, pi.pinv_neg);
        uint32_t t1 = mont_mul(x, ka[o], pi.p, pi.pinv_neg);
        buf[o + stride] = t0 >= pi.p ? t0 - pi.p : t0;
        buf[o + 2 * stride] = t1 >= pi.p ? t1 - pi.p : t1;
    }
}

__global__ void reduce_rows_kernel(uint32_t* __restrict__ a, int N,
                                   const PrimeInfo* __restrict__ pinfo) {
    const int j = blockIdx.y;
    const uint32_t p = pinfo[j].p;
    const size_t off = (size_t)j * N;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x)
        a[off + i] = reduce_4p(a[off + i], p);
}

// rows [z][P][N] (any 32-bit residues) -> x * c_j mod p_j in [0, p): folds the CRT constant
// c_j = (Q/p_j)^-1 N^-1 2^32 into a resident operand (the product and the inverse NTT are
// linear, so the CRT input arrives already multiplied by it)
__global__ void scale_rows_kernel(uint32_t* __restrict__ a, int P, int N, const PrimeInfo* __restrict__ pinfo,
                                  const uint32_t* __restrict__ c, const uint32_t* __restrict__ c_sh) {
    const int j = blockIdx.y;
    const uint32_t p = pinfo[j].p, w = c[j], wsh = c_sh[j];
    const size_t off = ((size_t)blockIdx.z * P + j) * N;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x)
        a[off + i] = reduce_2p(mul_shoup_lazy(a[off + i], w, wsh, p), p);
}

// ---- CRT reconstruction -----------------------------------------------------------------------
// Exact c = sum_j y_j Q/p_j - v Q with y_j = r_j (Q/p_j)^-1 N^-1 2^32 mod p_j and
// v = round(sum_j y_j / p_j) (|c| < Q/8 by the prime-count margin, so the float64 estimate
// is exact).  Column t of c mod 2^(32T) is sum_j y_j M[t][j] + v negQ[t] + carry, scanned
// low to high; the kernel emits bits [shift, shift + out_bits) of c + 2^(shift-1).
constexpr int kCrtCols = 8;  // columns accumulated per pass (register blocking)

// Scan columns [tb0, T) of c + round, 8 at a time: every y_j (shared memory) meets 8 column
// constants (two broadcast 16-byte loads of row j of M) -> 8 exact 32x32->64 MACs; the
// accumulators are folded every 4 primes so a 64-bit register never overflows.  Emits bits
// [shift, shift+out_bits).  Returns true if the columns below shift/32 (present only when
// tb0 > 0, the truncated "fraction" window) are too close to a carry to be trusted.
__device__ __forceinline__ bool crt_scan(const uint32_t* __restrict__ ys, int TB, int P4,
                                         const uint32_t* __restrict__ Mtab, int W,
                                         const uint32_t* __restrict__ negQ, uint32_t v, int tb0,
                                         int shift, int out_bits, uint32_t* __restrict__ out,
                                         int N, int i) {
    const int sw = shift >> 5, sb = shift & 31;
    const int out_w = (out_bits + 31) >> 5;
    const uint32_t top_mask = (out_bits & 31) ? ((1u << (out_bits & 31)) - 1u) : 0xffffffffu;
    const int T = sw + out_w + (sb ? 1 : 0);
    const int round_col = shift > 0 ? ((shift - 1) >> 5) : -1;
    const uint32_t round_bit = shift > 0 ? (1u << ((shift - 1) & 31)) : 0u;
    uint64_t carry = 0;
    uint32_t prev = 0;
    bool amb = false;
    const uint32_t* y_base = ys + threadIdx.x;
    for (int tb = tb0; tb < T; tb += kCrtCols) {
        uint64_t acc[kCrtCols], top[kCrtCols];
#pragma unroll
        for (int g = 0; g < kCrtCols; ++g) {
            uint64_t x = (uint64_t)v * negQ[tb + g] + ((tb + g) == round_col ? round_bit : 0u);
            acc[g] = (uint32_t)x;
            top[g] = x >> 32;
        }
        const uint32_t* mrow = Mtab + tb;
        for (int j = 0; j < P4; j += 4) {
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
                const uint64_t y = y_base[(j + jj) * TB];
                const uint4 m0 = *reinterpret_cast<const uint4*>(mrow + (size_t)(j + jj) * W);
                const uint4 m1 = *reinterpret_cast<const uint4*>(mrow + (size_t)(j + jj) * W + 4);
                acc[0] += y * m0.x;
                acc[1] += y * m0.y;
                acc[2] += y * m0.z;
                acc[3] += y * m0.w;
                acc[4] += y * m1.x;
                acc[5] += y * m1.y;
                acc[6] += y * m1.z;
                acc[7] += y * m1.w;
            }
#pragma unroll
            for (int g = 0; g < kCrtCols; ++g) {
                top[g] += acc[g] >> 32;
                acc[g] &= 0xffffffffull;
            }
        }
#pragma unroll
        for (int g = 0; g < kCrtCols; ++g) {
            const int t = tb + g;
            if (t < T) {
                const uint64_t s = acc[g] + (carry & 0xffffffffull);
                const uint32_t word = (uint32_t)s;
                carry = top[g] + (s >> 32) + (carry >> 32);
                if (t < sw) {
                    // truncated window: ambiguous if an unseen carry of < 2^39 units of
                    // column tb0 could still ripple into column sw
                    if (t == tb0 + 1) amb = word >= 0xFFFFFF00u;
                    else if (t > tb0 + 1) amb = amb && (word == 0xffffffffu);
                } else if (sb == 0) {
                    const int u = t - sw;
                    out[(size_t)u * N + i] = (u == out_w - 1) ? (word & top_mask) : word;
                } else if (t > sw) {
                    const int u = t - sw - 1;
                    const uint32_t o = (prev >> sb) | (word << (32 - sb));
                    out[(size_t)u * N + i] = (u == out_w - 1) ? (o & top_mask) : o;
                }
                prev = word;
            }
        }
    }
    return tb0 > 0 && amb;
}

__global__ void __launch_bounds__(kCrtThreads) crt_kernel(
    const uint32_t* __restrict__ res, int P, int P4, int N, const PrimeInfo* __restrict__ pinfo,
    const uint32_t* __restrict__ Mtab, int W, const uint32_t* __restrict__ negQ,
    const uint32_t* __restrict__ cinv, const uint32_t* __restrict__ cinv_sh,
    const double* __restrict__ invp, int shift, int out_bits, int tb0, OutSet outs) {
    extern __shared__ uint32_t ys[];  // [P4][TB]
    const int TB = blockDim.x;
    const int i = blockIdx.x * TB + threadIdx.x;
    const uint32_t* r = res + (size_t)blockIdx.y * P * N;
    const int oy = blockIdx.y;
    uint32_t* out = oy == 0 ? outs.out[0] : oy == 1 ? outs.out[1] : oy == 2 ? outs.out[2] : outs.out[3];
    double S = 0.0;
    for (int j = 0; j < P; ++j) {
        uint32_t p = pinfo[j].p;
        uint32_t x = r[(size_t)j * N + i];
        uint32_t y = reduce_2p(mul_shoup_lazy(x, cinv[j], cinv_sh[j], p), p);
        ys[j * TB + threadIdx.x] = y;
        S += (double)y * invp[j];
    }
    for (int j = P; j < P4; ++j) ys[j * TB + threadIdx.x] = 0;
    const uint32_t v = (uint32_t)floor(S + 0.5);
    if (crt_scan(ys, TB, P4, Mtab, W, negQ, v, tb0, shift, out_bits, out, N, i))
        crt_scan(ys, TB, P4, Mtab, W, negQ, v, 0, shift, out_bits, out, N, i);  // exact rescan
}

// ---- device scratch ------------------------------------------------------------------------
struct Scratch {
    void* p = nullptr;
    cudaStream_t s;
    explicit Scratch(cudaStream_t st) : s(st) {}
    // a failed allocation also sets the runtime's last-error state; clear it, so the caller's
    // retry (_lib.call) does not see a stale out-of-memory at its next launch check
    cudaError_t alloc(size_t bytes) {
        const cudaError_t e = cudaMallocAsync(&p, bytes, s);
        if (e != cudaSuccess) {
            p = nullptr;
            (void)cudaGetLastError();
        }
        return e;
    }
    ~Scratch() {
        if (p) cudaFreeAsync(p, s);
    }
    uint32_t* u32() { return static_cast<uint32_t*>(p); }
};

// out[k][j] = out[k][j] + 2^(32 kSplitW) hi[k][j] mod p_j, lazily in [0, 4p): the residues of an
// operand wider than the tensor-core ModUp takes, from the residues of its low kSplitW words
// (unsigned) and of its high words (the operand's own signedness) -- ModUp is linear
constexpr int kSplitW = 64;
__global__ void modup_combine_kernel(uint32_t* __restrict__ out, const uint32_t* __restrict__ hi, int N, int P,
                                     const PrimeInfo* __restrict__ pinfo,
                                     const uint32_t* __restrict__ modup_tab) {
    const int j = blockIdx.y, k = blockIdx.z;
    const uint32_t p = pinfo[j].p;
    const uint32_t c = modup_tab[(size_t)j * HG_MODUP_WMAX + kSplitW];   // 2^(32 kSplitW) mod p
    const uint32_t c_sh = (uint32_t)(((uint64_t)c << 32) / p);
    const size_t row = ((size_t)k * P + j) * N;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) {
        uint32_t lo = out[row + i];
        lo = min(lo, lo - 2 * p);                                  // [0, 2p)
        out[row + i] = lo + mul_shoup_lazy(hi[row + i], c, c_sh, p);   // + [0, 2p)
    }
}

int launch_modup(hg_ctx* ctx, const OperandSet& ops, int nops, int P, uint32_t* out,
                 int64_t kinv, cudaStream_t st) {
    int maxw = 0;
    for (int k = 0; k < nops; ++k) {
        int w = words_for_bits(ops.bits[k]);
        if (w > maxw) maxw = w;
        if (ops.bits[k] < 1 || w > HG_MODUP_WMAX - 1)
            return hg_fail(HG_EINVAL, "operand width out of range");
    }
    size_t smem = (size_t)maxw * kModupThreads * 4;
    static std::atomic<uint64_t> attr_set{0};
    if (hg_first_on_device(attr_set, ctx->device)) {
        cudaFuncSetAttribute(modup_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        cudaFuncSetAttribute(crt_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    }
    const int N = ctx->N;
    int threads = N < kModupThreads ? N : kModupThreads;
    smem = (size_t)maxw * threads * 4;
    dim3 grid(N / threads, nops);
    double macs = 0.0;
    for (int k = 0; k < nops; ++k) macs += (double)words_for_bits(ops.bits[k]) * P * N;
    if (!getenv("HG_NO_UMMA") && !getenv("HG_NO_MMA")) {
        HgTimed tm(ctx, st, HG_K_MODUP, macs);
        if (maxw > kSplitW && kinv == 0 && N >= 128 && !getenv("HG_NO_MODUP_SPLIT")) {
            // operands wider than the tensor-core kernel takes (switching keys, l + L bits): low
            // kSplitW words unsigned into `out`, the high words (signed as the operand) into
            // scratch, then out += 2^(32 kSplitW) hi mod p.  (Not under an automorphism: the
            // negation acts on the whole value.)
            const uint32_t* wl[4];
            const uint32_t* wh[4];
            int bl[4], bh[4], sl[4], sh[4];
            for (int k = 0; k < nops; ++k) {
                const bool wide = words_for_bits(ops.bits[k]) > kSplitW;
                wl[k] = ops.words[k];
                bl[k] = wide ? 32 * kSplitW : ops.bits[k];
                sl[k] = wide ? 0 : ops.is_signed[k];
                wh[k] = wide ? ops.words[k] + (size_t)kSplitW * N : ops.words[k];   // narrow: in bounds, cleared below
                bh[k] = wide ? ops.bits[k] - 32 * kSplitW : 1;   // narrow operands: a 1-bit zero-free dummy
                sh[k] = wide ? ops.is_signed[k] : 0;
            }
            void* hi = nullptr;
            if (cudaMallocAsync(&hi, (size_t)nops * P * N * 4, st) != cudaSuccess) {
                cudaGetLastError();
                return hg_fail(HG_ENOMEM, "ModUp split: scratch allocation failed");
            }
            int h = hg_modup_umma_launch(ctx, wl, bl, sl, nops, P, out, 0, st);
            if (h == 1) h = hg_modup_umma_launch(ctx, wh, bh, sh, nops, P, (uint32_t*)hi, 0, st);
            if (h == 1) {
                // narrow operands' high "part" must contribute 0: clear those rows
                for (int k = 0; k < nops; ++k)
                    if (words_for_bits(ops.bits[k]) <= kSplitW)
                        cudaMemsetAsync((uint32_t*)hi + (size_t)k * P * N, 0, (size_t)P * N * 4, st);
                modup_combine_kernel<<<dim3((N + 255) / 256 < 64 ? (N + 255) / 256 : 64, P, nops), 256, 0, st>>>(
                    out, (const uint32_t*)hi, N, P, ctx->d_pinfo, ctx->d_modup);
                cudaFreeAsync(hi, st);
                HG_LAUNCH_CHECK(ctx);
                return HG_OK;
            }
            cudaFreeAsync(hi, st);
            if (h < 0) return -h;
        } else {
            int h = hg_modup_umma_launch(ctx, ops.words, ops.bits, ops.is_signed, nops, P, out, kinv, st);
            if (h < 0) return -h;
            if (h == 1) return HG_OK;
        }
    }
    if (!getenv("HG_NO_MMA")) {
        HgTimed tm(ctx, st, HG_K_MODUP, macs);
        int h = hg_modup_mma_launch(ctx, ops.words, ops.bits, ops.is_signed, nops, P, out, kinv, st);
        if (h < 0) return -h;
        if (h == 1) return HG_OK;
    }
    {
        HgTimed tm(ctx, st, HG_K_MODUP, macs);
        if (maxw <= 8)
            modup_reg_kernel<8><<<grid, threads, 0, st>>>(ops, N, ctx->d_pinfo, ctx->d_modup, P, out, kinv);
        else if (maxw <= 16)
            modup_reg_kernel<16><<<grid, threads, 0, st>>>(ops, N, ctx->d_pinfo, ctx->d_modup, P, out, kinv);
        else if (maxw <= 32)
            modup_reg_kernel<32><<<grid, threads, 0, st>>>(ops, N, ctx->d_pinfo, ctx->d_modup, P, out, kinv);
        else if (maxw <= 48)
            modup_reg_kernel<48><<<grid, threads, 0, st>>>(ops, N, ctx->d_pinfo, ctx->d_modup, P, out, kinv);
        else if (maxw <= 64)
            modup_reg_kernel<64><<<grid, threads, 0, st>>>(ops, N, ctx->d_pinfo, ctx->d_modup, P, out, kinv);
        else
            modup_kernel<<<grid, threads, smem, st>>>(ops, N, ctx->log_n, ctx->d_pinfo, ctx->d_modup,
                                                      P, out, kinv);
    }
    HG_LAUNCH_CHECK(ctx);
    return HG_OK;
}

// columns below shift/32 only feed the carry: keep two of them (plus alignment) as a
// truncated fixed-point window instead of scanning all of them (exact rescan on doubt)
int crt_tb0(int shift) {
    const int sw = shift >> 5;
    return sw >= 2 ? ((sw - 2) & ~(kCrtCols - 1)) : 0;
}

bool crt_pipe_enabled(hg_ctx* ctx) {
    static const bool off = getenv("HG_NO_UMMA") || getenv("HG_NO_MMA") || getenv("HG_NO_PIPE");
    return ctx->N >= 128 && !off;
}

// true when launch_crt can take a CrtFinish (the pipelined tcgen05 kernel runs this window)
bool crt_finish_ok(hg_ctx* ctx, int P, int shift, int out_bits) {
    if (!crt_pipe_enabled(ctx) || getenv("HG_NO_FUSE")) return false;
    const CrtTable* tab = nullptr;
    if (hg_get_crt(ctx, P, &tab)) return false;
    return hg_crt_umma_pipe_ok(tab, ctx->N, shift, out_bits, crt_tb0(shift));
}

// true when the residues of this window may arrive prescaled (see scale_rows_kernel): the
// fused key/tensor product feeds the pipelined CRT
bool crt_prescale_ok(hg_ctx* ctx, int P, int shift, int out_bits) {
    if (!crt_pipe_enabled(ctx) || !fuse_pointwise() || getenv("HG_NO_PRESCALE")) return false;
    const CrtTable* tab = nullptr;
    if (hg_get_crt(ctx, P, &tab)) return false;
    return hg_crt_umma_pipe_ok(tab, ctx->N, shift, out_bits, crt_tb0(shift));
}

dim3 pw_grid(int N, int rows);

int prescale_rows(hg_ctx* ctx, uint32_t* rows, int nrows, int P, cudaStream_t st) {
    const CrtTable* tab = nullptr;
    if (int rc = hg_get_crt(ctx, P, &tab)) return rc;
    dim3 grid = pw_grid(ctx->N, P);
    grid.z = nrows;
    scale_rows_kernel<<<grid, 256, 0, st>>>(rows, P, ctx->N, ctx->d_pinfo, tab->d_cinv, tab->d_cinv_sh);
    HG_LAUNCH_CHECK(ctx);
    return HG_OK;
}

int launch_crt(hg_ctx* ctx, const uint32_t* res, int nouts, int P, int shift, int out_bits,
               const OutSet& outs, cudaStream_t st, const CrtFinish* finish = nullptr,
               bool prescaled = false) {
    const CrtTable* tab = nullptr;
    int rc = hg_get_crt(ctx, P, &tab);
    if (rc) return rc;
    int sw = shift >> 5;
    int T = sw + words_for_bits(out_bits) + ((shift & 31) ? 1 : 0);
    if (T > tab->W) return hg_fail(HG_ERANGE, "CRT window exceeds table width");
    const int tb0 = crt_tb0(shift);
    const int N = ctx->N;
    const int threads = N < kCrtThreads ? N : kCrtThreads;
    size_t smem = (size_t)tab->P4 * threads * 4;
    dim3 grid(N / threads, nouts);
    if (crt_pipe_enabled(ctx) && hg_crt_umma_pipe_ok(tab, N, shift, out_bits, tb0)) {
        // persistent warp-specialised tcgen05 path
        HgTimed tm(ctx, st, HG_K_CRT, (double)nouts * N * (double)P * (T - tb0));
        return hg_crt_umma_pipe_launch(ctx, tab, res, nouts, P, shift, out_bits, tb0, outs.out, st,
                                       finish, prescaled);
    }
    if (finish) return hg_fail(HG_EINVAL, "fused CRT finish needs the pipelined kernel");
    if (prescaled) return hg_fail(HG_EINVAL, "prescaled CRT residues need the pipelined kernel");
    if (nouts > 4) {   // the older kernels take 4 outputs per launch
        OutSet lo{}, hi{};
        for (int k = 0; k < 4; ++k) lo.out[k] = outs.out[k];
        for (int k = 4; k < nouts; ++k) hi.out[k - 4] = outs.out[k];
        if ((rc = launch_crt(ctx, res, 4, P, shift, out_bits, lo, st))) return rc;
        return launch_crt(ctx, res + (size_t)4 * P * N, nouts - 4, P, shift, out_bits, hi, st);
    }
    if (N >= 128 && !getenv("HG_NO_UMMA") && !getenv("HG_NO_MMA") &&
        hg_crt_umma_smem(tab->P32) <= 220 * 1024) {
        // tcgen05 path (UTCIMMA, accumulators in TMEM)
        HgTimed tm(ctx, st, HG_K_CRT, (double)nouts * N * (double)P * (T - tb0));
        return hg_crt_umma_launch(ctx, tab, res, nouts, P, shift, out_bits, tb0, outs.out, st);
    }
    if (N >= 64 && !getenv("HG_NO_MMA")) {
        // tensor-core path: work counted as 32x32-bit MACs, like the integer-pipe kernel
        HgTimed tm(ctx, st, HG_K_CRT, (double)nouts * N * (double)P * (T - tb0));
        return hg_crt_mma_launch(ctx, tab, res, nouts, P, shift, out_bits, tb0, outs.out, st);
    }
    {
        HgTimed tm(ctx, st, HG_K_CRT, (double)nouts * N * (double)P * (T - tb0));
        crt_kernel<<<grid, threads, smem, st>>>(res, P, tab->P4, N, ctx->d_pinfo, tab->d_M,
                                                tab->W, tab->d_negQ, tab->d_cinv, tab->d_cinv_sh,
                                                tab->d_invp, shift, out_bits, tb0, outs);
    }
    HG_LAUNCH_CHECK(ctx);
    return HG_OK;
}

dim3 pw_grid(int N, int rows) { return dim3((N + 255) / 256 < 64 ? (N + 255) / 256 : 64, rows); }

// Tensor with a resident (prepared) left operand: A0, A1 = NTT residues [P][N] in [0, 4p);
// buf = [B0 | B1 | (D2)] each [P][N] -> [D0 | D1 | D2].
__global__ void pw_tensor_prep_kernel(const uint32_t* __restrict__ A0, const uint32_t* __restrict__ A1,
                                      uint32_t* __restrict__ buf, int P, int N,
                                      const PrimeInfo* __restrict__ pinfo) {
    const int j = blockIdx.y;
    const PrimeInfo pi = pinfo[j];
    const size_t stride = (size_t)P * N;
    const size_t off = (size_t)j * N;
    const uint32_t p2 = pi.p << 1;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) {
        const size_t o = off + i;
        uint32_t a0 = A0[o], a1 = A1[o], b0 = buf[o], b1 = buf[o + stride];
        a0 = a0 >= p2 ? a0 - p2 : a0;
        a1 = a1 >= p2 ? a1 - p2 : a1;
        b0 = b0 >= p2 ? b0 - p2 : b0;
        b1 = b1 >= p2 ? b1 - p2 : b1;
        uint32_t d0 = mont_mul(a0, b0, pi.p, pi.pinv_neg);
        uint32_t d1 = mont_mul(a0, b1, pi.p, pi.pinv_neg) + mont_mul(a1, b0, pi.p, pi.pinv_neg);
        uint32_t d2 = mont_mul(a1, b1, pi.p, pi.pinv_neg);
        d0 = d0 >= pi.p ? d0 - pi.p : d0;
        d1 = d1 >= p2 ? d1 - p2 : d1;
        d1 = d1 >= pi.p ? d1 - pi.p : d1;
        d2 = d2 >= pi.p ? d2 - pi.p : d2;
        buf[o] = d0;
        buf[o + stride] = d1;
        buf[o + 2 * stride] = d2;
    }
}

int magnitude_bits(const hg_operand& o) { return o.signed_rep ? o.bits - 1 : o.bits; }

int primes_for_product(hg_ctx* ctx, double mag_bits, int window_bits) {
    // |c| <= N 2^mag ; need Q > 8|c| (2 bits of margin beyond the sign)
    (void)window_bits;  // CRT tables are at least HG_MODUP_WMAX words wide
    return hg_primes_for_bits(ctx, mag_bits + ctx->log_n + 3.0);
}

}  // namespace

// ---- public product API --------------------------------------------------------------------------
extern "C" int hg_poly_mul(hg_ctx* ctx, uint32_t* out, int out_bits, hg_operand a,
                           hg_operand b, void* stream) {
    if (!ctx || !out || !a.words || !b.words || out_bits < 1)
        return hg_fail(HG_EINVAL, "hg_poly_mul: bad arguments");
    cudaStream_t st = (cudaStream_t)stream;
    const int N = ctx->N;
    int P = primes_for_product(ctx, magnitude_bits(a) + magnitude_bits(b), out_bits);
    if (P < 0) return hg_fail(HG_ERANGE, "product exceeds the NTT prime basis");
    Scratch buf(st);
    HG_CUDA_TRY(buf.alloc((size_t)2 * P * N * 4));
    OperandSet ops{};
    ops.words[0] = a.words; ops.bits[0] = a.bits; ops.is_signed[0] = a.signed_rep;
    ops.words[1] = b.words; ops.bits[1] = b.bits; ops.is_signed[1] = b.signed_rep;
    int rc = launch_modup(ctx, ops, 2, P, buf.u32(), 0, st);
    if (rc) return rc;
    rc = hg_ntt_launch(ctx, buf.u32(), 2 * P, P, 0, true, st);
    if (rc) return rc;
    rc = fuse_pointwise() ? hg_intt_fused(ctx, 3, buf.u32(), buf.u32(), buf.u32() + (size_t)P * N,
                                          nullptr, nullptr, P, st)
                          : -1;
    if (rc > 0) return rc;
    if (rc < 0) {
        const int tpw = hg_timer_begin(ctx, st, HG_K_POINTWISE);
        pw_mul_kernel<<<pw_grid(N, P), 256, 0, st>>>(buf.u32(), buf.u32() + (size_t)P * N, P, N,
                                                     ctx->d_pinfo);
        hg_timer_end(ctx, tpw, st, HG_K_POINTWISE, (double)N * P);
        HG_LAUNCH_CHECK(ctx);
        rc = hg_ntt_launch(ctx, buf.u32(), P, P, 0, false, st);
        if (rc) return rc;
    }
    OutSet outs{};
    outs.out[0] = out;
    return launch_crt(ctx, buf.u32(), 1, P, 0, out_bits, outs, st);
}

extern "C" int hg_poly_tensor(hg_ctx* ctx, uint32_t* d0, uint32_t* d1, uint32_t* d2,
                              int out_bits, hg_operand a0, hg_operand a1, hg_operand b0,
                              hg_operand b1, void* stream) {
    if (!ctx || !d0 || !d1 || !d2 || out_bits < 1)
        return hg_fail(HG_EINVAL, "hg_poly_tensor: bad arguments");
    cudaStream_t st = (cudaStream_t)stream;
    const int N = ctx->N;
    int ma = magnitude_bits(a0) > magnitude_bits(a1) ? magnitude_bits(a0) : magnitude_bits(a1);
    int mb = magnitude_bits(b0) > magnitude_bits(b1) ? magnitude_bits(b0) : magnitude_bits(b1);
    int P = primes_for_product(ctx, ma + mb + 1, out_bits);  // +1: d1 is a sum of two products
    if (P < 0) return hg_fail(HG_ERANGE, "tensor product exceeds the NTT prime basis");
    Scratch buf(st);
    HG_CUDA_TRY(buf.alloc((size_t)4 * P * N * 4));
    OperandSet ops{};
    const hg_operand in[4] = {a0, a1, b0, b1};
    for (int k = 0; k < 4; ++k) {
        ops.words[k] = in[k].words; ops.bits[k] = in[k].bits; ops.is_signed[k] = in[k].signed_rep;
    }
    int rc = launch_modup(ctx, ops, 4, P, buf.u32(), 0, st);
    if (rc) return rc;
    rc = hg_ntt_launch(ctx, buf.u32(), 4 * P, P, 0, true, st);
    if (rc) return rc;
    {
        const size_t sp = (size_t)P * N;
        uint32_t* b = buf.u32();
        rc = fuse_pointwise() ? hg_intt_fused(ctx, 2, b, b, b + sp, b + 2 * sp, b + 3 * sp, P, st) : -1;
    }
    if (rc > 0) return rc;
    if (rc < 0) {
        const int tpw = hg_timer_begin(ctx, st, HG_K_POINTWISE);
        pw_tensor_kernel<<<pw_grid(N, P), 256, 0, st>>>(buf.u32(), P, N, ctx->d_pinfo);
        hg_timer_end(ctx, tpw, st, HG_K_POINTWISE, (double)N * P);
        HG_LAUNCH_CHECK(ctx);
        rc = hg_ntt_launch(ctx, buf.u32(), 3 * P, P, 0, false, st);
        if (rc) return rc;
    }
    OutSet outs{};
    outs.out[0] = d0; outs.out[1] = d1; outs.out[2] = d2;
    return launch_crt(ctx, buf.u32(), 3, P, 0, out_bits, outs, st);
}

// ---- keys and key switching ------------------------------------------------------------------------
extern "C" int hg_key_prepare(hg_ctx* ctx, const uint32_t* kb, const uint32_t* ka, int key_bits,
                              int level, int big_l, void* stream, hg_key** out) {
    if (!ctx || !kb || !ka || !out || level < 1 || big_l < 1 || level + big_l > key_bits)
        return hg_fail(HG_EINVAL, "hg_key_prepare: bad arguments");
    cudaStream_t st = (cudaStream_t)stream;
    const int N = ctx->N;
    const int kbits = level + big_l;
    // x canonical (level bits) times centered key (kbits-1 magnitude); window [L, L+level)
    int P = primes_for_product(ctx, (double)level + (kbits - 1), kbits + 1);
    if (P < 0) return hg_fail(HG_ERANGE, "key switch exceeds the NTT prime basis");
    hg_key* key = new hg_key();
    key->ctx = ctx;
    key->level = level;
    key->big_l = big_l;
    key->P = P;
    key->bytes = (size_t)2 * P * N * 4;
    const auto t_alloc = std::chrono::steady_clock::now();
    key->d_kb = (uint32_t*)hg_arena_alloc(ctx, key->bytes);
    if (!key->d_kb) {
        delete key;
        return hg_fail(HG_ENOMEM, "key allocation failed");
    }
    key->d_ka = key->d_kb + (size_t)P * N;
    if (getenv("HG_DEBUG_BUILD"))
        fprintf(stderr, "[hg build] key P=%d alloc %.2f ms\n", P,
                std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_alloc).count());
    OperandSet ops{};
    ops.words[0] = kb; ops.bits[0] = kbits; ops.is_signed[0] = 1;   // reduce_to(l+L), centered
    ops.words[1] = ka; ops.bits[1] = kbits; ops.is_signed[1] = 1;
    int rc = launch_modup(ctx, ops, 2, P, key->d_kb, 0, st);
    if (!rc) rc = hg_ntt_launch(ctx, key->d_kb, 2 * P, P, 0, true, st);
    if (!rc && crt_prescale_ok(ctx, P, big_l, level)) {
        rc = prescale_rows(ctx, key->d_kb, 2, P, st);   // d_ka follows d_kb
        key->prescaled = rc == HG_OK;
    } else if (!rc) {
        reduce_rows_kernel<<<pw_grid(N, P), 256, 0, st>>>(key->d_kb, N, ctx->d_pinfo);
        ctx->launches++;
        reduce_rows_kernel<<<pw_grid(N, P), 256, 0, st>>>(key->d_ka, N, ctx->d_pinfo);
        HG_LAUNCH_CHECK(ctx);
    }
    if (rc) {
        cudaStreamSynchronize(st);   // launches that did go out must finish before reuse
        hg_arena_free(ctx, key->d_kb);
        delete key;
        return rc;
    }
    *out = key;
    return HG_OK;
}

extern "C" int hg_key_destroy(hg_key* key) {
    if (!key) return HG_OK;
    cudaDeviceSynchronize();   // the arena reuses the memory at once: no reader may be queued
    hg_arena_free(key->ctx, key->d_kb);
    delete key;
    return HG_OK;
}

// stream-ordered destruction: the key's memory returns to the arena once the work queued on
// `stream` (the stream its readers were issued on) has finished -- no host synchronisation
extern "C" int hg_key_release(hg_key* key, void* stream) {
    if (!key) return HG_OK;
    int rc = hg_arena_free_after(key->ctx, key->d_kb, (cudaStream_t)stream);
    delete key;
    return rc;
}

extern "C" size_t hg_key_device_bytes(const hg_key* key) { return key ? key->bytes : 0; }

static int64_t inverse_mod_2n(int64_t k, int64_t n2) {
    // k odd, n2 a power of two: Newton iteration for the inverse mod 2^64, then reduce
    uint64_t x = (uint64_t)k;
    uint64_t inv = x;
    for (int it = 0; it < 6; ++it) inv *= 2 - x * inv;
    return (int64_t)(inv & (uint64_t)(n2 - 1));
}

static int keyswitch_impl(hg_ctx* ctx, const hg_key* key, const uint32_t* x, int64_t automorph_k,
                          uint32_t* out0, uint32_t* out1, cudaStream_t st, const CrtFinish* fin);

extern "C" int hg_keyswitch(hg_ctx* ctx, const hg_key* key, const uint32_t* x,
                            int64_t automorph_k, uint32_t* out0, uint32_t* out1, void* stream) {
    if (!ctx || !key || !x || !out0 || !out1 || key->ctx != ctx)
        return hg_fail(HG_EINVAL, "hg_keyswitch: bad arguments");
    return keyswitch_impl(ctx, key, x, automorph_k, out0, out1, (cudaStream_t)stream, nullptr);
}

// out = window [L, L+level) of x * (kb, ka), x read through x -> x^k; `fin` (optional) fuses
// the caller's add / rescale into the CRT epilogue
static int keyswitch_impl(hg_ctx* ctx, const hg_key* key, const uint32_t* x, int64_t automorph_k,
                          uint32_t* out0, uint32_t* out1, cudaStream_t st, const CrtFinish* fin) {
    const int N = ctx->N;
    const int P = key->P;
    int64_t kinv = 0;
    if (automorph_k != 1) {
        int64_t n2 = 2ll * N;
        int64_t k = ((automorph_k % n2) + n2) % n2;
        if ((k & 1) == 0) return hg_fail(HG_EINVAL, "automorphism exponent must be odd");
        kinv = inverse_mod_2n(k, n2);
    }
    Scratch buf(st);
    HG_CUDA_TRY(buf.alloc((size_t)3 * P * N * 4));
    OperandSet ops{};
    ops.words[0] = x; ops.bits[0] = key->level; ops.is_signed[0] = 0;  // canonical rep
    int rc = launch_modup(ctx, ops, 1, P, buf.u32(), kinv, st);
    if (rc) return rc;
    rc = hg_ntt_launch(ctx, buf.u32(), P, P, 0, true, st);
    if (rc) return rc;
    uint32_t* t = buf.u32() + (size_t)P * N;
    rc = fuse_pointwise() ? hg_intt_fused(ctx, 1, t, buf.u32(), key->d_kb, key->d_ka, nullptr, P, st) : -1;
    if (rc > 0) return rc;
    if (rc < 0) {
        const int tpw = hg_timer_begin(ctx, st, HG_K_POINTWISE);
        pw_key2_kernel<<<pw_grid(N, P), 256, 0, st>>>(buf.u32(), key->d_kb, key->d_ka, P, N,
                                                      ctx->d_pinfo);
        hg_timer_end(ctx, tpw, st, HG_K_POINTWISE, (double)N * P);
        HG_LAUNCH_CHECK(ctx);
        rc = hg_ntt_launch(ctx, t, 2 * P, P, 0, false, st);
        if (rc) return rc;
    }
    OutSet outs{};
    outs.out[0] = out0; outs.out[1] = out1;
    return launch_crt(ctx, t, 2, P, key->big_l, key->level, outs, st, fin, key->prescaled);
}

// ---- fused scheme ops ------------------------------------------------------------------------------
// relinearise d2 with evk, add to (d0, d1), rescale (or not) into (out0, out1)
static int ct_mult_finish(hg_ctx* ctx, const hg_key* evk, uint32_t* d0, uint32_t* d1,
                          uint32_t* d2, uint32_t* e0, uint32_t* e1, int level, int rescale_bits,
                          uint32_t* out0, uint32_t* out1, cudaStream_t st) {
    if (crt_finish_ok(ctx, evk->P, evk->big_l, level)) {
        // relinearise, add (d0, d1) and rescale in the key switch's CRT epilogue
        CrtFinish fin;
        fin.add[0] = d0;
        fin.add[1] = d1;
        fin.post = rescale_bits;
        return keyswitch_impl(ctx, evk, d2, 1, out0, out1, st, &fin);
    }
    int rc = hg_keyswitch(ctx, evk, d2, 1, e0, e1, st);
    if (rc) return rc;
    if (rescale_bits == 0) {
        rc = hg_ew_add(ctx, out0, d0, e0, level, false, st);
        if (!rc) rc = hg_ew_add(ctx, out1, d1, e1, level, false, st);
        return rc;
    }
    rc = hg_ew_add(ctx, d0, d0, e0, level, false, st);
    if (!rc) rc = hg_ew_add(ctx, d1, d1, e1, level, false, st);
    if (!rc) rc = hg_ew_divide_round(ctx, out0, level - rescale_bits, d0, level, rescale_bits, st);
    if (!rc) rc = hg_ew_divide_round(ctx, out1, level - rescale_bits, d1, level, rescale_bits, st);
    return rc;
}

extern "C" int hg_ct_mult(hg_ctx* ctx, const hg_key* evk, const uint32_t* a0, const uint32_t* a1,
                          const uint32_t* b0, const uint32_t* b1, int level, int rescale_bits,
                          uint32_t* out0, uint32_t* out1, void* stream) {
    if (!ctx || !evk || evk->level != level || rescale_bits < 0 || rescale_bits >= level)
        return hg_fail(HG_EINVAL, "hg_ct_mult: bad arguments (evk must be prepared at the level)");
    cudaStream_t st = (cudaStream_t)stream;
    const int N = ctx->N;
    const int W = words_for_bits(level);
    Scratch buf(st);
    HG_CUDA_TRY(buf.alloc((size_t)5 * W * N * 4));
    uint32_t* d0 = buf.u32();
    uint32_t* d1 = d0 + (size_t)W * N;
    uint32_t* d2 = d1 + (size_t)W * N;
    uint32_t* e0 = d2 + (size_t)W * N;
    uint32_t* e1 = e0 + (size_t)W * N;
    hg_operand o[4] = {{a0, level, 1}, {a1, level, 1}, {b0, level, 1}, {b1, level, 1}};
    int rc = hg_poly_tensor(ctx, d0, d1, d2, level, o[0], o[1], o[2], o[3], stream);
    if (rc) return rc;
    return ct_mult_finish(ctx, evk, d0, d1, d2, e0, e1, level, rescale_bits, out0, out1, st);
}

// ---- resident (prepared) left operands ----------------------------------------------------------
struct hg_ctprep {
    hg_ctx* ctx = nullptr;
    int level = 0;
    int P = 0;
    uint32_t* d_res = nullptr;   // [2][P][N] forward-NTT residues of c0, c1 (centered reps)
    size_t bytes = 0;
    bool prescaled = false;      // residues carry the tensor CRT constants (scale_rows_kernel)
};


// both operands centered at `level` bits, d1 is a sum of two products; a sum of `terms`
// tensor products grows by ceil(log2 terms) bits
static int tensor_sum_primes(hg_ctx* ctx, int level, int terms) {
    int extra = 0;
    while ((1 << extra) < terms) ++extra;
    return primes_for_product(ctx, 2.0 * (level - 1) + 1 + extra, level);
}

extern "C" int hg_ct_prepare(hg_ctx* ctx, const uint32_t* c0, const uint32_t* c1, int level,
                             void* stream, hg_ctprep** out) {
    return hg_ct_prepare_sum(ctx, c0, c1, level, 1, stream, out);
}

extern "C" int hg_ct_prepare_sum(hg_ctx* ctx, const uint32_t* c0, const uint32_t* c1, int level,
                                 int terms, void* stream, hg_ctprep** out) {
    if (!ctx || !c0 || !c1 || !out || level < 2 || terms < 1)
        return hg_fail(HG_EINVAL, "hg_ct_prepare: bad arguments");
    cudaStream_t st = (cudaStream_t)stream;
    const int N = ctx->N;
    const int P = tensor_sum_primes(ctx, level, terms);
    if (P < 0) return hg_fail(HG_ERANGE, "tensor product exceeds the NTT prime basis");
    hg_ctprep* pr = new hg_ctprep();
    pr->ctx = ctx;
    pr->level = level;
    pr->P = P;
    pr->bytes = (size_t)2 * P * N * 4;
    pr->d_res = (uint32_t*)hg_arena_alloc(ctx, pr->bytes);
    if (!pr->d_res) {
        delete pr;
        return hg_fail(HG_ENOMEM, "prepared operand allocation failed");
    }
    OperandSet ops{};
    ops.words[0] = c0; ops.bits[0] = level; ops.is_signed[0] = 1;
    ops.words[1] = c1; ops.bits[1] = level; ops.is_signed[1] = 1;
    int rc = launch_modup(ctx, ops, 2, P, pr->d_res, 0, st);
    if (!rc) rc = hg_ntt_launch(ctx, pr->d_res, 2 * P, P, 0, true, st);
    if (!rc && crt_prescale_ok(ctx, P, 0, level)) {
        rc = prescale_rows(ctx, pr->d_res, 2, P, st);
        pr->prescaled = rc == HG_OK;
    }
    if (rc) {
        cudaStreamSynchronize(st);
        hg_arena_free(ctx, pr->d_res);
        delete pr;
        return rc;
    }
    *out = pr;
    return HG_OK;
}

extern "C" int hg_ctprep_destroy(hg_ctprep* pr) {
    if (!pr) return HG_OK;
    cudaDeviceSynchronize();
    hg_arena_free(pr->ctx, pr->d_res);
    delete pr;
    return HG_OK;
}

/* As hg_key_release for a prepared operand. */
extern "C" int hg_ctprep_release(hg_ctprep* pr, void* stream) {
    if (!pr) return HG_OK;
    int rc = hg_arena_free_after(pr->ctx, pr->d_res, (cudaStream_t)stream);
    delete pr;
    return rc;
}

extern "C" size_t hg_ctprep_device_bytes(const hg_ctprep* pr) { return pr ? pr->bytes : 0; }

extern "C" int hg_ct_mult_prepared(hg_ctx* ctx, const hg_key* evk, const hg_ctprep* a,
                                   const uint32_t* b0, const uint32_t* b1, int level,
                                   int rescale_bits, uint32_t* out0, uint32_t* out1, void* stream) {
    if (!ctx || !evk || !a || a->ctx != ctx || a->level != level || evk->level != level ||
        rescale_bits < 0 || rescale_bits >= level)
        return hg_fail(HG_EINVAL, "hg_ct_mult_prepared: operand/key level mismatch");
    cudaStream_t st = (cudaStream_t)stream;
    const int N = ctx->N;
    const int W = words_for_bits(level);
    const int P = a->P;
    Scratch res(st), buf(st);
    HG_CUDA_TRY(res.alloc((size_t)3 * P * N * 4));
    HG_CUDA_TRY(buf.alloc((size_t)5 * W * N * 4));
    OperandSet ops{};
    ops.words[0] = b0; ops.bits[0] = level; ops.is_signed[0] = 1;
    ops.words[1] = b1; ops.bits[1] = level; ops.is_signed[1] = 1;
    int rc = launch_modup(ctx, ops, 2, P, res.u32(), 0, st);
    if (rc) return rc;
    rc = hg_ntt_launch(ctx, res.u32(), 2 * P, P, 0, true, st);
    if (rc) return rc;
    rc = fuse_pointwise() ? hg_intt_fused(ctx, 2, res.u32(), a->d_res, a->d_res + (size_t)P * N,
                                          res.u32(), res.u32() + (size_t)P * N, P, st)
                          : -1;
    if (rc > 0) return rc;
    if (rc < 0) {
        const int tpw = hg_timer_begin(ctx, st, HG_K_POINTWISE);
        pw_tensor_prep_kernel<<<pw_grid(N, P), 256, 0, st>>>(a->d_res, a->d_res + (size_t)P * N,
                                                             res.u32(), P, N, ctx->d_pinfo);
        hg_timer_end(ctx, tpw, st, HG_K_POINTWISE, (double)N * P);
        HG_LAUNCH_CHECK(ctx);
        rc = hg_ntt_launch(ctx, res.u32(), 3 * P, P, 0, false, st);
        if (rc) return rc;
    }
    uint32_t* d0 = buf.u32();
    uint32_t* d1 = d0 + (size_t)W * N;
    uint32_t* d2 = d1 + (size_t)W * N;
    uint32_t* e0 = d2 + (size_t)W * N;
    uint32_t* e1 = e0 + (size_t)W * N;
    OutSet outs{};
    outs.out[0] = d0; outs.out[1] = d1; outs.out[2] = d2;
    rc = launch_crt(ctx, res.u32(), 3, P, 0, level, outs, st, nullptr, a->prescaled);
    if (rc) return rc;
    return ct_mult_finish(ctx, evk, d0, d1, d2, e0, e1, level, rescale_bits, out0, out1, st);
}

// `count` products with resident left operands, up to four per group of launches: ModUps of the
// right operands two items at a time, one forward NTT over all of the group's rows (rows of a
// prime adjacent: twiddles shared), 6-output tensor CRTs, and for the relinearisation one
// ModUp of all d2, one forward NTT over [G][P'][N] (two rows per block instead of one), one
// batched key product fused into the inverse NTT and one 2G-output CRT with the add + rescale
// finish.  Each output is identical to hg_ct_mult_prepared's.
extern "C" int hg_ct_mult_prepared_batch(hg_ctx* ctx, const hg_key* evk, int count,
                                         const hg_ctprep* const* a, const uint32_t* const* b0s,
                                         const uint32_t* const* b1s, int level, int rescale_bits,
                                         uint32_t* const* out0s, uint32_t* const* out1s, void* stream) {
    if (!ctx || !evk || count < 0 || (count && (!a || !b0s || !b1s || !out0s || !out1s)) ||
        evk->level != level || rescale_bits < 0 || rescale_bits >= level)
        return hg_fail(HG_EINVAL, "hg_ct_mult_prepared_batch: bad arguments");
    const int N = ctx->N;
    const int W = words_for_bits(level);
    const int Pk = evk->P;
    const bool fused = fuse_pointwise() && crt_finish_ok(ctx, Pk, evk->big_l, level);
    static const int gmax = hg_env_group("HG_BATCH_G", 4, 1, 4);
    int rc;
    for (int g0 = 0; g0 < count;) {
        int G = count - g0 < gmax ? count - g0 : gmax;
        if (G > 4) G = 4;
        bool ok = fused && G > 1;
        for (int g = 0; ok && g < G; ++g) {
            const hg_ctprep* ag = a[g0 + g];
            ok = ag && ag->ctx == ctx && ag->level == level && ag->P == a[g0]->P &&
                 ag->prescaled == a[g0]->prescaled;
        }
        if (!ok) {
            for (int g = 0; g < G; ++g)
                if ((rc = hg_ct_mult_prepared(ctx, evk, a[g0 + g], b0s[g0 + g], b1s[g0 + g], level,
                                              rescale_bits, out0s[g0 + g], out1s[g0 + g], stream)))
                    return rc;
            g0 += G;
            continue;
        }
        cudaStream_t st = (cudaStream_t)stream;
        const int P = a[g0]->P;
        const size_t plane = (size_t)P * N, kplane = (size_t)Pk * N, wn = (size_t)W * N;
        Scratch res(st), tens(st), kres(st), buf(st);
        HG_CUDA_TRY(res.alloc((size_t)2 * G * plane * 4));     // [G items][b0, b1][P][N]
        HG_CUDA_TRY(tens.alloc((size_t)3 * G * plane * 4));    // [G][d0, d1, d2][P][N]
        HG_CUDA_TRY(kres.alloc((size_t)3 * G * kplane * 4));   // x [G][P'][N], products [G][2][P'][N]
        HG_CUDA_TRY(buf.alloc((size_t)3 * G * wn * 4));        // (d0_g, d1_g) addends, then d2_g
        for (int h = 0; h < G; h += 2) {                        // ModUp: two items (4 polys) per launch
            const int gh = G - h < 2 ? G - h : 2;
            OperandSet ops{};
            for (int k = 0; k < gh; ++k) {
                ops.words[2 * k] = b0s[g0 + h + k]; ops.bits[2 * k] = level; ops.is_signed[2 * k] = 1;
                ops.words[2 * k + 1] = b1s[g0 + h + k]; ops.bits[2 * k + 1] = level; ops.is_signed[2 * k + 1] = 1;
            }
            if ((rc = launch_modup(ctx, ops, 2 * gh, P, res.u32() + (size_t)2 * h * plane, 0, st))) return rc;
        }
        if ((rc = hg_ntt_launch(ctx, res.u32(), 2 * G * P, P, 0, true, st))) return rc;
        for (int g = 0; g < G; ++g) {
            const hg_ctprep* ag = a[g0 + g];
            const uint32_t* bg = res.u32() + (size_t)2 * g * plane;
            rc = hg_intt_fused(ctx, 2, tens.u32() + (size_t)3 * g * plane, ag->d_res, ag->d_res + plane,
                               bg, bg + plane, P, st);
            if (rc) return rc < 0 ? hg_fail(HG_EINVAL, "fused tensor product not available") : rc;
        }
        uint32_t* d = buf.u32();
        for (int h = 0; h < G; h += 2) {                        // tensor CRT: two items (6 outputs) per launch
            const int gh = G - h < 2 ? G - h : 2;
            OutSet touts{};
            for (int k = 0; k < gh; ++k) {
                const int g = h + k;
                touts.out[3 * k] = d + (size_t)(2 * g) * wn;            // d0_g
                touts.out[3 * k + 1] = d + (size_t)(2 * g + 1) * wn;    // d1_g
                touts.out[3 * k + 2] = d + (size_t)(2 * G + g) * wn;    // d2_g
            }
            if ((rc = launch_crt(ctx, tens.u32() + (size_t)3 * h * plane, 3 * gh, P, 0, level, touts, st,
                                 nullptr, a[g0]->prescaled)))
                return rc;
        }
        // relinearise all d2 together; the finish adds (d0_g, d1_g) and rescales
        OperandSet kops{};
        for (int g = 0; g < G; ++g) {
            kops.words[g] = d + (size_t)(2 * G + g) * wn; kops.bits[g] = level; kops.is_signed[g] = 0;   // canonical
        }
        if ((rc = launch_modup(ctx, kops, G, Pk, kres.u32(), 0, st))) return rc;
        if ((rc = hg_ntt_launch(ctx, kres.u32(), G * Pk, Pk, 0, true, st))) return rc;
        uint32_t* t = kres.u32() + (size_t)G * kplane;
        rc = hg_intt_fused(ctx, 1, t, kres.u32(), evk->d_kb, evk->d_ka, nullptr, Pk, st, G);
        if (rc) return rc < 0 ? hg_fail(HG_EINVAL, "batched key product not available") : rc;
        CrtFinish fin;
        for (int k = 0; k < 2 * G; ++k) fin.add[k] = d + (size_t)k * wn;   // d0_0 d1_0 d0_1 d1_1 ...
        fin.post = rescale_bits;
        OutSet kouts{};
        for (int g = 0; g < G; ++g) {
            kouts.out[2 * g] = out0s[g0 + g];
            kouts.out[2 * g + 1] = out1s[g0 + g];
        }
        if ((rc = launch_crt(ctx, t, 2 * G, Pk, evk->big_l, level, kouts, st, &fin, evk->prescaled))) return rc;
        g0 += G;
    }
    return HG_OK;
}

// `count` products of ciphertext pairs (a_i (x) b_i, relinearised, rescaled), up to four per group
// of launches: one ModUp per item's four polynomials, one forward NTT over all rows of the
// group, then the same tensor CRT / batched key switch / finish as hg_ct_mult_prepared_batch.
// Each output is identical to hg_ct_mult's.
extern "C" int hg_ct_mult_batch(hg_ctx* ctx, const hg_key* evk, int count, const uint32_t* const* a0s,
                                const uint32_t* const* a1s, const uint32_t* const* b0s,
                                const uint32_t* const* b1s, int level, int rescale_bits,
                                uint32_t* const* out0s, uint32_t* const* out1s, void* stream) {
    if (!ctx || !evk || count < 0 || (count && (!a0s || !a1s || !b0s || !b1s || !out0s || !out1s)) ||
        evk->level != level || rescale_bits < 0 || rescale_bits >= level)
        return hg_fail(HG_EINVAL, "hg_ct_mult_batch: bad arguments");
    const int N = ctx->N;
    const int W = words_for_bits(level);
    const int Pk = evk->P;
    const bool fused = fuse_pointwise() && crt_finish_ok(ctx, Pk, evk->big_l, level);
    const int P = tensor_sum_primes(ctx, level, 1);
    const bool prescale = fused && P > 0 && crt_prescale_ok(ctx, P, 0, level);
    int rc;
    for (int g0 = 0; g0 < count;) {
        const int G = count - g0 < 4 ? count - g0 : 4;
        if (!fused || G == 1 || P < 0) {
            for (int g = 0; g < G; ++g)
                if ((rc = hg_ct_mult(ctx, evk, a0s[g0 + g], a1s[g0 + g], b0s[g0 + g], b1s[g0 + g], level,
                                     rescale_bits, out0s[g0 + g], out1s[g0 + g], stream)))
                    return rc;
            g0 += G;
            continue;
        }
        cudaStream_t st = (cudaStream_t)stream;
        const size_t plane = (size_t)P * N, kplane = (size_t)Pk * N, wn = (size_t)W * N;
        Scratch res(st), tens(st), kres(st), buf(st);
        HG_CUDA_TRY(res.alloc((size_t)4 * G * plane * 4));     // [G items][a0, a1, b0, b1][P][N]
        HG_CUDA_TRY(tens.alloc((size_t)3 * G * plane * 4));
        HG_CUDA_TRY(kres.alloc((size_t)3 * G * kplane * 4));
        HG_CUDA_TRY(buf.alloc((size_t)3 * G * wn * 4));
        for (int g = 0; g < G; ++g) {
            OperandSet ops{};
            const uint32_t* src[4] = {a0s[g0 + g], a1s[g0 + g], b0s[g0 + g], b1s[g0 + g]};
            for (int k = 0; k < 4; ++k) { ops.words[k] = src[k]; ops.bits[k] = level; ops.is_signed[k] = 1; }
            if ((rc = launch_modup(ctx, ops, 4, P, res.u32() + (size_t)4 * g * plane, 0, st))) return rc;
        }
        if ((rc = hg_ntt_launch(ctx, res.u32(), 4 * G * P, P, 0, true, st))) return rc;
        // every tensor term has exactly one a factor: carrying the CRT constants on a0, a1
        // lets the CRT skip its own constant product (as a prepared operand does)
        if (prescale)
            for (int g = 0; g < G; ++g)
                if ((rc = prescale_rows(ctx, res.u32() + (size_t)4 * g * plane, 2, P, st))) return rc;
        for (int g = 0; g < G; ++g) {
            const uint32_t* r = res.u32() + (size_t)4 * g * plane;
            rc = hg_intt_fused(ctx, 2, tens.u32() + (size_t)3 * g * plane, r, r + plane, r + 2 * plane,
                               r + 3 * plane, P, st);
            if (rc) return rc < 0 ? hg_fail(HG_EINVAL, "fused tensor product not available") : rc;
        }
        uint32_t* d = buf.u32();
        for (int h = 0; h < G; h += 2) {
            const int gh = G - h < 2 ? G - h : 2;
            OutSet touts{};
            for (int k = 0; k < gh; ++k) {
                const int g = h + k;
                touts.out[3 * k] = d + (size_t)(2 * g) * wn;
                touts.out[3 * k + 1] = d + (size_t)(2 * g + 1) * wn;
                touts.out[3 * k + 2] = d + (size_t)(2 * G + g) * wn;
            }
            if ((rc = launch_crt(ctx, tens.u32() + (size_t)3 * h * plane, 3 * gh, P, 0, level, touts, st,
                                 nullptr, prescale)))
                return rc;
        }
        OperandSet kops{};
        for (int g = 0; g < G; ++g) {
            kops.words[g] = d + (size_t)(2 * G + g) * wn; kops.bits[g] = level; kops.is_signed[g] = 0;
        }
        if ((rc = launch_modup(ctx, kops, G, Pk, kres.u32(), 0, st))) return rc;
        if ((rc = hg_ntt_launch(ctx, kres.u32(), G * Pk, Pk, 0, true, st))) return rc;
        uint32_t* t = kres.u32() + (size_t)G * kplane;
        rc = hg_intt_fused(ctx, 1, t, kres.u32(), evk->d_kb, evk->d_ka, nullptr, Pk, st, G);
        if (rc) return rc < 0 ? hg_fail(HG_EINVAL, "batched key product not available") : rc;
        CrtFinish fin;
        for (int k = 0; k < 2 * G; ++k) fin.add[k] = d + (size_t)k * wn;
        fin.post = rescale_bits;
        OutSet kouts{};
        for (int g = 0; g < G; ++g) {
            kouts.out[2 * g] = out0s[g0 + g];
            kouts.out[2 * g + 1] = out1s[g0 + g];
        }
        if ((rc = launch_crt(ctx, t, 2 * G, Pk, evk->big_l, level, kouts, st, &fin, evk->prescaled))) return rc;
        g0 += G;
    }
    return HG_OK;
}

// ---- inner products over prepared operands ------------------------------------------------------
// acc[q] += A[q][b] (x) B[b] for QG weight sets at once: one thread per (prime, coefficient),
// the B residues of every b read once, the accumulators in registers.  Montgomery products of
// operands reduced to [0, 2p) (the same products the fused tensor kernel forms), sums kept in
// [0, 2p) and reduced to [0, p) on the way out.
template <int QG>
__global__ void __launch_bounds__(256) inner_acc_kernel(const uint32_t* const* __restrict__ a_tab, int nq,
                                                        int nb, const uint32_t* __restrict__ resb,
                                                        uint32_t* __restrict__ out, int P, int N,
                                                        const PrimeInfo* __restrict__ pinfo) {
    const int j = blockIdx.y;
    const PrimeInfo pi = pinfo[j];
    const uint32_t p = pi.p, p2 = p << 1;
    const size_t plane = (size_t)P * N;
    const int q0 = blockIdx.z * QG;
    const int nqg = nq - q0 < QG ? nq - q0 : QG;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) {
        const size_t o = (size_t)j * N + i;
        uint32_t acc[QG][3];
#pragma unroll
        for (int q = 0; q < QG; ++q) acc[q][0] = acc[q][1] = acc[q][2] = 0;
        for (int b = 0; b < nb; ++b) {
            uint32_t b0 = resb[(size_t)(2 * b) * plane + o], b1 = resb[(size_t)(2 * b + 1) * plane + o];
            b0 = min(b0, b0 - p2); b0 = min(b0, b0 - p2);     // [0, 4p) -> [0, 2p)
            b1 = min(b1, b1 - p2); b1 = min(b1, b1 - p2);
#pragma unroll
            for (int q = 0; q < QG; ++q) {
                if (q >= nqg) break;
                const uint32_t* a = a_tab[(size_t)(q0 + q) * nb + b];
                uint32_t a0 = a[o], a1 = a[plane + o];
                a0 = min(a0, a0 - p2); a0 = min(a0, a0 - p2);
                a1 = min(a1, a1 - p2); a1 = min(a1, a1 - p2);
                uint32_t t;
                t = acc[q][0] + mont_mul(a0, b0, p, pi.pinv_neg);
                acc[q][0] = min(t, t - p2);
                t = acc[q][1] + mont_mul(a0, b1, p, pi.pinv_neg);
                t = min(t, t - p2);
                t += mont_mul(a1, b0, p, pi.pinv_neg);
                acc[q][1] = min(t, t - p2);
                t = acc[q][2] + mont_mul(a1, b1, p, pi.pinv_neg);
                acc[q][2] = min(t, t - p2);
            }
        }
#pragma unroll
        for (int q = 0; q < QG; ++q) {
            if (q >= nqg) break;
            uint32_t* dst = out + (size_t)(q0 + q) * 3 * plane + o;
#pragma unroll
            for (int r = 0; r < 3; ++r) dst[(size_t)r * plane] = min(acc[q][r], acc[q][r] - p);
        }
    }
}

extern "C" int hg_ct_inner_prepared(hg_ctx* ctx, const hg_key* evk, int nq, int nb,
                                    const hg_ctprep* const* a, const uint32_t* const* b0s,
                                    const uint32_t* const* b1s, int level, int rescale_bits,
                                    uint32_t* const* out0s, uint32_t* const* out1s, void* stream) {
    if (!ctx || !evk || nq < 1 || nb < 1 || !a || !b0s || !b1s || !out0s || !out1s ||
        evk->level != level || rescale_bits < 0 || rescale_bits >= level)
        return hg_fail(HG_EINVAL, "hg_ct_inner_prepared: bad arguments");
    const int P = a[0]->P;
    const bool prescaled = a[0]->prescaled;
    for (int k = 0; k < nq * nb; ++k)
        if (!a[k] || a[k]->ctx != ctx || a[k]->level != level || a[k]->P != P || a[k]->prescaled != prescaled)
            return hg_fail(HG_EINVAL, "hg_ct_inner_prepared: operands differ in level / basis");
    if (P < tensor_sum_primes(ctx, level, nb))
        return hg_fail(HG_EINVAL, "hg_ct_inner_prepared: operands prepared for fewer summed terms");
    cudaStream_t st = (cudaStream_t)stream;
    const int N = ctx->N;
    const int W = words_for_bits(level);
    const size_t plane = (size_t)P * N;
    Scratch resb(st), acc(st), tab(st), buf(st);
    HG_CUDA_TRY(resb.alloc((size_t)2 * nb * plane * 4));
    HG_CUDA_TRY(acc.alloc((size_t)3 * nq * plane * 4));
    HG_CUDA_TRY(tab.alloc((size_t)nq * nb * sizeof(uint32_t*)));
    HG_CUDA_TRY(buf.alloc((size_t)5 * W * N * 4));
    std::vector<const uint32_t*> host(nq * nb);
    for (int k = 0; k < nq * nb; ++k) host[k] = a[k]->d_res;
    HG_CUDA_TRY(cudaMemcpyAsync(tab.u32(), host.data(), host.size() * sizeof(uint32_t*),
                                cudaMemcpyHostToDevice, st));
    // forward residues of every b: [nb][2][P][N]
    for (int b0 = 0; b0 < nb; b0 += 2) {
        const int g = nb - b0 < 2 ? nb - b0 : 2;
        OperandSet ops{};
        for (int k = 0; k < g; ++k) {
            ops.words[2 * k] = b0s[b0 + k]; ops.bits[2 * k] = level; ops.is_signed[2 * k] = 1;
            ops.words[2 * k + 1] = b1s[b0 + k]; ops.bits[2 * k + 1] = level; ops.is_signed[2 * k + 1] = 1;
        }
        if (int rc = launch_modup(ctx, ops, 2 * g, P, resb.u32() + (size_t)2 * b0 * plane, 0, st)) return rc;
    }
    if (int rc = hg_ntt_launch(ctx, resb.u32(), 2 * nb * P, P, 0, true, st)) return rc;
    {
        constexpr int QG = 4;
        dim3 grid = pw_grid(N, P);
        grid.z = (nq + QG - 1) / QG;
        const int tpw = hg_timer_begin(ctx, st, HG_K_POINTWISE);
        inner_acc_kernel<QG><<<grid, 256, 0, st>>>(reinterpret_cast<const uint32_t* const*>(tab.u32()), nq, nb,
                                                   resb.u32(), acc.u32(), P, N, ctx->d_pinfo);
        hg_timer_end(ctx, tpw, st, HG_K_POINTWISE, (double)nq * nb * 4.0 * plane * 4);
        HG_LAUNCH_CHECK(ctx);
    }
    if (int rc = hg_ntt_launch(ctx, acc.u32(), 3 * nq * P, P, 0, false, st)) return rc;
    uint32_t* d0 = buf.u32();
    uint32_t* d1 = d0 + (size_t)W * N;
    uint32_t* d2 = d1 + (size_t)W * N;
    uint32_t* e0 = d2 + (size_t)W * N;
    uint32_t* e1 = e0 + (size_t)W * N;
    for (int q = 0; q < nq; ++q) {
        OutSet outs{};
        outs.out[0] = d0; outs.out[1] = d1; outs.out[2] = d2;
        if (int rc = launch_crt(ctx, acc.u32() + (size_t)3 * q * plane, 3, P, 0, level, outs, st, nullptr, prescaled))
            return rc;
        if (int rc = ct_mult_finish(ctx, evk, d0, d1, d2, e0, e1, level, rescale_bits, out0s[q], out1s[q], st))
            return rc;
    }
    return HG_OK;
}

extern "C" int hg_ct_automorph(hg_ctx* ctx, const hg_key* key, const uint32_t* c0,
                               const uint32_t* c1, int level, int64_t k, uint32_t* out0,
                               uint32_t* out1, void* stream) {
    if (!ctx || !key || key->level != level)
        return hg_fail(HG_EINVAL, "hg_ct_automorph: bad arguments (key must be prepared at the level)");
    cudaStream_t st = (cudaStream_t)stream;
    const int N = ctx->N;
    const int W = words_for_bits(level);
    Scratch buf(st);
    HG_CUDA_TRY(buf.alloc((size_t)2 * W * N * 4));
    uint32_t* a0 = buf.u32();
    uint32_t* e0 = a0 + (size_t)W * N;
    int rc = hg_ew_automorphism(ctx, a0, c0, level, k, st);
    if (rc) return rc;
    rc = hg_keyswitch(ctx, key, c1, k, e0, out1, stream);
    if (rc) return rc;
    return hg_ew_add(ctx, out0, a0, e0, level, false, st);
}

// `count` rotations by the same automorphism and key at one level, up to 4 per group of
// launches: one ModUp of the 4 c1 gathers, one forward NTT over [4][P][N] (twiddle loads
// shared by the rows of a prime), one batched key product fused into the inverse NTT and one
// 8-output CRT -- instead of 4 separate chains.  Each output is identical to hg_ct_automorph's.
static int automorph_batch_impl(hg_ctx* ctx, const hg_key* key, int count, const uint32_t* const* c0s,
                                const uint32_t* const* c1s, int level, int64_t k, uint32_t* const* out0s,
                                uint32_t* const* out1s, void* stream, bool acc);

extern "C" int hg_ct_automorph_batch(hg_ctx* ctx, const hg_key* key, int count,
                                     const uint32_t* const* c0s, const uint32_t* const* c1s,
                                     int level, int64_t k, uint32_t* const* out0s,
                                     uint32_t* const* out1s, void* stream) {
    return automorph_batch_impl(ctx, key, count, c0s, c1s, level, k, out0s, out1s, stream, false);
}

// out_i = c_i + phi_k(c_i) key-switched: one step of the rotate-and-sum ladders (matrix.py
// rotate_sum: c += rot(c, 2^j)) without a separate ciphertext add per item
extern "C" int hg_ct_rotate_add_batch(hg_ctx* ctx, const hg_key* key, int count,
                                      const uint32_t* const* c0s, const uint32_t* const* c1s,
                                      int level, int64_t k, uint32_t* const* out0s,
                                      uint32_t* const* out1s, void* stream) {
    return automorph_batch_impl(ctx, key, count, c0s, c1s, level, k, out0s, out1s, stream, true);
}

static int automorph_batch_impl(hg_ctx* ctx, const hg_key* key, int count, const uint32_t* const* c0s,
                                const uint32_t* const* c1s, int level, int64_t k, uint32_t* const* out0s,
                                uint32_t* const* out1s, void* stream, bool acc) {
    if (!ctx || !key || key->level != level || count < 0 || (count && (!c0s || !c1s || !out0s || !out1s)))
        return hg_fail(HG_EINVAL, "hg_ct_automorph_batch: bad arguments (key must be prepared at the level)");
    cudaStream_t st = (cudaStream_t)stream;
    const int N = ctx->N;
    const int W = words_for_bits(level);
    const int P = key->P;
    const int64_t n2 = 2ll * N;
    const int64_t kk = ((k % n2) + n2) % n2;
    if ((kk & 1) == 0) return hg_fail(HG_EINVAL, "automorphism exponent must be odd");
    const int64_t kinv = kk == 1 ? 0 : inverse_mod_2n(kk, n2);
    int rc;
    static const int gmax = hg_env_group("HG_ROT_G", 4, 1, 8);   // 8: no gain measured
    const bool fin_ok = crt_finish_ok(ctx, P, key->big_l, level) && !getenv("HG_ROT_NO_FINISH");
    for (int g0 = 0; g0 < count; g0 += gmax) {
        int G = count - g0 < gmax ? count - g0 : gmax;
        if (G > 8) G = 8;
        if (!acc && (G == 1 || !fuse_pointwise())) {
            for (int g = 0; g < G; ++g)
                if ((rc = hg_ct_automorph(ctx, key, c0s[g0 + g], c1s[g0 + g], level, k, out0s[g0 + g],
                                          out1s[g0 + g], stream)))
                    return rc;
            continue;
        }
        if (acc && !fuse_pointwise()) {
            for (int g = 0; g < G; ++g) {
                Scratch t2(st);
                HG_CUDA_TRY(t2.alloc((size_t)2 * W * N * 4));
                uint32_t* r0 = t2.u32();
                uint32_t* r1 = r0 + (size_t)W * N;
                if ((rc = hg_ct_automorph(ctx, key, c0s[g0 + g], c1s[g0 + g], level, k, r0, r1, stream))) return rc;
                if ((rc = hg_ew_add(ctx, out0s[g0 + g], c0s[g0 + g], r0, level, false, st))) return rc;
                if ((rc = hg_ew_add(ctx, out1s[g0 + g], c1s[g0 + g], r1, level, false, st))) return rc;
            }
            continue;
        }
        for (int g = 0; g < G; ++g)
            if (out0s[g0 + g] == c0s[g0 + g] || out0s[g0 + g] == c1s[g0 + g] || out1s[g0 + g] == c1s[g0 + g] ||
                out1s[g0 + g] == c0s[g0 + g])
                return hg_fail(HG_EINVAL, "hg_ct_automorph_batch: outputs must not alias inputs");
        Scratch res(st), buf(st);
        HG_CUDA_TRY(res.alloc((size_t)3 * G * P * N * 4));   // x residues [G][P][N], products [G][2][P][N]
        HG_CUDA_TRY(buf.alloc((size_t)(acc ? 3 : 2) * G * W * N * 4));   // automorphed c0, e0 per item (+ e1 with acc)
        for (int h = 0; h < G; h += 4) {   // ModUp: up to 4 gathered c1 per launch
            const int gh = G - h < 4 ? G - h : 4;
            OperandSet ops{};
            for (int g = 0; g < gh; ++g) {
                ops.words[g] = c1s[g0 + h + g]; ops.bits[g] = level; ops.is_signed[g] = 0;   // canonical rep
            }
            if ((rc = launch_modup(ctx, ops, gh, P, res.u32() + (size_t)h * P * N, kinv, st))) return rc;
        }
        if ((rc = hg_ntt_launch(ctx, res.u32(), G * P, P, 0, true, st))) return rc;
        uint32_t* t = res.u32() + (size_t)G * P * N;
        rc = hg_intt_fused(ctx, 1, t, res.u32(), key->d_kb, key->d_ka, nullptr, P, st, G);
        if (rc) return rc < 0 ? hg_fail(HG_EINVAL, "batched key product not available") : rc;
        if (fin_ok) {   // (phi(c0) [+ c0], [c1]) added in the CRT epilogue, written to the outputs
            for (int h = 0; h < G; h += 4) {
                const int gh = G - h < 4 ? G - h : 4;
                uint32_t* ad = buf.u32() + (size_t)2 * h * W * N;
                if ((rc = hg_ew_automorph_addends(ctx, ad, c0s + g0 + h, c1s + g0 + h, gh, level, k, acc, st)))
                    return rc;
                CrtFinish fin;
                for (int q = 0; q < 2 * gh; ++q) fin.add[q] = ad + (size_t)q * W * N;
                OutSet outs{};
                for (int g = 0; g < gh; ++g) {
                    outs.out[2 * g] = out0s[g0 + h + g];
                    outs.out[2 * g + 1] = out1s[g0 + h + g];
                }
                if ((rc = launch_crt(ctx, t + (size_t)2 * h * P * N, 2 * gh, P, key->big_l, level, outs, st,
                                     &fin, key->prescaled)))
                    return rc;
            }
            continue;
        }
        for (int h = 0; h < G; h += 4) {   // CRT: up to 8 outputs (4 items) per launch
            const int gh = G - h < 4 ? G - h : 4;
            OutSet outs{};
            for (int g = 0; g < gh; ++g) {
                outs.out[2 * g] = buf.u32() + (size_t)(2 * (h + g) + 1) * W * N;   // e0
                outs.out[2 * g + 1] = acc ? buf.u32() + (size_t)(2 * G + h + g) * W * N : out1s[g0 + h + g];
            }
            if ((rc = launch_crt(ctx, t + (size_t)2 * h * P * N, 2 * gh, P, key->big_l, level, outs, st,
                                 nullptr, key->prescaled)))
                return rc;
        }
        for (int g = 0; g < G; ++g) {
            uint32_t* a0 = buf.u32() + (size_t)(2 * g) * W * N;
            if ((rc = hg_ew_automorphism(ctx, a0, c0s[g0 + g], level, k, st))) return rc;
            if (acc) {   // out0 = c0 + (phi(c0) + e0), out1 = c1 + e1 (exact mod 2^level)
                if ((rc = hg_ew_add(ctx, a0, a0, a0 + (size_t)W * N, level, false, st))) return rc;
                if ((rc = hg_ew_add(ctx, out0s[g0 + g], c0s[g0 + g], a0, level, false, st))) return rc;
                if ((rc = hg_ew_add(ctx, out1s[g0 + g], c1s[g0 + g], buf.u32() + (size_t)(2 * G + g) * W * N,
                                    level, false, st)))
                    return rc;
            } else if ((rc = hg_ew_add(ctx, out0s[g0 + g], a0, a0 + (size_t)W * N, level, false, st))) {
                return rc;
            }
        }
    }
    return HG_OK;
}

// ---- plaintext products with the rescale fused into the CRT window -------------------------------
// HeEngine.mult_plain = mult_plain then rescale by the plaintext scale (ckks.py:147-163, 197-224,
// 315-317): out = divide_round(c * m mod 2^level, bits) = bits [bits, level) of (c*m + 2^(bits-1))
// (reducing mod 2^level first does not change those bits).  The ciphertext polys are read as
// centered level-bit values, the plaintext through its caller-chosen (compact) operand.
namespace {
int plain_primes(hg_ctx* ctx, int level, const hg_operand* ms, int count) {
    int mb = 1;
    for (int i = 0; i < count; ++i) mb = std::max(mb, magnitude_bits(ms[i]));
    return primes_for_product(ctx, (double)(level - 1) + mb, level);
}
bool plain_args_ok(int level, int rescale_bits) { return level >= 1 && rescale_bits >= 1 && rescale_bits < level; }
}  // namespace

// One ciphertext times `count` plaintexts (replicate's one-hot masks, ccp_to_cp's column
// ranges: matrix.py:79-96, 196-209): c's ModUp and forward NTT run once for all of them; each
// group of up to 4 plaintexts is one ModUp, one NTT, one fused pointwise/inverse pass and one CRT.
extern "C" int hg_ct_mult_plain_many(hg_ctx* ctx, const uint32_t* c0, const uint32_t* c1, int level,
                                     int count, const hg_operand* ms, int rescale_bits,
                                     uint32_t* const* out0s, uint32_t* const* out1s, void* stream) {
    if (!ctx || !c0 || !c1 || count < 0 || (count && (!ms || !out0s || !out1s)) ||
        !plain_args_ok(level, rescale_bits))
        return hg_fail(HG_EINVAL, "hg_ct_mult_plain_many: bad arguments");
    if (count == 0) return HG_OK;
    for (int i = 0; i < count; ++i)
        if (!ms[i].words || ms[i].bits < 1 || !out0s[i] || !out1s[i])
            return hg_fail(HG_EINVAL, "hg_ct_mult_plain_many: bad plaintext or output");
    cudaStream_t st = (cudaStream_t)stream;
    const int N = ctx->N;
    const int P = plain_primes(ctx, level, ms, count);
    if (P < 0) return hg_fail(HG_ERANGE, "plaintext product exceeds the NTT prime basis");
    if (!fuse_pointwise()) return hg_fail(HG_EINVAL, "hg_ct_mult_plain_many needs the fused inverse NTT");
    const size_t plane = (size_t)P * N;
    const int G = count < 4 ? count : 4;
    Scratch cres(st), mres(st), prod(st);
    HG_CUDA_TRY(cres.alloc(2 * plane * 4));
    HG_CUDA_TRY(mres.alloc((size_t)G * plane * 4));
    HG_CUDA_TRY(prod.alloc((size_t)2 * G * plane * 4));
    OperandSet cops{};
    cops.words[0] = c0; cops.bits[0] = level; cops.is_signed[0] = 1;
    cops.words[1] = c1; cops.bits[1] = level; cops.is_signed[1] = 1;
    int rc = launch_modup(ctx, cops, 2, P, cres.u32(), 0, st);
    if (!rc) rc = hg_ntt_launch(ctx, cres.u32(), 2 * P, P, 0, true, st);
    if (rc) return rc;
    // the shared factor enters the Montgomery products reduced to [0, p)
    reduce_rows_kernel<<<pw_grid(N, P), 256, 0, st>>>(cres.u32(), N, ctx->d_pinfo);
    ctx->launches++;
    reduce_rows_kernel<<<pw_grid(N, P), 256, 0, st>>>(cres.u32() + plane, N, ctx->d_pinfo);
    HG_LAUNCH_CHECK(ctx);
    for (int g0 = 0; g0 < count; g0 += G) {
        const int gh = count - g0 < G ? count - g0 : G;
        OperandSet mops{};
        for (int g = 0; g < gh; ++g) {
            mops.words[g] = ms[g0 + g].words; mops.bits[g] = ms[g0 + g].bits;
            mops.is_signed[g] = ms[g0 + g].signed_rep;
        }
        if ((rc = launch_modup(ctx, mops, gh, P, mres.u32(), 0, st))) return rc;
        if ((rc = hg_ntt_launch(ctx, mres.u32(), gh * P, P, 0, true, st))) return rc;
        // out rows per plaintext: (m c0, m c1), the key-switch form with c as the shared "key"
        rc = hg_intt_fused(ctx, 1, prod.u32(), mres.u32(), cres.u32(), cres.u32() + plane, nullptr, P, st, gh);
        if (rc) return rc < 0 ? hg_fail(HG_EINVAL, "fused plaintext product not available") : rc;
        OutSet outs{};
        for (int g = 0; g < gh; ++g) {
            outs.out[2 * g] = out0s[g0 + g];
            outs.out[2 * g + 1] = out1s[g0 + g];
        }
        if ((rc = launch_crt(ctx, prod.u32(), 2 * gh, P, rescale_bits, level - rescale_bits, outs, st)))
            return rc;
    }
    return HG_OK;
}

// `count` ciphertexts times one plaintext: m's ModUp and NTT run once; up to 2 ciphertexts (4
// polys) per ModUp launch, 4 (8 outputs) per fused pass and CRT.
extern "C" int hg_ct_mult_plain_batch(hg_ctx* ctx, int count, const uint32_t* const* c0s,
                                      const uint32_t* const* c1s, int level, hg_operand m,
                                      int rescale_bits, uint32_t* const* out0s,
                                      uint32_t* const* out1s, void* stream) {
    if (!ctx || count < 0 || (count && (!c0s || !c1s || !out0s || !out1s)) || !m.words || m.bits < 1 ||
        !plain_args_ok(level, rescale_bits))
        return hg_fail(HG_EINVAL, "hg_ct_mult_plain_batch: bad arguments");
    if (count == 0) return HG_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const int N = ctx->N;
    const int P = plain_primes(ctx, level, &m, 1);
    if (P < 0) return hg_fail(HG_ERANGE, "plaintext product exceeds the NTT prime basis");
    if (!fuse_pointwise()) return hg_fail(HG_EINVAL, "hg_ct_mult_plain_batch needs the fused inverse NTT");
    const size_t plane = (size_t)P * N;
    const int G = count < 4 ? count : 4;
    Scratch mres(st), cres(st);
    HG_CUDA_TRY(mres.alloc(plane * 4));
    HG_CUDA_TRY(cres.alloc((size_t)2 * G * plane * 4));
    OperandSet mops{};
    mops.words[0] = m.words; mops.bits[0] = m.bits; mops.is_signed[0] = m.signed_rep;
    int rc = launch_modup(ctx, mops, 1, P, mres.u32(), 0, st);
    if (!rc) rc = hg_ntt_launch(ctx, mres.u32(), P, P, 0, true, st);
    if (rc) return rc;
    reduce_rows_kernel<<<pw_grid(N, P), 256, 0, st>>>(mres.u32(), N, ctx->d_pinfo);
    HG_LAUNCH_CHECK(ctx);
    for (int g0 = 0; g0 < count; g0 += G) {
        const int gh = count - g0 < G ? count - g0 : G;
        for (int h = 0; h < gh; h += 2) {
            const int k = gh - h < 2 ? gh - h : 2;
            OperandSet ops{};
            for (int q = 0; q < k; ++q) {
                ops.words[2 * q] = c0s[g0 + h + q]; ops.bits[2 * q] = level; ops.is_signed[2 * q] = 1;
                ops.words[2 * q + 1] = c1s[g0 + h + q]; ops.bits[2 * q + 1] = level; ops.is_signed[2 * q + 1] = 1;
            }
            if ((rc = launch_modup(ctx, ops, 2 * k, P, cres.u32() + (size_t)2 * h * plane, 0, st))) return rc;
        }
        if ((rc = hg_ntt_launch(ctx, cres.u32(), 2 * gh * P, P, 0, true, st))) return rc;
        // every poly times the shared plaintext, in place (each block reads its chunk first)
        rc = hg_intt_fused(ctx, 5, cres.u32(), cres.u32(), mres.u32(), nullptr, nullptr, P, st, 2 * gh);
        if (rc) return rc < 0 ? hg_fail(HG_EINVAL, "fused plaintext product not available") : rc;
        OutSet outs{};
        for (int g = 0; g < gh; ++g) {
            outs.out[2 * g] = out0s[g0 + g];
            outs.out[2 * g + 1] = out1s[g0 + g];
        }
        if ((rc = launch_crt(ctx, cres.u32(), 2 * gh, P, rescale_bits, level - rescale_bits, outs, st)))
            return rc;
    }
    return HG_OK;
}
