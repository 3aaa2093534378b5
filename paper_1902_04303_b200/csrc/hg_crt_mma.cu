// hg_crt_mma.cu -- CRT reconstruction on the tensor cores (int8 mma.sync, SASS IMMA.16832).
//
// Column t of the exact product is  col_t = sum_j y_j * M[j][t]  (y_j < 2^30, M 32-bit words
// of Q/p_j).  Splitting both into bytes,
//     col_t = sum_{q,r} 2^(8(q+r)) * sum_j yb[j][q] * mb[j][t][r],
// which is ONE u8 x u8 -> s32 GEMM with rows (coefficient n, byte q), K = primes j and columns
// (column t, byte r): C[(n,q)][(t,r)] = sum_j yb * mb  (< 320 * 255^2 < 2^25, exact in s32).
// Each 16-row m-tile holds 4 coefficients x 4 byte planes (row = q*4 + n), so a C fragment
// lane owns the four products (q0, r0), (q0, r0+1), (q0+2, r0), (q0+2, r0+1) of one (n, t):
// they fold into one u64 "digit" of weight 2^(8(q0+r0)).  A per-coefficient lane then runs the
// exact carry chain over the columns, adds v * (-Q) and the rounding bit, checks the truncated
// carry window and emits bits [shift, shift+out_bits) -- identical output to crt_kernel.
#include "hg_internal.cuh"

namespace {

constexpr int kCoefs = 64;        // coefficients per CTA (16 m-tiles)
constexpr int kWarps = 8;         // 2 m-tiles (8 coefficients) per warp
constexpr int kColBlock = 8;      // output columns per accumulation pass (4 n8-tiles)

__device__ __forceinline__ void mma_u8(int (&c)[4], const uint32_t (&a)[4], uint2 b) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};\n"
        : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b.x), "r"(b.y));
}

struct Outs4 {
    uint32_t* out[4];
};

// exact column scan for one coefficient from the byte planes (rare fallback path)
__device__ void crt_rescan_exact(const uint8_t* ybase, int rs_bytes, int P, int W,
                                 const uint32_t* __restrict__ Mtab, const uint32_t* __restrict__ negQ,
                                 uint32_t v, int shift, int out_bits, uint32_t* __restrict__ out,
                                 int N, int i) {
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
            uint32_t y = (uint32_t)ybase[j] | ((uint32_t)ybase[rs_bytes * 4 + j] << 8) |
                         ((uint32_t)ybase[rs_bytes * 8 + j] << 16) |
                         ((uint32_t)ybase[rs_bytes * 12 + j] << 24);
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

__global__ void __launch_bounds__(kWarps * 32) crt_mma_kernel(
    const uint32_t* __restrict__ res, int P, int P32, int N, const PrimeInfo* __restrict__ pinfo,
    const uint2* __restrict__ Bfrag, const uint32_t* __restrict__ Mtab, int W,
    const uint32_t* __restrict__ negQ, const uint32_t* __restrict__ cinv,
    const uint32_t* __restrict__ cinv_sh, const double* __restrict__ invp, int shift,
    int out_bits, int tb0, int rs_words, Outs4 outs) {
    extern __shared__ __align__(16) uint8_t smem[];
    // byte planes: row (mt*4 + q)*4 + n, row stride rs_words (= 4 mod 32 words: conflict-free)
    uint32_t* yb = reinterpret_cast<uint32_t*>(smem);
    const int rs_bytes = rs_words * 4;
    uint64_t* part = reinterpret_cast<uint64_t*>(smem + (size_t)kCoefs * 4 * rs_bytes);  // [8][8][8][4]
    uint32_t* vsm = reinterpret_cast<uint32_t*>(part + kWarps * 8 * kColBlock * 4);
    double* ssm = reinterpret_cast<double*>(vsm + kCoefs);  // [4][64]
    uint2* bsm = reinterpret_cast<uint2*>(ssm + 4 * kCoefs);  // B fragments of one column block

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int cb = blockIdx.x * kCoefs;
    const int oy = blockIdx.y;
    const uint32_t* r = res + (size_t)oy * P * N;
    uint32_t* out = oy == 0 ? outs.out[0] : oy == 1 ? outs.out[1] : oy == 2 ? outs.out[2] : outs.out[3];

    // ---- phase 1: y_j = r_j * cinv_j mod p_j -> byte planes; S = sum y_j / p_j ----------------
    {
        const int n = tid & 63, jg = tid >> 6;
        const int mt = n >> 2, nl = n & 3;
        double S = 0.0;
        // 4 quads (16 residues) per thread in flight before any of them is consumed
        for (int jb = jg * 4; jb < P32; jb += 64) {
            uint32_t xr[4][4];
#pragma unroll
            for (int qd = 0; qd < 4; ++qd)
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int j = jb + 16 * qd + u;
                    xr[qd][u] = j < P ? __ldcs(r + (size_t)j * N + cb + n) : 0u;
                }
#pragma unroll
            for (int qd = 0; qd < 4; ++qd) {
                const int j4 = jb + 16 * qd;
                if (j4 >= P32) break;
                uint32_t y[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int j = j4 + u;
                    y[u] = 0;
                    if (j < P) {
                        const uint32_t p = pinfo[j].p;
                        y[u] = reduce_2p(mul_shoup_lazy(xr[qd][u], cinv[j], cinv_sh[j], p), p);
                        S += (double)y[u] * invp[j];
                    }
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const uint32_t w = __byte_perm(__byte_perm(y[0] >> (8 * q), y[1] >> (8 * q), 0x0040),
                                                   __byte_perm(y[2] >> (8 * q), y[3] >> (8 * q), 0x0040),
                                                   0x5410);
                    yb[((mt * 4 + q) * 4 + nl) * rs_words + (j4 >> 2)] = w;
                }
            }
        }
        ssm[jg * kCoefs + n] = S;
    }
    __syncthreads();
    if (tid < kCoefs) {
        const double S = ssm[tid] + ssm[kCoefs + tid] + ssm[2 * kCoefs + tid] + ssm[3 * kCoefs + tid];
        vsm[tid] = (uint32_t)floor(S + 0.5);
    }
    __syncthreads();

    // ---- phase 2/3: GEMM over column blocks + per-coefficient carry chain --------------------
    const int sw = shift >> 5, sb = shift & 31;
    const int out_w = (out_bits + 31) >> 5;
    const uint32_t top_mask = (out_bits & 31) ? ((1u << (out_bits & 31)) - 1u) : 0xffffffffu;
    const int T = sw + out_w + (sb ? 1 : 0);
    const int round_col = shift > 0 ? ((shift - 1) >> 5) : -1;
    const uint32_t round_bit = shift > 0 ? (1u << ((shift - 1) & 31)) : 0u;
    const int nks = P32 >> 5;
    const int q0 = lane >> 4, nl = (lane >> 2) & 3, kq = (lane & 3) * 4;
    const int s0 = q0 + 2 * (lane & 1);
    // chain state (lanes 0..7: coefficient warp*8 + lane)
    uint64_t carry = 0;
    uint32_t prev = 0;
    bool amb = false;
    const int my_coef = warp * 8 + (lane & 7);
    const uint32_t my_v = vsm[my_coef];
    uint64_t* wpart = part + (size_t)warp * 8 * kColBlock * 4;
    for (int tb = tb0; tb < T; tb += kColBlock) {
        int acc[2][4][4];
#pragma unroll
        for (int m = 0; m < 2; ++m)
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int e = 0; e < 4; ++e) acc[m][i][e] = 0;
        // stage this column block's B fragments (4 n-tiles x nks x 32 lanes) in shared memory
        __syncthreads();
        {
            const uint2* src = Bfrag + (size_t)(tb >> 1) * nks * 32;
            for (int e = tid; e < 4 * nks * 32; e += kWarps * 32) bsm[e] = __ldg(src + e);
        }
        __syncthreads();
        const uint2* bt = bsm + lane;
        for (int ks = 0; ks < nks; ++ks) {
            uint32_t a[2][4];
#pragma unroll
            for (int m = 0; m < 2; ++m) {
                const int mt = warp * 2 + m;
                const uint8_t* row_lo = smem + (size_t)((mt * 4 + q0) * 4 + nl) * rs_bytes + ks * 32 + kq;
                const uint8_t* row_hi = row_lo + (size_t)8 * rs_bytes;  // q0 + 2
                a[m][0] = *reinterpret_cast<const uint32_t*>(row_lo);
                a[m][1] = *reinterpret_cast<const uint32_t*>(row_hi);
                a[m][2] = *reinterpret_cast<const uint32_t*>(row_lo + 16);
                a[m][3] = *reinterpret_cast<const uint32_t*>(row_hi + 16);
            }
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const uint2 b = bt[(i * nks + ks) * 32];
                mma_u8(acc[0][i], a[0], b);
                mma_u8(acc[1][i], a[1], b);
            }
        }
        // fold each lane's four products into one digit of weight 2^(8 s0)
#pragma unroll
        for (int m = 0; m < 2; ++m)
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const uint64_t val = (uint64_t)(uint32_t)acc[m][i][0] +
                                     ((uint64_t)(uint32_t)acc[m][i][1] << 8) +
                                     ((uint64_t)(uint32_t)acc[m][i][2] << 16) +
                                     ((uint64_t)(uint32_t)acc[m][i][3] << 24);
                const int cw = m * 4 + nl;
                const int ti = i * 2 + ((lane & 3) >> 1);
                wpart[(cw * kColBlock + ti) * 4 + s0] = val;
            }
        __syncwarp();
        // parallel combine: lane -> (coefficient lane/4, columns 2(lane%4), +1); each column
        // value becomes (lo32, hi) with value = hi * 2^32 + lo32 (hi < 2^43)
        {
            const int cw = lane >> 2;
            const uint32_t cv = vsm[warp * 8 + cw];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int ti = (lane & 3) * 2 + h;
                const int t = tb + ti;
                uint64_t* pp = wpart + (size_t)(cw * kColBlock + ti) * 4;
                const uint64_t x0 = pp[0] + (pp[1] << 8);   // < 2^57
                const uint64_t x1 = pp[2] + (pp[3] << 8);   // weight 2^16
                const uint64_t extra = (uint64_t)cv * negQ[t] + (t == round_col ? round_bit : 0u);
                const uint64_t lo = (x0 & 0xffffffffull) + ((x1 & 0xffffull) << 16) + (extra & 0xffffffffull);
                pp[0] = lo & 0xffffffffull;
                pp[1] = (lo >> 32) + (x0 >> 32) + (x1 >> 16) + (extra >> 32);
            }
        }
        __syncwarp();
        if (lane < 8) {
            const ulonglong2* pp = reinterpret_cast<const ulonglong2*>(wpart + (size_t)lane * kColBlock * 4);
            ulonglong2 cv[kColBlock];
#pragma unroll
            for (int ti = 0; ti < kColBlock; ++ti) cv[ti] = pp[2 * ti];   // all loads first
            uint32_t words[kColBlock];
#pragma unroll
            for (int ti = 0; ti < kColBlock; ++ti) {   // the serial part: 3 adds per column
                const uint64_t lo = cv[ti].x + (carry & 0xffffffffull);
                words[ti] = (uint32_t)lo;
                carry = cv[ti].y + (lo >> 32) + (carry >> 32);
            }
            // columns past T carried garbage into `carry`; it is never used after the last block
#pragma unroll
            for (int ti = 0; ti < kColBlock; ++ti) {
                const int t = tb + ti;
                if (t >= T) break;
                const uint32_t word = words[ti];
                if (t < sw) {
                    if (t == tb0 + 1) amb = word >= 0xFFFFFF00u;
                    else if (t > tb0 + 1) amb = amb && (word == 0xffffffffu);
                } else if (sb == 0) {
                    const int u = t - sw;
                    out[(size_t)u * N + cb + my_coef] = (u == out_w - 1) ? (word & top_mask) : word;
                } else if (t > sw) {
                    const int u = t - sw - 1;
                    const uint32_t o = (prev >> sb) | (word << (32 - sb));
                    out[(size_t)u * N + cb + my_coef] = (u == out_w - 1) ? (o & top_mask) : o;
                }
                prev = word;
            }
        }
        __syncwarp();
    }
    if (lane < 8 && tb0 > 0 && amb) {
        const int mt = my_coef >> 2, n4 = my_coef & 3;
        const uint8_t* ybase = smem + (size_t)((mt * 4 + 0) * 4 + n4) * rs_bytes;
        crt_rescan_exact(ybase, rs_bytes, P, W, Mtab, negQ, my_v, shift, out_bits, out, N,
                         cb + my_coef);
    }
}

}  // namespace

// Byte-split fragment table of M for the mma path: for n-tile nt (columns t = 2nt, 2nt+1,
// bytes r = 0..3), k-step ks and lane L: b0 = bytes r of M[k][t] for k = 32ks + 4(L%4) + 0..3,
// col = L/4 -> (t = 2nt + col/4, r = col%4); b1 = the same 16 primes further.
int hg_crt_build_fragments(const CrtTable& t, int P, int P32, std::vector<uint32_t>& out,
                           const std::vector<uint32_t>& M) {
    const int W = t.W, nks = P32 / 32, ntiles = W / 2;
    out.assign((size_t)ntiles * nks * 32 * 2, 0u);
    for (int nt = 0; nt < ntiles; ++nt)
        for (int ks = 0; ks < nks; ++ks)
            for (int L = 0; L < 32; ++L) {
                const int col = L / 4;
                const int tt = 2 * nt + col / 4, rr = col % 4;
                for (int half = 0; half < 2; ++half) {
                    uint32_t word = 0;
                    for (int bi = 0; bi < 4; ++bi) {
                        const int k = ks * 32 + (L % 4) * 4 + bi + 16 * half;
                        uint32_t byte = 0;
                        if (k < P && tt < W) byte = (M[(size_t)k * W + tt] >> (8 * rr)) & 0xffu;
                        word |= byte << (8 * bi);
                    }
                    out[(((size_t)nt * nks + ks) * 32 + L) * 2 + half] = word;
                }
            }
    return HG_OK;
}

int hg_crt_mma_launch(hg_ctx* ctx, const CrtTable* tab, const uint32_t* res, int nouts, int P,
                      int shift, int out_bits, int tb0, uint32_t* const* outs_in, cudaStream_t st) {
    const int P32 = tab->P32;
    int rs_words = P32 / 4;
    rs_words += (4 - rs_words) & 31;
    const size_t smem = (size_t)kCoefs * 4 * rs_words * 4 + (size_t)kWarps * 8 * kColBlock * 4 * 8 +
                        kCoefs * 4 + 4 * kCoefs * 8 + (size_t)4 * (P32 / 32) * 32 * 8;
    static std::atomic<uint64_t> attr_set{0};
    if (hg_first_on_device(attr_set, ctx->device))
        cudaFuncSetAttribute(crt_mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    Outs4 o{};
    for (int k = 0; k < nouts; ++k) o.out[k] = outs_in[k];
    const int N = ctx->N;
    dim3 grid(N / kCoefs, nouts);
    if (int rc = hg_crt_ensure_fallback(ctx, tab)) return rc;
    crt_mma_kernel<<<grid, kWarps * 32, smem, st>>>(res, P, P32, N, ctx->d_pinfo, tab->d_Bfrag,
                                                    tab->d_M, tab->W, tab->d_negQ, tab->d_cinv,
                                                    tab->d_cinv_sh, tab->d_invp, shift, out_bits,
                                                    tb0, rs_words, o);
    HG_LAUNCH_CHECK(ctx);
    return HG_OK;
}
