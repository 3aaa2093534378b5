// hg_modup_mma.cu -- ModUp (radix-2^32 words -> residues mod 30-bit primes) on the tensor cores.
//
// r_j(a) = sum_w a_w 2^(32w) mod p_j.  With a_w split into bytes a_{w,q} and the constants
// D(j,w,q) = 2^(32w+8q) mod p_j split into bytes d_r:
//     r_j = sum_r 2^(8r) * sum_{(w,q)} a_{w,q} * d_r(j,w,q)   (mod p_j)
// i.e. one u8 x u8 -> s32 GEMM: rows = coefficients, K = (word, byte) -- so an A fragment
// register IS an input word, no byte shuffling --, columns = (prime j, byte r).  Column sums
// are < 4W * 255^2 < 2^26; the four r-partials of a (coefficient, prime) sit in two adjacent
// lanes, are merged with one shuffle into a < 2^50 integer and reduced mod p_j.
#include "hg_internal.cuh"

namespace {

constexpr int kWarps = 4;
constexpr int kMt = 2;                       // m-tiles (16 coefficients each) per warp
constexpr int kCoefs = kWarps * kMt * 16;    // 128 coefficients per CTA

struct OpSet4 {
    const uint32_t* words[4];
    int bits[4];
    int is_signed[4];
};

__device__ __forceinline__ void mma_u8(int (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                       uint32_t a3, uint2 b) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};\n"
        : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b.x), "r"(b.y));
}

// KS = number of 8-word k-steps held in registers (W <= 8 KS)
template <int KS>
__global__ void __launch_bounds__(kWarps * 32) modup_mma_kernel(
    OpSet4 ops, int N, const PrimeInfo* __restrict__ pinfo, const uint32_t* __restrict__ modup_tab,
    const uint2* __restrict__ Bm, int ks_stride, int P, uint32_t* __restrict__ out,
    int64_t automorph_kinv) {
    const int op = blockIdx.y;
    const uint32_t* in = op == 0 ? ops.words[0] : op == 1 ? ops.words[1] : op == 2 ? ops.words[2] : ops.words[3];
    const int bits = op == 0 ? ops.bits[0] : op == 1 ? ops.bits[1] : op == 2 ? ops.bits[2] : ops.bits[3];
    const int is_signed = op == 0 ? ops.is_signed[0] : op == 1 ? ops.is_signed[1]
                        : op == 2 ? ops.is_signed[2] : ops.is_signed[3];
    const int W = (bits + 31) >> 5;
    const uint32_t top_mask = (bits & 31) ? ((1u << (bits & 31)) - 1u) : 0xffffffffu;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int c0 = blockIdx.x * kCoefs + warp * (kMt * 16);

    // A fragments: coefficient rows n = c0 + 16m + lane/4 (+8), words 8ks + lane%4 (+4)
    uint32_t a[kMt][KS][4];
    uint32_t any[kMt][2], sgn[kMt][2], neg[kMt][2];
#pragma unroll
    for (int m = 0; m < kMt; ++m)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int i = c0 + 16 * m + (lane >> 2) + 8 * h;
            int src = i;
            bool ng = false;
            if (automorph_kinv != 0) {
                int64_t j = ((int64_t)i * automorph_kinv) & ((2ll * N) - 1);
                if (j >= N) { ng = true; j -= N; }
                src = (int)j;
            }
            uint32_t an = 0, sg = 0;
#pragma unroll
            for (int ks = 0; ks < KS; ++ks)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int w = 8 * ks + (lane & 3) + 4 * e;
                    uint32_t v = 0;
                    if (w < W) {
                        v = __ldg(in + (size_t)w * N + src);
                        if (w == W - 1) {
                            v &= top_mask;
                            sg = is_signed ? (v >> ((bits - 1) & 31)) & 1u : 0u;
                        }
                    }
                    an |= v;
                    a[m][ks][h + 2 * e] = v;   // a0: (row, k), a1: (row+8, k), a2: (row, k+16), a3
                }
            // the four lanes of a coefficient share flags
            an |= __shfl_xor_sync(0xffffffffu, an, 1);
            an |= __shfl_xor_sync(0xffffffffu, an, 2);
            sg |= __shfl_xor_sync(0xffffffffu, sg, 1);
            sg |= __shfl_xor_sync(0xffffffffu, sg, 2);
            any[m][h] = an;
            sgn[m][h] = sg;
            neg[m][h] = ng;
        }

    uint32_t* outp = out + (size_t)op * P * N;
    const int ntiles = (P + 1) >> 1;
    // B fragments of n-tile nt+1 are loaded while n-tile nt is multiplied (register double
    // buffer): the L2 latency of the constant table hides behind the mma and the epilogue
    uint2 bnext[KS];
    {
        const uint2* bp = Bm + lane;
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) bnext[ks] = __ldg(bp + ks * 32);
    }
    for (int nt = 0; nt < ntiles; ++nt) {
        uint2 bcur[KS];
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) bcur[ks] = bnext[ks];
        if (nt + 1 < ntiles) {
            const uint2* bp = Bm + (size_t)(nt + 1) * ks_stride * 32 + lane;
#pragma unroll
            for (int ks = 0; ks < KS; ++ks) bnext[ks] = __ldg(bp + ks * 32);
        }
        int acc[kMt][4];
#pragma unroll
        for (int m = 0; m < kMt; ++m) acc[m][0] = acc[m][1] = acc[m][2] = acc[m][3] = 0;
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
#pragma unroll
            for (int m = 0; m < kMt; ++m)
                mma_u8(acc[m], a[m][ks][0], a[m][ks][1], a[m][ks][2], a[m][ks][3], bcur[ks]);
        }
        // lane: prime j = 2nt + (lane&3)/2, bytes r0 = 2(lane&1), +1; rows n, n+8
        const int j = 2 * nt + ((lane & 3) >> 1);
        const bool odd = lane & 1;
        const bool jok = j < P;
        PrimeInfo pi;
        if (jok) pi = pinfo[j];
        uint32_t pw = 0;
        bool need_pw = false;
#pragma unroll
        for (int m = 0; m < kMt; ++m)
#pragma unroll
            for (int h = 0; h < 2; ++h) need_pw |= (sgn[m][h] | neg[m][h]) != 0;
        if (jok && need_pw)
            pw = reduce_u64((uint64_t)modup_tab[(size_t)j * HG_MODUP_WMAX + (bits >> 5)] << (bits & 31), pi);
#pragma unroll
        for (int m = 0; m < kMt; ++m)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const uint64_t part = (uint64_t)(uint32_t)acc[m][2 * h] +
                                      ((uint64_t)(uint32_t)acc[m][2 * h + 1] << 8);   // < 2^35
                const uint64_t other = __shfl_xor_sync(0xffffffffu, part, 1);
                if (!odd && jok) {
                    const uint64_t v = part + (other << 16);   // < 2^51
                    uint32_t r = reduce_u64(v, pi);
                    if (sgn[m][h]) r = r >= pw ? r - pw : r + pi.p - pw;
                    if (neg[m][h] && any[m][h]) {
                        if (is_signed) r = r ? pi.p - r : 0;
                        else r = pw >= r ? pw - r : pw + pi.p - r;
                    }
                    const int i = c0 + 16 * m + (lane >> 2) + 8 * h;
                    outp[(size_t)j * N + i] = r;
                }
            }
    }
}

}  // namespace

// B fragments of D(j, w, q) = 2^(32w + 8q) mod p_j: n-tile nt = primes 2nt, 2nt+1 (cols
// col = lane/4 -> j = 2nt + col/4, r = col%4), k-step ks = words 8ks..8ks+7, lane L:
// b0 bytes i = byte r of D(j, 8ks + L%4, i), b1 = same for word + 4.
int hg_modup_build_fragments(hg_ctx* ctx) {
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (ctx->d_modup_frag) return HG_OK;
    const int P = ctx->nprimes, ntiles = (P + 1) / 2, nks = HG_MODUP_WMAX / 8;
    std::vector<uint32_t> frag((size_t)ntiles * nks * 32 * 2, 0u);
    for (int nt = 0; nt < ntiles; ++nt)
        for (int ks = 0; ks < nks; ++ks)
            for (int L = 0; L < 32; ++L) {
                const int col = L / 4, j = 2 * nt + col / 4, rr = col % 4;
                if (j >= P) continue;
                const uint64_t p = ctx->primes[j];
                for (int half = 0; half < 2; ++half) {
                    const int w = 8 * ks + (L % 4) + 4 * half;
                    uint32_t word = 0;
                    for (int i = 0; i < 4; ++i) {
                        // 2^(32w + 8i) mod p
                        uint64_t v = 1, base = 2, e = 32ull * w + 8ull * i;
                        while (e) {
                            if (e & 1) v = v * base % p;
                            base = base * base % p;
                            e >>= 1;
                        }
                        word |= (uint32_t)((v >> (8 * rr)) & 0xffu) << (8 * i);
                    }
                    frag[(((size_t)nt * nks + ks) * 32 + L) * 2 + half] = word;
                }
            }
    if (cudaMalloc(&ctx->d_modup_frag, frag.size() * 4) != cudaSuccess)
        return hg_fail(HG_ENOMEM, "modup fragment table");
    cudaMemcpy(ctx->d_modup_frag, frag.data(), frag.size() * 4, cudaMemcpyHostToDevice);
    ctx->modup_frag_ks = nks;
    return HG_OK;
}

// Returns 1 if handled (operands fit the register path), 0 to fall back, <0 on error.
int hg_modup_mma_launch(hg_ctx* ctx, const uint32_t* const* words, const int* bits,
                        const int* is_signed, int nops, int P, uint32_t* out, int64_t kinv,
                        cudaStream_t st) {
    int maxw = 0;
    for (int k = 0; k < nops; ++k) maxw = std::max(maxw, (bits[k] + 31) >> 5);
    if (ctx->N < kCoefs || maxw > 64) return 0;
    int rc = hg_modup_build_fragments(ctx);
    if (rc) return -rc;
    OpSet4 o{};
    for (int k = 0; k < nops; ++k) {
        o.words[k] = words[k];
        o.bits[k] = bits[k];
        o.is_signed[k] = is_signed[k];
    }
    dim3 grid(ctx->N / kCoefs, nops);
    const uint2* Bm = reinterpret_cast<const uint2*>(ctx->d_modup_frag);
    const int kss = ctx->modup_frag_ks;
#define HG_MODUP_CASE(K)                                                                     \
    case K:                                                                                  \
        modup_mma_kernel<K><<<grid, kWarps * 32, 0, st>>>(o, ctx->N, ctx->d_pinfo, ctx->d_modup, \
                                                          Bm, kss, P, out, kinv);            \
        break;
    switch ((maxw + 7) / 8) {  // exact k-step count: no padded mma, no early-exit branches
        HG_MODUP_CASE(1)
        HG_MODUP_CASE(2)
        HG_MODUP_CASE(3)
        HG_MODUP_CASE(4)
        HG_MODUP_CASE(5)
        HG_MODUP_CASE(6)
        HG_MODUP_CASE(7)
        HG_MODUP_CASE(8)
        default: return 0;
    }
#undef HG_MODUP_CASE
    ctx->launches.fetch_add(1, std::memory_order_relaxed);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return -hg_fail(HG_ECUDA, std::string("modup_mma launch: ") + cudaGetErrorString(e));
    return 1;
}
