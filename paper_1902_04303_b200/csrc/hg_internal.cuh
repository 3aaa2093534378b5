// hg_internal.cuh -- shared definitions for the sm_100a evaluator library.
//
// Arithmetic model: ring elements of Z_{2^l}[x]/(x^N+1) are stored
// limb-major in radix 2^32.  An exact negacyclic product (the reference's Kronecker
// big-int multiply, ring.py:46-58) is computed in an RNS basis of 30-bit NTT primes
// p = 1 mod 2^18:  ModUp (radix-2^32 -> residues), forward negacyclic NTT, pointwise
// Montgomery product, inverse NTT, and an exact CRT back to radix 2^32 that emits any
// bit window [shift, shift+bits) of (c + 2^(shift-1)) -- i.e. mod 2^k reduction and the
// divide_round of ckks._keyswitch / rescale fused into the reconstruction.
#pragma once

#include <cuda.h>   // CUtensorMap (encoded through the runtime's driver entry point)
#include <cuda_runtime.h>
#include <stdint.h>
#include <algorithm>
#include <cstdlib>
#include <map>
#include <mutex>
#include <string>
#include <vector>
#include <atomic>

#include "../../include/hegwas_b200.h"

#define HG_MAX_PRIMES 320
#define HG_MODUP_WMAX 192   // operands up to 6144 bits
#define HG_PRIME_SHIFT 18   // primes are 1 mod 2^18: negacyclic NTT up to N = 2^17

struct PrimeInfo {
    uint32_t p;         // the prime (< 2^30)
    uint32_t pinv_neg;  // -p^{-1} mod 2^32 (Montgomery)
    uint32_t c32;       // 2^32 mod p
    uint32_t c30;       // 2^30 mod p
    uint32_t c30_sh;    // floor(c30 * 2^32 / p) (Shoup companion)
    uint32_t ninv;      // N^{-1} mod p (unused by the fused CRT; kept for the raw iNTT)
    uint32_t ninv_sh;
    uint32_t pad;
};

// Per-P CRT reconstruction tables (P = number of primes of the basis prefix).
struct CrtTable {
    int P = 0;
    int P4 = 0;          // P rounded up to a multiple of 4 (row pitch of M)
    int W = 0;           // column words available (multiple of 8)
    uint32_t* d_M = nullptr;      // [P4][W]: word t of (Q/p_j mod 2^(32W)); zero padded
    uint32_t* d_negQ = nullptr;   // [W]: word t of (-Q mod 2^(32W))
    uint32_t* d_cinv = nullptr;   // [P]: (Q/p_j)^{-1} * N^{-1} * 2^32 mod p_j
    uint32_t* d_cinv_sh = nullptr;
    double* d_invp = nullptr;     // [P]: 1/p_j
    int P32 = 0;                  // P rounded up to 32 (mma K dimension)
    uint2* d_Bfrag = nullptr;     // byte-split M in mma B-fragment order (hg_crt_mma.cu)
    uint8_t* d_Bconv = nullptr;   // digit-layout B as a UMMA smem image (hg_crt_umma.cu)
    int P32p = 0;                 // (P + 1) rounded up to 32: K of the pipelined kernel
    uint8_t* d_Bpipe = nullptr;   // as d_Bconv with row P = -Q mod 2^(32W)
    std::vector<uint32_t> hM;     // host copy of M (source of the lazily built fallback images)
};

// Device arena for long-lived objects (prepared switching keys, prepared operands):
// cudaMalloc'd slabs carved first-fit with coalescing frees.  Growing a slab maps ~1 ms/GB
// against ~11 ms/GB for growing the stream-ordered pool allocation by allocation, and a
// cold P17 setup prepares ~55 GB of such objects.  Frees are immediate: callers free only
// once no queued work reads the object (hg_key_destroy / hg_ctprep_destroy synchronise).
struct DeviceArena {
    struct Slab {
        char* base = nullptr;
        size_t size = 0;
        std::map<size_t, size_t> free;   // offset -> length, disjoint and non-adjacent
    };
    std::vector<Slab> slabs;
    std::map<char*, std::pair<int, size_t>> live;   // ptr -> (slab, length)
    // stream-ordered frees: (object, event recorded on the stream that last used it); the
    // memory returns to the free lists once the event has completed
    std::vector<std::pair<void*, cudaEvent_t>> deferred;
    std::vector<cudaEvent_t> spare_events;
    std::mutex mu;
    size_t reserved = 0;
    size_t in_use = 0;
};
void* hg_arena_alloc(hg_ctx* ctx, size_t bytes);   // nullptr when the device is out of memory
void hg_arena_free(hg_ctx* ctx, void* p);
// free `p` once the work queued on `stream` so far has finished (no host synchronisation)
int hg_arena_free_after(hg_ctx* ctx, void* p, cudaStream_t stream);
int hg_arena_grow(hg_ctx* ctx, size_t bytes);        // one more slab of exactly `bytes`

struct hg_ctx {
    int log_n = 0;
    int N = 0;
    int device = 0;
    int nsm = 0;          // SM count of `device`
    int nprimes = 0;
    std::vector<uint32_t> primes;       // descending
    std::vector<double> prefix_bits;    // prefix_bits[P] = sum_{j<P} log2 p_j
    PrimeInfo* d_pinfo = nullptr;       // [nprimes]
    uint32_t* d_modup = nullptr;        // [nprimes][HG_MODUP_WMAX] : 2^(32w) mod p_j
    // twiddles (w, floor(w 2^32/p)) interleaved, lazily materialised for the first
    // `tw_ready` primes: [nprimes][N] uint2, forward psi^bitrev and inverse psi^-bitrev
    uint2* d_tw_fwd = nullptr;
    uint2* d_tw_inv = nullptr;
    int tw_ready = 0;
    // log_n = 17 cluster NTT: lane-transposed round-B twiddles (hg_ntt_cluster.cu), lazily built
    uint2* d_twc_fwd = nullptr;
    uint2* d_twc_inv = nullptr;
    int ntt_cluster = 0;   // NTT kernel variant (hg_set_ntt_variant; env HG_NTT_CLUSTER=0/1/2)
    uint32_t* d_modup_frag = nullptr;   // ModUp-on-tensor-cores B fragments (hg_modup_mma.cu)
    uint8_t* d_modup_umma = nullptr;    // ModUp tcgen05 B smem images (hg_modup_umma.cu)
    int modup_frag_ks = 0;
    std::map<int, CrtTable> crt;
    std::mutex mu;
    cudaStream_t upload_stream = nullptr;   // non-blocking: table uploads never drain the compute queue
    std::atomic<long long> launches{0};
    // live kernel timing (hg_set_kernel_timing)
    struct Timer {
        cudaEvent_t a = nullptr, b = nullptr;
        int kind = 0;
        double work = 0.0;
    };
    DeviceArena arena;             // prepared keys / operands
    int timing = 0;                // bitmask of timed kernel classes (1 << kind)
    std::vector<Timer> timers;     // recorded this window
    std::vector<Timer> spare;      // event pairs available for reuse
};

enum { HG_K_CRT = 0, HG_K_MODUP = 1, HG_K_NTT = 2, HG_K_POINTWISE = 3, HG_K_ELEMENTWISE = 4 };

// Bracket a launch with events when timing is enabled (returns -1 otherwise).
int hg_timer_begin(hg_ctx* ctx, cudaStream_t st, int kind);
void hg_timer_end(hg_ctx* ctx, int idx, cudaStream_t st, int kind, double work);
struct HgTimed {
    hg_ctx* ctx;
    cudaStream_t st;
    int kind;
    double work;
    int idx;
    HgTimed(hg_ctx* c, cudaStream_t s, int k, double w) : ctx(c), st(s), kind(k), work(w) {
        idx = hg_timer_begin(c, s, k);
    }
    ~HgTimed() { hg_timer_end(ctx, idx, st, kind, work); }
};

struct hg_key {
    hg_ctx* ctx = nullptr;
    int level = 0;      // input level l
    int big_l = 0;      // L
    int P = 0;          // primes of the keyswitch basis
    uint32_t* d_kb = nullptr;   // [P][N] NTT residues of kb mod 2^(l+L) (centered), in [0,p)
    uint32_t* d_ka = nullptr;
    size_t bytes = 0;
    // residues pre-multiplied by the key switch CRT constants (Q/p_j)^-1 N^-1 2^32: the
    // pipelined CRT then skips that product (set when that kernel covers the window)
    bool prescaled = false;
};

// ---- error plumbing ------------------------------------------------------------------
void hg_set_error(const std::string& msg);
int hg_fail(int code, const std::string& msg);
#define HG_CUDA_TRY(expr)                                                              \
    do {                                                                               \
        cudaError_t _e = (expr);                                                       \
        if (_e != cudaSuccess)                                                         \
            return hg_fail(HG_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
    } while (0)
#define HG_LAUNCH_CHECK(ctx)                                                           \
    do {                                                                               \
        (ctx)->launches.fetch_add(1, std::memory_order_relaxed);                       \
        cudaError_t _e = cudaGetLastError();                                           \
        if (_e != cudaSuccess)                                                         \
            return hg_fail(HG_ECUDA, std::string("kernel launch: ") + cudaGetErrorString(_e)); \
    } while (0)

static inline int words_for_bits(int bits) { return (bits + 31) >> 5; }

// Function attributes (dynamic shared memory limits) are per device: a process driving two
// GPUs must set them once on each.  True the first time `dev` is seen for this flag set.
static inline bool hg_first_on_device(std::atomic<uint64_t>& seen, int dev) {
    const uint64_t bit = 1ull << (dev & 63);
    return !(seen.fetch_or(bit) & bit);
}
// Clamp a group-size override from the environment (unset, 0 or negative -> default).
static inline int hg_env_group(const char* name, int dflt, int lo, int hi) {
    const char* s = getenv(name);
    int v = s ? atoi(s) : dflt;
    if (v <= 0) v = dflt;
    return v < lo ? lo : (v > hi ? hi : v);
}

// ---- host-side helpers (hg_context.cu) ----------------------------------------------
// 2-D uint32 tensor map (row pitch = inner * 4 bytes) for cp.async.bulk.tensor boxes
int hg_tmap_2d_u32(CUtensorMap* tm, const void* base, uint64_t inner, uint64_t outer,
                   uint32_t box_inner, uint32_t box_outer);
int hg_ensure_twiddles(hg_ctx* ctx, int P);
// one-round-trip length-2^17 transforms on 8-CTA clusters (hg_ntt_cluster.cu)
bool hg_ntt_cluster_ok(const hg_ctx* ctx, int P);
int hg_ntt_cluster(hg_ctx* ctx, uint32_t* data, int rows, int P, int prime_offset, bool forward,
                   cudaStream_t st);
int hg_intt_fused_cluster(hg_ctx* ctx, int pre, uint32_t* out, const uint32_t* i0, const uint32_t* i1,
                          const uint32_t* i2, const uint32_t* i3, int P, cudaStream_t st, int batch);
int hg_get_crt(hg_ctx* ctx, int P, const CrtTable** out);
// host -> device copy of a lazily built table on the context's private non-blocking stream: a
// plain cudaMemcpy would synchronise with the legacy default stream and so wait for every
// queued kernel (a first-use table build mid-pipeline would drain the GPU)
int hg_upload(hg_ctx* ctx, void* dst, const void* src, size_t bytes);
int hg_crt_ensure_fallback(hg_ctx* ctx, const CrtTable* tab);   // d_Bfrag / d_Bconv
int hg_primes_for_bits(const hg_ctx* ctx, double bits);   // -1 if too wide
int hg_crt_build_fragments(const CrtTable& t, int P, int P32, std::vector<uint32_t>& out,
                           const std::vector<uint32_t>& M);
int hg_crt_mma_launch(hg_ctx* ctx, const CrtTable* tab, const uint32_t* res, int nouts, int P,
                      int shift, int out_bits, int tb0, uint32_t* const* outs, cudaStream_t st);
int hg_crt_build_conv(const CrtTable& t, int P, int P32, std::vector<uint8_t>& out,
                      const std::vector<uint32_t>& M);
int hg_crt_build_pack4(const CrtTable& t, int P, int P32, std::vector<uint8_t>& out,
                       const std::vector<uint32_t>& M);
int hg_crt_umma_launch(hg_ctx* ctx, const CrtTable* tab, const uint32_t* res, int nouts, int P,
                       int shift, int out_bits, int tb0, uint32_t* const* outs, cudaStream_t st);
size_t hg_crt_umma_smem(int P32);
bool hg_crt_umma_pipe_ok(const CrtTable* tab, int N, int shift, int out_bits, int tb0);
// Optional fused finish of the pipelined CRT (see Emitter in hg_crt_umma.cu): per output k,
// out_k = bits [post, out_bits) of (window_k + add_k' + 2^(post-1)) mod 2^out_bits, where
// add_k' is add_k (out_bits wide, may be null) read through x -> x^k when kinv != 0.
struct CrtFinish {
    const uint32_t* add[8] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    int64_t kinv = 0;
    int post = 0;
};
int hg_crt_umma_pipe_launch(hg_ctx* ctx, const CrtTable* tab, const uint32_t* res, int nouts, int P,
                            int shift, int out_bits, int tb0, uint32_t* const* outs,
                            cudaStream_t st, const CrtFinish* finish = nullptr, bool prescaled = false);
int hg_modup_umma_launch(hg_ctx* ctx, const uint32_t* const* words, const int* bits,
                         const int* is_signed, int nops, int P, uint32_t* out, int64_t kinv,
                         cudaStream_t st);
int hg_modup_mma_launch(hg_ctx* ctx, const uint32_t* const* words, const int* bits,
                        const int* is_signed, int nops, int P, uint32_t* out, int64_t kinv,
                        cudaStream_t st);

// ---- device arithmetic --------------------------------------------------------------
// Shoup product a*w mod p for any a < 2^32, result in [0, 2p).
__device__ __forceinline__ uint32_t mul_shoup_lazy(uint32_t a, uint32_t w, uint32_t wsh,
                                                   uint32_t p) {
    uint32_t q = __umulhi(a, wsh);
    return a * w - q * p;
}
__device__ __forceinline__ uint32_t reduce_2p(uint32_t a, uint32_t p) {
    return a >= p ? a - p : a;
}
__device__ __forceinline__ uint32_t reduce_4p(uint32_t a, uint32_t p) {
    uint32_t p2 = p << 1;
    a = a >= p2 ? a - p2 : a;
    return a >= p ? a - p : a;
}
// Montgomery product a*b*2^-32 mod p; requires a*b < p*2^32; result in [0, 2p).
__device__ __forceinline__ uint32_t mont_mul(uint32_t a, uint32_t b, uint32_t p,
                                             uint32_t pinv_neg) {
    uint64_t t = (uint64_t)a * b;
    uint32_t m = (uint32_t)t * pinv_neg;
    uint64_t u = t + (uint64_t)m * p;
    return (uint32_t)(u >> 32);
}
// Reduce a 64-bit accumulator (any value) to [0, p) using 2^32 and 2^30 folds.
__device__ __forceinline__ uint32_t reduce_u64(uint64_t acc, const PrimeInfo& pi) {
    // fold 1: < 2^62 + 2^32 ; fold 2: < 2^61
    acc = (uint64_t)(uint32_t)(acc >> 32) * pi.c32 + (uint32_t)acc;
    acc = (uint64_t)(uint32_t)(acc >> 32) * pi.c32 + (uint32_t)acc;
    uint32_t a = (uint32_t)(acc >> 30);
    uint32_t b = (uint32_t)acc & 0x3fffffffu;
    uint32_t r = mul_shoup_lazy(a, pi.c30, pi.c30_sh, pi.p) + b;  // < 2p + 2^30 < 4p
    return reduce_4p(r, pi.p);
}
