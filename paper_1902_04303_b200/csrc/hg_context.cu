// hg_context.cu -- context creation: NTT prime basis, twiddles, base-conversion and CRT
// tables.  Host-side set-up only; kernels live in hg_ntt.cu / hg_rns.cu / hg_elementwise.cu.
#include "hg_internal.cuh"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>

// HG_DEBUG_BUILD=1: report host-side table builds (they run on first use of a prime count)
static void build_note(const char* what, int P, std::chrono::steady_clock::time_point t0) {
    static const bool on = getenv("HG_DEBUG_BUILD") != nullptr;
    if (!on) return;
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    fprintf(stderr, "[hg build] %s P=%d %.1f ms\n", what, P, ms);
}

static thread_local std::string g_last_error;

void hg_set_error(const std::string& msg) { g_last_error = msg; }
int hg_fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

extern "C" const char* hg_last_error(void) { return g_last_error.c_str(); }
extern "C" int hg_version(void) { return 1; }

// ---- 32-bit number theory (host) -------------------------------------------------------
static uint64_t mulmod64(uint64_t a, uint64_t b, uint64_t m) { return (a * b) % m; }
static uint64_t powmod(uint64_t b, uint64_t e, uint64_t m) {
    uint64_t r = 1 % m;
    b %= m;
    while (e) {
        if (e & 1) r = mulmod64(r, b, m);
        b = mulmod64(b, b, m);
        e >>= 1;
    }
    return r;
}
static bool is_prime_u32(uint32_t n) {
    if (n < 2) return false;
    for (uint32_t sp : {2u, 3u, 5u, 7u, 11u, 13u}) {
        if (n % sp == 0) return n == sp;
    }
    uint32_t d = n - 1;
    int s = 0;
    while ((d & 1) == 0) { d >>= 1; ++s; }
    for (uint32_t a : {2u, 7u, 61u}) {
        uint64_t x = powmod(a, d, n);
        if (x == 1 || x == n - 1) continue;
        bool comp = true;
        for (int r = 1; r < s; ++r) {
            x = mulmod64(x, x, n);
            if (x == n - 1) { comp = false; break; }
        }
        if (comp) return false;
    }
    return true;
}
static uint32_t shoup_of(uint32_t w, uint32_t p) {
    return (uint32_t)(((uint64_t)w << 32) / p);
}

// ---- context ----------------------------------------------------------------------------
extern "C" int hg_ctx_create(int log_n, int device, hg_ctx** out) {
    if (!out) return hg_fail(HG_EINVAL, "null output pointer");
    if (log_n < 2 || log_n > HG_PRIME_SHIFT - 1)
        return hg_fail(HG_EINVAL, "log_n must be in [2, 17] for the 30-bit NTT prime basis");
    HG_CUDA_TRY(cudaSetDevice(device));
    hg_ctx* ctx = new hg_ctx();
    ctx->log_n = log_n;
    ctx->N = 1 << log_n;
    ctx->device = device;
    HG_CUDA_TRY(cudaDeviceGetAttribute(&ctx->nsm, cudaDevAttrMultiProcessorCount, device));
    // primes p = k * 2^18 + 1 < 2^30, descending
    for (uint64_t k = ((1ull << 30) - 2) >> HG_PRIME_SHIFT; k >= 1 && ctx->primes.size() < HG_MAX_PRIMES; --k) {
        uint64_t p = (k << HG_PRIME_SHIFT) + 1;
        if (p >= (1ull << 30)) continue;
        if (p < (1ull << 26)) break;
        if (is_prime_u32((uint32_t)p)) ctx->primes.push_back((uint32_t)p);
    }
    ctx->nprimes = (int)ctx->primes.size();
    ctx->prefix_bits.assign(ctx->nprimes + 1, 0.0);
    for (int j = 0; j < ctx->nprimes; ++j)
        ctx->prefix_bits[j + 1] = ctx->prefix_bits[j] + std::log2((double)ctx->primes[j]);

    std::vector<PrimeInfo> pinfo(ctx->nprimes);
    std::vector<uint32_t> modup((size_t)ctx->nprimes * HG_MODUP_WMAX);
    for (int j = 0; j < ctx->nprimes; ++j) {
        uint32_t p = ctx->primes[j];
        PrimeInfo& pi = pinfo[j];
        pi.p = p;
        // -p^{-1} mod 2^32 by Newton iteration
        uint32_t inv = p;  // correct to 3 bits for odd p
        for (int it = 0; it < 5; ++it) inv *= 2u - p * inv;
        pi.pinv_neg = (uint32_t)(0u - inv);
        pi.c32 = (uint32_t)((1ull << 32) % p);
        pi.c30 = (uint32_t)((1ull << 30) % p);
        pi.c30_sh = shoup_of(pi.c30, p);
        pi.ninv = (uint32_t)powmod(ctx->N, p - 2, p);
        pi.ninv_sh = shoup_of(pi.ninv, p);
        pi.pad = 0;
        uint64_t v = 1;
        for (int w = 0; w < HG_MODUP_WMAX; ++w) {
            modup[(size_t)j * HG_MODUP_WMAX + w] = (uint32_t)v;
            v = mulmod64(v, pi.c32, p);
        }
    }
    size_t tw_bytes = (size_t)ctx->nprimes * ctx->N * sizeof(uint2);
    if (cudaMalloc(&ctx->d_pinfo, sizeof(PrimeInfo) * ctx->nprimes) != cudaSuccess ||
        cudaMalloc(&ctx->d_modup, modup.size() * sizeof(uint32_t)) != cudaSuccess ||
        cudaMalloc(&ctx->d_tw_fwd, tw_bytes) != cudaSuccess ||
        cudaMalloc(&ctx->d_tw_inv, tw_bytes) != cudaSuccess) {
        hg_ctx_destroy(ctx);
        return hg_fail(HG_ENOMEM, "context allocation failed");
    }
    cudaMemcpy(ctx->d_pinfo, pinfo.data(), sizeof(PrimeInfo) * ctx->nprimes, cudaMemcpyHostToDevice);
    cudaMemcpy(ctx->d_modup, modup.data(), modup.size() * sizeof(uint32_t), cudaMemcpyHostToDevice);
    // keep freed stream-ordered allocations cached in the pool (residue scratch is reused
    // every op; returning it to the driver would serialise on cudaFree)
    cudaStreamCreateWithFlags(&ctx->upload_stream, cudaStreamNonBlocking);   // created once: no lock in hg_upload
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        hg_ctx_destroy(ctx);
        return hg_fail(HG_ECUDA, std::string("context upload: ") + cudaGetErrorString(e));
    }
    if (const char* v = getenv("HG_NTT_CLUSTER")) ctx->ntt_cluster = (v[0] == '1' || v[0] == '2') ? v[0] - '0' : 0;
    *out = ctx;
    return HG_OK;
}

// ---- device arena (hg_internal.cuh) ---------------------------------------------------
static constexpr size_t kArenaAlign = 2u << 20;      // 2 MB: slab and object granularity
static constexpr size_t kArenaSlab = 8ull << 30;     // default growth step

int hg_arena_grow(hg_ctx* ctx, size_t bytes) {
    bytes = (bytes + kArenaAlign - 1) & ~(kArenaAlign - 1);
    char* base = nullptr;
    if (cudaMalloc(&base, bytes) != cudaSuccess) {
        cudaGetLastError();
        return hg_fail(HG_ENOMEM, "device arena: cudaMalloc of " + std::to_string(bytes >> 20) + " MB failed");
    }
    std::lock_guard<std::mutex> g(ctx->arena.mu);
    DeviceArena::Slab s;
    s.base = base;
    s.size = bytes;
    s.free[0] = bytes;
    ctx->arena.slabs.push_back(std::move(s));
    ctx->arena.reserved += bytes;
    return HG_OK;
}

static void* arena_take(DeviceArena& a, size_t bytes) {
    for (size_t i = 0; i < a.slabs.size(); ++i) {
        auto& fl = a.slabs[i].free;
        for (auto it = fl.begin(); it != fl.end(); ++it) {
            if (it->second < bytes) continue;
            const size_t off = it->first, len = it->second;
            fl.erase(it);
            if (len > bytes) fl[off + bytes] = len - bytes;
            char* p = a.slabs[i].base + off;
            a.live[p] = {(int)i, bytes};
            a.in_use += bytes;
            return p;
        }
    }
    return nullptr;
}

static void arena_free_locked(DeviceArena& a, void* ptr);

// return deferred frees whose events have completed (block: wait for all of them)
static void arena_reclaim_locked(DeviceArena& a, bool block) {
    size_t k = 0;
    for (auto& d : a.deferred) {
        const cudaError_t q = block ? cudaEventSynchronize(d.second) : cudaEventQuery(d.second);
        if (q == cudaSuccess) {
            arena_free_locked(a, d.first);
            a.spare_events.push_back(d.second);
        } else {
            if (q != cudaErrorNotReady) cudaGetLastError();
            a.deferred[k++] = d;
        }
    }
    a.deferred.resize(k);
}

int hg_arena_free_after(hg_ctx* ctx, void* ptr, cudaStream_t stream) {
    if (!ptr) return HG_OK;
    std::lock_guard<std::mutex> g(ctx->arena.mu);
    DeviceArena& a = ctx->arena;
    cudaEvent_t ev;
    if (!a.spare_events.empty()) {
        ev = a.spare_events.back();
        a.spare_events.pop_back();
    } else if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) {
        cudaGetLastError();
        cudaStreamSynchronize(stream);   // no event: order the free the slow way
        arena_free_locked(a, ptr);
        return HG_OK;
    }
    cudaEventRecord(ev, stream);
    a.deferred.emplace_back(ptr, ev);
    arena_reclaim_locked(a, false);
    return HG_OK;
}

void* hg_arena_alloc(hg_ctx* ctx, size_t bytes) {
    if (!bytes) bytes = 1;
    bytes = (bytes + kArenaAlign - 1) & ~(kArenaAlign - 1);
    {
        std::lock_guard<std::mutex> g(ctx->arena.mu);
        arena_reclaim_locked(ctx->arena, false);
        if (void* p = arena_take(ctx->arena, bytes)) return p;
        if (!ctx->arena.deferred.empty()) {   // before growing: wait for pending frees
            arena_reclaim_locked(ctx->arena, true);
            if (void* p = arena_take(ctx->arena, bytes)) return p;
        }
    }
    // grow by a default slab (or exactly the request when the device is nearly full)
    if (hg_arena_grow(ctx, bytes > kArenaSlab ? bytes : kArenaSlab) != HG_OK &&
        hg_arena_grow(ctx, bytes) != HG_OK)
        return nullptr;
    std::lock_guard<std::mutex> g(ctx->arena.mu);
    return arena_take(ctx->arena, bytes);
}

void hg_arena_free(hg_ctx* ctx, void* ptr) {
    if (!ptr) return;
    std::lock_guard<std::mutex> g(ctx->arena.mu);
    arena_free_locked(ctx->arena, ptr);
}

static void arena_free_locked(DeviceArena& a, void* ptr) {
    auto it = a.live.find((char*)ptr);
    if (it == a.live.end()) return;
    const int si = it->second.first;
    size_t off = (size_t)((char*)ptr - a.slabs[si].base), len = it->second.second;
    a.in_use -= len;
    a.live.erase(it);
    auto& fl = a.slabs[si].free;
    auto nx = fl.lower_bound(off);
    if (nx != fl.end() && off + len == nx->first) {   // merge with the following hole
        len += nx->second;
        nx = fl.erase(nx);
    }
    if (nx != fl.begin()) {                           // merge with the preceding hole
        auto pv = std::prev(nx);
        if (pv->first + pv->second == off) {
            pv->second += len;
            return;
        }
    }
    fl[off] = len;
}

extern "C" int hg_pool_reserve(hg_ctx* ctx, size_t bytes, void* stream) {
    (void)stream;
    if (!ctx) return hg_fail(HG_EINVAL, "hg_pool_reserve: null context");
    if (!bytes) return HG_OK;
    return hg_arena_grow(ctx, bytes);
}

extern "C" size_t hg_pool_trim(hg_ctx* ctx) {
    if (!ctx) return 0;
    std::lock_guard<std::mutex> g(ctx->arena.mu);
    DeviceArena& a = ctx->arena;
    arena_reclaim_locked(a, true);
    size_t released = 0;
    std::vector<DeviceArena::Slab> keep;
    std::vector<int> remap(a.slabs.size(), -1);
    for (size_t i = 0; i < a.slabs.size(); ++i) {
        auto& sl = a.slabs[i];
        const bool empty = sl.free.size() == 1 && sl.free.begin()->first == 0 && sl.free.begin()->second == sl.size;
        if (empty) {
            cudaFree(sl.base);
            released += sl.size;
        } else {
            remap[i] = (int)keep.size();
            keep.push_back(std::move(sl));
        }
    }
    for (auto& kv : a.live) kv.second.first = remap[kv.second.first];
    a.slabs = std::move(keep);
    a.reserved -= released;
    return released;
}

extern "C" size_t hg_pool_bytes(const hg_ctx* ctx, int in_use) {
    if (!ctx) return 0;
    return in_use ? ctx->arena.in_use : ctx->arena.reserved;
}

extern "C" int hg_ctx_destroy(hg_ctx* ctx) {
    if (!ctx) return HG_OK;
    if (ctx->upload_stream) cudaStreamDestroy(ctx->upload_stream);
    cudaFree(ctx->d_pinfo);
    cudaFree(ctx->d_modup);
    cudaFree(ctx->d_tw_fwd);
    cudaFree(ctx->d_tw_inv);
    cudaFree(ctx->d_twc_fwd);
    cudaFree(ctx->d_twc_inv);
    cudaFree(ctx->d_modup_frag);
    cudaFree(ctx->d_modup_umma);
    for (auto& sl : ctx->arena.slabs) cudaFree(sl.base);
    for (auto& kv : ctx->crt) {
        cudaFree(kv.second.d_M);
        cudaFree(kv.second.d_negQ);
        cudaFree(kv.second.d_cinv);
        cudaFree(kv.second.d_cinv_sh);
        cudaFree(kv.second.d_invp);
        cudaFree(kv.second.d_Bfrag);
        cudaFree(kv.second.d_Bconv);
        cudaFree(kv.second.d_Bpipe);
    }
    delete ctx;
    return HG_OK;
}

extern "C" int hg_ctx_max_product_bits(const hg_ctx* ctx) {
    return ctx ? (int)std::floor(ctx->prefix_bits[ctx->nprimes]) : 0;
}
extern "C" int hg_ctx_num_primes(const hg_ctx* ctx) { return ctx ? ctx->nprimes : 0; }
extern "C" int hg_ctx_primes(const hg_ctx* ctx, uint32_t* out) {
    if (!ctx || !out) return hg_fail(HG_EINVAL, "null argument");
    std::memcpy(out, ctx->primes.data(), ctx->primes.size() * sizeof(uint32_t));
    return HG_OK;
}
extern "C" long long hg_launch_count(const hg_ctx* ctx) { return ctx ? ctx->launches.load() : 0; }

// ---- live kernel timing ----------------------------------------------------------------------
int hg_timer_begin(hg_ctx* ctx, cudaStream_t st, int kind) {
    if (!(ctx->timing & (1 << kind))) return -1;
    std::lock_guard<std::mutex> lk(ctx->mu);
    hg_ctx::Timer t;
    if (!ctx->spare.empty()) {
        t = ctx->spare.back();
        ctx->spare.pop_back();
    } else {
        cudaEventCreate(&t.a);
        cudaEventCreate(&t.b);
    }
    cudaEventRecord(t.a, st);
    ctx->timers.push_back(t);
    return (int)ctx->timers.size() - 1;
}

void hg_timer_end(hg_ctx* ctx, int idx, cudaStream_t st, int kind, double work) {
    if (idx < 0) return;
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (idx >= (int)ctx->timers.size()) return;
    hg_ctx::Timer& t = ctx->timers[idx];
    cudaEventRecord(t.b, st);
    t.kind = kind;
    t.work = work;
}

extern "C" int hg_set_kernel_timing(hg_ctx* ctx, int enabled) {
    if (!ctx) return hg_fail(HG_EINVAL, "null context");
    HG_CUDA_TRY(cudaDeviceSynchronize());
    std::lock_guard<std::mutex> lk(ctx->mu);
    for (auto& t : ctx->timers) ctx->spare.push_back(t);
    ctx->timers.clear();
    ctx->timing = enabled == 1 ? 0x1f : (enabled < 0 ? 0 : enabled >> 1);
    return HG_OK;
}

extern "C" int hg_kernel_stats(hg_ctx* ctx, int kind, double* ms, long long* launches,
                               double* work) {
    if (!ctx || !ms || !launches || !work) return hg_fail(HG_EINVAL, "null argument");
    std::lock_guard<std::mutex> lk(ctx->mu);
    double tot = 0.0, w = 0.0;
    long long n = 0;
    for (auto& t : ctx->timers) {
        if (t.kind != kind) continue;
        HG_CUDA_TRY(cudaEventSynchronize(t.b));
        float e = 0.f;
        HG_CUDA_TRY(cudaEventElapsedTime(&e, t.a, t.b));
        tot += e;
        w += t.work;
        ++n;
    }
    *ms = tot;
    *launches = n;
    *work = w;
    return HG_OK;
}

extern "C" int hg_sync(hg_ctx* ctx, void* stream) {
    (void)ctx;
    HG_CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream));
    return HG_OK;
}

int hg_primes_for_bits(const hg_ctx* ctx, double bits) {
    for (int P = 1; P <= ctx->nprimes; ++P)
        if (ctx->prefix_bits[P] >= bits) return P;
    return -1;
}

// ---- twiddles ----------------------------------------------------------------------------
// psi_rev[k] = psi^bitrev(k), ipsi_rev[k] = psi^-bitrev(k) for a primitive 2N-th root psi
// (merged negacyclic Cooley-Tukey forward / Gentleman-Sande inverse).
// psi^bitrev(k) and psi^-bitrev(k) with their Shoup companions, one thread per (prime, k)
__global__ void twiddle_kernel(uint2* __restrict__ fwd, uint2* __restrict__ inv,
                               const uint32_t* __restrict__ roots, const uint32_t* __restrict__ primes,
                               int logn) {
    const int N = 1 << logn;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= N) return;
    const int j = blockIdx.y;
    const uint64_t p = primes[j], root = roots[j];
    auto pw = [&](uint32_t e) {
        uint64_t r = 1, b = root;
        while (e) {
            if (e & 1) r = r * b % p;
            b = b * b % p;
            e >>= 1;
        }
        return (uint32_t)r;
    };
    const uint32_t e = __brev((uint32_t)k) >> (32 - logn);
    const uint32_t w = pw(e);
    const uint32_t iw = e == 0 ? 1u : (uint32_t)(p - pw(N - e));   // psi^-e = -psi^(N-e)
    const size_t o = (size_t)j * N + k;
    fwd[o] = make_uint2(w, (uint32_t)(((uint64_t)w << 32) / p));
    inv[o] = make_uint2(iw, (uint32_t)(((uint64_t)iw << 32) / p));
}

int hg_ensure_twiddles(hg_ctx* ctx, int P) {
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (P <= ctx->tw_ready) return HG_OK;
    const auto t_start = std::chrono::steady_clock::now();
    const int N = ctx->N;
    // materialise every prime at once (the tables are allocated for all of them)
    const int j0 = ctx->tw_ready, j1 = ctx->nprimes;
    std::vector<uint32_t> roots(j1 - j0);
    for (int j = j0; j < j1; ++j) {
        uint32_t p = ctx->primes[j];
        uint64_t root = 0;
        for (uint64_t g = 2; g < p; ++g) {
            uint64_t cand = powmod(g, (p - 1) / (2ull * N), p);
            if (powmod(cand, N, p) == p - 1) { root = cand; break; }
        }
        if (!root) return hg_fail(HG_EINVAL, "no primitive 2N-th root");
        roots[j - j0] = (uint32_t)root;
    }
    uint32_t *d_roots = nullptr, *d_primes = nullptr;
    HG_CUDA_TRY(cudaMalloc(&d_roots, roots.size() * 4));
    HG_CUDA_TRY(cudaMalloc(&d_primes, roots.size() * 4));
    HG_CUDA_TRY(cudaMemcpy(d_roots, roots.data(), roots.size() * 4, cudaMemcpyHostToDevice));
    HG_CUDA_TRY(cudaMemcpy(d_primes, ctx->primes.data() + j0, roots.size() * 4, cudaMemcpyHostToDevice));
    const size_t off = (size_t)j0 * N;
    twiddle_kernel<<<dim3((N + 255) / 256, j1 - j0), 256>>>(ctx->d_tw_fwd + off, ctx->d_tw_inv + off, d_roots,
                                                         d_primes, ctx->log_n);
    HG_CUDA_TRY(cudaGetLastError());
    HG_CUDA_TRY(cudaDeviceSynchronize());
    cudaFree(d_roots);
    cudaFree(d_primes);
    ctx->tw_ready = j1;
    build_note("twiddles", j1, t_start);
    return HG_OK;
}

// ---- TMA tensor maps ------------------------------------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int hg_tmap_2d_u32(CUtensorMap* tm, const void* base, uint64_t inner, uint64_t outer,
                   uint32_t box_inner, uint32_t box_outer) {
    static EncodeTiledFn encode = nullptr;
    if (!encode) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !fn)
            return hg_fail(HG_ECUDA, "cuTensorMapEncodeTiled entry point unavailable");
        encode = (EncodeTiledFn)fn;
    }
    const cuuint64_t dims[2] = {inner, outer};
    const cuuint64_t strides[1] = {inner * 4};
    const cuuint32_t box[2] = {box_inner, box_outer};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = encode(tm, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, const_cast<void*>(base), dims, strides,
                        box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return hg_fail(HG_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    return HG_OK;
}

int hg_upload(hg_ctx* ctx, void* dst, const void* src, size_t bytes) {
    HG_CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->upload_stream));
    HG_CUDA_TRY(cudaStreamSynchronize(ctx->upload_stream));   // the copy only, not the compute queue
    return HG_OK;
}

// ---- CRT tables ---------------------------------------------------------------------------
// multiply a little-endian word array (truncated to W words) by a 32-bit value in place
static void mul_small_trunc(std::vector<uint32_t>& a, uint32_t m) {
    uint64_t carry = 0;
    for (size_t i = 0; i < a.size(); ++i) {
        uint64_t t = (uint64_t)a[i] * m + carry;
        a[i] = (uint32_t)t;
        carry = t >> 32;
    }
}

int hg_get_crt(hg_ctx* ctx, int P, const CrtTable** out) {
    {
        std::lock_guard<std::mutex> lk(ctx->mu);
        auto it = ctx->crt.find(P);
        if (it != ctx->crt.end()) { *out = &it->second; return HG_OK; }
    }
    const auto t_start = std::chrono::steady_clock::now();
    CrtTable t;
    t.P = P;
    t.P4 = (P + 3) & ~3;
    t.W = (int)std::ceil(ctx->prefix_bits[P] / 32.0) + 2;
    if (t.W < HG_MODUP_WMAX) t.W = HG_MODUP_WMAX;  // any emitted window up to 6144 bits
    t.W = (t.W + 7) & ~7;                          // 8-column blocks of the CRT kernel
    const int W = t.W;
    // M is prime-major: row j holds the words of Q/p_j mod 2^(32W) (rows >= P are zero)
    std::vector<uint32_t> M((size_t)W * t.P4, 0u), negQ(W, 0u), cinv(P), cinv_sh(P);
    std::vector<double> invp(P);
    // Q mod 2^(32W) and Q/p_j mod 2^(32W)
    std::vector<uint32_t> Q(W, 0u);
    Q[0] = 1;
    for (int i = 0; i < P; ++i) mul_small_trunc(Q, ctx->primes[i]);
    // negQ = 2^(32W) - Q
    {
        uint64_t borrow = 0;
        for (int w = 0; w < W; ++w) {
            uint64_t v = (uint64_t)0 - Q[w] - borrow;
            negQ[w] = (uint32_t)v;
            borrow = (Q[w] != 0 || borrow) ? 1 : 0;
        }
    }
    // W >= bits(Q)/32 + 2, so Q is exact in W words and Q/p_j is an exact multiword division
    for (int j = 0; j < P; ++j) {
        uint64_t qmodp = 1;
        uint32_t pj = ctx->primes[j];
        for (int i = 0; i < P; ++i)
            if (i != j) qmodp = mulmod64(qmodp, ctx->primes[i] % pj, pj);
        uint64_t rem = 0;
        for (int w = W - 1; w >= 0; --w) {
            const uint64_t cur = (rem << 32) | Q[w];
            M[(size_t)j * W + w] = (uint32_t)(cur / pj);
            rem = cur % pj;
        }
        uint64_t inv = powmod(qmodp, pj - 2, pj);
        uint64_t ninv = powmod(ctx->N % pj, pj - 2, pj);
        uint64_t r32 = (1ull << 32) % pj;
        uint64_t c = mulmod64(mulmod64(inv, ninv, pj), r32, pj);
        cinv[j] = (uint32_t)c;
        cinv_sh[j] = shoup_of((uint32_t)c, pj);
        invp[j] = 1.0 / (double)pj;
    }
    HG_CUDA_TRY(cudaMalloc(&t.d_M, M.size() * 4));
    HG_CUDA_TRY(cudaMalloc(&t.d_negQ, negQ.size() * 4));
    HG_CUDA_TRY(cudaMalloc(&t.d_cinv, P * 4));
    HG_CUDA_TRY(cudaMalloc(&t.d_cinv_sh, P * 4));
    HG_CUDA_TRY(cudaMalloc(&t.d_invp, P * 8));
    if (int rc = hg_upload(ctx, t.d_M, M.data(), M.size() * 4)) return rc;
    if (int rc = hg_upload(ctx, t.d_negQ, negQ.data(), negQ.size() * 4)) return rc;
    if (int rc = hg_upload(ctx, t.d_cinv, cinv.data(), P * 4)) return rc;
    if (int rc = hg_upload(ctx, t.d_cinv_sh, cinv_sh.data(), P * 4)) return rc;
    if (int rc = hg_upload(ctx, t.d_invp, invp.data(), P * 8)) return rc;
    t.P32 = (P + 31) & ~31;
    {
        std::vector<uint8_t> conv;
        // (the fallback kernels' B images are built on their first use: hg_crt_ensure_fallback)
        // pipelined kernel: one more K row (slot P) carries -Q, so v * (-Q) comes out of the GEMM
        t.P32p = (P + 1 + 31) & ~31;
        std::vector<uint32_t> Mp((size_t)W * t.P32p, 0u);
        std::copy(M.begin(), M.begin() + (size_t)W * P, Mp.begin());
        std::copy(negQ.begin(), negQ.end(), Mp.begin() + (size_t)W * P);
        hg_crt_build_pack4(t, P + 1, t.P32p, conv, Mp);
        HG_CUDA_TRY(cudaMalloc(&t.d_Bpipe, conv.size()));
        if (int rc = hg_upload(ctx, t.d_Bpipe, conv.data(), conv.size())) return rc;
    }
    t.hM = std::move(M);
    std::lock_guard<std::mutex> lk(ctx->mu);
    auto ins = ctx->crt.emplace(P, t);
    if (!ins.second) {  // another thread won the race
        cudaFree(t.d_M); cudaFree(t.d_negQ); cudaFree(t.d_cinv); cudaFree(t.d_cinv_sh); cudaFree(t.d_invp);
        cudaFree(t.d_Bfrag);
        cudaFree(t.d_Bconv);
        cudaFree(t.d_Bpipe);
    }
    *out = &ins.first->second;
    build_note("crt", P, t_start);
    return HG_OK;
}

int hg_crt_ensure_fallback(hg_ctx* ctx, const CrtTable* ctab) {
    std::lock_guard<std::mutex> lk(ctx->mu);
    CrtTable* t = const_cast<CrtTable*>(ctab);
    if (t->d_Bfrag && t->d_Bconv) return HG_OK;
    std::vector<uint32_t> frag;
    hg_crt_build_fragments(*t, t->P, t->P32, frag, t->hM);
    HG_CUDA_TRY(cudaMalloc(&t->d_Bfrag, frag.size() * 4));
    if (int rc = hg_upload(ctx, t->d_Bfrag, frag.data(), frag.size() * 4)) return rc;
    std::vector<uint8_t> conv;
    hg_crt_build_conv(*t, t->P, t->P32, conv, t->hM);
    HG_CUDA_TRY(cudaMalloc(&t->d_Bconv, conv.size()));
    if (int rc = hg_upload(ctx, t->d_Bconv, conv.data(), conv.size())) return rc;
    return HG_OK;
}
