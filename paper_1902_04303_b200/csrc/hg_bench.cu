// hg_bench.cu -- integer-pipe roofline probe: the exact lazy Harvey butterfly (Shoup
// modmul + add/sub) the NTT kernels execute -- hgntt::fwd_bfly itself, so the probe carries the
// kernels' instruction mix (IMAD.HI + 2 IMAD on the fma pipe, VIADDMNMX + 2 IADD3 on the alu
// pipe) --, register resident, 8 independent chains per thread, enough CTAs to fill all SMs.  The measured butterflies/s is the integer-pipe
// "peak" that NTT kernel throughput is reported against (MEASURED_PEAKS.json has no
// integer figure).
#include "hg_ntt_common.cuh"

namespace {

__global__ void __launch_bounds__(256) modmul_probe_kernel(int iters, uint32_t p, uint32_t w,
                                                           uint32_t wsh, uint32_t* sink) {
    uint32_t x[8], y[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        x[k] = (threadIdx.x * 2654435761u + k * 40503u) % p;
        y[k] = (blockIdx.x * 97u + k * 7919u + threadIdx.x) % p;
    }
    const uint2 tw = make_uint2(w, wsh);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < 8; ++k) hgntt::fwd_bfly(x[k], y[k], tw, p);
    }
    uint32_t acc = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) acc ^= x[k] ^ y[k];
    if (acc == 0x12345678u) sink[0] = acc;  // keep the chains live
}

}  // namespace

extern "C" int hg_bench_modmul(hg_ctx* ctx, int iters, uint32_t* sink, double* ops_out,
                               void* stream) {
    if (!ctx || !sink || iters < 1) return hg_fail(HG_EINVAL, "hg_bench_modmul: bad arguments");
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
    const int blocks = sms * 8, threads = 256;
    uint32_t p = ctx->primes[0];
    uint32_t w = 123456789u % p;
    uint32_t wsh = (uint32_t)(((uint64_t)w << 32) / p);
    modmul_probe_kernel<<<blocks, threads, 0, (cudaStream_t)stream>>>(iters, p, w, wsh, sink);
    HG_LAUNCH_CHECK(ctx);
    if (ops_out) *ops_out = (double)blocks * threads * 8.0 * iters;
    return HG_OK;
}

// ---- base-conversion MAC probe: 32x32->64 multiply-accumulate with the CRT kernel's
// fold-every-4 exact accumulation, 8 independent accumulators per thread. ---------------
namespace {
__global__ void __launch_bounds__(256) mac_probe_kernel(int iters, uint32_t* sink) {
    uint64_t acc[8];
    uint64_t top[8];
    uint32_t y[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        acc[k] = 0;
        top[k] = 0;
        y[k] = (threadIdx.x * 2654435761u + k * 40503u) & 0x3fffffffu;
    }
    uint32_t m = blockIdx.x * 97u + 12345u;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
#pragma unroll
            for (int k = 0; k < 8; ++k) acc[k] += (uint64_t)y[k] * (m + r);
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            top[k] += acc[k] >> 32;
            acc[k] = (uint32_t)acc[k];
        }
        m = m * 1664525u + 1013904223u;
    }
    uint64_t s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s ^= acc[k] ^ top[k];
    if ((uint32_t)s == 0x12345678u) sink[0] = (uint32_t)s;
}
}  // namespace

extern "C" int hg_bench_mac(hg_ctx* ctx, int iters, uint32_t* sink, double* ops_out,
                            void* stream) {
    if (!ctx || !sink || iters < 1) return hg_fail(HG_EINVAL, "hg_bench_mac: bad arguments");
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
    const int blocks = sms * 8, threads = 256;
    mac_probe_kernel<<<blocks, threads, 0, (cudaStream_t)stream>>>(iters, sink);
    HG_LAUNCH_CHECK(ctx);
    if (ops_out) *ops_out = (double)blocks * threads * 8.0 * 4.0 * iters;
    return HG_OK;
}
