#include <cstdint>
#include <cstdio>
__global__ void imma_probe(int iters, int* out) {
    uint32_t a[4] = {threadIdx.x, threadIdx.x * 3u, 7u, 9u};
    uint32_t b[2] = {threadIdx.x ^ 5u, 11u};
    int c[8][4] = {};
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k)
        asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                     : "+r"(c[k][0]), "+r"(c[k][1]), "+r"(c[k][2]), "+r"(c[k][3])
                     : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
    }
    int s = 0;
    for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1] + c[k][2] + c[k][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void dfma_probe(int iters, double* out) {
    double a[8], x = threadIdx.x * 1e-3, y = 1.0000001;
    for (int k = 0; k < 8; ++k) a[k] = k;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = fma(a[k], y, x);
    double s = 0; for (int k = 0; k < 8; ++k) s += a[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void imadhi_probe(int iters, uint32_t* out) {
    uint32_t a[8], m = threadIdx.x * 2654435761u;
    for (int k = 0; k < 8; ++k) a[k] = k * 7919u + threadIdx.x;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = __umulhi(a[k], m) + a[k];
    uint32_t s = 0; for (int k = 0; k < 8; ++k) s += a[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void imad_probe(int iters, uint32_t* out) {
    uint32_t a[8], m = threadIdx.x * 2654435761u;
    for (int k = 0; k < 8; ++k) a[k] = k * 7919u + threadIdx.x;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = a[k] * m + k;
    uint32_t s = 0; for (int k = 0; k < 8; ++k) s += a[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void imadwide_probe(int iters, uint64_t* out) {
    uint64_t a[8]; uint32_t m = threadIdx.x * 2654435761u;
    for (int k = 0; k < 8; ++k) a[k] = k * 7919u + threadIdx.x;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = (uint64_t)(uint32_t)a[k] * m + a[k];
    uint64_t s = 0; for (int k = 0; k < 8; ++k) s += a[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    int *o; cudaMalloc(&o, 1 << 26);
    cudaEvent_t s, e; cudaEventCreate(&s); cudaEventCreate(&e);
    int blocks = 148 * 8, thr = 128, iters = 20000; float ms;
    for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(s); imma_probe<<<blocks, thr>>>(iters, o); cudaEventRecord(e); cudaEventSynchronize(e);
    cudaEventElapsedTime(&ms, s, e);
    double ops = 2.0 * 16 * 8 * 32 * 8.0 * iters * blocks * (thr / 32);
    printf("IMMA u8 m16n8k32: %.1f TOPS (%.2f ms)\n", ops / ms / 1e9, ms);
    cudaEventRecord(s); dfma_probe<<<blocks, thr>>>(iters, (double*)o); cudaEventRecord(e); cudaEventSynchronize(e);
    cudaEventElapsedTime(&ms, s, e);
    printf("DFMA: %.1f G/s = %.1f /clk/SM @1.965GHz\n", 8.0 * iters * blocks * thr / ms / 1e6, 8.0 * iters * blocks * thr / ms / 1e6 / 148 / 1.965);
    cudaEventRecord(s); imadhi_probe<<<blocks, thr>>>(iters, (uint32_t*)o); cudaEventRecord(e); cudaEventSynchronize(e);
    cudaEventElapsedTime(&ms, s, e);
    printf("IMAD.HI+IADD: %.1f G/s = %.1f /clk/SM\n", 8.0 * iters * blocks * thr / ms / 1e6, 8.0 * iters * blocks * thr / ms / 1e6 / 148 / 1.965);
    cudaEventRecord(s); imad_probe<<<blocks, thr>>>(iters, (uint32_t*)o); cudaEventRecord(e); cudaEventSynchronize(e);
    cudaEventElapsedTime(&ms, s, e);
    printf("IMAD: %.1f G/s = %.1f /clk/SM\n", 8.0 * iters * blocks * thr / ms / 1e6, 8.0 * iters * blocks * thr / ms / 1e6 / 148 / 1.965);
    cudaEventRecord(s); imadwide_probe<<<blocks, thr>>>(iters, (uint64_t*)o); cudaEventRecord(e); cudaEventSynchronize(e);
    cudaEventElapsedTime(&ms, s, e);
    printf("IMAD.WIDE acc: %.1f G/s = %.1f /clk/SM\n", 8.0 * iters * blocks * thr / ms / 1e6, 8.0 * iters * blocks * thr / ms / 1e6 / 148 / 1.965);
    }
    return 0;
}
