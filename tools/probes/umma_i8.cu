// Standalone probe: tcgen05.mma kind::i8 (u8 x u8 -> s32), M=128, N=256, K=128 bytes,
// A/B K-major SWIZZLE_NONE in shared memory, D in TMEM, read back with tcgen05.ld.
// Validates the descriptor encodings used by hg_crt_umma.cu.   nvcc -arch=sm_100a
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;  // version = 1 (sm100)
    // base_offset 0, lbo_mode 0, layout_type 0 (SWIZZLE_NONE)
    return d;
}

// A: M x K (row-major bytes), core-matrix layout: core(g, c) = rows 8g..8g+7, bytes 16c..16c+15
__global__ void umma_probe(const uint8_t* A, const uint8_t* B, int* D, int M, int N, int K) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t tmem_base;
    __shared__ __align__(8) uint64_t mbar;
    uint8_t* sa = smem;
    uint8_t* sb = smem + M * K;
    const int tid = threadIdx.x;
    const int KC = K / 16;
    // stage A, B into core-matrix layout
    for (int idx = tid; idx < M * K / 16; idx += blockDim.x) {
        int r = idx / KC, c = idx % KC;
        int g = r / 8, rr = r % 8;
        const uint4 v = *reinterpret_cast<const uint4*>(A + r * K + c * 16);
        *reinterpret_cast<uint4*>(sa + ((g * KC + c) * 8 + rr) * 16) = v;
    }
    for (int idx = tid; idx < N * K / 16; idx += blockDim.x) {
        int r = idx / KC, c = idx % KC;
        int g = r / 8, rr = r % 8;
        const uint4 v = *reinterpret_cast<const uint4*>(B + r * K + c * 16);
        *reinterpret_cast<uint4*>(sb + ((g * KC + c) * 8 + rr) * 16) = v;
    }
    if (tid / 32 == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"((uint32_t)__cvta_generic_to_shared(&tmem_base)), "n"(256));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"((uint32_t)__cvta_generic_to_shared(&mbar)));
    }
    asm volatile("fence.proxy.async.shared::cta;\n");
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t tmem = tmem_base;
    if (tid == 0) {
        // idesc: c_format S32 (2) bits 4-5, a/b format u8 (0), K-major, N>>3 at 17, M>>4 at 24
        uint32_t idesc = (2u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
        const uint32_t a0 = (uint32_t)__cvta_generic_to_shared(sa);
        const uint32_t b0 = (uint32_t)__cvta_generic_to_shared(sb);
        for (int k = 0; k < K / 32; ++k) {
            uint64_t da = smem_desc(a0 + k * 2 * 128, 128, KC * 128);
            uint64_t db = smem_desc(b0 + k * 2 * 128, 128, KC * 128);
            uint32_t acc = k > 0;
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                         "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                         ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(acc));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"((uint32_t)__cvta_generic_to_shared(&mbar)));
    }
    // wait for the MMA
    {
        uint32_t done = 0;
        while (!done) {
            asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
                         : "=r"(done) : "r"((uint32_t)__cvta_generic_to_shared(&mbar)), "r"(0));
        }
    }
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    // each warp reads its 32 lanes; thread = row
    const int warp = tid / 32;
    const int row = warp * 32 + (tid & 31);
    for (int c0 = 0; c0 < N; c0 += 8) {
        uint32_t v[8];
        uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + c0;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                     : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;\n");
        for (int j = 0; j < 8; ++j) D[row * N + c0 + j] = (int)v[j];
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(256));
}

int main() {
    const int M = 128, N = 256, K = 128;
    std::vector<uint8_t> A(M * K), B(N * K);
    for (auto& x : A) x = rand() & 0xff;
    for (auto& x : B) x = rand() & 0xff;
    uint8_t *dA, *dB;
    int* dD;
    CK(cudaMalloc(&dA, M * K));
    CK(cudaMalloc(&dB, N * K));
    CK(cudaMalloc(&dD, M * N * 4));
    CK(cudaMemcpy(dA, A.data(), M * K, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, B.data(), N * K, cudaMemcpyHostToDevice));
    size_t smem = M * K + N * K;
    CK(cudaFuncSetAttribute(umma_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    umma_probe<<<1, 128, smem>>>(dA, dB, dD, M, N, K);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    std::vector<int> D(M * N);
    CK(cudaMemcpy(D.data(), dD, M * N * 4, cudaMemcpyDeviceToHost));
    long bad = 0;
    for (int i = 0; i < M; ++i)
        for (int j = 0; j < N; ++j) {
            long s = 0;
            for (int k = 0; k < K; ++k) s += (long)A[i * K + k] * B[j * K + k];
            if (s != D[i * N + j]) {
                if (bad < 5) printf("mismatch (%d,%d): got %d want %ld\n", i, j, D[i * N + j], s);
                ++bad;
            }
        }
    printf("UMMA i8 probe: %ld mismatches of %d\n", bad, M * N);
    return bad != 0;
}
