// tmabench.cu -- HBM -> shared streaming through TMA bulk copies
// (cp.async.bulk + mbarrier), per-warp rings, no compute: the ceiling of the
// staged GEMV pipeline for a given slot size / ring depth / warp count.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmabench tmabench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void stream(const char* __restrict__ src, int64_t bytes_per_cta, int slot, int ring, unsigned* out) {
    extern __shared__ __align__(1024) char smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
    char* buf = smem + 1024;
    uint64_t* mb = bars + warp * ring;
    char* mybuf = buf + (size_t)warp * ring * slot;
    if (lane == 0) {
        for (int s = 0; s < ring; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&mb[s])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    const int64_t per_warp = bytes_per_cta / nw;
    const char* base = src + blockIdx.x * bytes_per_cta + warp * per_warp;
    const int n = (int)(per_warp / slot);
    auto issue = [&](int e) {
        const int s = e % ring;
        if (lane == 0) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&mb[s])), "r"(slot) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                             sa(mybuf + (size_t)s * slot)),
                         "l"(base + (int64_t)e * slot), "r"(slot), "r"(sa(&mb[s]))
                         : "memory");
        }
    };
    for (int e = 0; e < ring && e < n; ++e) issue(e);
    unsigned acc = 0;
    for (int e = 0; e < n; ++e) {
        const int s = e % ring;
        const uint32_t ph = (e / ring) & 1;
        asm volatile(
            "{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n" ::"r"(
                sa(&mb[s])),
            "r"(ph)
            : "memory");
        acc += reinterpret_cast<const unsigned*>(mybuf + (size_t)s * slot)[lane];
        __syncwarp();
        if (e + ring < n) issue(e + ring);
    }
    if (acc == 0x1234567u) out[0] = acc;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int64_t per_cta = 4ll << 20;  // 4 MiB per CTA -> 592 MiB per launch
    char* d;
    unsigned* out;
    cudaMalloc(&d, per_cta * sms);
    cudaMemset(d, 1, per_cta * sms);
    cudaMalloc(&out, 4);
    cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int warps : {4, 8, 16})
        for (int slot : {2048, 4096, 8192, 16384})
            for (int ring : {2, 4, 8}) {
                const size_t smem = 1024 + (size_t)warps * ring * slot;
                if (smem > 200 * 1024) continue;
                stream<<<sms, warps * 32, smem>>>(d, per_cta, slot, ring, out);
                cudaEventRecord(a);
                stream<<<sms, warps * 32, smem>>>(d, per_cta, slot, ring, out);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                printf("warps %2d slot %5d ring %d (in flight %4zu KB/SM): %6.0f GB/s\n", warps, slot, ring,
                       (size_t)warps * ring * slot / 1024, per_cta * sms / (ms * 1e-3) / 1e9);
            }
    printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
