// membench2.cu -- achievable HBM read bandwidth on this B200 for a few access
// patterns (1 GiB per launch, so launch overhead is amortised).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o membench2 membench2.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint4 ldna(const uint4* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}
__device__ __forceinline__ void ld256(const void* p, uint32_t (&r)[8]) {
    asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "l"(p));
}

template <int U>
__global__ void gs(const uint4* __restrict__ s, int64_t n, unsigned* out) {
    unsigned acc = 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    for (; i + (U - 1) * stride < n; i += U * stride) {
        uint4 v[U];
#pragma unroll
        for (int k = 0; k < U; ++k) v[k] = ldna(s + i + k * stride);
#pragma unroll
        for (int k = 0; k < U; ++k) acc ^= v[k].x + v[k].y + v[k].z + v[k].w;
    }
    for (; i < n; i += stride) {
        uint4 v = ldna(s + i);
        acc ^= v.x + v.w;
    }
    if (acc == 0x1234567u) out[0] = acc;
}

template <int U>
__global__ void gs256(const uint4* __restrict__ s, int64_t n2, unsigned* out) {
    unsigned acc = 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    for (; i + (U - 1) * stride < n2; i += U * stride) {
        uint32_t v[U][8];
#pragma unroll
        for (int k = 0; k < U; ++k) ld256(s + 2 * (i + k * stride), v[k]);
#pragma unroll
        for (int k = 0; k < U; ++k) acc ^= v[k][0] + v[k][3] + v[k][5] + v[k][7];
    }
    if (acc == 0x1234567u) out[0] = acc;
}

// the GEMV's pattern: CTA-contiguous block ranges, warps round-robin over
// 512 B blocks, B loads in flight per warp
template <int B>
__global__ void ctablk(const uint4* __restrict__ s, int64_t nblocks, unsigned* out) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int64_t per = (nblocks + gridDim.x - 1) / gridDim.x;
    const int64_t b0 = blockIdx.x * per, b1 = min(nblocks, b0 + per);
    unsigned acc = 0;
    for (int64_t b = b0 + warp; b < b1; b += (int64_t)nw * B) {
        uint4 v[B];
#pragma unroll
        for (int k = 0; k < B; ++k)
            v[k] = (b + (int64_t)k * nw < b1) ? ldna(s + (b + (int64_t)k * nw) * 32 + lane) : make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int k = 0; k < B; ++k) acc ^= v[k].x + v[k].y + v[k].z + v[k].w;
    }
    if (acc == 0x1234567u) out[0] = acc;
}
// grid-interleaved blocks: block j of the whole array goes to CTA j % G
template <int B>
__global__ void gridblk(const uint4* __restrict__ s, int64_t nblocks, unsigned* out) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int64_t stride = (int64_t)gridDim.x * nw;
    unsigned acc = 0;
    for (int64_t b = (int64_t)blockIdx.x * nw + warp; b < nblocks; b += stride * B) {
        uint4 v[B];
#pragma unroll
        for (int k = 0; k < B; ++k)
            v[k] = (b + k * stride < nblocks) ? ldna(s + (b + k * stride) * 32 + lane) : make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int k = 0; k < B; ++k) acc ^= v[k].x + v[k].y + v[k].z + v[k].w;
    }
    if (acc == 0x1234567u) out[0] = acc;
}

template <typename F>
float timeit(F f, int reps = 10) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    f(0);
    f(1);
    cudaEventRecord(a);
    for (int i = 0; i < reps; ++i) f(i);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms / reps;
}

int main() {
    const int64_t bytes = 1ll << 30;
    uint4* d;
    unsigned* out;
    cudaMalloc(&d, 2 * bytes);
    cudaMemset(d, 1, 2 * bytes);
    cudaMalloc(&out, 4);
    const int64_t n = bytes / 16;
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    auto gb = [&](float ms) { return bytes / (ms * 1e-3) / 1e9; };
    for (int t : {256, 512, 1024})
        for (int bpsm : {1, 2, 4, 8}) {
            if (t * bpsm > 2048) continue;
            int g = sms * bpsm;
            float a4 = timeit([&](int i) { gs<4><<<g, t>>>(d + (i & 1) * n, n, out); });
            float a8 = timeit([&](int i) { gs<8><<<g, t>>>(d + (i & 1) * n, n, out); });
            float b2 = timeit([&](int i) { gs256<2><<<g, t>>>(d + (i & 1) * n, n / 2, out); });
            float b4 = timeit([&](int i) { gs256<4><<<g, t>>>(d + (i & 1) * n, n / 2, out); });
            printf("threads %4d x %d/SM: v4 u4 %6.0f  v4 u8 %6.0f  v8 u2 %6.0f  v8 u4 %6.0f GB/s\n", t, bpsm, gb(a4),
                   gb(a8), gb(b2), gb(b4));
        }
    const int64_t nb = bytes / 512;
    for (int t : {512, 640, 768}) {
        int g = sms;
        float c8 = timeit([&](int i) { ctablk<8><<<g, t>>>(d + (i & 1) * n, nb, out); });
        float c4 = timeit([&](int i) { ctablk<4><<<g, t>>>(d + (i & 1) * n, nb, out); });
        float g8 = timeit([&](int i) { gridblk<8><<<g, t>>>(d + (i & 1) * n, nb, out); });
        float g4 = timeit([&](int i) { gridblk<4><<<g, t>>>(d + (i & 1) * n, nb, out); });
        printf("threads %4d x 1/SM: cta-contig B8 %6.0f B4 %6.0f | grid-interleaved B8 %6.0f B4 %6.0f GB/s\n", t,
               gb(c8), gb(c4), gb(g8), gb(g4));
    }
    float c = timeit([&](int i) {
        cudaMemcpyAsync(d + (i & 1) * n, d + ((i + 1) & 1) * n, bytes, cudaMemcpyDeviceToDevice);
    });
    printf("cudaMemcpy D2D 1 GiB: %6.0f GB/s (read+write)\n", 2 * gb(c));
    printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
