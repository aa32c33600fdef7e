// membench.cu -- HBM streaming micro-benchmark mirroring the GEMV's access
// pattern (512 B blocks, one 16 B load per lane), to find the achievable read
// bandwidth for each load flavour / occupancy. Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o membench membench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE>
__device__ __forceinline__ uint4 ld(const uint4* p) {
    uint4 r;
    if constexpr (MODE == 0)
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    else if constexpr (MODE == 1)
        asm volatile("ld.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    else if constexpr (MODE == 2)
        asm volatile("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    else
        asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}

// blocks of 512 B; CTA c owns a contiguous block range; warps round-robin.
template <int MODE, int BATCH>
__global__ void stream(const uint4* __restrict__ src, int64_t nblocks, unsigned* out, int prefetch) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int64_t per = (nblocks + gridDim.x - 1) / gridDim.x;
    const int64_t b0 = blockIdx.x * per, b1 = min(nblocks, b0 + per);
    if (prefetch && threadIdx.x == 0) {
        const char* p = reinterpret_cast<const char*>(src + b0 * 32);
        int64_t bytes = (b1 - b0) * 512;
        while (bytes > 0) {
            unsigned n = bytes > 65536 ? 65536u : (unsigned)bytes;
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(n) : "memory");
            p += n; bytes -= n;
        }
    }
    unsigned acc = 0;
    for (int64_t b = b0 + warp; b < b1; b += (int64_t)nw * BATCH) {
        uint4 v[BATCH];
#pragma unroll
        for (int k = 0; k < BATCH; ++k)
            if (b + (int64_t)k * nw < b1) v[k] = ld<MODE>(src + (b + (int64_t)k * nw) * 32 + lane);
            else v[k] = make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int k = 0; k < BATCH; ++k) acc ^= v[k].x + v[k].y * 3 + v[k].z * 5 + v[k].w * 7;
    }
    if (acc == 0x12345678u) out[0] = acc;
}

template <int MODE, int BATCH>
float run(const uint4* d, int64_t nblocks, unsigned* out, int grid, int threads, int prefetch, int copies, int64_t copy_blocks) {
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    for (int i = 0; i < 3; ++i) stream<MODE, BATCH><<<grid, threads>>>(d + (i % copies) * copy_blocks * 32, nblocks, out, prefetch);
    cudaEventRecord(a);
    const int reps = 20;
    for (int i = 0; i < reps; ++i) stream<MODE, BATCH><<<grid, threads>>>(d + (i % copies) * copy_blocks * 32, nblocks, out, prefetch);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    return ms / reps;
}

int main() {
    const int64_t bytes_per = 64ll << 20;  // 64 MiB per launch
    const int copies = 4;                  // rotate 256 MiB > L2
    const int64_t nblocks = bytes_per / 512;
    uint4* d; unsigned* out;
    cudaMalloc(&d, bytes_per * copies);
    cudaMemset(d, 1, bytes_per * copies);
    cudaMalloc(&out, 4);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    printf("SMs %d, %lld MiB per launch\n", sms, (long long)(bytes_per >> 20));
    struct Cfg { int threads, ctas_per_sm; };
    Cfg cfgs[] = {{512, 1}, {640, 1}, {768, 1}, {1024, 1}, {256, 4}, {512, 2}};
    for (auto c : cfgs) {
        for (int pf = 0; pf < 2; ++pf) {
            float t0 = run<0, 8>(d, nblocks, out, sms * c.ctas_per_sm, c.threads, pf, copies, nblocks);
            float t1 = run<1, 8>(d, nblocks, out, sms * c.ctas_per_sm, c.threads, pf, copies, nblocks);
            float t2 = run<2, 8>(d, nblocks, out, sms * c.ctas_per_sm, c.threads, pf, copies, nblocks);
            float t3 = run<3, 8>(d, nblocks, out, sms * c.ctas_per_sm, c.threads, pf, copies, nblocks);
            float t4 = run<0, 4>(d, nblocks, out, sms * c.ctas_per_sm, c.threads, pf, copies, nblocks);
            float t5 = run<0, 16>(d, nblocks, out, sms * c.ctas_per_sm, c.threads, pf, copies, nblocks);
            auto gbs = [&](float ms) { return bytes_per / (ms * 1e-3) / 1e9; };
            printf("threads %4d x %d/SM prefetch %d | nc.na b8 %7.0f | plain b8 %7.0f | na b8 %7.0f | nc b8 %7.0f | nc.na b4 %7.0f | nc.na b16 %7.0f GB/s\n",
                   c.threads, c.ctas_per_sm, pf, gbs(t0), gbs(t1), gbs(t2), gbs(t3), gbs(t4), gbs(t5));
        }
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("status %s\n", cudaGetErrorString(e));
    return 0;
}
