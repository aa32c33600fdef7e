// mma.sync m16n8k16 (f16 -> f32) issue rate on one SM: W warps, each running
// CH independent accumulator chains; prints HMMA per SM-cycle.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o hmma_rate hmma_rate.cu && ./hmma_rate
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int CH>
__global__ void hmma_loop(int iters, float* out, long long* cyc) {
    float c[CH][4];
    for (int k = 0; k < CH; ++k)
        for (int j = 0; j < 4; ++j) c[k][j] = 0.f;
    uint32_t a0 = threadIdx.x * 0x00010001u, a1 = a0 ^ 0x3c003c00u, a2 = a0 + 7, a3 = a1 + 9;
    uint32_t b0 = 0x3c00bc00u ^ threadIdx.x, b1 = 0xbc003c00u;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < CH; ++k)
            asm volatile(
                "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                "{%0,%1,%2,%3};"
                : "+f"(c[k][0]), "+f"(c[k][1]), "+f"(c[k][2]), "+f"(c[k][3])
                : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    __syncthreads();
    long long t1 = clock64();
    float s = 0.f;
    for (int k = 0; k < CH; ++k) s += c[k][0] + c[k][1] + c[k][2] + c[k][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int CH>
void run(int warps) {
    const int iters = 4096;
    float* out;
    long long* cyc;
    cudaMalloc(&out, 148 * warps * 32 * sizeof(float));
    cudaMalloc(&cyc, 148 * sizeof(long long));
    hmma_loop<CH><<<148, warps * 32>>>(16, out, cyc);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    hmma_loop<CH><<<148, warps * 32>>>(iters, out, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    long long c0;
    cudaMemcpy(&c0, cyc, sizeof(c0), cudaMemcpyDeviceToHost);
    const double hmma_per_sm = (double)iters * CH * warps;
    printf("warps/SM %2d chains %d: %.3f HMMA per SM-cycle (%.0f cycles), %.0f TFLOP/s f16 dense over 148 SMs\n", warps,
           CH, hmma_per_sm / c0, (double)c0, hmma_per_sm * 148 * 4096 * 2 / (ms * 1e-3) / 1e12);
    cudaFree(out);
    cudaFree(cyc);
}

int main() {
    for (int w : {4, 8, 16, 32}) {
        run<1>(w);
        run<2>(w);
        run<4>(w);
        run<8>(w);
    }
    return 0;
}
