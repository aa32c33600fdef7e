// pdlfloor.cu -- the floor of a chain of dependent launches on this GPU: empty
// kernels (griddepcontrol.wait + launch_dependents) back to back in a CUDA
// graph, with / without programmatic dependent launch, 148 CTAs, with and
// without a 16-CTA cluster, and with 227 KB of dynamic shared memory.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pdlfloor pdlfloor.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void empty_kernel(int* p) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;");
    if (p && threadIdx.x == 0 && blockIdx.x == 0) atomicAdd(p, 1);
}

static float chain(int n, bool pdl, int cluster, int smem, int threads, cudaStream_t st) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cluster > 1 ? 112 : 148);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    int na = 0;
    if (pdl) {
        at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    if (cluster > 1) {
        at[na].id = cudaLaunchAttributeClusterDimension;
        at[na].val.clusterDim.x = cluster;
        at[na].val.clusterDim.y = 1;
        at[na].val.clusterDim.z = 1;
        ++na;
    }
    cfg.attrs = at;
    cfg.numAttrs = na;
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < n; ++i) cudaLaunchKernelEx(&cfg, empty_kernel, (int*)nullptr);
    cudaStreamEndCapture(st, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, st);
    cudaStreamSynchronize(st);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, st);
    for (int r = 0; r < 10; ++r) cudaGraphLaunch(ge, st);
    cudaEventRecord(b, st);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
    return ms * 1e3f / (10 * n);
}

int main() {
    cudaStream_t st;
    cudaStreamCreate(&st);
    cudaFuncSetAttribute(empty_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(empty_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int pdl : {0, 1})
        for (int cl : {1, 16})
            for (int smem : {0, 113 * 1024, 227 * 1024})
                printf("pdl %d cluster %2d smem %6d: %.2f us per launch\n", pdl, cl, smem,
                       chain(50, pdl, cl, smem, 288, st));
    printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
