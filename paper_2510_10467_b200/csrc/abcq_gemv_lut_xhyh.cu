// abcq_gemv_lut_xhyh.cu -- instantiation unit (x __half, y __half) of the LUT GEMV
// kernel; split out so nvcc compiles the dtype combinations in parallel.
#include "abcq_gemv_batch.cuh"

namespace abcq {
template <>
int launch_batch_xy_inst<__half, __half>(const BatchArgs& a, int sd, bool asym, int grid, cudaStream_t st) {
    return launch_batch_xy<__half, __half>(a, sd, asym, grid, st);
}
}  // namespace abcq
