// abcq_gemv_lut_xhyf.cu -- instantiation unit (x __half, y float) of the LUT GEMV
// kernel; split out so nvcc compiles the dtype combinations in parallel.
#include "abcq_gemv_batch.cuh"

namespace abcq {
template <>
int launch_batch_xy_inst<__half, float>(const BatchArgs& a, int sd, bool asym, int grid, cudaStream_t st) {
    return launch_batch_xy<__half, float>(a, sd, asym, grid, st);
}
}  // namespace abcq
