// abcq_gemv_lut_xfyf.cu -- instantiation unit (x float, y float) of the LUT GEMV
// kernel; split out so nvcc compiles the dtype combinations in parallel.
#include "abcq_gemv_batch.cuh"

namespace abcq {
template <>
int launch_batch_xy_inst<float, float>(const BatchArgs& a, int sd, bool asym, int grid, cudaStream_t st) {
    return launch_batch_xy<float, float>(a, sd, asym, grid, st);
}
}  // namespace abcq
