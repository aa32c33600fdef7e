// abcq_gemv_lut_xfyf.cu -- instantiation unit (x float, y float) of the LUT GEMV kernel;
// split out so nvcc compiles the four dtype combinations in parallel.
#include "abcq_gemv_lut.cuh"
#include "abcq_gemv_lut_direct.cuh"

namespace abcq {
template <>
int launch_lut_xy<float, float>(const LutArgs& a, int sd, bool asym, int grid, cudaStream_t st) {
    return launch_st<float, float>(a, sd, asym, grid, st);
}
}  // namespace abcq
