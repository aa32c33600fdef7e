// abcq_gemv_lut_xfyh.cu -- instantiation unit (x float, y __half) of the LUT GEMV kernel;
// split out so nvcc compiles the four dtype combinations in parallel.
#include "abcq_gemv_lut.cuh"
#include "abcq_gemv_lut_direct.cuh"

namespace abcq {
template <>
int launch_lut_xy<float, __half>(const LutArgs& a, int sd, bool asym, int grid, cudaStream_t st) {
    return launch_st<float, __half>(a, sd, asym, grid, st);
}
}  // namespace abcq
