// abcq_gemv_lut_xhyf.cu -- instantiation unit (x __half, y float) of the LUT GEMV kernel;
// split out so nvcc compiles the four dtype combinations in parallel.
#include "abcq_gemv_lut.cuh"
#include "abcq_gemv_lut_direct.cuh"

namespace abcq {
template <>
int launch_lut_xy<__half, float>(const LutArgs& a, int sd, bool asym, int grid, cudaStream_t st) {
    return launch_st<__half, float>(a, sd, asym, grid, st);
}
}  // namespace abcq
