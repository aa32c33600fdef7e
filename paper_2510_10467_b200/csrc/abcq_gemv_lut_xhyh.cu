// abcq_gemv_lut_xhyh.cu -- instantiation unit (x __half, y __half) of the LUT GEMV kernel;
// split out so nvcc compiles the four dtype combinations in parallel.
#include "abcq_gemv_lut.cuh"
#include "abcq_gemv_lut_direct.cuh"

namespace abcq {
template <>
int launch_lut_xy<__half, __half>(const LutArgs& a, int sd, bool asym, int grid, cudaStream_t st) {
    return launch_st<__half, __half>(a, sd, asym, grid, st);
}
}  // namespace abcq
