// abcq_gemv_generic.cu -- any-layout, any-group-size GEMV on sm_100a.
//
// Covers what the tiled LUT kernel does not: group sizes other than 128
// (tests/test_gemv.py:25-36 uses g=32 and a ragged g=40; acceptance uses
// g=25), the ROWMAJOR (reference) plane layout, and GemvEngine.naive
// semantics (gemv.py:170-186). One warp per row; the warp decodes the sign
// bits of a group column-parallel, reduces, and lane 0 accumulates
//   naive=0: s_g in f32, acc += f32(alpha*s_g) in f64    (numba kernel, gemv.py:86-95)
//   naive=1: s_g in f64, acc += alpha*s_g in f64          (gemv.py:178-182)
// and the asymmetric term offset . gx in f64 (gemv.py:183-185, 217-221).
// This is a correctness path for small or irregular shapes, not the hot path.
#include "abcq_common.cuh"
#include "abcq_internal.h"

namespace abcq {

struct GenArgs {
    const void* planes;
    int64_t plane_stride;  // bytes
    const void* alpha;
    const void* offset;
    const void* x;
    void* y;
    int rows, cols, g, p, layout, scale_dtype, x_dtype, y_dtype, naive;
};

// sign bit (1 -> +1) of plane i, row n, column k in either layout
__device__ __forceinline__ int code_bit(const GenArgs& a, int i, int n, int k) {
    const char* base = static_cast<const char*>(a.planes) + (int64_t)i * a.plane_stride;
    if (a.layout == ABCQ_LAYOUT_ROWMAJOR) {
        const uint32_t* w = reinterpret_cast<const uint32_t*>(base);
        return (w[(int64_t)n * words_per_row(a.cols) + (k >> 5)] >> (k & 31)) & 1;
    }
    const int NRT = n_row_tiles(a.rows);
    const int grp = k >> 7, s = grp >> 1, half = grp & 1;
    const int rt = n >> 4, r = n & 15;
    const int b = (k & 127) >> 3;     // reference byte within the group block
    const int j = (b - r) & 15;       // rotated storage position
    const unsigned char* blk = reinterpret_cast<const unsigned char*>(base) +
                               (((int64_t)s * NRT + rt) * 32 + half * 16 + r) * 16;
    return (blk[j] >> (k & 7)) & 1;
}

__device__ __forceinline__ float scale_at(const GenArgs& a, int i, int n, int grp) {
    if (a.layout == ABCQ_LAYOUT_ROWMAJOR) {
        const int G = group_count(a.cols, a.g);
        return load_any(a.alpha, a.scale_dtype, ((int64_t)i * a.rows + n) * G + grp);
    }
    const int NRT = n_row_tiles(a.rows);
    const int s = grp >> 1, half = grp & 1, rt = n >> 4, r = n & 15;
    const int64_t items = (int64_t)n_slices(a.cols) * NRT;
    return load_any(a.alpha, a.scale_dtype, ((int64_t)i * items + (int64_t)s * NRT + rt) * 32 + half * 16 + r);
}

__device__ __forceinline__ float offset_at(const GenArgs& a, int n, int grp) {
    if (a.layout == ABCQ_LAYOUT_ROWMAJOR) {
        const int G = group_count(a.cols, a.g);
        return load_any(a.offset, a.scale_dtype, (int64_t)n * G + grp);
    }
    const int NRT = n_row_tiles(a.rows);
    const int s = grp >> 1, half = grp & 1, rt = n >> 4, r = n & 15;
    return load_any(a.offset, a.scale_dtype, ((int64_t)s * NRT + rt) * 32 + half * 16 + r);
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__global__ void gemv_generic_kernel(const GenArgs a) {
    const int lane = threadIdx.x & 31;
    const int n = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (n >= a.rows) return;
    const int G = group_count(a.cols, a.g);
    double acc = 0.0;
    for (int i = 0; i < a.p; ++i) {
        for (int grp = 0; grp < G; ++grp) {
            const int lo = grp * a.g, hi = min(lo + a.g, a.cols);
            double part;
            if (a.naive) {
                double s = 0.0;
                for (int k = lo + lane; k < hi; k += 32) {
                    const double xv = load_any(a.x, a.x_dtype, k);
                    s += code_bit(a, i, n, k) ? xv : -xv;
                }
                part = warp_sum(s) * (double)scale_at(a, i, n, grp);
            } else {
                float s = 0.f;
                for (int k = lo + lane; k < hi; k += 32) {
                    const float xv = load_any(a.x, a.x_dtype, k);
                    s += code_bit(a, i, n, k) ? xv : -xv;
                }
                part = (double)(scale_at(a, i, n, grp) * warp_sum(s));
            }
            acc += part;
        }
    }
    if (a.offset) {
        for (int grp = 0; grp < G; ++grp) {
            const int lo = grp * a.g, hi = min(lo + a.g, a.cols);
            double gx = 0.0;
            for (int k = lo + lane; k < hi; k += 32) gx += load_any(a.x, a.x_dtype, k);
            acc += (double)offset_at(a, n, grp) * warp_sum(gx);
        }
    }
    if (lane == 0) store_any(a.y, a.y_dtype, n, (float)acc);
}

// bcq.dequantize (bcq.py:372-378 -> _dequant64 bcq.py:137-152): f64 sum, f32 cast
__global__ void dequantize_kernel(const GenArgs a, void* w, int w_dtype) {
    const int64_t total = (int64_t)a.rows * a.cols;
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < total;
         u += (int64_t)gridDim.x * blockDim.x) {
        const int n = (int)(u / a.cols), k = (int)(u - (int64_t)n * a.cols);
        const int grp = k / a.g;
        double v = 0.0;
        for (int i = 0; i < a.p; ++i)
            v += code_bit(a, i, n, k) ? (double)scale_at(a, i, n, grp) : -(double)scale_at(a, i, n, grp);
        if (a.offset) v += (double)offset_at(a, n, grp);
        store_any(w, w_dtype, u, (float)v);
    }
}

int launch_dequantize(const abcq_model_t* m, int p, void* w, int w_dtype, cudaStream_t st) {
    GenArgs a{};
    a.planes = m->planes;
    a.plane_stride = m->plane_stride_bytes;
    a.alpha = m->alpha[p];
    a.offset = m->asymmetric ? m->offset[p] : nullptr;
    a.rows = m->rows;
    a.cols = m->cols;
    a.g = m->group_size;
    a.p = p;
    a.layout = m->layout;
    a.scale_dtype = m->scale_dtype;
    const int64_t total = (int64_t)m->rows * m->cols;
    int64_t grid = ceil_div(total, 256);
    if (grid > 148 * 64) grid = 148 * 64;
    dequantize_kernel<<<(int)grid, 256, 0, st>>>(a, w, w_dtype);
    return (int)cudaGetLastError();
}

int launch_gemv_generic(const abcq_model_t* m, int p, const void* x, int x_dtype, void* y, int y_dtype,
                        int naive, cudaStream_t st) {
    GenArgs a;
    a.planes = m->planes;
    a.plane_stride = m->plane_stride_bytes;
    a.alpha = m->alpha[p];
    a.offset = m->asymmetric ? m->offset[p] : nullptr;
    a.x = x;
    a.y = y;
    a.rows = m->rows;
    a.cols = m->cols;
    a.g = m->group_size;
    a.p = p;
    a.layout = m->layout;
    a.scale_dtype = m->scale_dtype;
    a.x_dtype = x_dtype;
    a.y_dtype = y_dtype;
    a.naive = naive;
    const int warps = 8;
    const int grid = (int)ceil_div(m->rows, warps);
    gemv_generic_kernel<<<grid, warps * 32, 0, st>>>(a);
    return (int)cudaGetLastError();
}

}  // namespace abcq
