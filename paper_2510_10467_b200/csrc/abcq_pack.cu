// abcq_pack.cu -- reference packing -> B200 tiled layout (and back), scale-set
// tiling, and the bit-exact lookup-table builder.
//
// Reference anchors (paths under /root/reference/pkg/src/anybcq/):
//   packing.py:1-37     normative plane packing the input words follow
//   bcq.py:50-96        ScaleTensor alpha (p, N, G) / offset (N, G)
//   gemv.py:67-81       LookupTable.build
#include "abcq_common.cuh"
#include "abcq_internal.h"

namespace abcq {

// One thread per 16-byte lane block of the tiled layout.
__global__ void pack_planes_kernel(const uint32_t* __restrict__ words, int planes, int rows,
                                   int cols, uint4* __restrict__ out) {
    const int NRT = n_row_tiles(rows), NS = n_slices(cols), wpr = words_per_row(cols);
    const int64_t per_plane = (int64_t)NS * NRT * 32;
    const int64_t total = per_plane * planes;
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < total;
         u += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(u / per_plane);
        const int64_t rem = u - i * per_plane;
        const int blk = (int)(rem >> 5), lane = (int)(rem & 31);
        const int s = blk / NRT, rt = blk - s * NRT;
        const int half = lane >> 4, r = lane & 15;
        const int row = rt * kTileRows + r, g = 2 * s + half;
        uint32_t src[4] = {0u, 0u, 0u, 0u};
        if (row < rows) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int w = 4 * g + q;
                if (w < wpr) src[q] = words[((int64_t)i * rows + row) * wpr + w];
            }
        }
        // rotate the 16 bytes left by r: dst byte j = src byte (j + r) & 15
        uint32_t dst[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            uint32_t v = 0;
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const int sb = (4 * q + b + r) & 15;
                const uint32_t byte = (src[sb >> 2] >> (8 * (sb & 3))) & 0xFFu;
                v |= byte << (8 * b);
            }
            dst[q] = v;
        }
        out[u] = make_uint4(dst[0], dst[1], dst[2], dst[3]);
    }
}

__global__ void unpack_planes_kernel(const uint4* __restrict__ tiled, int planes, int rows,
                                     int cols, uint32_t* __restrict__ words) {
    const int NRT = n_row_tiles(rows), NS = n_slices(cols), wpr = words_per_row(cols);
    const int64_t per_plane = (int64_t)NS * NRT * 32;
    const int64_t total = per_plane * planes;
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < total;
         u += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(u / per_plane);
        const int64_t rem = u - i * per_plane;
        const int blk = (int)(rem >> 5), lane = (int)(rem & 31);
        const int s = blk / NRT, rt = blk - s * NRT;
        const int half = lane >> 4, r = lane & 15;
        const int row = rt * kTileRows + r, g = 2 * s + half;
        if (row >= rows) continue;
        const uint4 v = tiled[u];
        const uint32_t st[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int w = 4 * g + q;
            if (w >= wpr) continue;
            uint32_t word = 0;
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const int rb = 4 * q + b;        // reference byte
                const int j = (rb - r) & 15;     // stored position
                word |= ((st[j >> 2] >> (8 * (j & 3))) & 0xFFu) << (8 * b);
            }
            words[((int64_t)i * rows + row) * wpr + w] = word;
        }
    }
}

template <typename ST>
__global__ void pack_scales_kernel(const float* __restrict__ alpha, const float* __restrict__ offset,
                                   int p, int rows, int cols, ST* __restrict__ alpha_out,
                                   ST* __restrict__ offset_out) {
    const int NRT = n_row_tiles(rows), NS = n_slices(cols), G = group_count(cols, kGroup);
    const int64_t n_alpha = (int64_t)NS * NRT * p * 32;
    const int64_t n_off = offset ? (int64_t)NS * NRT * 32 : 0;
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n_alpha + n_off;
         u += (int64_t)gridDim.x * blockDim.x) {
        if (u < n_alpha) {
            const int64_t per_plane = (int64_t)NS * NRT * 32;  // element (i*items + item)*32 + lane
            const int i = (int)(u / per_plane);
            const int64_t q = u - i * per_plane;
            const int lane = (int)(q & 31);
            const int blk = (int)(q >> 5);
            const int s = blk / NRT, rt = blk - s * NRT;
            const int row = rt * kTileRows + (lane & 15), g = 2 * s + (lane >> 4);
            float v = 0.f;
            if (row < rows && g < G) v = alpha[((int64_t)i * rows + row) * G + g];
            alpha_out[u] = from_f32<ST>(v);
        } else {
            const int64_t o = u - n_alpha;
            const int lane = (int)(o & 31);
            const int blk = (int)(o >> 5);
            const int s = blk / NRT, rt = blk - s * NRT;
            const int row = rt * kTileRows + (lane & 15), g = 2 * s + (lane >> 4);
            float v = 0.f;
            if (row < rows && g < G) v = offset[(int64_t)row * G + g];
            offset_out[o] = from_f32<ST>(v);
        }
    }
}

// LookupTable.build (gemv.py:67-81): one thread per (chunk, entry); the
// sequential ascending-j evaluation reproduces the doubling's f32 rounding.
template <typename XT>
__global__ void lut_build_kernel(const XT* __restrict__ x, int cols, int mu, float* __restrict__ table) {
    const int chunks = (int)ceil_div(cols, mu);
    const int n = 1 << mu;
    const int64_t total = (int64_t)chunks * n;
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < total;
         u += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(u >> mu), t = (int)(u & (n - 1));
        float v = 0.f;
        for (int j = 0; j < mu; ++j) {
            const int k = c * mu + j;
            const float xj = k < cols ? to_f32<XT>(x[k]) : 0.f;
            v = ((t >> j) & 1) ? v + xj : v - xj;
        }
        table[u] = v;
    }
}

int probe_kernel_image() {
    cudaFuncAttributes fa;
    return (int)cudaFuncGetAttributes(&fa, pack_planes_kernel);
}

static int grid_for(int64_t work, int threads) {
    int64_t g = ceil_div(work, threads);
    if (g < 1) g = 1;
    if (g > 148 * 32) g = 148 * 32;
    return (int)g;
}

int launch_pack_planes(const uint32_t* words, int planes, int rows, int cols, void* out,
                       cudaStream_t st) {
    const int64_t total = (int64_t)planes * n_slices(cols) * n_row_tiles(rows) * 32;
    pack_planes_kernel<<<grid_for(total, 256), 256, 0, st>>>(words, planes, rows, cols,
                                                             static_cast<uint4*>(out));
    return (int)cudaGetLastError();
}

int launch_unpack_planes(const void* tiled, int planes, int rows, int cols, uint32_t* words,
                         cudaStream_t st) {
    const int64_t total = (int64_t)planes * n_slices(cols) * n_row_tiles(rows) * 32;
    unpack_planes_kernel<<<grid_for(total, 256), 256, 0, st>>>(static_cast<const uint4*>(tiled),
                                                               planes, rows, cols, words);
    return (int)cudaGetLastError();
}

int launch_pack_scales(const float* alpha, const float* offset, int p, int rows, int cols,
                       int scale_dtype, void* alpha_out, void* offset_out, cudaStream_t st) {
    const int64_t total = tiled_alpha_elems(rows, cols, p) + (offset ? tiled_offset_elems(rows, cols) : 0);
    if (scale_dtype == ABCQ_F16)
        pack_scales_kernel<__half><<<grid_for(total, 256), 256, 0, st>>>(
            alpha, offset, p, rows, cols, static_cast<__half*>(alpha_out), static_cast<__half*>(offset_out));
    else
        pack_scales_kernel<float><<<grid_for(total, 256), 256, 0, st>>>(
            alpha, offset, p, rows, cols, static_cast<float*>(alpha_out), static_cast<float*>(offset_out));
    return (int)cudaGetLastError();
}

int launch_lut_build(const void* x, int x_dtype, int cols, int mu, float* table, cudaStream_t st) {
    const int64_t total = ceil_div(cols, mu) << mu;
    if (x_dtype == ABCQ_F16)
        lut_build_kernel<__half><<<grid_for(total, 256), 256, 0, st>>>(static_cast<const __half*>(x), cols, mu, table);
    else
        lut_build_kernel<float><<<grid_for(total, 256), 256, 0, st>>>(static_cast<const float*>(x), cols, mu, table);
    return (int)cudaGetLastError();
}

}  // namespace abcq
