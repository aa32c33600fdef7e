// abcq_gemv_lut.cu -- sm_100a batch-1 bit-plane GEMV (the hot path).
//
// Replaces GemvEngine.lut + LookupTable.build + _lut_kernel
// (/root/reference/pkg/src/anybcq/gemv.py:67-95,188-222):
//
//   y[n] = sum_{i<p} sum_g alpha^(p)[i,n,g] * s(i,n,g)   (+ offset^(p)[n,g] * gx[g])
//   s(i,n,g) = sum_{c in g} T[c][byte(i,n,c)]             (mu = 8 chunk table)
//
// Design:
//  * work item = (256-col slice s, 16-row tile rt); items are ordered
//    slice-major and split evenly over a one-wave grid; every CTA owns a
//    contiguous item range, which spans at most two slices.
//  * each CTA builds the reference lookup table of its (<= 2) slices in
//    shared memory -- 32 chunks x 256 entries x f32 per slice, layout
//    [t][col] with a 256-byte t-row so that
//        address = PRMT(weight word, lane column bytes)  (= t<<8 | col*4)
//    costs ONE instruction per looked-up byte, and the pack-time byte
//    rotation (abcq_pack.cu) puts the 32 lanes on 32 distinct banks.
//  * weights never transit shared memory: 128-bit streaming loads straight
//    to registers, DEPTH elements in flight per warp, issued before the table
//    build so the build hides under the first DRAM round trip.
//  * per (plane, row, group): 16 lookups summed with packed FADD2, then one
//    FFMA by alpha; asymmetric offsets are one extra "element" per item.
//  * split over slices: each item writes a 16-row partial to an L2-resident
//    workspace; the last arriving warp of a row tile (per-tile counter) sums
//    the partials in fixed slice order (deterministic) and writes y.
#include "abcq_common.cuh"
#include "abcq_internal.h"

namespace abcq {

struct LutArgs {
    const uint4* planes;
    int64_t plane_stride_u4;  // uint4 units between planes
    const void* alpha;        // scale set p, tiled
    const void* offset;       // offsets of set p, tiled (ASYM)
    const void* x;
    void* y;
    float* partial;           // [NS][NRT*16]
    uint32_t* counters;       // [NRT]
    int rows, cols, NRT, NS, p, items;
};

constexpr int kWarps = 16;
constexpr int kDepth = 8;
constexpr int kTableBytes = 256 * 256;  // 256 t-rows x 64 cols x 4 B: two 32-col slots

// 16 lookups of one 16-byte lane block against table slot SLOT
template <int SLOT>
__device__ __forceinline__ float lut16(const uint4 w, const uint32_t (&rb)[4], const char* tbl) {
    const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
    unsigned long long acc[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        acc[h] = 0ull;
#pragma unroll
        for (int qq = 0; qq < 2; ++qq) {
            const int q = 2 * h + qq;
#pragma unroll
            for (int b = 0; b < 4; b += 2) {
                // byte0 <- lane column byte b of rb[q], byte1 <- weight byte b, bytes2,3 <- 0
                const uint32_t a0 = prmt(ww[q], rb[q], 0xCC00u | (b << 4) | (4 + b));
                const uint32_t a1 = prmt(ww[q], rb[q], 0xCC00u | ((b + 1) << 4) | (5 + b));
                const float v0 = *reinterpret_cast<const float*>(tbl + a0 + SLOT * 128);
                const float v1 = *reinterpret_cast<const float*>(tbl + a1 + SLOT * 128);
                acc[h] = fadd2(acc[h], pack2(v0, v1));
            }
        }
    }
    const float2 f = unpack2(fadd2(acc[0], acc[1]));
    return f.x + f.y;
}

template <typename XT>
__device__ __forceinline__ void load_x8(const XT* x, int k0, int cols, float xs[8]) {
#pragma unroll
    for (int j = 0; j < 8; ++j) xs[j] = (k0 + j < cols) ? to_f32<XT>(x[k0 + j]) : 0.f;
}

template <typename XT, typename YT, typename ST, bool ASYM>
__global__ void __launch_bounds__(kWarps * 32, 1) gemv_lut_kernel(const LutArgs a) {
    extern __shared__ __align__(128) char smem[];
    char* tbl = smem;                                          // kTableBytes
    float* csum = reinterpret_cast<float*>(smem + kTableBytes);  // [2][32] chunk sums (ASYM)

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int G = gridDim.x;
    const int it0 = (int)((int64_t)blockIdx.x * a.items / G);
    const int it1 = (int)((int64_t)(blockIdx.x + 1) * a.items / G);
    if (it0 >= it1) return;
    const int s0 = it0 / a.NRT;
    const int s1 = (it1 - 1) / a.NRT;  // == s0 or s0 + 1 (grid >= NS)
    const int split = (s0 + 1) * a.NRT;

    const int EP = a.p + (ASYM ? 1 : 0);  // elements per item
    const int first = it0 + warp;
    const int M = first < it1 ? (it1 - first + kWarps - 1) / kWarps : 0;
    const int E = M * EP;

    const uint4* __restrict__ planes = a.planes;
    const ST* __restrict__ alpha = static_cast<const ST*>(a.alpha);
    const ST* __restrict__ offs = static_cast<const ST*>(a.offset);

    // ---- element ring: issue the first DEPTH loads before building tables --
    uint4 wbuf[kDepth];
    ST sbuf[kDepth];
    int lm = 0, li = 0;  // load cursor (item, element)
    auto issue = [&](uint4& wd, ST& sd) {
        const int item = first + kWarps * lm;
        if (!ASYM || li < a.p) {
            wd = ldg_stream(planes + li * a.plane_stride_u4 + (int64_t)item * 32 + lane);
            sd = alpha[((int64_t)item * a.p + li) * 32 + lane];
        } else {
            sd = offs[(int64_t)item * 32 + lane];
        }
        if (++li == EP) { li = 0; ++lm; }
    };
#pragma unroll
    for (int d = 0; d < kDepth; ++d)
        if (d < E) issue(wbuf[d], sbuf[d]);

    // ---- build the lookup table(s): slot k holds slice s0 + k ---------------
    const XT* __restrict__ x = static_cast<const XT*>(a.x);
    const int nslots = (s1 != s0) ? 2 : 1;
    for (int slot = 0; slot < nslots; ++slot) {
        const int s = s0 + slot;
        for (int task = tid; task < 32 * 16; task += kWarps * 32) {
            const int c = task & 31, hi = task >> 5;
            float xs[8];
            load_x8<XT>(x, s * kSliceCols + 8 * c, a.cols, xs);
            float e[16];
            lut_chunk_entries16(xs, hi, e);
            float* col = reinterpret_cast<float*>(tbl) + slot * 32 + c;
#pragma unroll
            for (int t = 0; t < 16; ++t) col[(hi * 16 + t) * 64] = e[t];
            if (ASYM && hi == 15) csum[slot * 32 + c] = e[15];  // T[255] = chunk sum
        }
    }
    __syncthreads();

    // lane constants: column bytes for the 16 lookup steps (rotation r = lane & 15)
    const int half = lane >> 4, r = lane & 15;
    uint32_t rb[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        uint32_t v = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b) v |= (uint32_t)((half * 16 + ((4 * q + b + r) & 15)) * 4) << (8 * b);
        rb[q] = v;
    }
    float gx[2] = {0.f, 0.f};
    if (ASYM) {
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            float v = 0.f;
            for (int c = 0; c < 16; ++c) v += csum[k * 32 + half * 16 + c];
            gx[k] = v;
        }
    }

    // ---- main loop over this warp's elements --------------------------------
    YT* __restrict__ y = static_cast<YT*>(a.y);
    int cm = 0, ci = 0;  // consume cursor
    float yacc = 0.f;
    for (int e0 = 0; e0 < E; e0 += kDepth) {
#pragma unroll
        for (int d = 0; d < kDepth; ++d) {
            const int e = e0 + d;
            if (e < E) {
                const int item = first + kWarps * cm;
                const bool slot1 = item >= split;
                const float sc = to_f32<ST>(sbuf[d]);
                if (!ASYM || ci < a.p) {
                    const float s = slot1 ? lut16<1>(wbuf[d], rb, tbl) : lut16<0>(wbuf[d], rb, tbl);
                    yacc = fmaf(sc, s, yacc);
                } else {
                    yacc = fmaf(sc, slot1 ? gx[1] : gx[0], yacc);
                }
                if (e + kDepth < E) issue(wbuf[d], sbuf[d]);
                if (++ci == EP) {
                    // item done: combine the two groups of the slice, emit 16 rows
                    const float v = yacc + __shfl_down_sync(0xffffffffu, yacc, 16);
                    yacc = 0.f;
                    const int s = slot1 ? s1 : s0;
                    const int rt = item - s * a.NRT;
                    if (lane < 16) {
                        const int row = rt * kTileRows + lane;
                        if (a.NS == 1) {
                            if (row < a.rows) y[row] = from_f32<YT>(v);
                        } else {
                            a.partial[(int64_t)s * a.NRT * kTileRows + row] = v;
                        }
                    }
                    ci = 0;
                    ++cm;
                }
            }
        }
    }
    if (a.NS == 1 || M == 0) return;

    // ---- split-K completion: last arriving warp of a row tile reduces it ----
    __threadfence();
    __syncwarp();
    for (int mb = 0; mb < M; mb += 32) {
        const int m = mb + lane;
        bool won = false;
        int rt = 0;
        if (m < M) {
            const int item = first + kWarps * m;
            rt = item - (item >= split ? s1 : s0) * a.NRT;
            won = atomicAdd(&a.counters[rt], 1u) == (uint32_t)(a.NS - 1);
        }
        unsigned mask = __ballot_sync(0xffffffffu, won);
        while (mask) {
            const int src = __ffs(mask) - 1;
            mask &= mask - 1;
            const int rtw = __shfl_sync(0xffffffffu, rt, src);
            __threadfence();
            const int row = rtw * kTileRows + r;
            const float* pp = a.partial + row;
            const int64_t stride = (int64_t)a.NRT * kTileRows;
            float v0 = 0.f, v1 = 0.f;
            int s = half;
            for (; s + 2 < a.NS; s += 4) {  // fixed order: even/odd slices, ascending
                v0 += __ldcg(pp + s * stride);
                v1 += __ldcg(pp + (s + 2) * stride);
            }
            if (s < a.NS) v0 += __ldcg(pp + s * stride);
            float v = v0 + v1;
            v += __shfl_down_sync(0xffffffffu, v, 16);
            if (lane < 16 && row < a.rows) y[row] = from_f32<YT>(v);
            if (lane == 0) a.counters[rtw] = 0u;
        }
    }
}

size_t lut_workspace_bytes(const abcq_model_t* m) {
    const int NRT = n_row_tiles(m->rows), NS = n_slices(m->cols);
    if (NS <= 1) return 0;
    return (size_t)NS * NRT * kTileRows * sizeof(float) + (size_t)NRT * sizeof(uint32_t);
}

template <typename XT, typename YT, typename ST, bool ASYM>
static int launch_t(const LutArgs& a, int grid, cudaStream_t st) {
    auto kern = gemv_lut_kernel<XT, YT, ST, ASYM>;
    const int smem = kTableBytes + 2 * 32 * (int)sizeof(float);
    static bool attr_set = false;  // per instantiation
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return (int)e;
        attr_set = true;
    }
    kern<<<grid, kWarps * 32, smem, st>>>(a);
    return (int)cudaGetLastError();
}

template <typename XT, typename YT, typename ST>
static int launch_asym(const LutArgs& a, bool asym, int grid, cudaStream_t st) {
    return asym ? launch_t<XT, YT, ST, true>(a, grid, st) : launch_t<XT, YT, ST, false>(a, grid, st);
}
template <typename XT, typename YT>
static int launch_st(const LutArgs& a, int sd, bool asym, int grid, cudaStream_t st) {
    return sd == ABCQ_F16 ? launch_asym<XT, YT, __half>(a, asym, grid, st)
                          : launch_asym<XT, YT, float>(a, asym, grid, st);
}
template <typename XT>
static int launch_yt(const LutArgs& a, int yd, int sd, bool asym, int grid, cudaStream_t st) {
    return yd == ABCQ_F16 ? launch_st<XT, __half>(a, sd, asym, grid, st)
                          : launch_st<XT, float>(a, sd, asym, grid, st);
}

int launch_gemv_lut(const abcq_model_t* m, int p, const void* x, int x_dtype, void* y, int y_dtype,
                    void* ws, cudaStream_t st) {
    LutArgs a;
    a.rows = m->rows;
    a.cols = m->cols;
    a.NRT = n_row_tiles(m->rows);
    a.NS = n_slices(m->cols);
    a.p = p;
    a.items = a.NRT * a.NS;
    a.planes = static_cast<const uint4*>(m->planes);
    a.plane_stride_u4 = m->plane_stride_bytes / 16;
    a.alpha = m->alpha[p];
    a.offset = m->asymmetric ? m->offset[p] : nullptr;
    a.x = x;
    a.y = y;
    a.partial = static_cast<float*>(ws);
    a.counters = ws ? reinterpret_cast<uint32_t*>(static_cast<char*>(ws) +
                                                  (size_t)a.NS * a.NRT * kTileRows * sizeof(float))
                    : nullptr;
    int grid = num_sms();
    if (grid < a.NS) grid = a.NS;      // keeps every CTA within <= 2 slices
    if (grid > a.items) grid = a.items;
    const bool asym = m->asymmetric != 0;
    return x_dtype == ABCQ_F16 ? launch_yt<__half>(a, y_dtype, m->scale_dtype, asym, grid, st)
                               : launch_yt<float>(a, y_dtype, m->scale_dtype, asym, grid, st);
}

}  // namespace abcq
