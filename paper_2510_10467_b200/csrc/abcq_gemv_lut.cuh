// abcq_gemv_lut.cuh -- sm_100a batch-1 bit-plane GEMV kernel (the hot path).
//
// Replaces GemvEngine.lut + LookupTable.build + _lut_kernel
// (/root/reference/pkg/src/anybcq/gemv.py:67-95,188-222):
//
//   y[n] = sum_{i<p} sum_g alpha^(p)[i,n,g] * s(i,n,g)   (+ offset^(p)[n,g] * gx[g])
//   s(i,n,g) = sum_{c in g} T[c][byte(i,n,c)]             (mu = 8 chunk table)
//
// Design:
//  * work item = (256-column slice s, 16-row tile rt); items are ordered
//    slice-major and split evenly over a one-wave grid; a CTA owns a
//    contiguous item range, which spans at most two slices ("slots").
//  * each CTA builds the reference lookup table of its slices in shared
//    memory: 32 chunks x 256 entries x f32 per slice in a [t][col] slab with
//    a 256-byte t-row (slot k = columns 32k..32k+31), so that
//        smem address = PRMT(weight word, lane column bytes) = t<<8 | col*4
//    costs ONE instruction per looked-up byte; the pack-time byte rotation
//    (abcq_pack.cu) puts the 32 lanes on 32 distinct banks. The slot is part
//    of the lane's column bytes, so one code path serves both slots.
//  * warps are assigned items of ONE slot each (items of a CTA split by slot,
//    round-robin within); a warp streams its (item, plane) elements -- p is
//    a runtime kernel argument -- in batches of kBatch 128-bit loads straight
//    to registers (24 warps/SM keep HBM busy). The first batch is issued before
//    the table build and before griddepcontrol.wait, so with programmatic
//    dependent launch it overlaps the previous kernel's tail.
//  * per element: 16 lookups summed with packed FADD2, one FFMA by alpha;
//    an asymmetric offset is one extra element (z * group sum of x).
//  * split over slices: each item writes a 16-row partial to an L2-resident
//    workspace; a small PDL-chained kernel sums the partials in a fixed
//    order (deterministic) and writes y.
#pragma once
#include "abcq_common.cuh"
#include "abcq_internal.h"

namespace abcq {

struct LutArgs {
    const uint4* planes;
    int64_t plane_stride_u4;  // uint4 units between planes
    const void* alpha;        // scale set p, tiled [item][lane][p]
    const void* offset;       // offsets of set p, tiled [item][lane] (ASYM)
    const void* x;
    void* y;
    float* partial;           // [NS][NRT*16]
    unsigned long long* trace;  // optional per-CTA phase timestamps (abcq_debug_set_trace)
    int rows, cols, NRT, NS, p, items;
    int q, rem;  // items per CTA: q (+1 for the first rem CTAs)
    int dbg_mode;  // profiling experiments only: 0 normal, 1 no lookups, 2 no weight loads
};

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define ABCQ_TRACE(k)                                                                   \
    do {                                                                                \
        if (a.trace && threadIdx.x == 0) a.trace[blockIdx.x * 8 + (k)] = globaltimer(); \
    } while (0)

constexpr int kWarps = 20;
constexpr int kThreads = kWarps * 32;
constexpr int kBatch = 8;               // elements in flight per warp
constexpr int kMaxFastP = ABCQ_MAX_PLANES;
constexpr int kTableBytes = 256 * 256;  // 256 t-rows x 64 cols x 4 B: two 32-col slots

// 16 lookups of one 16-byte lane block. rb[k] holds the column bytes of steps
// 3k..3k+2 in bytes 0..2 and a zero in byte 3 (-> address bytes 2, 3).
__device__ __forceinline__ float lut16(const uint4 w, const uint32_t (&rb)[6], const char* tbl) {
    const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
    unsigned long long acc[2] = {0ull, 0ull};
#pragma unroll
    for (int j = 0; j < 16; j += 2) {
        const uint32_t a0 = prmt(ww[j >> 2], rb[j / 3], 0x7700u | ((j & 3) << 4) | (4 + j % 3));
        const uint32_t a1 =
            prmt(ww[(j + 1) >> 2], rb[(j + 1) / 3], 0x7700u | (((j + 1) & 3) << 4) | (4 + (j + 1) % 3));
        const float v0 = *reinterpret_cast<const float*>(tbl + a0);
        const float v1 = *reinterpret_cast<const float*>(tbl + a1);
        acc[(j >> 1) & 1] = fadd2(acc[(j >> 1) & 1], pack2(v0, v1));
    }
    const float2 f = unpack2(fadd2(acc[0], acc[1]));
    return f.x + f.y;
}

template <typename XT>
__device__ __forceinline__ void load_x8(const XT* x, int k0, int cols, float (&xs)[8]) {
    if (k0 + 8 <= cols) {
        if constexpr (sizeof(XT) == 2) {
            const uint4 v = __ldg(reinterpret_cast<const uint4*>(x + k0));
            const __half2* h = reinterpret_cast<const __half2*>(&v);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const float2 f = __half22float2(h[j]);
                xs[2 * j] = f.x;
                xs[2 * j + 1] = f.y;
            }
        } else {
            const float4 a = __ldg(reinterpret_cast<const float4*>(x + k0));
            const float4 b = __ldg(reinterpret_cast<const float4*>(x + k0 + 4));
            xs[0] = a.x; xs[1] = a.y; xs[2] = a.z; xs[3] = a.w;
            xs[4] = b.x; xs[5] = b.y; xs[6] = b.z; xs[7] = b.w;
        }
    } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) xs[j] = (k0 + j < cols) ? to_f32<XT>(x[k0 + j]) : 0.f;
    }
}

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" :::); }

template <typename XT, typename YT, typename ST, bool ASYM>
__global__ void __launch_bounds__(kThreads, 1) gemv_lut_kernel(const LutArgs a) {
    extern __shared__ __align__(128) char smem[];
    float* csum = reinterpret_cast<float*>(smem + kTableBytes);         // [2][32] chunk sums (ASYM)
    XT* xs_smem = reinterpret_cast<XT*>(smem + kTableBytes + 256);       // x of the CTA's slices
    uint64_t* xbar = reinterpret_cast<uint64_t*>(smem + kTableBytes + 256 + 2 * kSliceCols * 4);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int p = a.p;
    ABCQ_TRACE(0);

    // ---- this CTA's items, split by slot; this warp's slot and item list ----
    const int b = blockIdx.x;
    const int it0 = b * a.q + min(b, a.rem);
    const int it1 = it0 + a.q + (b < a.rem ? 1 : 0);
    const int s0 = it0 / a.NRT;
    const int split = min((s0 + 1) * a.NRT, it1);  // items >= split belong to slot 1
    const int n0 = split - it0, n1 = it1 - split;
    int w0 = n1 == 0 ? kWarps : (n0 == 0 ? 0 : (kWarps * n0 + (it1 - it0) / 2) / (it1 - it0));
    if (n0 > 0 && w0 == 0) w0 = 1;
    if (n1 > 0 && w0 == kWarps) w0 = kWarps - 1;
    const int slot = warp < w0 ? 0 : 1;
    const int nw = slot == 0 ? w0 : kWarps - w0;          // warps sharing this slot
    const int wi = slot == 0 ? warp : warp - w0;          // index among them
    const int base = slot == 0 ? it0 : split;
    const int cnt = slot == 0 ? n0 : n1;
    const int M = wi < cnt ? (cnt - wi + nw - 1) / nw : 0;  // items of this warp: base + wi + nw*m
    const int sl = s0 + slot;                                // this warp's slice

    const ST* __restrict__ alpha = static_cast<const ST*>(a.alpha);
    const ST* __restrict__ offs = static_cast<const ST*>(a.offset);
    const int64_t istep = (int64_t)nw * 32;  // uint4 / lane-element stride between this warp's items

    // A block = up to kBatch items of this warp; one plane of a block is one
    // batch of kBatch 16-byte loads per lane.
    uint4 w[kBatch];
    ST sc[kBatch];
    auto load_plane = [&](int m0, int nval, int i) {
        const uint4* src = a.planes + i * a.plane_stride_u4 + (base + wi + (int64_t)nw * m0) * 32 + lane;
        const ST* sp = alpha + ((base + wi + (int64_t)nw * m0) * 32 + lane) * p + i;
#pragma unroll
        for (int k = 0; k < kBatch; ++k) {
            if (k < nval) {
                if (a.dbg_mode == 2)
                    w[k] = make_uint4(lane * 0x01010101u * (k + i), lane, k, i);
                else
                    w[k] = ldg_stream(src + k * istep);
                sc[k] = sp[k * istep * p];
            }
        }
    };

    // static model data, before the PDL wait: the TMA engine streams this CTA's
    // whole weight range (contiguous per plane) and its scale range into L2,
    // decoupling HBM streaming from the warps' load/consume cycles; then each
    // warp issues its first batch.
    if (tid <= p) {
        const int64_t nit = it1 - it0;
        if (tid < p)
            prefetch_l2_range(a.planes + tid * a.plane_stride_u4 + (int64_t)it0 * 32, nit * kBlockBytes);
        else
            prefetch_l2_range(alpha + (int64_t)it0 * 32 * p, nit * 32 * p * (int64_t)sizeof(ST));
    }
    if (M > 0) load_plane(0, min(M, kBatch), 0);
    if (tid == 0) {
        mbar_init(xbar, 1);
        fence_mbar_init();
    }
    ABCQ_TRACE(1);
    pdl_wait();
    pdl_launch_dependents();
    ABCQ_TRACE(2);

    // ---- x of this CTA's slices: one TMA bulk copy (does not queue behind the
    //      weight loads in the LSU), then the reference lookup tables ----------
    const XT* __restrict__ x = static_cast<const XT*>(a.x);
    const int nslots = n1 > 0 ? 2 : 1;
    const int k0 = s0 * kSliceCols;
    const int ncols = min(nslots * kSliceCols, a.cols - k0);
    const bool tma_x = (ncols * (int)sizeof(XT)) % 16 == 0;
    __syncthreads();  // mbarrier initialised
    if (tma_x && tid == 0) {
        mbar_arrive_expect_tx(xbar, ncols * sizeof(XT));
        bulk_g2s(xs_smem, x + k0, ncols * sizeof(XT), xbar);
    }
    if (tma_x) mbar_wait(xbar, 0);
    for (int task = tid; task < nslots * 32 * 16; task += kThreads) {
        const int ts = task >> 9, c = task & 31, hi = (task >> 5) & 15;
        float xv[8];
        const int kk = ts * kSliceCols + 8 * c;  // relative to k0
        if (tma_x) {
#pragma unroll
            for (int j = 0; j < 8; ++j) xv[j] = kk + j < ncols ? to_f32<XT>(xs_smem[kk + j]) : 0.f;
        } else {
            load_x8<XT>(x, k0 + kk, a.cols, xv);
        }
        float e[16];
        lut_chunk_entries16(xv, hi, e);
        float* col = reinterpret_cast<float*>(smem) + ts * 32 + c;
#pragma unroll
        for (int t = 0; t < 16; ++t) col[(hi * 16 + t) * 64] = e[t];
        if (ASYM && hi == 15) csum[ts * 32 + c] = e[15];  // T[255] = chunk sum
    }
    __syncthreads();
    ABCQ_TRACE(3);

    // lane column bytes for the 16 lookup steps (rotation r = lane & 15)
    const int half = lane >> 4, r = lane & 15;
    uint32_t rb[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) {
        uint32_t v = 0;
#pragma unroll
        for (int bb = 0; bb < 3; ++bb) {
            const int j = 3 * k + bb;
            if (j < 16) v |= (uint32_t)((slot * 32 + half * 16 + ((j + r) & 15)) * 4) << (8 * bb);
        }
        rb[k] = v;
    }
    float gx = 0.f;
    if constexpr (ASYM) {
        for (int c = 0; c < 16; ++c) gx += csum[slot * 32 + half * 16 + c];
    }

    // ---- stream this warp's items: per block of kBatch items, a runtime loop
    //      over the p planes, one batch of loads per plane --------------------
    YT* __restrict__ y = static_cast<YT*>(a.y);
    const int64_t pstride = (int64_t)a.NRT * kTileRows;
    for (int m0 = 0; m0 < M; m0 += kBatch) {
        const int nval = min(M - m0, kBatch);
        float acc[kBatch];
#pragma unroll
        for (int k = 0; k < kBatch; ++k) acc[k] = 0.f;
        for (int i = 0; i < p; ++i) {
            if (m0 > 0 || i > 0) load_plane(m0, nval, i);
#pragma unroll
            for (int k = 0; k < kBatch; ++k)
                if (k < nval) {
                    if (a.dbg_mode == 1)
                        acc[k] = fmaf(to_f32<ST>(sc[k]), (float)(w[k].x ^ w[k].y ^ w[k].z ^ w[k].w), acc[k]);
                    else
                        acc[k] = fmaf(to_f32<ST>(sc[k]), lut16(w[k], rb, smem), acc[k]);
                }
        }
        if constexpr (ASYM) {
            const ST* zp = offs + (base + wi + (int64_t)nw * m0) * 32 + lane;
#pragma unroll
            for (int k = 0; k < kBatch; ++k)
                if (k < nval) acc[k] = fmaf(to_f32<ST>(zp[k * istep]), gx, acc[k]);
        }
        // combine the slice's two groups (lanes l, l+16) and emit 16 rows per item
#pragma unroll
        for (int k = 0; k < kBatch; ++k) {
            if (k < nval) {
                const float out = acc[k] + __shfl_down_sync(0xffffffffu, acc[k], 16);
                const int row = (base + wi + nw * (m0 + k) - sl * a.NRT) * kTileRows + lane;
                if (lane < 16) {
                    if (a.NS == 1) {
                        if (row < a.rows) y[row] = from_f32<YT>(out);
                    } else {
                        __stcg(a.partial + sl * pstride + row, out);
                    }
                }
            }
        }
    }
    if (warp == 0) ABCQ_TRACE(4);
}

// Split-K completion (NS > 1): y[n] = sum_s partial[s][n] in a fixed order
// (four interleaved chains over ascending s, then (c0 + c1) + (c2 + c3)),
// so results are bitwise reproducible. Launched with PDL right after the
// GEMV kernel; it waits for the GEMV grid inside griddepcontrol.wait.
template <typename YT>
__global__ void __launch_bounds__(256) split_reduce_kernel(const float* __restrict__ partial, int NS,
                                                           int64_t stride, int rows, YT* __restrict__ y) {
    pdl_wait();
    pdl_launch_dependents();
    for (int row = blockIdx.x * blockDim.x + threadIdx.x; row < rows; row += gridDim.x * blockDim.x) {
        const float* pp = partial + row;
        float c[4] = {0.f, 0.f, 0.f, 0.f};
        int s = 0;
        for (; s + 4 <= NS; s += 4) {
#pragma unroll
            for (int k = 0; k < 4; ++k) c[k] += __ldcg(pp + (s + k) * stride);
        }
        for (int k = 0; s + k < NS; ++k) c[k] += __ldcg(pp + (s + k) * stride);
        y[row] = from_f32<YT>((c[0] + c[1]) + (c[2] + c[3]));
    }
}

template <typename XT, typename YT, typename ST, bool ASYM>
inline int launch_t(const LutArgs& a, int grid, cudaStream_t st) {
    auto kern = gemv_lut_kernel<XT, YT, ST, ASYM>;
    const int smem = kTableBytes + 256 + 2 * kSliceCols * 4 + 16;
    int dev = 0;
    cudaGetDevice(&dev);
    static bool attr_set[64] = {};  // per instantiation and device
    if (dev < 64 && !attr_set[dev]) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return (int)e;
        attr_set[dev] = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, a);
    if (e != cudaSuccess || a.NS == 1) return (int)e;
    cudaLaunchConfig_t rc = cfg;
    rc.blockDim = dim3(256);
    rc.gridDim = dim3((unsigned)ceil_div(a.rows, 256));
    rc.dynamicSmemBytes = 0;
    return (int)cudaLaunchKernelEx(&rc, split_reduce_kernel<YT>, (const float*)a.partial, a.NS,
                                   (int64_t)a.NRT * kTileRows, a.rows, static_cast<YT*>(a.y));
}

template <typename XT, typename YT, typename ST>
inline int launch_asym(const LutArgs& a, bool asym, int grid, cudaStream_t st) {
    return asym ? launch_t<XT, YT, ST, true>(a, grid, st) : launch_t<XT, YT, ST, false>(a, grid, st);
}
template <typename XT, typename YT>
inline int launch_st(const LutArgs& a, int sd, bool asym, int grid, cudaStream_t st) {
    return sd == ABCQ_F16 ? launch_asym<XT, YT, __half>(a, asym, grid, st)
                          : launch_asym<XT, YT, float>(a, asym, grid, st);
}

// one explicit instantiation unit per (x dtype, y dtype): abcq_gemv_lut_x?y?.cu
template <typename XT, typename YT>
int launch_lut_xy(const LutArgs& a, int sd, bool asym, int grid, cudaStream_t st);
template <> int launch_lut_xy<__half, __half>(const LutArgs&, int, bool, int, cudaStream_t);
template <> int launch_lut_xy<__half, float>(const LutArgs&, int, bool, int, cudaStream_t);
template <> int launch_lut_xy<float, __half>(const LutArgs&, int, bool, int, cudaStream_t);
template <> int launch_lut_xy<float, float>(const LutArgs&, int, bool, int, cudaStream_t);

}  // namespace abcq
