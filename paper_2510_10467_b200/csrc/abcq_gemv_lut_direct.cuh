// abcq_gemv_lut_direct.cuh -- register-direct variant of the batch-1 LUT GEMV.
//
// Same math, layout and tables as abcq_gemv_lut.cuh; differs in how weights
// reach the lookups: the TMA engine prefetches the CTA's (contiguous) weight
// and scale ranges into L2 (cp.async.bulk.prefetch.L2), and warps load their
// 16-byte lane blocks straight into registers (no shared-memory staging, so
// the shared-memory port only serves table lookups). Each warp keeps one
// batch of kDBatch loads in flight; 20 warps per SM hide the L2 latency.
#pragma once
#include "abcq_gemv_lut.cuh"

namespace abcq {

constexpr int kDWarps = 20;
constexpr int kDThreads = kDWarps * 32;
constexpr int kDBatch = 8;

template <typename ST, bool ASYM>
constexpr int lut_direct_smem_bytes() {
    return kTableBytes + kXBytes + 256;
}

template <typename XT, typename YT, typename ST, bool ASYM>
__global__ void __launch_bounds__(kDThreads, 1) gemv_lut_direct_kernel(const LutArgs a) {
    extern __shared__ __align__(128) char smem[];
    float* xs_smem = reinterpret_cast<float*>(smem + kTableBytes);
    float* csum = reinterpret_cast<float*>(smem + kTableBytes + kXBytes);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int p = a.p;
    ABCQ_TRACE(0);

    // ---- this CTA's items, split by segment; this warp's segment and items --
    const int b = blockIdx.x;
    const int it0 = b * a.q + min(b, a.rem);
    const int it1 = it0 + a.q + (b < a.rem ? 1 : 0);
    const int s0 = it0 / a.NRT;
    const int split = min((s0 + 1) * a.NRT, it1);
    const int n0 = split - it0, n1 = it1 - split;
    int w0 = n1 == 0 ? kDWarps : (n0 == 0 ? 0 : (kDWarps * n0 + (it1 - it0) / 2) / (it1 - it0));
    if (n0 > 0 && w0 == 0) w0 = 1;
    if (n1 > 0 && w0 == kDWarps) w0 = kDWarps - 1;
    const int seg = warp < w0 ? 0 : 1;
    const int nw = seg == 0 ? w0 : kDWarps - w0;
    const int wi = seg == 0 ? warp : warp - w0;
    const int base = seg == 0 ? it0 : split;
    const int cnt = seg == 0 ? n0 : n1;
    const int M = wi < cnt ? (cnt - wi + nw - 1) / nw : 0;  // items base + wi + nw*m
    const int sl = s0 + seg;

    const ST* __restrict__ alpha = static_cast<const ST*>(a.alpha);
    const ST* __restrict__ offs = static_cast<const ST*>(a.offset);

    // static model data, before the PDL wait: the TMA engine streams the CTA's
    // weight and scale ranges HBM -> L2 at full rate, independent of the warps
    if (tid < 2 * p + 1) {
        const int64_t nit = it1 - it0;
        if (tid < p)
            prefetch_l2_range(a.planes + tid * a.plane_stride_u4 + (int64_t)it0 * 32, nit * kBlockBytes);
        else if (tid < 2 * p)
            prefetch_l2_range(alpha + ((int64_t)(tid - p) * a.items + it0) * 32, nit * 32 * (int64_t)sizeof(ST));
        else if (ASYM)
            prefetch_l2_range(offs + (int64_t)it0 * 32, nit * 32 * (int64_t)sizeof(ST));
    }
    ABCQ_TRACE(1);
    pdl_wait();
    pdl_launch_dependents();
    ABCQ_TRACE(2);

    // ---- x -> smem, then the lookup tables (x loads go out before any weight
    //      load, so they do not queue behind them in the LSU) ----------------
    const XT* __restrict__ x = static_cast<const XT*>(a.x);
    const int nseg = n1 > 0 ? 2 : 1;
    const int k0 = s0 * kSliceCols;
    if (tid < nseg * 32) {
        float xv[8];
        load_x8<XT>(x, k0 + 8 * tid, a.cols, xv);
#pragma unroll
        for (int j = 0; j < 8; ++j) xs_smem[8 * tid + j] = xv[j];
    }
    __syncthreads();
    for (int task = tid; task < nseg * 32 * 16; task += kDThreads) {
        const int ts = task >> 9, c = task & 31, hi = (task >> 5) & 15;
        float xv[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) xv[j] = xs_smem[ts * kSliceCols + 8 * c + j];
        float e[16];
        lut_chunk_entries16(xv, hi, e);
        float* col = reinterpret_cast<float*>(smem) + ts * 32 + c;
#pragma unroll
        for (int t = 0; t < 16; ++t) col[(hi * 16 + t) * 64] = e[t];
        if (ASYM && hi == 15) csum[ts * 32 + c] = e[15];
    }
    __syncthreads();
    ABCQ_TRACE(3);

    const int half = lane >> 4, r = lane & 15;
    uint32_t rb[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) {
        uint32_t v = 0;
#pragma unroll
        for (int bb = 0; bb < 3; ++bb) {
            const int j = 3 * k + bb;
            if (j < 16) v |= (uint32_t)((seg * 32 + half * 16 + ((j + r) & 15)) * 4) << (8 * bb);
        }
        rb[k] = v;
    }
    float gx = 0.f;
    if constexpr (ASYM) {
        for (int c = 0; c < 16; ++c) gx += csum[seg * 32 + half * 16 + c];
    }

    // ---- stream: per block of kDBatch items, a runtime loop over the planes --
    YT* __restrict__ y = static_cast<YT*>(a.y);
    const int64_t pstride = (int64_t)a.NRT * kTileRows;
    const int64_t istep = (int64_t)nw * 32;
    uint4 w[kDBatch];
    ST sc[kDBatch];
    for (int m0 = 0; m0 < M; m0 += kDBatch) {
        const int nval = min(M - m0, kDBatch);
        const int64_t item0 = base + wi + (int64_t)nw * m0;
        float acc[kDBatch];
#pragma unroll
        for (int k = 0; k < kDBatch; ++k) acc[k] = 0.f;
        for (int i = 0; i < p; ++i) {
            const uint4* src = a.planes + i * a.plane_stride_u4 + item0 * 32 + lane;
            const ST* sp = alpha + ((int64_t)i * a.items + item0) * 32 + lane;
#pragma unroll
            for (int k = 0; k < kDBatch; ++k) {
                if (k < nval) {
                    w[k] = ldg_stream(src + k * istep);
                    sc[k] = sp[k * istep];
                }
            }
#pragma unroll
            for (int k = 0; k < kDBatch; ++k)
                if (k < nval) acc[k] = fmaf(to_f32<ST>(sc[k]), lut16<0>(w[k], rb, smem), acc[k]);
        }
        if constexpr (ASYM) {
            const ST* zp = offs + item0 * 32 + lane;
#pragma unroll
            for (int k = 0; k < kDBatch; ++k)
                if (k < nval) acc[k] = fmaf(to_f32<ST>(zp[k * istep]), gx, acc[k]);
        }
#pragma unroll
        for (int k = 0; k < kDBatch; ++k) {
            if (k < nval) {
                const float out = acc[k] + __shfl_down_sync(0xffffffffu, acc[k], 16);
                const int row = (int)(item0 + k * nw - sl * a.NRT) * kTileRows + lane;
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

template <typename XT, typename YT, typename ST, bool ASYM>
int launch_direct_t(const LutArgs& a, int grid, cudaStream_t st) {
    auto kern = gemv_lut_direct_kernel<XT, YT, ST, ASYM>;
    constexpr int smem = lut_direct_smem_bytes<ST, ASYM>();
    int dev = 0;
    cudaGetDevice(&dev);
    static bool attr_set[64] = {};
    if (dev < 64 && !attr_set[dev]) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return (int)e;
        attr_set[dev] = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kDThreads);
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
    rc.blockDim = dim3(64);
    rc.gridDim = dim3((unsigned)ceil_div(a.rows, 64));
    rc.dynamicSmemBytes = 0;
    return (int)cudaLaunchKernelEx(&rc, split_reduce_kernel<YT>, (const float*)a.partial, a.NS,
                                   (int64_t)a.NRT * kTileRows, a.rows, static_cast<YT*>(a.y), a.trace);
}

}  // namespace abcq
