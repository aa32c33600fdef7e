// abcq_gemm_mixedp.cu -- small-batch (B <= 16) bit-plane GEMM with a
// per-request precision p_b, on the tensor cores (mma.sync m16n8k16, f16 in,
// f32 accumulate).
//
// Reference semantics: the CLI `gemv` loops GemvEngine.lut over the rows of x
// (/root/reference/pkg/src/anybcq/cli.py:122-126) and the service serves one
// precision per request (service/server.py:188-206); this kernel computes all
// requests in one pass over the planes:
//   Y[b][n] = sum_{i < p_b} sum_g alpha^(p_b)[i,n,g] * sum_{k in g} s_i[n,k] X[b][k]
//             (+ offset^(p_b)[n,g] * sum_{k in g} X[b][k])
// Each plane is read ONCE for the whole batch (planes up to max p_b); plane i's
// per-group partial sums are shared by every request with p_b > i and scaled by
// that request's own scale set (scale sets differ per precision,
// progressive.py:32-79).
//
// Mapping: Y^T (requests x rows) = X (requests x K) . W^T. A = X fragment
// (16 requests x 16 k, fp16, kept in registers for the warp's slice); B = the
// sign bits of 8 weight rows, expanded to +-1 fp16 through a 16-entry nibble
// table in shared memory (a lane's B fragment is one nibble per row and
// k-step); C = 16 requests x 8 rows, reset per 128-column group, scaled by
// alpha^(p_b) and accumulated. Weight blocks (tiled layout, rotated bytes) are
// un-rotated through a per-warp shared-memory scratch.
// This is a dense contraction (2*B flops per weight bit), hence tensor cores;
// the batch-1 path is the LUT kernel.
#include "abcq_common.cuh"
#include "abcq_internal.h"

namespace abcq {

constexpr int kGWarps = 8;
constexpr int kMaxBatch = 16;
constexpr int kMaxStagePlanes = 4;  // planes staged per item (p_max > 4 loads the rest in rounds)
constexpr int kMaxSets = 4;         // distinct precisions whose scales are staged with the planes

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(smem_dst)),
                 "l"(src)
                 : "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

struct GemmArgs {
    const uint4* planes;
    int64_t plane_stride_u4;
    const void* alpha[ABCQ_MAX_PLANES + 1];   // scale set per precision (tiled [i][item][lane])
    const void* offset[ABCQ_MAX_PLANES + 1];  // offsets per precision (asymmetric)
    const __half* x;  // (B, cols) fp16
    float* partial;   // [NS][B][NRT*16]
    int p_of[kMaxBatch];
    int set_of[kMaxBatch];  // request -> index of its precision in pset (-1: not staged)
    int pset[kMaxSets];     // distinct precisions of the batch (first kMaxSets)
    int npset;
    int rows, cols, NRT, NS, items, B, pmax;
};

// dynamic shared memory of the GEMM kernel
struct GemmSmem {
    uint4 stage[kGWarps][2][kMaxStagePlanes][32];              // plane blocks, double-buffered
    uint4 sc[kGWarps][2][kMaxStagePlanes][kMaxSets][8];         // their scales (<= 128 B per set)
    unsigned char scratch[kGWarps][512];                        // per-warp un-rotated block
};

__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

template <typename ST, bool ASYM>
__global__ void __launch_bounds__(kGWarps * 32) gemm_mixedp_kernel(const GemmArgs a) {
    __shared__ __align__(16) uint2 nib_tab[16];  // nibble -> {half2, half2}
    // per-warp double buffer of an item's plane blocks and their scales, filled
    // with cp.async (group-tracked, so the next item streams in while this one
    // computes)
    extern __shared__ __align__(16) char gsmem[];
    GemmSmem& S = *reinterpret_cast<GemmSmem*>(gsmem);
    auto& stage = S.stage;
    auto& scratch = S.scratch;

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x < 16) {
        const int n = threadIdx.x;
        auto h = [](int bit) -> uint32_t { return bit ? 0x3C00u : 0xBC00u; };  // +1 / -1 in fp16
        nib_tab[n] = make_uint2(h(n & 1) | (h((n >> 1) & 1) << 16), h((n >> 2) & 1) | (h((n >> 3) & 1) << 16));
    }
    __syncthreads();

    const int g = lane >> 2, t = lane & 3;
    const int gw = blockIdx.x * kGWarps + warp, W = gridDim.x * kGWarps;
    // this warp's slice and row tiles: warps cycle over slices first
    const int s = gw % a.NS;
    const int wps = W / a.NS + (gw % a.NS < W % a.NS ? 1 : 0);  // warps on slice s
    const int widx = gw / a.NS;
    if (widx >= a.NRT) return;
    const int B = a.B;

    // A fragments (X) of the whole 256-column slice: 16 k-steps x 4 regs
    uint32_t xa[16][4];
    float gxs[2][2];  // per group: sum of x over the group for requests g, g+8 (asymmetric)
    {
        const int k0 = s * kSliceCols;
#pragma unroll
        for (int ks = 0; ks < 16; ++ks) {
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int req = g + ((r & 1) ? 8 : 0);
                const int k = k0 + ks * 16 + 2 * t + ((r & 2) ? 8 : 0);
                uint32_t v = 0;
                if (req < B) {
                    const __half* xp = a.x + (int64_t)req * a.cols + k;
                    if (k + 1 < a.cols && (a.cols & 1) == 0) {
                        v = __ldg(reinterpret_cast<const unsigned int*>(xp));  // (k, k+1) as one 32-bit load
                    } else {
                        const __half lo = k < a.cols ? xp[0] : __float2half(0.f);
                        const __half hi = k + 1 < a.cols ? xp[1] : __float2half(0.f);
                        v = (uint32_t)__half_as_ushort(lo) | ((uint32_t)__half_as_ushort(hi) << 16);
                    }
                }
                xa[ks][r] = v;
            }
        }
        if (ASYM) {
#pragma unroll
            for (int gg = 0; gg < 2; ++gg)
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    const int req = g + 8 * q;
                    float sum = 0.f;
                    if (req < B)
                        for (int k = k0 + gg * 128; k < min(k0 + gg * 128 + 128, a.cols); ++k)
                            sum += __half2float(a.x[(int64_t)req * a.cols + k]);
                    gxs[gg][q] = sum;
                }
        }
    }
    const int preq0 = g < B ? a.p_of[g] : 0, preq1 = g + 8 < B ? a.p_of[g + 8] : 0;
    const int set0 = g < B ? a.set_of[g] : -1, set1 = g + 8 < B ? a.set_of[g + 8] : -1;
    const int64_t pstride = (int64_t)B * a.NRT * kTileRows;

    // issue the cp.async copies of item rt's planes [i0, i0 + n) into buffer bf
    constexpr int kScChunks = 32 * (int)sizeof(ST) / 16;  // 16-byte pieces of one plane-item's 32 scales
    auto stage_item = [&](int rt, int bf, int i0) {
        if (rt < a.NRT) {
            const int item = s * a.NRT + rt;
            for (int i = i0; i < min(a.pmax, i0 + kMaxStagePlanes); ++i) {
                cp_async16(&stage[warp][bf][i - i0][lane], a.planes + i * a.plane_stride_u4 + (int64_t)item * 32 + lane);
                const int k = lane / kScChunks, c = lane % kScChunks;  // set k, chunk c
                if (k < a.npset && i < a.pset[k]) {
                    const ST* al = static_cast<const ST*>(a.alpha[a.pset[k]]) + ((int64_t)i * a.items + item) * 32;
                    cp_async16(&S.sc[warp][bf][i - i0][k][c], reinterpret_cast<const char*>(al) + 16 * c);
                }
            }
        }
        cp_async_commit();
    };
    int buf = 0;
    stage_item(widx, 0, 0);
    for (int rt = widx; rt < a.NRT; rt += wps, buf ^= 1) {
        const int item = s * a.NRT + rt;
        // accumulators: requests {g, g+8} x tile rows {2t, 2t+1, 8+2t, 8+2t+1}
        float y[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
        for (int i = 0; i < a.pmax; ++i) {
            if (i % kMaxStagePlanes == 0) {
                // planes [i, i+4) of this item are (being) staged in `buf`: prefetch the
                // next round (more planes of this item, or the next item) into buf^1
                if (i + kMaxStagePlanes < a.pmax) stage_item(rt, buf ^ 1, i + kMaxStagePlanes);
                else stage_item(rt + wps, buf ^ 1, 0);
                cp_async_wait<1>();
                __syncwarp();
            }
            // un-rotate this plane's 512-byte block into logical row-major bytes:
            // lane (half, r) holds group (2s + half) bytes of row r rotated by r
            const uint4 blk = stage[warp][buf][i % kMaxStagePlanes][lane];
            const ST* scs = reinterpret_cast<const ST*>(&S.sc[warp][buf][i % kMaxStagePlanes][0][0]);  // [set][32]
            if (i % kMaxStagePlanes == kMaxStagePlanes - 1 && i + 1 < a.pmax) buf ^= 1;  // next round staged in buf^1
            {
                const int half = lane >> 4, r = lane & 15;
                const uint32_t wv[4] = {blk.x, blk.y, blk.z, blk.w};
#pragma unroll
                for (int j = 0; j < 16; ++j)  // stored byte j = logical byte (j + r) & 15
                    scratch[warp][r * 32 + half * 16 + ((j + r) & 15)] = (unsigned char)(wv[j >> 2] >> (8 * (j & 3)));
            }
            __syncwarp();
            // rows g and g+8 of the tile: 32 logical bytes each
            uint32_t rowb[2][8];
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const uint4 lo = *reinterpret_cast<const uint4*>(&scratch[warp][(g + 8 * q) * 32]);
                const uint4 hi = *reinterpret_cast<const uint4*>(&scratch[warp][(g + 8 * q) * 32 + 16]);
                rowb[q][0] = lo.x; rowb[q][1] = lo.y; rowb[q][2] = lo.z; rowb[q][3] = lo.w;
                rowb[q][4] = hi.x; rowb[q][5] = hi.y; rowb[q][6] = hi.z; rowb[q][7] = hi.w;
            }
            __syncwarp();
#pragma unroll
            for (int gg = 0; gg < 2; ++gg) {  // two 128-column groups of the slice
                float c[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const int ks = gg * 8 + kk;
#pragma unroll
                    for (int q = 0; q < 2; ++q) {  // q: weight rows g (0-7 tile) / g+8 (8-15 tile)
                        const uint32_t hw = rowb[q][ks >> 1] >> (16 * (ks & 1));  // bytes 2ks, 2ks+1
                        const uint32_t nib = ((hw >> (2 * t)) & 3u) | ((hw >> (8 + 2 * t - 2)) & 0xCu);
                        const uint2 bf = nib_tab[nib];
                        mma16816(c[q], xa[ks], bf.x, bf.y);
                    }
                }
                // scale: C[q] holds requests {g, g+8} x rows {q*8 + 2t, q*8 + 2t + 1}
#pragma unroll
                for (int q = 0; q < 2; ++q) {
#pragma unroll
                    for (int e2 = 0; e2 < 2; ++e2) {
                        const int tr = q * 8 + 2 * t + e2;  // tile row
                        const int lane_sc = gg * 16 + tr;   // scale lane in the tiled layout
#pragma unroll
                        for (int rq = 0; rq < 2; ++rq) {
                            // branch-free: lanes serve different requests (precisions)
                            const int pr = rq ? preq1 : preq0;
                            const int k = rq ? set1 : set0;
                            float av = to_f32<ST>(scs[max(k, 0) * (8 * 16 / (int)sizeof(ST)) + lane_sc]);  // staged
                            if (k < 0 && i < pr) {  // (precisions beyond kMaxSets: global load)
                                const ST* al = static_cast<const ST*>(a.alpha[pr]);
                                av = to_f32<ST>(al[((int64_t)i * a.items + item) * 32 + lane_sc]);
                            }
                            av = i < pr ? av : 0.f;
                            y[rq][q * 2 + e2] = fmaf(av, c[q][rq * 2 + e2], y[rq][q * 2 + e2]);
                        }
                    }
                }
                if (ASYM && i == 0) {
#pragma unroll
                    for (int q = 0; q < 2; ++q)
#pragma unroll
                        for (int e2 = 0; e2 < 2; ++e2)
#pragma unroll
                            for (int rq = 0; rq < 2; ++rq) {
                                const int pr = rq ? preq1 : preq0;
                                if (pr > 0) {
                                    const ST* of = static_cast<const ST*>(a.offset[pr]);
                                    const float zv = to_f32<ST>(of[(int64_t)item * 32 + gg * 16 + q * 8 + 2 * t + e2]);
                                    y[rq][q * 2 + e2] = fmaf(zv, gxs[gg][rq], y[rq][q * 2 + e2]);
                                }
                            }
                }
            }
        }
        // partial[s][req][row]
#pragma unroll
        for (int rq = 0; rq < 2; ++rq) {
            const int req = g + 8 * rq;
            if (req < B) {
#pragma unroll
                for (int q = 0; q < 2; ++q)
#pragma unroll
                    for (int e2 = 0; e2 < 2; ++e2) {
                        const int row = rt * kTileRows + q * 8 + 2 * t + e2;
                        a.partial[s * pstride + (int64_t)req * a.NRT * kTileRows + row] = y[rq][q * 2 + e2];
                    }
            }
        }
    }
}

// Y[b][row] = sum_s partial[s][b][row] in ascending s
template <typename YT>
__global__ void gemm_reduce_kernel(const float* __restrict__ partial, int NS, int B, int NRT, int rows,
                                   YT* __restrict__ y) {
    const int64_t n = (int64_t)B * rows;
    const int64_t pstride = (int64_t)B * NRT * kTileRows;
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n; u += (int64_t)gridDim.x * blockDim.x) {
        const int b = (int)(u / rows), row = (int)(u - (int64_t)b * rows);
        const float* pp = partial + (int64_t)b * NRT * kTileRows + row;
        float c[4] = {0.f, 0.f, 0.f, 0.f};
        int s = 0;
        for (; s + 4 <= NS; s += 4)
#pragma unroll
            for (int k = 0; k < 4; ++k) c[k] += pp[(s + k) * pstride];
        for (int k = 0; s + k < NS; ++k) c[k] += pp[(s + k) * pstride];
        y[(int64_t)b * rows + row] = from_f32<YT>((c[0] + c[1]) + (c[2] + c[3]));
    }
}

size_t gemm_workspace_bytes(const abcq_model_t* m, int B) {
    return (size_t)n_slices(m->cols) * B * n_row_tiles(m->rows) * kTileRows * sizeof(float);
}

int launch_gemm_mixedp(const abcq_model_t* m, int B, const int* p_host, const void* x, void* y, int y_dtype,
                       void* ws, cudaStream_t st) {
    GemmArgs a{};
    a.planes = static_cast<const uint4*>(m->planes);
    a.plane_stride_u4 = m->plane_stride_bytes / 16;
    for (int p = 0; p <= ABCQ_MAX_PLANES; ++p) {
        a.alpha[p] = m->alpha[p];
        a.offset[p] = m->asymmetric ? m->offset[p] : nullptr;
    }
    a.x = static_cast<const __half*>(x);
    a.partial = static_cast<float*>(ws);
    a.rows = m->rows;
    a.cols = m->cols;
    a.NRT = n_row_tiles(m->rows);
    a.NS = n_slices(m->cols);
    a.items = a.NRT * a.NS;
    a.B = B;
    a.pmax = 0;
    a.npset = 0;
    for (int b = 0; b < B; ++b) {
        a.p_of[b] = p_host[b];
        a.pmax = a.pmax > p_host[b] ? a.pmax : p_host[b];
        int k = 0;
        while (k < a.npset && a.pset[k] != p_host[b]) ++k;
        if (k == a.npset && a.npset < kMaxSets) a.pset[a.npset++] = p_host[b];
        a.set_of[b] = k < a.npset ? k : -1;
    }
    const int grid = num_sms() * 2;
    const size_t smem = sizeof(GemmSmem);
    auto go = [&](auto kern) -> cudaError_t {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        kern<<<grid, kGWarps * 32, smem, st>>>(a);
        return cudaGetLastError();
    };
    cudaError_t e0;
    if (m->scale_dtype == ABCQ_F16)
        e0 = m->asymmetric ? go(gemm_mixedp_kernel<__half, true>) : go(gemm_mixedp_kernel<__half, false>);
    else
        e0 = m->asymmetric ? go(gemm_mixedp_kernel<float, true>) : go(gemm_mixedp_kernel<float, false>);
    if (e0 != cudaSuccess) return (int)e0;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return (int)e;
    const int64_t n = (int64_t)B * m->rows;
    const int rg = (int)ceil_div(n, 256) < 148 * 8 ? (int)ceil_div(n, 256) : 148 * 8;
    if (y_dtype == ABCQ_F16)
        gemm_reduce_kernel<__half><<<rg, 256, 0, st>>>(a.partial, a.NS, B, a.NRT, m->rows, static_cast<__half*>(y));
    else
        gemm_reduce_kernel<float><<<rg, 256, 0, st>>>(a.partial, a.NS, B, a.NRT, m->rows, static_cast<float*>(y));
    return (int)cudaGetLastError();
}

}  // namespace abcq
