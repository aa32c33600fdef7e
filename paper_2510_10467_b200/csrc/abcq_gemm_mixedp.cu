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
// (16 requests x 16 k, fp16; the CTA's slice of X is staged in shared memory
// once and read with ldmatrix, one 128-column group at a time); B = the
// sign bits of 8 weight rows, expanded to +-1 fp16 through a 16-entry nibble
// table in shared memory (a lane's B fragment is one nibble per row and
// k-step); C = 16 requests x 8 rows, reset per 128-column group, scaled by
// alpha^(p_b) and accumulated. Weight blocks (tiled layout, rotated bytes) are
// read straight from the staging buffer and un-rotated in registers.
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
    int overflow;           // some request's precision is not among pset (its scales are read from global)
    int rows, cols, NRT, NS, items, B, pmax;
    int cps;  // CTAs per slice (each takes every cps-th group of kGWarps row tiles)
};

// dynamic shared memory of the GEMM kernel
constexpr int kXPitch = 256 + 8;  // halves per staged X row: 528 B, ldmatrix rows hit distinct banks
struct GemmSmem {
    uint4 stage[kGWarps][2][kMaxStagePlanes][32];              // plane blocks, double-buffered
    uint4 sc[kGWarps][2][kMaxStagePlanes][kMaxSets][8];         // their scales (<= 128 B per set)
    __align__(16) __half xs[kMaxBatch][kXPitch];                // the CTA's X slice (16 requests x 256 k)
};

__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void ldmatrix_x4(uint32_t (&r)[4], const void* smem) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"((uint32_t)__cvta_generic_to_shared(smem)));
}

// One 16-byte lane chunk of a tiled block holds a row's group bytes rotated by
// the row index r (stored byte j = logical byte (j + r) & 15); undo it in
// registers: logical = stored rotated left by r bytes. K2 = bit 3 of r (a
// compile-time word swap), k1 = bit 2, sh = 8 * (r & 3).
template <bool K2>
__device__ __forceinline__ void unrotate16(const uint4 v, bool k1, int sh, uint32_t (&o)[4]) {
    uint32_t w0 = v.x, w1 = v.y, w2 = v.z, w3 = v.w;
    if (K2) {  // R[m] = S[m - 2]
        uint32_t t0 = w0, t1 = w1;
        w0 = w2; w1 = w3; w2 = t0; w3 = t1;
    }
    if (k1) {  // R[m] = S[m - 1]
        uint32_t t = w3;
        w3 = w2; w2 = w1; w1 = w0; w0 = t;
    }
    o[0] = __funnelshift_l(w3, w0, sh);
    o[1] = __funnelshift_l(w0, w1, sh);
    o[2] = __funnelshift_l(w1, w2, sh);
    o[3] = __funnelshift_l(w2, w3, sh);
}

__device__ __forceinline__ uint2 lds64(uint32_t addr) {
    uint2 v;
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr));
    return v;
}

template <typename ST>
__device__ __forceinline__ float2 ld_scale2(const ST* p);
template <>
__device__ __forceinline__ float2 ld_scale2<__half>(const __half* p) {
    return __half22float2(*reinterpret_cast<const __half2*>(p));
}
template <>
__device__ __forceinline__ float2 ld_scale2<float>(const float* p) {
    return *reinterpret_cast<const float2*>(p);
}

template <typename ST, bool ASYM>
__global__ void __launch_bounds__(kGWarps * 32) gemm_mixedp_kernel(const GemmArgs a) {
    __shared__ __align__(128) uint2 nib_tab[16];  // nibble -> {half2, half2}; 128-aligned: address = base | 8*nibble
    // per-warp double buffer of an item's plane blocks and their scales, filled
    // with cp.async (group-tracked, so the next item streams in while this one
    // computes); the CTA's X slice, read as A fragments with ldmatrix
    extern __shared__ __align__(16) char gsmem[];
    GemmSmem& S = *reinterpret_cast<GemmSmem*>(gsmem);
    auto& stage = S.stage;

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x < 16) {
        const int n = threadIdx.x;
        auto h = [](int bit) -> uint32_t { return bit ? 0x3C00u : 0xBC00u; };  // +1 / -1 in fp16
        nib_tab[n] = make_uint2(h(n & 1) | (h((n >> 1) & 1) << 16), h((n >> 2) & 1) | (h((n >> 3) & 1) << 16));
    }

    const int g = lane >> 2, t = lane & 3;
    const int B = a.B;
    const int preq0 = g < B ? a.p_of[g] : 0, preq1 = g + 8 < B ? a.p_of[g + 8] : 0;
    const int set0 = g < B ? a.set_of[g] : -1, set1 = g + 8 < B ? a.set_of[g + 8] : -1;
    // element offsets of the lane's two requests' staged scale sets
    const int soff0 = max(set0, 0) * (8 * 16 / (int)sizeof(ST)), soff1 = max(set1, 0) * (8 * 16 / (int)sizeof(ST));
    const int64_t pstride = (int64_t)B * a.NRT * kTileRows;
    const bool xvec = (a.cols & 7) == 0 && (reinterpret_cast<uintptr_t>(a.x) & 15) == 0;
    // this lane's ldmatrix row address inside the X slice (matrix lane>>3: rows +8, k +8)
    const int xrow = (lane & 7) + ((lane >> 3) & 1) * 8, xcol = (lane >> 4) * 8;
    const int tstride = a.cps * kGWarps;  // tiles per slice step of a warp
    const uint32_t nib_base = (uint32_t)__cvta_generic_to_shared(nib_tab);
    const bool rk1 = (g >> 2) & 1;  // bit 2 of the lane's rows g, g+8 (their rotations)
    const int rsh = 8 * (g & 3);

    // units = (slice, chunk of the slice's row tiles); a CTA's warps share the slice
    for (int u = blockIdx.x; u < a.NS * a.cps; u += gridDim.x) {
        const int s = u % a.NS, chunk = u / a.NS;
        const int k0 = s * kSliceCols;
        __syncthreads();  // the previous unit's X reads are done (and nib_tab is written)
        // X slice -> shared, k permuted inside each 16-column k-step so that the four
        // k a lane feeds the MMA (2t, 2t+1, 2t+8, 2t+9) are weight bits 4t..4t+3, one
        // contiguous nibble: MMA k = m holds column 4*((m & 7) >> 1) + 2*(m >> 3) + (m & 1),
        // i.e. the low 8 MMA columns take the column pairs (0,1),(4,5),(8,9),(12,13)
        // and the high 8 take (2,3),(6,7),(10,11),(14,15).
        for (int cidx = threadIdx.x; cidx < kMaxBatch * 16; cidx += blockDim.x) {
            const int req = cidx >> 4, ks = cidx & 15, kc = ks * 16, k = k0 + kc;
            uint32_t e[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};  // column pairs of the k-step
            if (req < B) {
                const __half* xp = a.x + (int64_t)req * a.cols + k;
                if (xvec && k + 16 <= a.cols) {
                    const uint4 v0 = __ldg(reinterpret_cast<const uint4*>(xp));
                    const uint4 v1 = __ldg(reinterpret_cast<const uint4*>(xp) + 1);
                    e[0] = v0.x; e[1] = v0.y; e[2] = v0.z; e[3] = v0.w;
                    e[4] = v1.x; e[5] = v1.y; e[6] = v1.z; e[7] = v1.w;
                } else {
#pragma unroll
                    for (int j = 0; j < 16; ++j)
                        if (k + j < a.cols) e[j >> 1] |= (uint32_t)__half_as_ushort(xp[j]) << (16 * (j & 1));
                }
            }
            *reinterpret_cast<uint4*>(&S.xs[req][kc]) = make_uint4(e[0], e[2], e[4], e[6]);
            *reinterpret_cast<uint4*>(&S.xs[req][kc + 8]) = make_uint4(e[1], e[3], e[5], e[7]);
        }
        __syncthreads();
        float gxs[2][2];  // per group: sum of x over the group for requests g, g+8 (asymmetric)
        if (ASYM) {
#pragma unroll
            for (int gg = 0; gg < 2; ++gg)
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    float sum = 0.f;  // lanes t split the group's 128 columns, fixed order
                    for (int k = 0; k < 32; ++k) sum += __half2float(S.xs[g + 8 * q][gg * 128 + t * 32 + k]);
                    sum += __shfl_xor_sync(0xffffffffu, sum, 1);
                    sum += __shfl_xor_sync(0xffffffffu, sum, 2);
                    gxs[gg][q] = sum;
                }
        }

        // issue the cp.async copies of tile rt's planes [i0, i0 + n) into buffer bf
        constexpr int kScChunks = 32 * (int)sizeof(ST) / 16;  // 16-byte pieces of one plane-item's 32 scales
        auto stage_item = [&](int rt, int bf, int i0) {
            if (rt < a.NRT) {
                const int item = s * a.NRT + rt;
                for (int i = i0; i < min(a.pmax, i0 + kMaxStagePlanes); ++i) {
                    cp_async16(&stage[warp][bf][i - i0][lane], a.planes + i * a.plane_stride_u4 + (int64_t)item * 32 + lane);
                    const int k = lane / kScChunks, c = lane % kScChunks;  // set k, chunk c
                    if (k < a.npset) {
                        if (i < a.pset[k]) {
                            const ST* al = static_cast<const ST*>(a.alpha[a.pset[k]]) + ((int64_t)i * a.items + item) * 32;
                            cp_async16(&S.sc[warp][bf][i - i0][k][c], reinterpret_cast<const char*>(al) + 16 * c);
                        } else {  // plane i is beyond this set's precision: scale 0
                            S.sc[warp][bf][i - i0][k][c] = make_uint4(0u, 0u, 0u, 0u);
                        }
                    }
                }
            }
            cp_async_commit();
        };
        int buf = 0;
        const int rt0 = chunk * kGWarps + warp;
        stage_item(rt0, 0, 0);
        for (int rt = rt0; rt < a.NRT; rt += tstride) {
            const int item = s * a.NRT + rt;
            // accumulators: requests {g, g+8} x tile rows {2t, 2t+1, 8+2t, 8+2t+1}
            float y[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
            for (int i0 = 0; i0 < a.pmax; i0 += kMaxStagePlanes, buf ^= 1) {
                // planes [i0, i0+4) of this tile are (being) staged in `buf`: prefetch the
                // next round (more planes of this tile, or the next tile) into buf^1
                if (i0 + kMaxStagePlanes < a.pmax) stage_item(rt, buf ^ 1, i0 + kMaxStagePlanes);
                else stage_item(rt + tstride, buf ^ 1, 0);
                cp_async_wait<1>();
                __syncwarp();
                const int np = min(kMaxStagePlanes, a.pmax - i0);
#pragma unroll
                for (int gg = 0; gg < 2; ++gg) {  // two 128-column groups of the slice
                    uint32_t xa[8][4];            // A fragments of this group's 8 k-steps
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk) ldmatrix_x4(xa[kk], &S.xs[xrow][gg * 128 + kk * 16 + xcol]);
                    for (int ii = 0; ii < np; ++ii) {
                        const int i = i0 + ii;
                        // rows g and g+8 of the tile: their 16 group bytes (lane chunk gg*16 + row)
                        uint32_t rowb[2][4];
                        unrotate16<false>(stage[warp][buf][ii][gg * 16 + g], rk1, rsh, rowb[0]);
                        unrotate16<true>(stage[warp][buf][ii][gg * 16 + g + 8], rk1, rsh, rowb[1]);
                        const ST* scs = reinterpret_cast<const ST*>(&S.sc[warp][buf][ii][0][0]);  // [set][32]
                        float c[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
                        for (int kk = 0; kk < 8; ++kk) {
#pragma unroll
                            for (int q = 0; q < 2; ++q) {  // q: weight rows g (0-7 tile) / g+8 (8-15 tile)
                                // weight bits 4t..4t+3 of k-step kk (see the X permutation), as
                                // the byte offset 8 * nibble of its table entry
                                const uint32_t w = rowb[q][kk >> 1];
                                const uint32_t off = (kk & 1) ? (w >> (13 + 4 * t)) & 0x78u : ((w << 3) >> (4 * t)) & 0x78u;
                                const uint2 bf = lds64(nib_base | off);
                                mma16816(c[q], xa[kk], bf.x, bf.y);
                            }
                        }
                        // scale: C[q] holds requests {g, g+8} x rows {q*8 + 2t, q*8 + 2t + 1};
                        // staged sets are zero beyond their precision, so no masking
                        if (!a.overflow) {
#pragma unroll
                            for (int q = 0; q < 2; ++q)
#pragma unroll
                                for (int rq = 0; rq < 2; ++rq) {
                                    const float2 av = ld_scale2<ST>(scs + (rq ? soff1 : soff0) + gg * 16 + q * 8 + 2 * t);
                                    y[rq][q * 2] = fmaf(av.x, c[q][rq * 2], y[rq][q * 2]);
                                    y[rq][q * 2 + 1] = fmaf(av.y, c[q][rq * 2 + 1], y[rq][q * 2 + 1]);
                                }
                        } else {
#pragma unroll
                            for (int q = 0; q < 2; ++q) {
#pragma unroll
                                for (int e2 = 0; e2 < 2; ++e2) {
                                    const int lane_sc = gg * 16 + q * 8 + 2 * t + e2;  // scale lane in the tiled layout
#pragma unroll
                                    for (int rq = 0; rq < 2; ++rq) {
                                        const int pr = rq ? preq1 : preq0;
                                        const int k = rq ? set1 : set0;
                                        float av = to_f32<ST>(scs[(rq ? soff1 : soff0) + lane_sc]);
                                        if (k < 0 && i < pr) {  // precisions beyond kMaxSets: global load
                                            const ST* al = static_cast<const ST*>(a.alpha[pr]);
                                            av = to_f32<ST>(al[((int64_t)i * a.items + item) * 32 + lane_sc]);
                                        }
                                        av = i < pr ? av : 0.f;
                                        y[rq][q * 2 + e2] = fmaf(av, c[q][rq * 2 + e2], y[rq][q * 2 + e2]);
                                    }
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
                                            const float zv =
                                                to_f32<ST>(of[(int64_t)item * 32 + gg * 16 + q * 8 + 2 * t + e2]);
                                            y[rq][q * 2 + e2] = fmaf(zv, gxs[gg][rq], y[rq][q * 2 + e2]);
                                        }
                                    }
                        }
                    }
                }
                __syncwarp();  // all lanes are done with `buf` before it is refilled
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
        cp_async_wait<0>();
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
        if (a.set_of[b] < 0) a.overflow = 1;
    }
    const size_t smem = sizeof(GemmSmem);
    auto go = [&](auto kern) -> cudaError_t {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        int per_sm = 0;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kGWarps * 32, smem);
        if (e != cudaSuccess) return e;
        // CTAs share a slice (its X staged once); slices get equal CTA counts
        const int G = num_sms() * (per_sm > 0 ? per_sm : 1);
        const int tile_groups = (int)ceil_div(a.NRT, kGWarps);
        a.cps = G / a.NS > 1 ? G / a.NS : 1;
        if (a.cps > tile_groups) a.cps = tile_groups;
        const int units = a.NS * a.cps;
        const int grid = units < G ? units : G;
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
