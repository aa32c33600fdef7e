// abcq_gemv_lut.cuh -- sm_100a batch-1 bit-plane GEMV kernel (the hot path).
//
// Replaces GemvEngine.lut + LookupTable.build + _lut_kernel
// (/root/reference/pkg/src/anybcq/gemv.py:67-95,188-222):
//
//   y[n] = sum_{i<p} sum_g alpha^(p)[i,n,g] * s(i,n,g)   (+ offset^(p)[n,g] * gx[g])
//   s(i,n,g) = sum_{c in g} T[c][byte(i,n,c)]             (mu = 8 chunk table)
//
// Design:
//  * work item = (256-column slice s, 16-row tile rt) = one 512-byte block per
//    plane; items are ordered slice-major and split evenly over a one-wave
//    grid; a CTA owns a contiguous item range spanning at most two slices
//    ("segments"). For every plane that range is ONE contiguous byte range.
//  * TMA bulk-copy pipeline: a producer warp streams stages of
//    (kChunk items x one plane) -- weights, that plane's scales, and (plane 0,
//    asymmetric) the offsets -- global -> shared through the TMA engine into a
//    kStages-deep ring (mbarrier full/empty). ~100 KB per SM stay in flight
//    continuously, independent of the consumers' issue; weights are static
//    model data, so the producer never waits on the previous kernel (PDL).
//  * consumers (16 warps) build the reference lookup table of the CTA's
//    slices in shared memory -- 32 chunks x 256 entries x f32 per slice in a
//    [t][col] slab with a 256-byte t-row, segment k = columns 32k..32k+31 --
//    so that smem address = PRMT(weight word, lane column bytes) = t<<8|col*4
//    costs ONE instruction per looked-up byte; the pack-time byte rotation
//    (abcq_pack.cu) puts the 32 lanes on 32 distinct banks.
//  * p is a runtime kernel argument: stages run chunk-major, plane-minor; a
//    warp owns 2 items of every chunk and keeps their accumulators across the
//    p plane stages. Per element: 16 lookups summed with packed FADD2, one
//    FFMA by alpha; asymmetric offsets: one FFMA with the group sum of x.
//  * split over slices: each item writes a 16-row partial to an L2-resident
//    workspace; a small PDL-chained kernel sums the partials in a fixed
//    order (deterministic) and writes y.
#pragma once
#include <type_traits>

#include "abcq_common.cuh"
#include "abcq_internal.h"

namespace abcq {

struct LutArgs {
    const uint4* planes;
    int64_t plane_stride_u4;  // uint4 units between planes
    const void* alpha;        // scale set p, tiled [i][item][lane]
    const void* offset;       // offsets of set p, tiled [item][lane] (ASYM)
    const void* x;
    void* y;
    float* partial;           // [NS][NRT*16]
    unsigned long long* trace;  // optional per-CTA phase timestamps (abcq_debug_set_trace)
    int rows, cols, NRT, NS, p, items;
    int q, rem;                 // items per CTA: q (+1 for the first rem CTAs)
    int dbg_mode;               // profiling experiments only (0 = normal)
};

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
constexpr int kTraceCtas = 160;  // per launch slot: CTA stamps [0, 148), reduce kernel at 159
#define ABCQ_TRACE(k)                                                                   \
    do {                                                                                \
        if (a.trace && threadIdx.x == 0) a.trace[blockIdx.x * 8 + (k)] = globaltimer(); \
    } while (0)

constexpr int kConsumerWarps = 16;
constexpr int kConsumers = kConsumerWarps * 32;
constexpr int kThreads = kConsumers + 32;  // + one producer warp
constexpr int kChunk = 32;                 // items per stage
constexpr int kItemsPerWarp = kChunk / kConsumerWarps;
constexpr int kStages = 6;
constexpr int kMaxFastP = ABCQ_MAX_PLANES;
constexpr int kTableBytes = 256 * 256;  // 256 t-rows x 64 cols x 4 B: two 32-col segments
constexpr int kXBytes = 2 * kSliceCols * 4;

template <typename ST, bool ASYM>
struct StageGeom {
    static constexpr int kW = kChunk * kBlockBytes;            // weights
    static constexpr int kA = kChunk * 32 * (int)sizeof(ST);  // scales of one plane
    static constexpr int kZ = ASYM ? kChunk * 32 * (int)sizeof(ST) : 0;
    static constexpr int kBytes = kW + kA + kZ;
};

template <typename ST, bool ASYM>
constexpr int lut_smem_bytes() {
    return kTableBytes + kXBytes + 256 /*csum*/ + kStages * StageGeom<ST, ASYM>::kBytes + 2 * kStages * 8;
}

// 16 lookups of one 16-byte lane block. rb[k] holds the column bytes of steps
// 3k..3k+2 in bytes 0..2 and a zero in byte 3 (-> address bytes 2, 3); SEG
// selects the table segment through the load's immediate offset. Four packed
// FADD2 chains keep the dependent-add depth at 2.
template <int SEG>
__device__ __forceinline__ float lut16(const uint4 w, const uint32_t (&rb)[6], const char* tbl) {
    const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
    unsigned long long acc[4];
#pragma unroll
    for (int j = 0; j < 16; j += 2) {
        const uint32_t a0 = prmt(ww[j >> 2], rb[j / 3], 0x7700u | ((j & 3) << 4) | (4 + j % 3));
        const uint32_t a1 =
            prmt(ww[(j + 1) >> 2], rb[(j + 1) / 3], 0x7700u | (((j + 1) & 3) << 4) | (4 + (j + 1) % 3));
        const float v0 = *reinterpret_cast<const float*>(tbl + a0 + SEG * 128);
        const float v1 = *reinterpret_cast<const float*>(tbl + a1 + SEG * 128);
        const int ch = (j >> 1) & 3;
        acc[ch] = j < 8 ? pack2(v0, v1) : fadd2(acc[ch], pack2(v0, v1));
    }
    const float2 f = unpack2(fadd2(fadd2(acc[0], acc[1]), fadd2(acc[2], acc[3])));
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
__device__ __forceinline__ void consumer_sync() { asm volatile("bar.sync 1, %0;" ::"n"(kConsumers) : "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}

// Chunk c of a CTA: segment 0 = items [it0, split), segment 1 = [split, it1),
// each cut into kChunk-item chunks.
struct ChunkMap {
    int it0, split, it1, nc0, nchunks;
    __device__ __forceinline__ void get(int c, int& start, int& cnt, int& seg) const {
        if (c < nc0) {
            seg = 0;
            start = it0 + c * kChunk;
            cnt = min(kChunk, split - start);
        } else {
            seg = 1;
            start = split + (c - nc0) * kChunk;
            cnt = min(kChunk, it1 - start);
        }
    }
};

template <typename XT, typename YT, typename ST, bool ASYM>
__global__ void __launch_bounds__(kThreads, 1) gemv_lut_kernel(const LutArgs a) {
    using SG = StageGeom<ST, ASYM>;
    extern __shared__ __align__(128) char smem[];
    float* xs_smem = reinterpret_cast<float*>(smem + kTableBytes);
    float* csum = reinterpret_cast<float*>(smem + kTableBytes + kXBytes);  // [2][32] chunk sums
    char* stages = smem + kTableBytes + kXBytes + 256;
    uint64_t* full = reinterpret_cast<uint64_t*>(stages + kStages * SG::kBytes);
    uint64_t* empty = full + kStages;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int p = a.p;
    ABCQ_TRACE(0);

    const int b = blockIdx.x;
    ChunkMap cm;
    cm.it0 = b * a.q + min(b, a.rem);
    cm.it1 = cm.it0 + a.q + (b < a.rem ? 1 : 0);
    const int s0 = cm.it0 / a.NRT;
    cm.split = min((s0 + 1) * a.NRT, cm.it1);
    cm.nc0 = (cm.split - cm.it0 + kChunk - 1) / kChunk;
    cm.nchunks = cm.nc0 + (cm.it1 - cm.split + kChunk - 1) / kChunk;
    const int nseg = cm.it1 > cm.split ? 2 : 1;
    const int T = cm.nchunks * p;  // stages of this CTA

    if (tid == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kConsumerWarps);
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (warp == kConsumerWarps) {
        // ---------------- producer warp: TMA bulk copies of static model data
        if (lane == 0) {
            const ST* alpha = static_cast<const ST*>(a.alpha);
            const ST* offs = static_cast<const ST*>(a.offset);
            int c = 0, i = 0;
            for (int k = 0; k < T; ++k) {
                const int slot = k % kStages;
                if (k >= kStages) mbar_wait(&empty[slot], ((k / kStages) - 1) & 1);
                int start, cnt, seg;
                cm.get(c, start, cnt, seg);
                char* st = stages + slot * SG::kBytes;
                const uint32_t wb = cnt * kBlockBytes, ab = cnt * 32 * (uint32_t)sizeof(ST);
                const bool z = ASYM && i == 0;
                mbar_arrive_expect_tx(&full[slot], wb + ab + (z ? ab : 0));
                bulk_g2s(st, a.planes + i * a.plane_stride_u4 + (int64_t)start * 32, wb, &full[slot]);
                bulk_g2s(st + SG::kW, alpha + ((int64_t)i * a.items + start) * 32, ab, &full[slot]);
                if (z) bulk_g2s(st + SG::kW + SG::kA, offs + (int64_t)start * 32, ab, &full[slot]);
                if (++i == p) {
                    i = 0;
                    ++c;
                }
            }
        }
        return;
    }

    // -------------------- consumer warps --------------------------------------
    ABCQ_TRACE(1);
    pdl_wait();  // x (and y / the workspace) belong to the previous kernel
    pdl_launch_dependents();
    ABCQ_TRACE(2);

    // the reference lookup tables of the CTA's slices: thread (c, hi) loads the
    // 8 x values of chunk c straight into registers and writes 16 entries
    const XT* __restrict__ x = static_cast<const XT*>(a.x);
    const int k0 = s0 * kSliceCols;
    for (int task = tid; task < nseg * 32 * 16; task += kConsumers) {
        const int ts = task >> 9, c = task & 31, hi = (task >> 5) & 15;
        float xv[8];
        load_x8<XT>(x, k0 + ts * kSliceCols + 8 * c, a.cols, xv);
        float e[16];
        lut_chunk_entries16(xv, hi, e);
        float* col = reinterpret_cast<float*>(smem) + ts * 32 + c;
#pragma unroll
        for (int t = 0; t < 16; ++t) col[(hi * 16 + t) * 64] = e[t];
        if (ASYM && hi == 15) csum[ts * 32 + c] = e[15];  // T[255] = chunk sum
    }
    consumer_sync();
    ABCQ_TRACE(3);

    // lane column bytes for the 16 lookup steps (rotation r = lane & 15);
    // segment 1 adds 32 columns through the load's immediate offset
    const int half = lane >> 4, r = lane & 15;
    uint32_t rb[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) {
        uint32_t v = 0;
#pragma unroll
        for (int bb = 0; bb < 3; ++bb) {
            const int j = 3 * k + bb;
            if (j < 16) v |= (uint32_t)((half * 16 + ((j + r) & 15)) * 4) << (8 * bb);
        }
        rb[k] = v;
    }
    float gx0 = 0.f, gx1 = 0.f;
    if constexpr (ASYM) {
        for (int c = 0; c < 16; ++c) {
            gx0 += csum[half * 16 + c];
            gx1 += csum[32 + half * 16 + c];
        }
    }

    YT* __restrict__ y = static_cast<YT*>(a.y);
    const int64_t pstride = (int64_t)a.NRT * kTileRows;
    float acc[kItemsPerWarp];
#pragma unroll
    for (int j = 0; j < kItemsPerWarp; ++j) acc[j] = 0.f;

    // one stage (kChunk items x plane i) for this warp's items, segment SEG
    auto consume = [&](auto seg_tag, const char* st, int cnt, int i) {
        constexpr int SEG = decltype(seg_tag)::value;
        const float gxs = SEG ? gx1 : gx0;
#pragma unroll
        for (int j = 0; j < kItemsPerWarp; ++j) {
            const int it = kItemsPerWarp * warp + j;
            if (it < cnt) {
                const uint4 wv = *reinterpret_cast<const uint4*>(st + it * kBlockBytes + lane * 16);
                const float sc = to_f32<ST>(reinterpret_cast<const ST*>(st + SG::kW)[it * 32 + lane]);
                acc[j] = fmaf(sc, lut16<SEG>(wv, rb, smem), acc[j]);
                if constexpr (ASYM) {
                    if (i == 0) {
                        const float z =
                            to_f32<ST>(reinterpret_cast<const ST*>(st + SG::kW + SG::kA)[it * 32 + lane]);
                        acc[j] = fmaf(z, gxs, acc[j]);
                    }
                }
            }
        }
    };

    int c = 0, i = 0;
    for (int k = 0; k < T; ++k) {
        const int slot = k % kStages;
        int start, cnt, seg;
        cm.get(c, start, cnt, seg);
        mbar_wait(&full[slot], (k / kStages) & 1);
        const char* st = stages + slot * SG::kBytes;
        if (seg)
            consume(std::integral_constant<int, 1>{}, st, cnt, i);
        else
            consume(std::integral_constant<int, 0>{}, st, cnt, i);
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
        if (++i == p) {
            // chunk done: combine the slice's two groups (lanes l, l+16), emit 16 rows per item
            const int sl = s0 + seg;
#pragma unroll
            for (int j = 0; j < kItemsPerWarp; ++j) {
                const int it = kItemsPerWarp * warp + j;
                const float out = acc[j] + __shfl_down_sync(0xffffffffu, acc[j], 16);
                acc[j] = 0.f;
                if (it < cnt && lane < 16) {
                    const int row = (start + it - sl * a.NRT) * kTileRows + lane;
                    if (a.NS == 1) {
                        if (row < a.rows) y[row] = from_f32<YT>(out);
                    } else {
                        __stcg(a.partial + sl * pstride + row, out);
                    }
                }
            }
            i = 0;
            ++c;
        }
    }
    if (warp == 0) ABCQ_TRACE(4);
}

// Split-K completion (NS > 1): y[n] = sum_s partial[s][n] in a fixed order
// (four interleaved chains over ascending s, then (c0 + c1) + (c2 + c3)),
// so results are bitwise reproducible. Launched with PDL right after the
// GEMV kernel; it waits for the GEMV grid inside griddepcontrol.wait.
template <typename YT>
__global__ void __launch_bounds__(64) split_reduce_kernel(const float* __restrict__ partial, int NS,
                                                          int64_t stride, int rows, YT* __restrict__ y,
                                                          unsigned long long* trace) {
    if (trace && blockIdx.x == 0 && threadIdx.x == 0) trace[(kTraceCtas - 1) * 8 + 0] = globaltimer();
    pdl_wait();
    pdl_launch_dependents();
    if (trace && blockIdx.x == 0 && threadIdx.x == 0) trace[(kTraceCtas - 1) * 8 + 1] = globaltimer();
    const int row = blockIdx.x * blockDim.x + threadIdx.x;
    if (row < rows) {
        const float* pp = partial + row;
        float c[4] = {0.f, 0.f, 0.f, 0.f};
        for (int s0 = 0; s0 < NS; s0 += 16) {  // 16 loads in flight, fixed summation order
            float v[16];
#pragma unroll
            for (int k = 0; k < 16; ++k) v[k] = s0 + k < NS ? __ldcg(pp + (s0 + k) * stride) : 0.f;
#pragma unroll
            for (int k = 0; k < 16; ++k) c[k & 3] += v[k];
        }
        y[row] = from_f32<YT>((c[0] + c[1]) + (c[2] + c[3]));
    }
    if (trace && blockIdx.x == 0 && threadIdx.x == 0) trace[(kTraceCtas - 1) * 8 + 2] = globaltimer();
}

template <typename XT, typename YT, typename ST, bool ASYM>
inline int launch_t(const LutArgs& a, int grid, cudaStream_t st) {
    auto kern = gemv_lut_kernel<XT, YT, ST, ASYM>;
    constexpr int smem = lut_smem_bytes<ST, ASYM>();
    static_assert(smem <= 227 * 1024, "shared memory budget");
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
    rc.blockDim = dim3(64);
    rc.gridDim = dim3((unsigned)ceil_div(a.rows, 64));
    rc.dynamicSmemBytes = 0;
    return (int)cudaLaunchKernelEx(&rc, split_reduce_kernel<YT>, (const float*)a.partial, a.NS,
                                   (int64_t)a.NRT * kTileRows, a.rows, static_cast<YT*>(a.y), a.trace);
}

template <typename XT, typename YT, typename ST, bool ASYM>
int launch_direct_t(const LutArgs& a, int grid, cudaStream_t st);  // abcq_gemv_lut_direct.cuh

template <typename XT, typename YT, typename ST>
inline int launch_asym(const LutArgs& a, bool asym, int grid, cudaStream_t st) {
    if (a.dbg_mode == 11)  // variant experiment: register-direct kernel
        return asym ? launch_direct_t<XT, YT, ST, true>(a, grid, st) : launch_direct_t<XT, YT, ST, false>(a, grid, st);
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
