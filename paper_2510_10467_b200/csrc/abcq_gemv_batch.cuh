// abcq_gemv_batch.cuh -- persistent bit-plane GEMV over a list of independent
// jobs (one job = one GemvEngine.lut call, /root/reference/pkg/src/anybcq/
// gemv.py:188-222). A single GEMV is a batch of one. Building blocks (layout,
// lookup, table, TMA helpers) live in abcq_gemv_lut.cuh; DESIGN.md §3.1.
//
// One CTA per SM (a co-resident grid) of kWarps warps. Every warp is its own
// producer and consumer: it owns a contiguous run of items of each job and a
// private kRing-deep ring of shared-memory slots; lane 0 streams
// (kK items x one plane) of weights + that plane's scales (+ offsets) per slot
// with TMA bulk copies (cp.async.bulk ... mbarrier::complete_tx), the warp
// consumes slot e while slots e+1..e+kRing-1 are in flight. No cross-warp
// synchronisation on the streaming path; the slot stream runs on across job
// boundaries (weights are static, so it starts before the PDL wait).
// Per job the warps rebuild the reference lookup table from x (one CTA
// barrier); with split over slices (NS > 1) items store 16-row partials, and
// after the last job every CTA completes an even share of every job's row
// tiles (arrival counters, fixed-order sums -> bitwise reproducible).
#pragma once
#include "abcq_gemv_lut.cuh"

namespace abcq {

constexpr int kMaxJobs = 16;
constexpr int kWarps = 16;
constexpr int kBThreads = kWarps * 32;
constexpr int kK = 4;  // items per slot

struct Job {
    const uint4* planes;
    int64_t plane_stride_u4;
    const void* alpha;   // scale set p, tiled [i][item][lane]
    const void* offset;  // offsets of set p, tiled [item][lane] (asymmetric)
    const void* x;
    void* y;
    float* partial;      // [NS][NRT*16]
    uint32_t* counters;  // [NRT] arrival counters, self-resetting
    int rows, cols, NRT, NS, p, items, q, rem;
};

// kernel parameter: NJ job slots (1, 4 or 16 -- the smallest that fits)
template <int NJ>
struct KArgs {
    Job jobs[NJ];
    int n_jobs;
    int fused;
    int dbg;  // profiling experiments: 1 = skip the lookups
    unsigned long long* trace;
};

struct BatchArgs {
    Job jobs[kMaxJobs];
    int n_jobs;
    int fused;  // 1: in-kernel split-K completion; 0: split_reduce_kernel follows
    int dbg;
    unsigned long long* trace;  // optional per-CTA stamps (abcq_debug_set_trace)
};

template <typename ST, bool ASYM>
struct SlotGeom {
    static constexpr int kW = kK * kBlockBytes;           // weights
    static constexpr int kA = kK * 32 * (int)sizeof(ST);  // scales of one plane
    static constexpr int kZ = ASYM ? kK * 32 * (int)sizeof(ST) : 0;
    static constexpr int kBytes = kW + kA + kZ;
    // slots fit around the table window: [0x400+1024, 0x10000) and
    // [0x20000, 227 KiB - 0x400 of dynamic smem)
    static constexpr int kLow = (int)((kTableWindow - 0x400 - 1024) / kBytes);
    static constexpr int kHigh = (227 * 1024 - (int)(2 * kTableWindow - 0x400)) / kBytes;
    static constexpr int kRing = (kLow + kHigh) / kWarps < 6 ? (kLow + kHigh) / kWarps : 6;
    static constexpr int kSmem =
        (int)(2 * kTableWindow - 0x400) + (kWarps * kRing > kLow ? kWarps * kRing - kLow : 0) * kBytes;
};

// This warp's items of job J in CTA b: the CTA's range [it0, it1) has <= 2
// segments (slices); warps split proportionally to the segment sizes, then
// each warp gets a contiguous run.
struct WarpRun {
    int lo, hi, seg, s0;  // items [lo, hi) of slice s0 + seg
    __device__ __forceinline__ int n() const { return hi - lo; }
};
__device__ __forceinline__ WarpRun warp_run(const Job& J, int b, int warp) {
    WarpRun r;
    const int it0 = b * J.q + min(b, J.rem);
    const int it1 = it0 + J.q + (b < J.rem ? 1 : 0);
    r.s0 = J.NRT > 0 ? it0 / J.NRT : 0;
    const int split = min((r.s0 + 1) * J.NRT, it1);
    const int n0 = split - it0, n1 = it1 - split, n = it1 - it0;
    int w0 = n1 == 0 ? kWarps : (n0 == 0 ? 0 : (kWarps * n0 + n / 2) / max(n, 1));
    if (n0 > 0 && w0 == 0) w0 = 1;
    if (n1 > 0 && w0 == kWarps) w0 = kWarps - 1;
    r.seg = warp < w0 ? 0 : 1;
    const int nw = r.seg ? kWarps - w0 : w0, wi = r.seg ? warp - w0 : warp;
    const int base = r.seg ? split : it0, cnt = r.seg ? n1 : n0;
    r.lo = base + (int)((int64_t)wi * cnt / max(nw, 1));
    r.hi = base + (int)((int64_t)(wi + 1) * cnt / max(nw, 1));
    return r;
}

// fixed-order sum of one row's NS slice partials (4 interleaved chains over
// ascending s, then (c0 + c1) + (c2 + c3)) -- shared by the fused completion
// and split_reduce_kernel so every path gives bitwise-identical y
__device__ __forceinline__ float reduce_row(const float* pp, int NS, int64_t stride) {
    float c[4] = {0.f, 0.f, 0.f, 0.f};
    for (int s0 = 0; s0 < NS; s0 += 16) {  // 16 loads in flight
        float v[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) v[k] = s0 + k < NS ? __ldcg(pp + (s0 + k) * stride) : 0.f;
#pragma unroll
        for (int k = 0; k < 16; ++k) c[k & 3] += v[k];
    }
    return (c[0] + c[1]) + (c[2] + c[3]);
}

#define ABCQ_BTRACE(k)                                                           \
    do {                                                                         \
        if (a.trace && lane == 0) a.trace[blockIdx.x * 8 + (k)] = globaltimer(); \
    } while (0)

template <int NJ, typename XT, typename YT, typename ST, bool ASYM>
__global__ void __launch_bounds__(kBThreads, 1) gemv_batch_kernel(const __grid_constant__ KArgs<NJ> a) {
    using SG = SlotGeom<ST, ASYM>;
    constexpr int R = SG::kRing;
    extern __shared__ __align__(1024) char smem[];
    // shared-memory map (window addresses): [base, 0x10000) = barriers, chunk
    // sums and the first slots; [0x10000, 0x20000) = the lookup table (absolute
    // address lookups, see lut16); [0x20000, ...) = the remaining slots
    const uint32_t tbl_off = kTableWindow - smem_addr(smem);
    float* csum = reinterpret_cast<float*>(smem);              // [2][32] chunk sums
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 256);  // [kWarps][R]
    float* table = reinterpret_cast<float*>(smem + tbl_off);
    const int nlow = (int)((tbl_off - 1024) / SG::kBytes);
    auto slot_ptr = [&](int g) -> char* {  // g = global slot index warp*R + s
        return g < nlow ? smem + 1024 + g * SG::kBytes : smem + tbl_off + kTableBytes + (g - nlow) * SG::kBytes;
    };

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int b = blockIdx.x, G = gridDim.x;
    if (warp == 0) ABCQ_BTRACE(0);
    uint64_t* mybar = bars + warp * R;
    if (lane == 0) {
        for (int s = 0; s < R; ++s) mbar_init(&mybar[s], 1);
        fence_mbar_init();
    }
    __syncwarp();

    // ---- this warp's slot stream: over jobs j, chunks of kK items, planes i --
    // issue cursor: element (job j, chunk start c, plane i) with its source
    // pointers kept in registers and advanced incrementally (the job table in
    // parameter space is only read when the cursor enters a new job)
    struct Cur {
        int j, hi, c, i, p;
        const char* w;   // planes + i*plane_stride + c*512   (bytes)
        const ST* al;    // alpha + (i*items + c)*32
        const ST* z;     // offset + c*32
        int64_t pst;     // plane stride (bytes)
        int64_t ast;     // items*32: scale elements per plane
    };
    auto cur_job = [&](Cur& k, int j) {
        for (; j < a.n_jobs; ++j) {
            const Job& J = a.jobs[j];
            const WarpRun r = warp_run(J, b, warp);
            if (r.n() > 0) {
                k.j = j;
                k.hi = r.hi;
                k.c = r.lo;
                k.i = 0;
                k.p = J.p;
                k.pst = J.plane_stride_u4 * 16;
                k.ast = (int64_t)J.items * 32;
                k.w = reinterpret_cast<const char*>(J.planes) + (int64_t)r.lo * kBlockBytes;
                k.al = static_cast<const ST*>(J.alpha) + (int64_t)r.lo * 32;
                k.z = ASYM ? static_cast<const ST*>(J.offset) + (int64_t)r.lo * 32 : nullptr;
                return;
            }
        }
        k.j = a.n_jobs;  // exhausted
    };
    auto advance = [&](Cur& k) {
        if (++k.i < k.p) {
            k.w += k.pst;
            k.al += k.ast;
        } else {
            k.i = 0;
            k.c += kK;
            if (k.c >= k.hi) {
                cur_job(k, k.j + 1);
            } else {
                k.w += kK * kBlockBytes - (k.p - 1) * k.pst;
                k.al += kK * 32 - (k.p - 1) * k.ast;
                if constexpr (ASYM) k.z += kK * 32;
            }
        }
    };
    // issue the TMA copies of the cursor's element into slot s (lane 0 only)
    auto issue = [&](const Cur& k, int s) {
        const int cnt = min(kK, k.hi - k.c);
        char* st = slot_ptr(warp * R + s);
        const uint32_t wb = cnt * kBlockBytes, ab = cnt * 32 * (uint32_t)sizeof(ST);
        const bool z = ASYM && k.i == 0;
        if (lane == 0) {
            mbar_arrive_expect_tx(&mybar[s], wb + ab + (z ? ab : 0));
            bulk_g2s(st, k.w, wb, &mybar[s]);
            bulk_g2s(st + SG::kW, k.al, ab, &mybar[s]);
            if (z) bulk_g2s(st + SG::kW + SG::kA, k.z, ab, &mybar[s]);
        }
    };

    Cur ic;  // issue cursor: runs R elements ahead of consumption
    cur_job(ic, 0);
    // static model data: fill the ring before waiting on the previous kernel
    for (int s = 0; s < R && ic.j < a.n_jobs; ++s) {
        issue(ic, s);
        advance(ic);
    }
    pdl_wait();  // x, y and the workspace belong to the previous kernel
    pdl_launch_dependents();

    const int half = lane >> 4, r = lane & 15;
    uint32_t rb[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) {
        uint32_t v = 0;
#pragma unroll
        for (int bb = 0; bb < 3; ++bb) {
            const int jj = 3 * k + bb;
            if (jj < 16) v |= (uint32_t)((half * 16 + ((jj + r) & 15)) * 4) << (8 * bb);
        }
        rb[k] = v | ((kTableWindow >> 16) << 24);  // byte 3 -> address byte 2
    }

    // x values of this thread's table tasks (chunk tid&31 of up to 2 slices)
    static_assert(kBThreads == 512, "table build maps one thread to (chunk, hi) of a slice");
    float xpre[2][8];
    int xpre_job = -1;
    auto prefetch_x = [&](int jn) {
        const Job& Jn = a.jobs[jn];
        const int it0 = b * Jn.q + min(b, Jn.rem);
        const int sn = Jn.NRT > 0 ? it0 / Jn.NRT : 0;
        const XT* __restrict__ xn = static_cast<const XT*>(Jn.x);
#pragma unroll
        for (int ts = 0; ts < 2; ++ts)  // slice sn + 1 may not exist: load_x8 zero-fills past cols
            load_x8<XT>(xn, (sn + ts) * kSliceCols + 8 * (tid & 31), Jn.cols, xpre[ts]);
        xpre_job = jn;
    };

    int e = 0;  // consumed elements (slot = e % R, phase = (e / R) & 1)
    for (int j = 0; j < a.n_jobs; ++j) {
        const Job& J = a.jobs[j];
        const int it0 = b * J.q + min(b, J.rem), it1 = it0 + J.q + (b < J.rem ? 1 : 0);
        if (it1 <= it0) continue;  // no items for this CTA: nothing to build or stream
        const WarpRun wr = warp_run(J, b, warp);
        const int s0 = wr.s0;
        const int nseg = it1 > min((s0 + 1) * J.NRT, it1) ? 2 : 1;
        // ---- lookup tables of job j's slices (one CTA barrier each side) ------
        // thread (c, hi) of task ts builds 16 entries of chunk c from 8 x values;
        // they were prefetched into registers while the previous job streamed
        if (xpre_job != j) prefetch_x(j);
        if (j > 0) __syncthreads();  // every warp is done with the previous table
#pragma unroll
        for (int ts = 0; ts < 2; ++ts) {
            if (ts < nseg) {
                const int c = tid & 31, hi = tid >> 5;
                float ev[16];
                lut_chunk_entries16(xpre[ts], hi, ev);
                float* col = table + ts * 32 + c;
#pragma unroll
                for (int t = 0; t < 16; ++t) col[(hi * 16 + t) * 64] = ev[t];
                if (ASYM && hi == 15) csum[ts * 32 + c] = ev[15];  // T[255] = chunk sum
            }
        }
        __syncthreads();
        for (int jn = j + 1; jn < a.n_jobs; ++jn) {  // x of the next job this CTA works on
            const Job& Jn = a.jobs[jn];
            if (Jn.q + (b < Jn.rem ? 1 : 0) > 0) {
                prefetch_x(jn);
                break;
            }
        }
        if (j < 3 && warp == 0) ABCQ_BTRACE(1 + 2 * j);
        if (wr.n() == 0) continue;
        float gx = 0.f;
        if constexpr (ASYM) {
            for (int c = 0; c < 16; ++c) gx += csum[wr.seg * 32 + half * 16 + c];
        }

        // ---- stream this warp's elements of job j -------------------------------
        YT* __restrict__ y = static_cast<YT*>(J.y);
        const int64_t pstride = (int64_t)J.NRT * kTileRows;
        const int sl = s0 + wr.seg;
        auto run = [&](auto seg_tag) {
            constexpr int SEG = decltype(seg_tag)::value;
            for (int c = wr.lo; c < wr.hi; c += kK) {
                const int cnt = min(kK, wr.hi - c);
                float acc[kK];
#pragma unroll
                for (int q = 0; q < kK; ++q) acc[q] = 0.f;
                for (int i = 0; i < J.p; ++i, ++e) {
                    const int s = e % R;
                    mbar_wait(&mybar[s], (e / R) & 1);
                    const char* st = slot_ptr(warp * R + s);
                    if (a.dbg != 1) {
                        // a slot's kK elements are independent: load them all, then
                        // look up -- no per-element branch in the full-slot case, so
                        // the scheduler interleaves the four lookup chains
                        auto elems = [&](auto n_tag) {
                            constexpr int N = decltype(n_tag)::value;
                            uint4 wv[N];
                            float sc[N];
#pragma unroll
                            for (int q = 0; q < N; ++q) {
                                wv[q] = *reinterpret_cast<const uint4*>(st + q * kBlockBytes + lane * 16);
                                sc[q] = to_f32<ST>(reinterpret_cast<const ST*>(st + SG::kW)[q * 32 + lane]);
                            }
#pragma unroll
                            for (int q = 0; q < N; ++q) acc[q] = fmaf(sc[q], lut16<SEG>(wv[q], rb), acc[q]);
                            if constexpr (ASYM) {
                                if (i == 0) {
#pragma unroll
                                    for (int q = 0; q < N; ++q)
                                        acc[q] = fmaf(to_f32<ST>(reinterpret_cast<const ST*>(st + SG::kW + SG::kA)[q * 32 + lane]),
                                                      gx, acc[q]);
                                }
                            }
                        };
                        if (cnt == kK) {
                            elems(std::integral_constant<int, kK>{});
                        } else {
                            if (cnt == 1) elems(std::integral_constant<int, 1>{});
                            else if (cnt == 2) elems(std::integral_constant<int, 2>{});
                            else elems(std::integral_constant<int, 3>{});
                        }
                    }
                    __syncwarp();  // every lane has consumed slot s
                    if (ic.j < a.n_jobs) {  // refill it with the element R ahead
                        issue(ic, s);
                        advance(ic);
                    }
                }
                // chunk done: combine the slice's two groups (lanes l, l+16), emit 16 rows per item
#pragma unroll
                for (int q = 0; q < kK; ++q) {
                    const float out = acc[q] + __shfl_down_sync(0xffffffffu, acc[q], 16);
                    if (q < cnt && lane < 16) {
                        const int row = (c + q - sl * J.NRT) * kTileRows + lane;
                        if (J.NS == 1) {
                            if (row < J.rows) y[row] = from_f32<YT>(out);
                        } else {
                            __stcg(J.partial + sl * pstride + row, out);
                        }
                    }
                }
            }
        };
        if (wr.seg)
            run(std::integral_constant<int, 1>{});
        else
            run(std::integral_constant<int, 0>{});
        if (j < 3 && warp == 0) ABCQ_BTRACE(2 + 2 * j);
    }

    if (!a.fused) return;
    // ---- split-K completion of every job (NS > 1), after all streams --------
    // 1. publish: one fence per warp, then per-row-tile arrival counters
    __syncwarp();
    if (lane == 0) __threadfence();
    __syncwarp();
    for (int j = 0; j < a.n_jobs; ++j) {
        const Job& J = a.jobs[j];
        if (J.NS <= 1) continue;
        const WarpRun wr = warp_run(J, b, warp);
        for (int it = wr.lo + lane; it < wr.hi; it += 32) atomicAdd(&J.counters[it - (wr.s0 + wr.seg) * J.NRT], 1u);
    }
    // 2. this CTA reduces an even share of every job's row tiles once all NS
    //    slices arrived; (job, row) pairs of all jobs are spread over the
    //    threads so the batch pays ONE latency round, not one per job
    //    (thread per row, reduce_row order -> bitwise equal to the unfused path)
    {
        int total = 0;
        for (int j = 0; j < a.n_jobs; ++j) {
            const Job& J = a.jobs[j];
            if (J.NS > 1) total += ((int)((int64_t)(b + 1) * J.NRT / G) - (int)((int64_t)b * J.NRT / G)) * kTileRows;
        }
        for (int f = tid; f < total; f += kBThreads) {
            int j = 0, lr = f;
            for (;; ++j) {  // locate job j and local row lr of flat index f
                const Job& J = a.jobs[j];
                if (J.NS <= 1) continue;
                const int n = ((int)((int64_t)(b + 1) * J.NRT / G) - (int)((int64_t)b * J.NRT / G)) * kTileRows;
                if (lr < n) break;
                lr -= n;
            }
            const Job& J = a.jobs[j];
            const int rt_lo = (int)((int64_t)b * J.NRT / G);
            const int rt = rt_lo + lr / kTileRows;
            const uint32_t* cptr = J.counters + rt;
            uint32_t seen;
            do {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(cptr) : "memory");
            } while (seen < (uint32_t)J.NS);
            const int row = rt_lo * kTileRows + lr;
            const float v = reduce_row(J.partial + row, J.NS, (int64_t)J.NRT * kTileRows);
            if (row < J.rows) static_cast<YT*>(J.y)[row] = from_f32<YT>(v);
        }
    }
    __syncthreads();  // every counter of this CTA's share was consumed
    for (int j = 0; j < a.n_jobs; ++j) {
        const Job& J = a.jobs[j];
        if (J.NS <= 1) continue;
        const int rt_lo = (int)((int64_t)b * J.NRT / G), rt_hi = (int)((int64_t)(b + 1) * J.NRT / G);
        for (int rt = rt_lo + tid; rt < rt_hi; rt += kBThreads) J.counters[rt] = 0u;  // self-reset
    }
    if (warp == 0) ABCQ_BTRACE(7);
}

// Split-K completion as a separate PDL-chained kernel (single GEMVs)
template <typename YT>
__global__ void __launch_bounds__(64) split_reduce_kernel(const float* __restrict__ partial, int NS,
                                                          int64_t stride, int rows, YT* __restrict__ y) {
    pdl_wait();
    pdl_launch_dependents();
    const int row = blockIdx.x * blockDim.x + threadIdx.x;
    if (row < rows) y[row] = from_f32<YT>(reduce_row(partial + row, NS, stride));
}

template <int NJ, typename XT, typename YT, typename ST, bool ASYM>
int launch_batch_nj(const BatchArgs& ba, int grid, cudaStream_t st) {
    KArgs<NJ> a;
    for (int j = 0; j < ba.n_jobs; ++j) a.jobs[j] = ba.jobs[j];
    a.n_jobs = ba.n_jobs;
    a.fused = ba.fused;
    a.dbg = ba.dbg;
    a.trace = ba.trace;
    auto kern = gemv_batch_kernel<NJ, XT, YT, ST, ASYM>;
    constexpr int smem = SlotGeom<ST, ASYM>::kSmem;
    static_assert(smem <= 227 * 1024, "shared memory budget");
    static_assert(SlotGeom<ST, ASYM>::kRing >= 2, "ring too shallow");
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
    cfg.blockDim = dim3(kBThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, a);
    if (e != cudaSuccess || a.fused) return (int)e;
    for (int j = 0; j < a.n_jobs; ++j) {  // unfused: one reduce kernel per split job
        const Job& J = a.jobs[j];
        if (J.NS <= 1) continue;
        cudaLaunchConfig_t rc = cfg;
        rc.blockDim = dim3(64);
        rc.gridDim = dim3((unsigned)ceil_div(J.rows, 64));
        rc.dynamicSmemBytes = 0;
        e = cudaLaunchKernelEx(&rc, split_reduce_kernel<YT>, (const float*)J.partial, J.NS,
                               (int64_t)J.NRT * kTileRows, J.rows, static_cast<YT*>(J.y));
        if (e != cudaSuccess) return (int)e;
    }
    return 0;
}

template <typename XT, typename YT, typename ST, bool ASYM>
int launch_batch_t(const BatchArgs& a, int grid, cudaStream_t st) {
    if (a.n_jobs <= 1) return launch_batch_nj<1, XT, YT, ST, ASYM>(a, grid, st);
    if (a.n_jobs <= 4) return launch_batch_nj<4, XT, YT, ST, ASYM>(a, grid, st);
    return launch_batch_nj<kMaxJobs, XT, YT, ST, ASYM>(a, grid, st);
}

template <typename XT, typename YT>
int launch_batch_xy(const BatchArgs& a, int sd, bool asym, int grid, cudaStream_t st) {
    if (sd == ABCQ_F16)
        return asym ? launch_batch_t<XT, YT, __half, true>(a, grid, st)
                    : launch_batch_t<XT, YT, __half, false>(a, grid, st);
    return asym ? launch_batch_t<XT, YT, float, true>(a, grid, st) : launch_batch_t<XT, YT, float, false>(a, grid, st);
}

// one explicit instantiation unit per (x dtype, y dtype): abcq_gemv_lut_x?y?.cu
template <typename XT, typename YT>
int launch_batch_xy_inst(const BatchArgs& a, int sd, bool asym, int grid, cudaStream_t st);
template <> int launch_batch_xy_inst<__half, __half>(const BatchArgs&, int, bool, int, cudaStream_t);
template <> int launch_batch_xy_inst<__half, float>(const BatchArgs&, int, bool, int, cudaStream_t);
template <> int launch_batch_xy_inst<float, __half>(const BatchArgs&, int, bool, int, cudaStream_t);
template <> int launch_batch_xy_inst<float, float>(const BatchArgs&, int, bool, int, cudaStream_t);

}  // namespace abcq
