// abcq_gemv_batch.cuh -- persistent bit-plane GEMV over a list of independent
// jobs (one job = one GemvEngine.lut call, /root/reference/pkg/src/anybcq/
// gemv.py:188-222). A single GEMV is a batch of one. Building blocks (layout,
// lookup, table, TMA helpers) live in abcq_gemv_lut.cuh; DESIGN.md §3.1.
//
// One CTA per SM (a co-resident grid) of kWarps warps. The batch's items form
// one sequence split into cost-balanced CTA ranges (host-computed, see "Work
// schedule"); a range is processed in rounds of one (job, slice) piece each,
// the round's lookup table double-buffered and built by a builder group while
// the previous round streams. Every warp is its own producer and consumer: a
// private ring of SlotGeom::kRing shared-memory slots, lane 0 streaming
// (SlotGeom::kK items x one plane) of weights + that plane's scales (+
// offsets) per slot with TMA bulk copies (cp.async.bulk ...
// mbarrier::complete_tx); the warp consumes slot e while the later slots are
// in flight, and the slot stream runs on across rounds and jobs (weights are
// static: it starts before the PDL wait). Jobs split over slices (NS > 1)
// store 16-row partials; the split-K sums are completed in a fixed order
// (bitwise reproducible) by trailing CTAs of this grid (small batches) or by
// ONE PDL-chained batch_reduce_kernel.
#pragma once
#include "abcq_gemv_lut.cuh"

namespace abcq {

constexpr int kMaxJobs = kMaxBatchJobs;
constexpr int kWarps = 16;
constexpr int kBThreads = kWarps * 32;

struct Job {
    const uint4* planes;
    int64_t plane_stride_u4;
    const void* alpha;   // scale set p, tiled [i][item][lane]
    const void* offset;  // offsets of set p, tiled [item][lane] (asymmetric)
    const void* x;
    void* y;
    float* partial;      // [NRT][NS][16]: a row tile's slice partials are one contiguous run
    int rows, cols, NRT, NS, p, items;
    int glu;        // x = [g ; u] (2*cols f16): input f16(silu(g) * u) (ABCQ_F16_SILU_GLU)
    int nrm;        // input f16(f16(x + res) * inv_rms * nw) (abcq_gemv_add_rmsnorm; single-job launches)
    const __half* res;  // residual added to x (may be NULL)
    const __half* nw;   // RMSNorm weight
    __half* xo;         // x + res written back (the residual stream; may be NULL)
    float eps;
    uint32_t* arrive;   // CTAs done streaming this job (split jobs; self-resetting)
    uint32_t* reduced;  // reduce blocks done with this job (self-resetting)
    int ncta;           // CTAs whose range touches this job
    int ibase;      // first item of this job in the batch's item sequence
    int w;          // cost units per item: p blocks + the item's share of a table build
    int64_t ubase;  // first cost unit of this job (sum of items * w before it)
};

// norm epilogue (abcq_gemv_rmsnorm_out; a single split job with f16 y):
// stream += y; h = rmsnorm(stream) * w in the block completing the job last
struct Epi {
    __half* x;        // residual stream (updated in place); NULL: no epilogue
    const __half* w;  // RMSNorm weight
    __half* h;
    float eps;
};

// fused all-gather (abcq_gemv_batch_peer): every completed y row is also
// stored into each peer rank's gathered buffer at the same offset
// (symmetric layout, peer memory over NVLink). Publication is deferred by one
// launch: the NEXT peer launch (or abcq_peer_wait) -- once its PDL wait has
// seen this launch complete -- fences at system scope and writes the epoch
// into slot [rank] of every rank's signal array, from the GEMV grid's last
// CTA (the partition's remainder: it has slack), so the ~1.5 us system-scope
// fence is off the critical path (at the end of this launch it cost ~3 us
// per launch with the completion counting it needed)
constexpr int kMaxPeers = 8;
struct Peers {
    int n;                     // ranks (0: no peer outputs)
    int rank;                  // this rank (its own buffer is local_base: not stored twice)
    const char* local_base;    // this rank's gathered buffer
    char* base[kMaxPeers];     // rank q's gathered buffer
    uint32_t* sig[kMaxPeers];  // rank q's signal slots [n]
    uint32_t* state;           // this rank's [0] epochs published, [1] a launch awaits publication
};

// publish the previous peer launch (its grid, and everything before it, has
// completed: the caller is past its PDL wait), then mark this one pending
__device__ __forceinline__ void peer_publish(const Peers& P, bool mark_pending) {
    volatile uint32_t* st = P.state;
    if (st[1]) {
        __threadfence_system();
        const uint32_t e = st[0] + 1u;
        st[0] = e;
        for (int k = 0; k < P.n; ++k)
            asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(P.sig[k] + P.rank), "r"(e) : "memory");
    }
    st[1] = mark_pending ? 1u : 0u;
}

// kernel parameter: NJ job slots (1, 8 or 32 -- the smallest that fits)
constexpr int kMaxGrid = 192;  // CTAs (one per SM)

template <int NJ>
struct KArgs {
    Job jobs[NJ];
    int cta_it[kMaxGrid + 1];  // CTA b owns batch items [cta_it[b], cta_it[b+1]) (host-computed)
    uint32_t cta_split[kMaxGrid];      // CTA b: bit j set = its range touches split job j (host-computed)
    unsigned char cta_j0[kMaxGrid];    // CTA b: job of its first item (job scans start there)
    int main_ctas;             // GEMV CTAs; CTAs beyond them complete the split-K sums
    int n_jobs;
    int total_items;
    int64_t total_units;
    int prefill;  // ring slots issued before the PDL wait
    int dbg;      // profiling experiments: 1 = skip the lookups
    unsigned long long* trace;
    unsigned long long* rtrace;  // per-warp round stamps of CTA rtrace_cta (profiling), or NULL
    int rtrace_cta;
    Epi ep;                      // norm epilogue of job 0 (abcq_gemv_rmsnorm_out), ep.x == NULL: none
    Peers pe;                    // fused all-gather (abcq_gemv_batch_peer), pe.n == 0: none
};

struct BatchArgs {
    Job jobs[kMaxJobs];
    int cta_it[kMaxGrid + 1];
    uint32_t cta_split[kMaxGrid];      // CTA b: bit j set = its range touches split job j (host-computed)
    unsigned char cta_j0[kMaxGrid];    // CTA b: job of its first item (job scans start there)
    int main_ctas;
    int n_jobs;
    int total_items;
    int64_t total_units;
    int prefill;
    int dbg;
    unsigned long long* trace;  // optional per-CTA stamps (abcq_debug_set_trace)
    unsigned long long* rtrace;
    int rtrace_cta;
    Epi ep;
    Peers pe;
};

template <typename ST, bool ASYM>
struct SlotGeom {
    // items per slot: 8 (per-slot wait/issue/cursor work amortised over 8
    // blocks) where a 2-deep ring of them fits, else 4. (Weights loaded
    // straight to registers after an L2 prefetch instead of TMA staging were
    // measured 16% slower: the L2 latency lands on every slot.)
    static constexpr int kK = (sizeof(ST) == 4 && ASYM) ? 4 : 8;
    static constexpr int kW = kK * kBlockBytes;  // weights
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

// ---------------------------------------------------------------------------
// Work schedule. The batch's items (job-major, then slice-major as stored) form
// one sequence; an item of job j costs w_j units: its p_j 512-byte blocks plus
// its share of a piece's fixed cost (table build, barrier: ~kPieceBlocks
// blocks' worth, spread over the NRT items of a slice), so CTAs that cross
// many small slices get fewer bytes. CTA b owns the items whose first cost
// unit lies in [b*U/G, (b+1)*U/G). A CTA's range is cut into "rounds" of at
// most two pieces, a piece being the range's items of one (job, slice): one
// lookup-table build (two 32-column table segments) and one CTA barrier per
// round. Within a round the warps split the cost evenly; a warp's run may
// cover the tail of piece 0 and the head of piece 1 (two sub-runs).
// ---------------------------------------------------------------------------
struct Piece {
    int j, s, lo, hi;  // job, slice, batch items [lo, hi)
};
struct Round {
    Piece pc[2];
    int nseg, end;  // pc[1] valid iff nseg == 2; end = pc[nseg-1].hi
};
struct WarpRun {
    int lo, hi;  // batch items; sub-run k = [lo, hi) intersected with piece k
};

// the schedule slot of this CTA: its index, or reversed under debug mode 33
// (placement experiment: does a slow range follow the work or the SM?)
template <int NJ>
__device__ __forceinline__ int cta_slot(const KArgs<NJ>& a) {
    return a.dbg == 33 ? a.main_ctas - 1 - (int)blockIdx.x : (int)blockIdx.x;
}
template <int NJ>
__device__ __forceinline__ Piece piece_at(const KArgs<NJ>& a, int g, int it1) {
    Piece P;
    P.j = a.cta_j0[cta_slot(a)];  // g >= this CTA's first item: no scan from job 0 (param-space loads miss)
    while (P.j + 1 < a.n_jobs && a.jobs[P.j + 1].ibase <= g) ++P.j;
    const Job& J = a.jobs[P.j];
    P.s = (g - J.ibase) / J.NRT;
    P.lo = g;
    P.hi = min(J.ibase + (P.s + 1) * J.NRT, it1);
    return P;
}
template <int NJ>
__device__ __forceinline__ Round make_round(const KArgs<NJ>& a, int g, int it1) {
    // one piece per round: round r's table lives in table half r & 1, built
    // while round r-1 streams (see the kernel), so rounds cost no barrier
    Round R;
    R.pc[0] = piece_at(a, g, it1);
    R.pc[1] = R.pc[0];
    R.nseg = 1;
    R.end = R.pc[0].hi;
    return R;
}
template <int NJ>
__device__ __forceinline__ WarpRun warp_run(const KArgs<NJ>& a, const Round& R, int warp) {
    const int p0 = a.jobs[R.pc[0].j].p, p1 = a.jobs[R.pc[1].j].p;
    const int c0 = (R.pc[0].hi - R.pc[0].lo) * p0;
    const int c = c0 + (R.nseg == 2 ? (R.pc[1].hi - R.pc[1].lo) * p1 : 0);
    auto item_at = [&](int pos) -> int {  // first item starting at or after cost pos
        if (pos <= c0) return R.pc[0].lo + (pos + p0 - 1) / p0;
        return R.pc[1].lo + (pos - c0 + p1 - 1) / p1;
    };
    WarpRun w;
    w.lo = item_at((int)(((int64_t)warp * c) >> 4));  // kWarps == 16: shifts, no 64-bit division
    w.hi = item_at((int)(((int64_t)(warp + 1) * c) >> 4));
    return w;
}
static_assert(kWarps == 16, "warp_run divides by kWarps with a shift");
// Chunk-aligned split of a one-piece round (default; debug mode 32 = the cost
// split above): the piece's ceil(n / KK) slot-sized chunks go to the warps in
// rank order -- rank = (warp - off) mod 16, off = the CTA's chunk count before
// this piece, so successive short pieces land on successive warps -- one
// chunk per rank while there are fewer chunks than warps, else contiguous
// runs of floor / ceil(chunks / 16). Every slot but a piece's last is full:
// in the saturated memory system a warp's share of HBM bandwidth follows its
// bytes in flight, and the cost split left warps of short pieces (k / v
// slices of a few row tiles per CTA) with half-filled slots streaming at
// half rate (per-round stamps, tools/layer_probe.py --rtrace). Warps without
// a chunk run on into the next round (its table is already built). A CTA's
// last round keeps the cost split when it is the CTA's only round or the
// launch is a single GEMV: no round follows for idle warps, and more warps
// with part-filled slots keep more bytes in flight (single-GEMV CTAs of one
// short piece: decode p3 2.21 -> 2.28 ms/token with chunks; the two-piece
// CTAs of a 4096 x 14336 GEMV: p3 12.8 -> 13.1 us). In a batch the last
// round is chunked too (bench step 60.6 -> 60.0 us).
template <int KK>
__device__ __forceinline__ WarpRun warp_run_chunks(const Round& R, int warp, int it0) {
    const int lo = R.pc[0].lo, n = R.pc[0].hi - lo;
    const int c = (n + KK - 1) / KK;
    const int off = ((lo - it0) / KK) & 15;
    const int w = (warp - off) & 15;
    int c0, c1;
    if (c <= 16) {
        c0 = min(w, c);
        c1 = min(w + 1, c);
    } else {
        c0 = (w * c) >> 4;
        c1 = ((w + 1) * c) >> 4;
    }
    WarpRun r;
    r.lo = lo + min(c0 * KK, n);
    r.hi = lo + min(c1 * KK, n);
    return r;
}
__device__ __forceinline__ int sub_lo(const WarpRun& w, const Round& R, int k) {
    return k == 0 ? w.lo : max(w.lo, R.pc[0].hi);
}
__device__ __forceinline__ int sub_hi(const WarpRun& w, const Round& R, int k) {
    return k == 0 ? min(w.hi, R.pc[0].hi) : (R.nseg == 2 ? w.hi : w.lo);
}

// Split-K order (every completion path): row r's NS slice partials are summed
// as 4 chains, chain m = slices s = m (mod 4) in ascending s, each chain
// zero-padded to whole 16-slice blocks, then (c0 + c1) + (c2 + c3) -- so every
// path gives bitwise-identical y. Partials of row tile rt: partial[(rt*NS + s)*16 + r].
__device__ __forceinline__ const float* partial_row(const Job& J, int row) {
    return J.partial + ((int64_t)(row >> 4) * J.NS) * kTileRows + (row & 15);
}

// 16 entries of chunk c of the lookup table, t = u + 16*h (h = 0..15), from the
// chunk's 8 x values: the shared prefix over x0..x3 (bits of u) once, then the
// binary tree over x4..x7 -- every entry keeps the reference's f32 rounding
// sequence ((((0 -/+ x0) -/+ x1) ...) -/+ x7) (gemv.py:67-81), 34 adds
__device__ __forceinline__ void lut_chunk_column16(const float (&xs)[8], int u, float (&leaf)[16]) {
    float v = 0.f;
#pragma unroll
    for (int j = 0; j < 4; ++j) v = ((u >> j) & 1) ? v + xs[j] : v - xs[j];
    leaf[0] = v;
#pragma unroll
    for (int j = 4; j < 8; ++j) {
        const int n = 1 << (j - 4);  // leaves so far: index = bits 4..j-1 of t
#pragma unroll
        for (int k = n - 1; k >= 0; --k) {
            leaf[k + n] = leaf[k] + xs[j];
            leaf[k] = leaf[k] - xs[j];
        }
    }
}

constexpr int kReduceTPR = 2;  // threads per row: thread h sums chains 2h, 2h+1
constexpr int kReduceThreads = 1024;
constexpr int kReduceRPT = 2;  // rows per thread of the standalone reduce kernel
constexpr int kReduceRows = kReduceThreads / kReduceTPR * kReduceRPT;  // rows per block
// (few, fat blocks: the bench batch's reduce is one block per SM, and the
// block dispatch of hundreds of 1024-thread blocks onto the SMs the GEMV
// grid frees was measured at ~5 us)

// one reduce block: rows [blk*RPB, (blk+1)*RPB) of the blk-th block's job
// (blocks laid out job by job), kReduceTPR threads per row (blockDim.x == kReduceTPR*RPB).
// RELEASE: let the dependent grid launch once this block's job has arrived --
// not earlier, or the next kernel's CTAs take the SMs that the remaining
// reduce blocks of this grid still need.
template <int NJ, typename YT, int RPB, int RPT, bool RELEASE, bool PRE_WAIT = false>
__device__ __forceinline__ int reduce_rows(const KArgs<NJ>& a, int blk) {
    constexpr int rpb = RPB;
    // blocks laid out job by job, jobs of more than 16 slices first: their
    // completion is the longest, and the blocks reach SMs in index order as
    // the GEMV CTAs retire (debug mode 29: plain job order)
    int j = -1, nbj = 0;
    for (int pass = (a.dbg == 29 ? 1 : 0); pass < 2 && j < 0; ++pass) {
        for (int jj = 0; jj < a.n_jobs; ++jj) {
            const Job& J = a.jobs[jj];
            if (J.NS <= 1 || (pass == 0 && J.NS <= 16) || (pass == 1 && a.dbg != 29 && J.NS > 16)) continue;
            nbj = (J.rows + rpb - 1) / rpb;
            if (blk < nbj) {
                j = jj;
                break;
            }
            blk -= nbj;
        }
    }
    if (j < 0) {
        if (PRE_WAIT) pdl_wait();
        if (RELEASE) pdl_launch_dependents();
        return -1;
    }
    const Job& J = a.jobs[j];
    if (PRE_WAIT) pdl_wait();  // (after the param-space job scan: y may still be read by the previous kernel)
    // wait for this job's CTA arrivals only (acquire), so the reduction
    // overlaps the GEMV CTAs still streaming other jobs
    if (threadIdx.x == 0) {
        if (a.trace && j < 32) atomicMax(&a.trace[156 * 8 + j], globaltimer());  // last task start of job j
        uint32_t seen;
        for (;;) {  // relaxed polling, one acquire fence once the count is complete
            asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(J.arrive) : "memory");
            if (seen >= (uint32_t)J.ncta) break;
            __nanosleep(20);
        }
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        if (a.trace) {
            const unsigned long long t = globaltimer();
            atomicMin(&a.trace[148 * 8 + 1], t);
            if (j < 32) atomicMax(&a.trace[164 * 8 + j], t);  // last block of job j past its wait
        }
    }
    __syncthreads();
    if (RELEASE) pdl_launch_dependents();
    constexpr int CPT = 4 / kReduceTPR;  // chains per thread
    constexpr int kSpan = RPB / RPT;     // rows between a thread's rows
    const int sub = threadIdx.x % kReduceTPR;
    int row[RPT];
    const float* pp[RPT];
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
        row[q] = blk * rpb + q * kSpan + threadIdx.x / kReduceTPR;
        pp[q] = partial_row(J, row[q] < J.rows ? row[q] : 0);
    }
    const int nterm = 4 * ((J.NS + 15) / 16);  // terms per chain, zero-padded to whole 16-slice blocks
    float c[RPT][CPT];
#pragma unroll
    for (int q = 0; q < RPT; ++q)
#pragma unroll
        for (int u = 0; u < CPT; ++u) c[q][u] = 0.f;
    // loads per row in flight: 32 for one row per thread (the trailing CTAs of
    // single GEMVs: a 56-slice down projection's sums in one L2 round trip),
    // 16 for the separate kernel's two rows per thread
    constexpr int KB = RPT == 1 ? 32 : 16;
    for (int b0 = 0; b0 < nterm; b0 += KB / CPT) {
        float v[RPT][KB];
#pragma unroll
        for (int q = 0; q < RPT; ++q)
#pragma unroll
            for (int k = 0; k < KB; ++k) {  // chain sub*CPT + k%CPT, term b0 + k/CPT
                const int term = b0 + k / CPT, s = term * 4 + sub * CPT + k % CPT;
                v[q][k] = (term < nterm && s < J.NS) ? __ldcg(pp[q] + s * kTileRows) : 0.f;
            }
#pragma unroll
        for (int q = 0; q < RPT; ++q)
#pragma unroll
            for (int k = 0; k < KB; ++k)
                if (b0 + k / CPT < nterm) c[q][k % CPT] += v[q][k];
    }
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
        float tot = c[q][0];
#pragma unroll
        for (int u = 1; u < CPT; ++u) tot += c[q][u];  // CPT == 2: c0+c1 | c2+c3
#pragma unroll
        for (int w = 1; w < kReduceTPR; w <<= 1) tot += __shfl_xor_sync(0xffffffffu, tot, w);  // (c0+c1)+(c2+c3)
        if (sub == 0 && row[q] < J.rows) {
            YT* yr = static_cast<YT*>(J.y) + row[q];
            const YT v = from_f32<YT>(tot);
            *yr = v;
            if (a.pe.n) {  // the same row into every peer's gathered buffer (NVLink stores)
                const int64_t off = reinterpret_cast<const char*>(yr) - a.pe.local_base;
                for (int k = 0; k < a.pe.n; ++k)
                    if (k != a.pe.rank) *reinterpret_cast<YT*>(a.pe.base[k] + off) = v;
            }
        }
    }
    const bool epi = j == 0 && a.ep.x != nullptr;
    if (epi) __threadfence();  // release the y rows to the block that runs the norm epilogue
    __syncthreads();
    if (threadIdx.x == 0) {
        if (a.trace) {  // profiling: last block end, per job
            const unsigned long long t = globaltimer();
            atomicMax(&a.trace[148 * 8 + 2], t);
            if (j < 32) atomicMax(&a.trace[149 * 8 + j], t);
        }
    }
    // (the job's norm epilogue, if any, runs in the block that completes it last)
    bool last = false;
    if (threadIdx.x == 0) {
        last = atomicAdd(J.reduced, 1u) == (uint32_t)(nbj - 1);
        if (last) {  // last block of job j: recycle
            *J.arrive = 0u;
            *J.reduced = 0u;
        }
    }
    if (epi) return __syncthreads_or(last) ? j : -1;  // (block-uniform)
    return -1;
}

// norm epilogue of job J (the block that completed its split-K sums last,
// 512 threads): stream += y; h = rmsnorm(stream) * w -- add_rmsnorm_kernel's
// arithmetic through the same helpers, so bitwise equal to that launch
__device__ __forceinline__ void rmsnorm_epilogue(const Job& J, const Epi& E, float* red) {
    __threadfence();  // acquire: every completion block's y rows
    float v[16];
    const int t = threadIdx.x;
    const float ss = rms_load(E.x, static_cast<const __half*>(J.y), J.rows, t, v);
    const float inv = rms_inv(ss, J.rows, E.eps, red);
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        const int i = (k < 8 ? 8 * t + k : 4096 + 8 * t + (k - 8));
        if (i < J.rows) {
            E.x[i] = __float2half_rn(v[k]);
            E.h[i] = __float2half_rn(v[k] * inv * __half2float(E.w[i]));
        }
    }
}

// profiling stamps (abcq_debug_set_trace; tools/layer_probe.py reads them):
// per CTA (8 slots of %globaltimer) 0 start, 1 release fence done, 2 first
// table ready, 3 streams done (max over warps), 4 arrivals issued, 5 all
// warps done, 6 = rounds, 7 past the PDL wait; per job (rows 149 / 156 / 160
// / 164 of the launch's slot): last row reduced, last reduce block started,
// last CTA arrival, last reduce block past its wait; row 148: reduce grid
// first start / first wait passed / end
#define ABCQ_BTRACE(k)                                                                   \
    do {                                                                                 \
        if (a.trace && lane == 0) atomicMax(&a.trace[blockIdx.x * 8 + (k)], globaltimer()); \
    } while (0)

template <int NJ, typename XT, typename YT, typename ST, bool ASYM, bool FUSED>
__global__ void __launch_bounds__(kBThreads, 1) gemv_batch_kernel(const __grid_constant__ KArgs<NJ> a) {
    if constexpr (FUSED) {
        if ((int)blockIdx.x >= a.main_ctas) {
            // trailing CTAs: split-K completion (they get SMs as GEMV CTAs
            // retire) -- for batches whose reduce fits one wave; larger ones
            // use the separate kernel (a trailing CTA needs a whole SM, and
            // the role's code in the kernel costs the streams ~7%)
            const int ej = reduce_rows<NJ, YT, kBThreads / kReduceTPR, 1, true, true>(a, blockIdx.x - a.main_ctas);
            if constexpr (std::is_same<YT, __half>::value) {
                extern __shared__ __align__(1024) char ep_smem[];
                if (ej >= 0) rmsnorm_epilogue(a.jobs[ej], a.ep, reinterpret_cast<float*>(ep_smem));
            }
            return;
        }
    }
    using SG = SlotGeom<ST, ASYM>;
    constexpr int kK = SG::kK;
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
    const int b = cta_slot(a), G = gridDim.x;
    if (warp == 0) ABCQ_BTRACE(0);
    uint64_t* mybar = bars + warp * R;
    if (lane == 0) {
        for (int s = 0; s < R; ++s) mbar_init(&mybar[s], 1);
        fence_mbar_init();
    }
    __syncwarp();
    const int it0 = a.cta_it[b], it1 = a.cta_it[b + 1];

    // ---- this warp's slot stream: rounds -> sub-runs -> chunks of SlotGeom::kK items ->
    // planes; the issue cursor keeps its source pointers in registers and
    // advances them incrementally (the job table in parameter space is read
    // only when the cursor enters a new sub-run)
    struct Cur {
        int rs, rend, mid, whi;  // round start / end, piece boundary, warp run end
        int hi, c, i, p;         // sub-run end, chunk start, plane, job precision
        const char* w;           // planes + i*plane_stride + item*512   (bytes)
        const ST* al;            // alpha + (i*items + item)*32
        const ST* z;             // offset + item*32
        int64_t pst;             // plane stride (bytes)
        int64_t ast;             // items*32: scale elements per plane
    };
    auto enter_sub = [&](Cur& k, int j, int lo, int hi) {
        const Job& J = a.jobs[j];
        const int loc = lo - J.ibase;
        k.hi = hi;
        k.c = lo;
        k.i = 0;
        k.p = J.p;
        k.pst = J.plane_stride_u4 * 16;
        k.ast = (int64_t)J.items * 32;
        k.w = reinterpret_cast<const char*>(J.planes) + (int64_t)loc * kBlockBytes;
        k.al = static_cast<const ST*>(J.alpha) + (int64_t)loc * 32;
        k.z = ASYM ? static_cast<const ST*>(J.offset) + (int64_t)loc * 32 : nullptr;
    };
    // first non-empty sub-run at or after round start rs (k.rs = it1: exhausted)
    auto enter_round = [&](Cur& k, int rs) {
        for (; rs < it1;) {
            const Round Rn = make_round(a, rs, it1);
            const WarpRun wr = (a.dbg == 32 || (Rn.end >= it1 && (a.n_jobs == 1 || Rn.pc[0].lo == it0))) ? warp_run(a, Rn, warp) : warp_run_chunks<kK>(Rn, warp, it0);
            k.rs = rs;
            k.rend = Rn.end;
            k.mid = Rn.pc[0].hi;
            k.whi = sub_hi(wr, Rn, 1);
            const int lo0 = sub_lo(wr, Rn, 0), hi0 = sub_hi(wr, Rn, 0);
            const int lo1 = sub_lo(wr, Rn, 1), hi1 = sub_hi(wr, Rn, 1);
            const bool first = lo0 < hi0;
            if (first || lo1 < hi1) {  // (selects, not an indexed Round: no local memory)
                enter_sub(k, first ? Rn.pc[0].j : Rn.pc[1].j, first ? lo0 : lo1, first ? hi0 : hi1);
                return;
            }
            rs = Rn.end;
        }
        k.rs = it1;
    };
    auto advance = [&](Cur& k) {
        if (++k.i < k.p) {
            k.w += k.pst;
            k.al += k.ast;
            return;
        }
        k.i = 0;
        k.c += kK;
        if (k.c < k.hi) {
            k.w += kK * kBlockBytes - (k.p - 1) * k.pst;
            k.al += kK * 32 - (k.p - 1) * k.ast;
            if constexpr (ASYM) k.z += kK * 32;
            return;
        }
        if (k.hi == k.mid && k.whi > k.mid) {  // sub-run 0 done, sub-run 1 follows
            const Round Rn = make_round(a, k.rs, it1);
            enter_sub(k, Rn.pc[1].j, k.mid, k.whi);
            return;
        }
        enter_round(k, k.rend);
    };
    const uint64_t pol = l2_evict_first_policy();
    const uint64_t pol_keep = l2_evict_last_policy();
    // issue the TMA copies of the cursor's element into slot s (lane 0 only)
    auto issue = [&](const Cur& k, int s) {
        const int cnt = min(kK, k.hi - k.c);
        char* st = slot_ptr(warp * R + s);
        const uint32_t wb = cnt * kBlockBytes, ab = cnt * 32 * (uint32_t)sizeof(ST);
        const bool z = ASYM && k.i == 0;
        if (lane == 0) {
            mbar_arrive_expect_tx(&mybar[s], wb + ab + (z ? ab : 0));
            bulk_g2s_hint(st, k.w, wb, &mybar[s], pol);
            bulk_g2s_hint(st + SG::kW, k.al, ab, &mybar[s], pol);
            if (z) bulk_g2s_hint(st + SG::kW + SG::kA, k.z, ab, &mybar[s], pol);
        }
    };

    Cur ic;  // issue cursor: runs R elements ahead of consumption
    enter_round(ic, it0);
    // static model data: fill the ring (a.prefill slots, default all) before
    // waiting on the previous kernel -- the weights land during the wait
    int s_fill = 0;
    for (; s_fill < a.prefill && s_fill < R && ic.rs < it1; ++s_fill) {
        issue(ic, s_fill);
        advance(ic);
    }
    // everything that reads only parameters / shared memory happens before the
    // PDL wait too: the first two rounds' pieces and x addresses, the lookup
    // column registers (param-space loads miss the constant cache at kernel start)
    const bool has0 = it0 < it1;
    Round R0, R1;
    bool has1 = false;
    const XT* xp0 = nullptr;
    const XT* xp1 = nullptr;
    int xk0 = 0, xk1 = 0, xc0 = 0, xc1 = 0, xg0 = 0, xg1 = 0;
    if (has0) {
        R0 = make_round(a, it0, it1);
        const Job& J0 = a.jobs[R0.pc[0].j];
        xp0 = static_cast<const XT*>(J0.x);
        xk0 = R0.pc[0].s * kSliceCols + 8 * (tid & 31);
        xc0 = J0.cols;
        xg0 = J0.glu;
        has1 = R0.end < it1;
        if (has1) {
            R1 = make_round(a, R0.end, it1);
            const Job& J1 = a.jobs[R1.pc[0].j];
            xp1 = static_cast<const XT*>(J1.x);
            xk1 = R1.pc[0].s * kSliceCols + 8 * (tid & 31);
            xc1 = J1.cols;
            xg1 = J1.glu;
        }
    }
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

    // ---- lookup tables: round r uses table half r & 1 (32 columns each) -----
    // Rounds 0 and 1 are built by the whole CTA up front. Round r+2's table is
    // built by the 4 warps of builder group r mod 4 (each 4 of the 16 entry
    // columns): they load its x when they enter round r, finish their round-r
    // work, wait until all warps are done with round r (a shared counter) and
    // build into the half round r used; the last builder publishes it. A warp
    // entering round r >= 2 only waits if that table is not ready yet -- no
    // CTA-wide barrier between rounds, fast warps run on into the next round.
    static_assert(kBThreads == 512 && kWarps == 16, "4 builder groups of 4 warps; 16 entry columns");
    volatile int* done = reinterpret_cast<volatile int*>(smem + 768);   // [2] warps done with round r (r & 1)
    volatile int* ready = reinterpret_cast<volatile int*>(smem + 776);  // [2] round whose table half h holds
    volatile int* bcnt = reinterpret_cast<volatile int*>(smem + 784);   // [2] builders done with half h
    auto build_entries = [&](const float (&xv)[8], int half_sel, int c, int u) {
        float ev[16];
        lut_chunk_column16(xv, u, ev);
        float* col = table + half_sel * 32 + c;
#pragma unroll
        for (int h = 0; h < 16; ++h) col[(u + 16 * h) * 64] = ev[h];
        if (ASYM && u == 15) csum[half_sel * 32 + c] = ev[15];  // T[255] = chunk sum
    };
    float* nrm_red = reinterpret_cast<float*>(smem + 800);  // [17]: RMSNorm statistics (norm input mode)
    auto load_job_x8 = [&](const Job& Jn, int k0, float (&xv)[8]) {
        if (Jn.nrm) {  // f16(f16(x + res) * inv * w): add_rmsnorm_kernel's expression, bitwise
            const float inv = nrm_red[16];
            const __half* xh = static_cast<const __half*>(Jn.x);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int i = k0 + j;
                float v = 0.f;
                if (i < Jn.cols) {
                    v = __half2float(xh[i]);
                    if (Jn.res) v = __half2float(__float2half_rn(v + __half2float(Jn.res[i])));
                    v = __half2float(__float2half_rn(v * inv * __half2float(Jn.nw[i])));
                }
                xv[j] = v;
            }
        } else {
            load_x8_any<XT>(static_cast<const XT*>(Jn.x), k0, Jn.cols, Jn.glu, xv);
        }
    };
    auto piece_x = [&](const Round& Rn, int c, float (&xv)[8]) {
        const Job& Jn = a.jobs[Rn.pc[0].j];
        load_job_x8(Jn, Rn.pc[0].s * kSliceCols + 8 * c, xv);
    };

    int e = 0;  // consumed elements (slot = e % R, phase = (e / R) & 1)
    int round = 0;
    pdl_wait();  // x, y and the workspace belong to the previous kernel
    pdl_launch_dependents();
    if (a.trace && tid == 0) a.trace[blockIdx.x * 8 + 7] = globaltimer();  // past the PDL wait
    if (a.pe.n && tid == 0 && (int)blockIdx.x == a.main_ctas - 1) peer_publish(a.pe, true);
    if (a.jobs[0].nrm) {  // RMSNorm statistics of the whole input (every CTA, bitwise as add_rmsnorm)
        const Job& J = a.jobs[0];
        float v[16];
        const float ss = rms_load(static_cast<const __half*>(J.x), J.res, J.cols, tid, v);
        rms_inv(ss, J.cols, J.eps, nrm_red);
        if (J.xo && blockIdx.x == 0) {  // the updated residual stream (one CTA writes it)
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                const int i = (k < 8 ? 8 * tid + k : 4096 + 8 * tid + (k - 8));
                if (i < J.cols) J.xo[i] = __float2half_rn(v[k]);
            }
        }
    }
    {
        float xv0[8], xv1[8];
        if (has0) {
            if (a.jobs[R0.pc[0].j].nrm) load_job_x8(a.jobs[R0.pc[0].j], xk0, xv0);
            else load_x8_any<XT>(xp0, xk0, xc0, xg0, xv0);
        }
        if (has1) {
            if (a.jobs[R1.pc[0].j].nrm) load_job_x8(a.jobs[R1.pc[0].j], xk1, xv1);
            else load_x8_any<XT>(xp1, xk1, xc1, xg1, xv1);
        }
        for (; s_fill < R && ic.rs < it1; ++s_fill) {  // rest of the ring, behind x
            issue(ic, s_fill);
            advance(ic);
        }
        if (has0) build_entries(xv0, 0, tid & 31, tid >> 5);
        if (has1) build_entries(xv1, 1, tid & 31, tid >> 5);
        if (tid == 0) {
            done[0] = done[1] = 0;
            bcnt[0] = bcnt[1] = 0;
            ready[0] = 0;
            ready[1] = 1;
        }
        __syncthreads();
    }
    if (warp == 0) ABCQ_BTRACE(2);
#define ABCQ_RTRACE(k)                                                                          \
    do {                                                                                        \
        if (a.rtrace && (int)blockIdx.x == a.rtrace_cta && lane == 0 && round < 32)             \
            a.rtrace[(warp * 32 + round) * 4 + (k)] = globaltimer();                            \
    } while (0)
    for (int rs = it0; rs < it1; ++round) {
        const Round Rd = make_round(a, rs, it1);
        ABCQ_RTRACE(0);
        if (round >= 2) {  // table of round `round` (built by the last warp of round-2)
            while (ready[round & 1] < round) __nanosleep(64);
            __threadfence_block();
        }
        ABCQ_RTRACE(1);
        const WarpRun wr = (a.dbg == 32 || (Rd.end >= it1 && (a.n_jobs == 1 || Rd.pc[0].lo == it0))) ? warp_run(a, Rd, warp) : warp_run_chunks<kK>(Rd, warp, it0);
        // builder of round+2's table? then fetch its x now (used after this round)
        const bool builder = (warp >> 2) == (round & 3);
        bool build_next = false;
        float bx[8];
        if (builder && Rd.end < it1) {
            const Round Rn1 = make_round(a, Rd.end, it1);
            if (Rn1.end < it1) {
                build_next = true;
                piece_x(make_round(a, Rn1.end, it1), lane, bx);
            }
        }

        // ---- stream this warp's elements of the round ---------------------------
        auto run = [&](auto seg_tag) {
            constexpr int SEG = decltype(seg_tag)::value;  // table half = round & 1
            const int lo = sub_lo(wr, Rd, 0), hi = sub_hi(wr, Rd, 0);
            if (lo >= hi) return;
            const Piece& P = Rd.pc[0];
            const Job& J = a.jobs[P.j];
            float gx = 0.f;
            if constexpr (ASYM) {
                for (int c = 0; c < 16; ++c) gx += csum[SEG * 32 + half * 16 + c];
            }
            YT* __restrict__ y = static_cast<YT*>(J.y);
            float* __restrict__ part = J.partial + (int64_t)P.s * kTileRows;  // + rt*NS*16 + r
            const int tile0 = J.ibase + P.s * J.NRT;  // batch item of row tile 0 of this slice
            const int p = J.p, NS = J.NS, rows = J.rows;
            for (int c = lo; c < hi; c += kK) {
                const int cnt = min(kK, hi - c);
                float acc[kK];
#pragma unroll
                for (int q = 0; q < kK; ++q) acc[q] = 0.f;
                for (int i = 0; i < p; ++i, ++e) {
                    const int s = e % R;
                    mbar_wait(&mybar[s], (e / R) & 1);
                    const char* st = slot_ptr(warp * R + s);
                    if (a.dbg != 1) {
                        // a slot's kK elements are independent: load them all, then
                        // look up -- no per-element branch in the full-slot case, so
                        // the scheduler interleaves the four lookup chains
                        auto elems = [&](auto q0_tag, auto n_tag) {  // items [Q0, Q0 + N) of the slot
                            constexpr int Q0 = decltype(q0_tag)::value, N = decltype(n_tag)::value;
                            uint4 wv[N];
                            float sc[N];
#pragma unroll
                            for (int q = 0; q < N; ++q) {
                                wv[q] = *reinterpret_cast<const uint4*>(st + (Q0 + q) * kBlockBytes + lane * 16);
                                sc[q] = to_f32<ST>(reinterpret_cast<const ST*>(st + SG::kW)[(Q0 + q) * 32 + lane]);
                            }
#pragma unroll
                            for (int q = 0; q < N; ++q) acc[Q0 + q] = fmaf(sc[q], lut16<SEG>(wv[q], rb), acc[Q0 + q]);
                            if constexpr (ASYM) {
                                if (i == 0) {
#pragma unroll
                                    for (int q = 0; q < N; ++q)
                                        acc[Q0 + q] = fmaf(
                                            to_f32<ST>(reinterpret_cast<const ST*>(st + SG::kW + SG::kA)[(Q0 + q) * 32 + lane]),
                                            gx, acc[Q0 + q]);
                                }
                            }
                        };
                        using I0 = std::integral_constant<int, 0>;
                        using I4 = std::integral_constant<int, 4>;
                        auto group = [&](auto q0_tag, int n) {  // n = 1..4 items from Q0
                            if (n == 4) elems(q0_tag, I4{});
                            else if (n == 3) elems(q0_tag, std::integral_constant<int, 3>{});
                            else if (n == 2) elems(q0_tag, std::integral_constant<int, 2>{});
                            else elems(q0_tag, std::integral_constant<int, 1>{});
                        };
                        if (cnt == kK) {
                            elems(I0{}, I4{});
                            if constexpr (kK == 8) elems(I4{}, I4{});
                        } else {
                            group(I0{}, cnt < 4 ? cnt : 4);
                            if constexpr (kK == 8) {
                                if (cnt > 4) group(I4{}, cnt - 4);
                            }
                        }
                    }
                    __syncwarp();  // every lane has consumed slot s
                    if (ic.rs < it1) {  // refill it with the element R ahead
                        issue(ic, s);
                        advance(ic);
                    }
                }
                // chunk done: combine the slice's two groups (lanes l, l+16), emit 16 rows per item
                float outv[kK];
#pragma unroll
                for (int q = 0; q < kK; ++q) outv[q] = acc[q] + __shfl_down_sync(0xffffffffu, acc[q], 16);
                if (NS == 1) {
#pragma unroll
                    for (int q = 0; q < kK; ++q) {
                        const int row = (c + q - tile0) * kTileRows + lane;
                        if (q < cnt && lane < 16 && row < rows) y[row] = from_f32<YT>(outv[q]);
                    }
                } else {
#pragma unroll
                    for (int q = 0; q < kK; ++q)
                        if (q < cnt && lane < 16)
                            st_f32_hint(part + (int64_t)(c + q - tile0) * NS * kTileRows + lane, outv[q], pol_keep);
                }
            }
        };
        if (round & 1)
            run(std::integral_constant<int, 1>{});
        else
            run(std::integral_constant<int, 0>{});
        // done with round `round`; builders fill round+2's table into this half
        __syncwarp();
        ABCQ_RTRACE(2);
        if (lane == 0) atomicAdd((int*)&done[round & 1], 1);
        if (build_next) {
            while (done[round & 1] < kWarps) __nanosleep(32);
            __threadfence_block();
            ABCQ_RTRACE(3);
#pragma unroll
            for (int k = 0; k < 4; ++k) build_entries(bx, round & 1, lane, (warp & 3) * 4 + k);
            __syncwarp();
            __threadfence_block();
            int old = 0;
            if (lane == 0) old = atomicAdd((int*)&bcnt[round & 1], 1);
            old = __shfl_sync(0xffffffffu, old, 0);
            if (old == 3 && lane == 0) {  // last of the 4 builders: recycle the counters, publish
                done[round & 1] = 0;
                bcnt[round & 1] = 0;
                __threadfence_block();
                ready[round & 1] = round + 2;
            }
        }
        rs = Rd.end;
    }

    ABCQ_BTRACE(3);
    // publish this CTA's split-K partials: one release per CTA, one arrival per
    // split job it touched -- the reduce kernel starts on a job as soon as all
    // of its CTAs arrived, while stragglers are still streaming other jobs
    // (per-warp release arrivals were measured slower: one hot counter)
    __syncthreads();
    if (a.trace && tid == 0) a.trace[blockIdx.x * 8 + 5] = globaltimer();  // all warps done
    if (warp == 0 && it0 < it1) {  // lane j signals job j (each lane: release fence, then its arrival)
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        if (a.trace && lane == 0) a.trace[blockIdx.x * 8 + 1] = globaltimer();  // fence done
        const uint32_t mask = a.cta_split[b];
        for (int j = lane; j < a.n_jobs; j += 32) {
            if ((mask >> j) & 1u) {
                asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(a.jobs[j].arrive) : "memory");
                if (a.trace && j < 32) atomicMax(&a.trace[160 * 8 + j], globaltimer());  // last arrival
            }
        }
    }
    if (a.trace && tid == 0) {
        a.trace[blockIdx.x * 8 + 6] = round;
        a.trace[blockIdx.x * 8 + 4] = globaltimer();  // CTA done (arrivals issued)
    }
}

// Split-K completion as ONE PDL-chained kernel for the whole batch: block k
// completes kReduceRows rows of one split job (blocks are laid out job by job,
// so the job lookup is block-uniform). Two threads per row: thread h sums
// chains 2h and 2h+1 of the split-K order (chain m = slices s = m mod 4,
// ascending, zero-padded to whole 16-slice blocks), up to 16 loads in flight;
// then (c0 + c1) + (c2 + c3) -- independent of the batch composition.
// Standalone split-K completion kernel (PDL-chained; debug mode 22): the
// default folds these blocks into the GEMV grid itself (trailing CTAs,
// gemv_batch_kernel) -- one launch per batch, no kernel boundary.
template <int NJ, typename YT>
__global__ void __launch_bounds__(kReduceThreads, 1) batch_reduce_kernel(const __grid_constant__ KArgs<NJ> a) {
    if (a.trace && threadIdx.x == 0) atomicMin(&a.trace[148 * 8 + 0], globaltimer());
    reduce_rows<NJ, YT, kReduceRows, kReduceRPT, true>(a, blockIdx.x);
    pdl_wait();  // the GEMV grid (y of unsplit jobs) completes before this grid does
}

template <int NJ, typename XT, typename YT, typename ST, bool ASYM>
int launch_batch_nj(const BatchArgs& ba, int grid, cudaStream_t st) {
    KArgs<NJ> a;
    for (int j = 0; j < ba.n_jobs; ++j) a.jobs[j] = ba.jobs[j];
    a.n_jobs = ba.n_jobs;
    a.main_ctas = grid;
    for (int i = 0; i <= grid && i <= kMaxGrid; ++i) a.cta_it[i] = ba.cta_it[i];
    for (int i = 0; i < grid && i < kMaxGrid; ++i) {
        a.cta_split[i] = ba.cta_split[i];
        a.cta_j0[i] = ba.cta_j0[i];
    }
    a.total_items = ba.total_items;
    a.total_units = ba.total_units;
    a.prefill = ba.prefill;
    a.dbg = ba.dbg;
    a.trace = ba.trace;
    a.rtrace = ba.rtrace;
    a.rtrace_cta = ba.rtrace_cta;
    a.ep = ba.ep;
    a.pe = ba.pe;
    int rblocks = 0;  // split-K completion blocks (rows / (kBThreads/4) per job)
    constexpr int kFusedRows = kBThreads / kReduceTPR;
    for (int j = 0; j < ba.n_jobs; ++j)
        if (ba.jobs[j].NS > 1) rblocks += (ba.jobs[j].rows + kFusedRows - 1) / kFusedRows;
    constexpr bool kCanFuse = NJ <= 8;  // fused variant instantiated for single GEMVs and small batches
    const bool fused = kCanFuse && ba.dbg != 22 && rblocks <= grid;
    if (ba.ep.x && (!fused || ba.n_jobs != 1 || ba.jobs[0].NS <= 1 || !std::is_same<YT, __half>::value))
        return (int)cudaErrorInvalidConfiguration;  // the norm epilogue runs in the trailing completion CTAs
    auto kern = fused ? gemv_batch_kernel<NJ, XT, YT, ST, ASYM, kCanFuse> : gemv_batch_kernel<NJ, XT, YT, ST, ASYM, false>;
    constexpr int smem = SlotGeom<ST, ASYM>::kSmem;
    static_assert(smem <= 227 * 1024, "shared memory budget");
    static_assert(SlotGeom<ST, ASYM>::kRing >= 2, "ring too shallow");
    int dev = 0;
    cudaGetDevice(&dev);
    static bool attr_set[64] = {};  // per instantiation and device
    if (dev < 64 && !attr_set[dev]) {
        // the reduce kernel keeps the GEMV's shared-memory carveout: an SM that
        // ran it must not be reconfigured before the next GEMV CTA can start
        cudaError_t e = cudaFuncSetAttribute(batch_reduce_kernel<NJ, YT>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                             cudaSharedmemCarveoutMaxShared);
        if (e != cudaSuccess) return (int)e;
        for (auto kf : {gemv_batch_kernel<NJ, XT, YT, ST, ASYM, kCanFuse>, gemv_batch_kernel<NJ, XT, YT, ST, ASYM, false>}) {
            e = cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            if (e != cudaSuccess) return (int)e;
            e = cudaFuncSetAttribute(kf, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
            if (e != cudaSuccess) return (int)e;
        }
        attr_set[dev] = true;
    }
    int sep_blocks = 0;  // blocks of the separate completion kernel
    for (int j = 0; j < ba.n_jobs; ++j)
        if (ba.jobs[j].NS > 1) sep_blocks += (ba.jobs[j].rows + kReduceRows - 1) / kReduceRows;
    if (a.pe.n) {
        for (int j = 0; j < ba.n_jobs; ++j)
            if (ba.jobs[j].NS <= 1) return (int)cudaErrorInvalidConfiguration;  // peer rows leave through the completion
    }
    cudaLaunchConfig_t cfg = {};
    const bool separate = !fused;
    cfg.gridDim = dim3(grid + (separate ? 0 : rblocks));
    cfg.blockDim = dim3(kBThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, a);
    if (e != cudaSuccess || !separate) return (int)e;
    const int nblocks = sep_blocks;  // one separate reduce launch
    if (nblocks == 0) return 0;
    cudaLaunchConfig_t rc = cfg;
    rc.blockDim = dim3(kReduceThreads);
    rc.gridDim = dim3((unsigned)nblocks);
    rc.dynamicSmemBytes = 0;
    return (int)cudaLaunchKernelEx(&rc, batch_reduce_kernel<NJ, YT>, a);
}

template <typename XT, typename YT, typename ST, bool ASYM>
int launch_batch_t(const BatchArgs& a, int grid, cudaStream_t st) {
    if (a.n_jobs <= 1) return launch_batch_nj<1, XT, YT, ST, ASYM>(a, grid, st);
    if (a.n_jobs <= 8) return launch_batch_nj<8, XT, YT, ST, ASYM>(a, grid, st);
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
