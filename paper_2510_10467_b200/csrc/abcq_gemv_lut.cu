// abcq_gemv_lut.cu -- host launchers of the sm_100a LUT GEMV (kernel:
// abcq_gemv_batch.cuh): single GEMV (abcq_gemv) and batches of independent
// GEMVs (abcq_gemv_batch) share one persistent, warp-specialised kernel.
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "abcq_gemv_batch.cuh"

namespace abcq {

unsigned long long* g_trace = nullptr;  // abcq_debug_set_trace (profiling aid)
int g_rtrace_cta = -1;
int g_dbg_mode = 0;                     // abcq_debug_set_mode (profiling experiments)
// fixed cost of a (job, slice) piece in 512-byte blocks (load-balance model;
// abcq_debug_set_mode(1000 + v) sets it to v)
int g_piece_blocks = 0;  // 0: by batch size (below)
int g_partition = 0;
int g_reserved_sms = 0;  // abcq_set_reserved_sms: SMs the persistent grid leaves to concurrent kernels  // 0: greedy fill with exact piece costs; 1: proportional (abcq_debug_set_mode(3000 + v))
int g_prefill = 8;  // ring slots issued before the PDL wait (all of them); abcq_debug_set_mode(2000 + v)
constexpr int kCostScale = 64;

static size_t align256(size_t v) { return (v + 255) & ~size_t(255); }

static size_t partial_bytes(const abcq_model_t* m) {
    const int NRT = n_row_tiles(m->rows), NS = n_slices(m->cols);
    if (NS <= 1) return 0;
    return align256((size_t)NS * NRT * kTileRows * sizeof(float));  // split-K partials
}
constexpr int kCounterStride = 32;  // one 128-byte line per counter: spinning readers and arrivals of
                                    // different jobs never share a line
constexpr size_t kCounterBytes = 2 * kMaxJobs * kCounterStride * sizeof(uint32_t);  // per job: CTA arrivals, reduce blocks done
static_assert(kCounterBytes % 256 == 0, "partials after the counters stay 256-byte aligned");

// workspace of a job list: (if any job is split) the self-resetting per-job
// counters FIRST -- at the same offset for every job list, so one zero-filled
// workspace serves every model and batch launched in order on a stream
// (partials are always written before they are read) -- then every split
// job's partials
size_t lut_jobs_workspace_bytes(const abcq_model_t* const* models, int n) {
    size_t tot = 0;
    for (int j = 0; j < n; ++j) tot += partial_bytes(models[j]);
    return tot ? tot + kCounterBytes : 0;
}
size_t lut_workspace_bytes(const abcq_model_t* m) { return lut_jobs_workspace_bytes(&m, 1); }

bool lut_supports(const abcq_model_t* m, int p) {
    return m->layout == ABCQ_LAYOUT_TILED && p <= kMaxFastP && n_slices(m->cols) <= num_sms();
}

int lut_max_jobs() { return kMaxJobs; }

// fill a Job from a model + call; ws points at this job's workspace region
static void make_job(Job& J, const abcq_model_t* m, int p, const void* x, void* y, char* ws) {
    J.rows = m->rows;
    J.cols = m->cols;
    J.NRT = n_row_tiles(m->rows);
    J.NS = n_slices(m->cols);
    J.p = p;
    J.items = J.NRT * J.NS;
    J.planes = static_cast<const uint4*>(m->planes);
    J.plane_stride_u4 = m->plane_stride_bytes / 16;
    J.alpha = m->alpha[p];
    J.offset = m->asymmetric ? m->offset[p] : nullptr;
    J.x = x;
    J.glu = 0;
    J.nrm = 0;
    J.res = nullptr;
    J.nw = nullptr;
    J.xo = nullptr;
    J.eps = 0.f;
    J.y = y;
    J.partial = reinterpret_cast<float*>(ws);
    J.ncta = 0;
}

template <typename XT>
static int launch_yt(const BatchArgs& a, int yd, int sd, bool asym, int grid, cudaStream_t st) {
    return yd == ABCQ_F16 ? launch_batch_xy_inst<XT, __half>(a, sd, asym, grid, st)
                          : launch_batch_xy_inst<XT, float>(a, sd, asym, grid, st);
}

int launch_gemv_jobs(const abcq_model_t* const* models, const int* ps, const void* const* xs, void* const* ys,
                     int n, const int* x_dtypes, int y_dtype, void* ws, cudaStream_t st, const NormIn* nin,
                     const NormOut* nout, const PeerOut* pout) {
    BatchArgs a;  // passed by value (kernel parameter space)
    // one CTA per SM, minus the SMs reserved for kernels that run beside the
    // GEMV (e.g. an NCCL collective on another stream overlapping it)
    int grid = num_sms() - g_reserved_sms;
    grid = grid < 1 ? 1 : (grid > kMaxGrid ? kMaxGrid : grid);
    // fixed cost of a (job, slice) piece in blocks: measured best 300 for
    // single GEMVs and decoder-sized groups, 130-160 for large batches (bench
    // step 60.4 -> 59.6 us; tools/ab_step.py / ab_small.py with modes 1xxx)
    const int piece_blocks = g_piece_blocks > 0 ? g_piece_blocks : (n >= 8 ? 150 : 300);
    char* w = static_cast<char*>(ws);
    int items = 0;
    int64_t units = 0;
    size_t part_total = 0;
    for (int j = 0; j < n; ++j) part_total += partial_bytes(models[j]);
    uint32_t* counters = part_total ? reinterpret_cast<uint32_t*>(w) : nullptr;
    if (part_total) w += kCounterBytes;  // (kCounterBytes: a multiple of 256, partials stay aligned)
    for (int j = 0; j < n; ++j) {
        make_job(a.jobs[j], models[j], ps[j], xs[j], ys[j], w);
        a.jobs[j].glu = x_dtypes[j] == ABCQ_F16_SILU_GLU;
        if (nin && j == 0) {
            a.jobs[0].nrm = 1;
            a.jobs[0].res = static_cast<const __half*>(nin->residual);
            a.jobs[0].nw = static_cast<const __half*>(nin->norm_w);
            a.jobs[0].xo = static_cast<__half*>(nin->x_out);
            a.jobs[0].eps = nin->eps;
        }
        w += partial_bytes(models[j]);
        a.jobs[j].arrive = counters ? counters + j * kCounterStride : nullptr;
        a.jobs[j].reduced = counters ? counters + (kMaxJobs + j) * kCounterStride : nullptr;
        Job& J = a.jobs[j];
        J.ibase = items;
        J.ubase = units;
        J.w = kCostScale * ps[j] + (int)ceil_div((int64_t)kCostScale * piece_blocks, J.NRT);
        items += J.items;
        units += (int64_t)J.items * J.w;
    }
    a.n_jobs = n;
    a.pe = Peers{};
    if (pout) {
        static_assert(kMaxPeers == kMaxPeerRanks, "peer slots");
        a.pe.n = pout->n;
        a.pe.rank = pout->rank;
        a.pe.local_base = static_cast<const char*>(pout->local_base);
        for (int k = 0; k < pout->n; ++k) {
            a.pe.base[k] = static_cast<char*>(pout->base[k]);
            a.pe.sig[k] = pout->sig[k];
        }
        a.pe.state = pout->state;
    }
    a.ep = Epi{nout ? static_cast<__half*>(nout->stream) : nullptr, nout ? static_cast<const __half*>(nout->norm_w) : nullptr,
               nout ? static_cast<__half*>(nout->h) : nullptr, nout ? nout->eps : 0.f};
    a.total_items = items;
    a.total_units = units;
    // CTA ranges: greedy fill against a common budget T, with exact piece
    // accounting -- an item of job j costs p_j blocks, and every (job, slice)
    // piece a CTA touches costs g_piece_blocks more (its table build and
    // round switch), however few of its items the CTA takes. The smallest T
    // that covers all items with `grid` CTAs is found by bisection (host
    // only; the kernel reads the ranges from its parameters).
    // the partition depends only on the job shapes and precisions: memoised
    // (the bisection costs tens of microseconds of host time per call)
    std::string key;
    key.reserve(16 + 12 * n);
    auto put = [&](int v) { key.append(reinterpret_cast<const char*>(&v), sizeof(v)); };
    put(grid);
    put(g_partition);
    put(piece_blocks);
    for (int j = 0; j < n; ++j) {
        put(a.jobs[j].rows);
        put(a.jobs[j].cols);
        put(a.jobs[j].p);
    }
    static std::mutex memo_mu;
    static std::unordered_map<std::string, std::vector<int>> memo;
    bool have = false;
    {
        std::lock_guard<std::mutex> lk(memo_mu);
        auto it = memo.find(key);
        if (it != memo.end()) {
            for (int b = 0; b <= grid; ++b) a.cta_it[b] = it->second[b];
            have = true;
        }
    }
    if (have) {
    } else if (g_partition == 0) {
        auto fill = [&](int64_t T, bool write) -> bool {  // all items placed within grid CTAs?
            int j = 0, g = 0;
            for (int b = 0; b < grid; ++b) {
                if (write) a.cta_it[b] = g;
                int64_t cost = 0;
                while (g < items) {
                    while (g >= a.jobs[j].ibase + a.jobs[j].items) ++j;
                    const Job& J = a.jobs[j];
                    const int loc = g - J.ibase, s = loc / J.NRT;
                    const int pend = J.ibase + (s + 1) * J.NRT;  // end of this piece
                    const int64_t start = (int64_t)piece_blocks * 64;
                    const int64_t per = (int64_t)J.p * 64;
                    if (cost > 0 && cost + start + per > T) break;  // next CTA takes this piece
                    cost += start;
                    int64_t take = (T - cost) / per;
                    if (take < 1) take = 1;
                    if (take > pend - g) take = pend - g;
                    cost += take * per;
                    g += (int)take;
                    if (cost >= T) break;
                }
            }
            if (write) a.cta_it[grid] = g;
            return g >= items;
        };
        int64_t lo = 1, hi = (int64_t)64 * (units / 64 + 1) + (int64_t)64 * piece_blocks * 4 * (items + 1);
        while (lo < hi) {
            const int64_t mid = lo + (hi - lo) / 2;
            if (fill(mid, false)) hi = mid;
            else lo = mid + 1;
        }
        fill(lo, true);
        a.cta_it[grid] = items;
    } else {
        // (partition 1: proportional split of the per-item cost sequence)
        auto first_item = [&](int64_t u) -> int {
            int j = 0;
            while (j + 1 < n && a.jobs[j + 1].ubase <= u) ++j;
            const Job& J = a.jobs[j];
            const int64_t loc = (u - J.ubase + J.w - 1) / J.w;
            return J.ibase + (int)(loc < J.items ? loc : J.items);
        };
        for (int b = 0; b <= grid; ++b) a.cta_it[b] = first_item((int64_t)b * units / grid);
    }
    if (!have) {
        std::lock_guard<std::mutex> lk(memo_mu);
        if (memo.size() > 4096) memo.clear();
        memo.emplace(key, std::vector<int>(a.cta_it, a.cta_it + grid + 1));
    }
    for (int b = 0; b < grid; ++b) {
        a.cta_split[b] = 0;
        a.cta_j0[b] = 0;
        while (a.cta_j0[b] + 1 < n && a.jobs[a.cta_j0[b] + 1].ibase <= a.cta_it[b]) ++a.cta_j0[b];
    }
    for (int j = 0; j < n; ++j) {  // CTAs whose range touches job j (arrivals its reduce waits for)
        Job& J = a.jobs[j];
        for (int b = 0; b < grid; ++b)
            if (a.cta_it[b] < J.ibase + J.items && a.cta_it[b + 1] > J.ibase && a.cta_it[b] < a.cta_it[b + 1]) {
                ++J.ncta;
                if (J.NS > 1) a.cta_split[b] |= 1u << j;
            }
    }
    a.prefill = g_prefill;
    a.dbg = (g_dbg_mode == 1 || g_dbg_mode == 22 || g_dbg_mode == 29 || g_dbg_mode == 32 || g_dbg_mode == 33 || g_dbg_mode == 37 || g_dbg_mode == 38) ? g_dbg_mode : 0;
    static unsigned trace_seq = 0;
    a.trace = g_trace ? g_trace + (size_t)(trace_seq++ % 16) * kTraceCtas * 8 : nullptr;
    // round trace: after the 16 launch slots, [warp][round < 32][4] stamps of CTA g_rtrace_cta
    a.rtrace = g_trace && g_rtrace_cta >= 0 ? g_trace + (size_t)16 * kTraceCtas * 8 : nullptr;
    a.rtrace_cta = g_rtrace_cta;
    const abcq_model_t* m = models[0];
    const bool asym = m->asymmetric != 0;
    return x_dtypes[0] != ABCQ_F32 ? launch_yt<__half>(a, y_dtype, m->scale_dtype, asym, grid, st)
                               : launch_yt<float>(a, y_dtype, m->scale_dtype, asym, grid, st);
}

int launch_gemv_lut(const abcq_model_t* m, int p, const void* x, int x_dtype, void* y, int y_dtype,
                    void* ws, cudaStream_t st) {
    return launch_gemv_jobs(&m, &p, &x, &y, 1, &x_dtype, y_dtype, ws, st);
}

int launch_gemv_add_rmsnorm(const abcq_model_t* m, int p, const NormIn& nin, void* y, int y_dtype, void* ws,
                            cudaStream_t st) {
    const int xd = ABCQ_F16;
    const void* x = nin.x;
    return launch_gemv_jobs(&m, &p, &x, &y, 1, &xd, y_dtype, ws, st, &nin);
}

int launch_gemv_rmsnorm_out(const abcq_model_t* m, int p, const void* x, int x_dtype, void* y, const NormOut& nout,
                            void* ws, cudaStream_t st) {
    return launch_gemv_jobs(&m, &p, &x, &y, 1, &x_dtype, ABCQ_F16, ws, st, nullptr, &nout);
}

// consumer side of the fused all-gather: publish this rank's pending launch,
// then wait (lane k polls rank k's slot with acquire loads at system scope)
// until every rank published this rank's epoch; gives up after timeout_ns and
// sets *err = 1 + k instead of hanging
__global__ void peer_wait_kernel(const Peers P, uint32_t* err, long long timeout_ns) {
    const int k = threadIdx.x;
    pdl_wait();  // the peer launch before it has completed (PDL-launched: it ramps under that grid's tail)
    if (k == 0) peer_publish(P, false);
    __syncwarp();
    if (k >= P.n) return;
    const uint32_t want = *reinterpret_cast<const volatile uint32_t*>(P.state);
    const uint32_t* slot = P.sig[P.rank] + k;
    const unsigned long long t0 = globaltimer();
    for (;;) {
        uint32_t v;
        asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(slot) : "memory");
        if ((int32_t)(v - want) >= 0) break;
        if ((long long)(globaltimer() - t0) > timeout_ns) {
            atomicCAS(err, 0u, 1u + (uint32_t)k);
            break;
        }
        __nanosleep(64);
    }
}

int launch_peer_wait(const PeerOut& po, uint32_t* err, long long timeout_ns, cudaStream_t st) {
    Peers P{};
    P.n = po.n;
    P.rank = po.rank;
    P.local_base = static_cast<const char*>(po.local_base);
    for (int k = 0; k < po.n; ++k) {
        P.base[k] = static_cast<char*>(po.base[k]);
        P.sig[k] = po.sig[k];
    }
    P.state = po.state;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(1);
    cfg.blockDim = dim3(32);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return (int)cudaLaunchKernelEx(&cfg, peer_wait_kernel, P, err, timeout_ns);
}

}  // namespace abcq
