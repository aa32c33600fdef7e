// abcq_gemv_cluster.cu -- host side of the cluster GEMV (kernel:
// abcq_gemv_cluster.cuh): launch geometry, occupancy queries, dispatch.
#include <mutex>

#include "abcq_gemv_cluster.cuh"

namespace abcq {

int g_cl_force = 0;  // abcq_debug_set_mode(5000 + 100*slots + 10*C + tcw): forced geometry (0 = automatic)
int g_cl_warps = 0;  // abcq_debug_set_mode(6000 + W): consumer warps per CTA (0 = automatic)

namespace cl {

// clusters of size C co-resident at one CTA per SM (queried once per device)
static int max_clusters(int C) {
    static std::mutex mu;
    static int cache[64][5] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    const int ci = C == 1 ? 0 : C == 2 ? 1 : C == 4 ? 2 : C == 8 ? 3 : 4;
    std::lock_guard<std::mutex> lk(mu);
    if (dev < 64 && cache[dev][ci]) return cache[dev][ci];
    int n = 0;
    if (C == 1) {
        n = num_sms();
    } else {
        auto kern = gemv_cluster_kernel<__half, __half, __half, false, 16>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem1);
        if (C > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(C * 64);
        cfg.blockDim = dim3(threads_of<16>());
        cfg.dynamicSmemBytes = kSmem1;  // one CTA per SM: the clusters one grid can spread over
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = C;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        if (cudaOccupancyMaxActiveClusters(&n, (const void*)kern, &cfg) != cudaSuccess || n <= 0) {
            cudaGetLastError();
            n = num_sms() / C;
        }
    }
    if (dev < 64) cache[dev][ci] = n;
    return n;
}

struct Geom {
    int C, M, slots, tc, ring, stage_bytes, part_off, xs_off, recv_off, ring_off, smem, W;
};

static bool plan(const abcq_model_t* m, int p, Geom& g) {
    const int NRT = n_row_tiles(m->rows), NS = n_slices(m->cols);
    const int esz = m->scale_dtype == ABCQ_F16 ? 2 : 4;
    const int zmul = m->asymmetric ? 2 : 1;
    int forced_slots = 0, forced_C = 0, forced_tcw = 0;
    if (g_cl_force) {
        forced_slots = g_cl_force / 100 % 10;
        forced_C = g_cl_force / 10 % 10;
        if (forced_C == 6) forced_C = 16;
        forced_tcw = g_cl_force % 10;
    }
    // cluster size: the largest C <= NS (fewest slices -- table builds -- per
    // CTA; measured best for every Llama shape, tools/cl_probe.py --sweep),
    // clusters: as many as fit one CTA per SM, rows split evenly over them
    int bc = 0, bm = 0;
    for (int C : {16, 8, 4, 2, 1}) {
        if (forced_C ? C != forced_C : C > NS) continue;
        const int Mmax = max_clusters(C);
        if (Mmax <= 0) continue;
        const int Tm = (int)ceil_div(NRT, Mmax);
        bc = C;
        bm = (int)ceil_div(NRT, Tm);
        break;
    }
    if (!bc) return false;
    const int Tm = (int)ceil_div(NRT, bm);
    const int part_bytes = (int)((Tm * 16 * 4 + 127) / 128 * 128);
    // one or two CTAs per SM: two when a CTA's whole stream is short (its
    // producers then prefetch during the previous GEMV; the ring is smaller)
    const int64_t cta_bytes = (int64_t)Tm * ceil_div(NS, bc) * p * kBlockBytes;
    int slots = forced_slots ? forced_slots : (cta_bytes <= 40 * 1024 ? 2 : 1);
    const int smem = slots == 2 ? kSmem2 : kSmem1;
    const int part_off = (int)(kTBase - kDynBase) + kTblBytes;
    const int Smax = (int)ceil_div(NS, bc);
    const int xs_off = part_off + part_bytes;
    const int xs_bytes = Smax * kSliceCols * 4;
    const int recv_off = xs_off + xs_bytes;
    const int recv_bytes = bc > 1 ? (Tm * 16 + 8) * 4 : 0;
    const int ring_off = (recv_off + recv_bytes + 127) / 128 * 128;
    // stage = (slice, chunk of tc tiles, all p planes); one or two tiles per consumer warp
    // consumer warps: 8 when two CTAs share an SM (register budget); alone, 16
    // for bands of >= 48 tiles up to p = 3, else 8 (16 warps x 2 tiles x p >= 4
    // planes make stages too large for a ring deeper than 2, and short bands
    // leave warps idle; tools/cl_probe.py)
    const int W = g_cl_warps ? g_cl_warps : (slots == 2 || p > 3 || Tm < 48 ? 8 : 16);
    int tcw = forced_tcw ? forced_tcw : kMaxTCW;
    if (tcw > kMaxTCW) tcw = kMaxTCW;
    const int nch = (int)ceil_div(Tm, W * tcw);
    const int tc = (int)ceil_div(Tm, nch);
    const int stage = (p * tc * (kBlockBytes + 32 * esz) + (zmul - 1) * tc * 32 * esz + 127) / 128 * 128;
    int ring = (smem - ring_off) / stage;
    if (ring > kMaxRing) ring = kMaxRing;
    if (ring < 1) return false;
    if (slots == 2 && W != 8) return false;
    g = Geom{bc, bm, slots, tc, ring, stage, part_off, xs_off, recv_off, ring_off, ring_off + ring * stage, W};
    return true;
}

template <typename XT, typename YT, typename ST, bool ASYM, int W>
static int launch_t(const Args& a, int smem, cudaStream_t st) {
    auto kern = gemv_cluster_kernel<XT, YT, ST, ASYM, W>;
    static bool attr_set[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 64 && !attr_set[dev]) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem1);
        if (e != cudaSuccess) return (int)e;
        e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
        if (e != cudaSuccess) return (int)e;
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return (int)e;
        attr_set[dev] = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(a.M * a.C);
    cfg.blockDim = dim3(threads_of<W>());
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    int na = 0;
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
    if (a.C > 1) {
        at[na].id = cudaLaunchAttributeClusterDimension;
        at[na].val.clusterDim.x = a.C;
        at[na].val.clusterDim.y = 1;
        at[na].val.clusterDim.z = 1;
        ++na;
    }
    cfg.attrs = at;
    cfg.numAttrs = na;
    return (int)cudaLaunchKernelEx(&cfg, kern, a);
}

template <typename XT, typename YT, int W>
static int launch_w(const Args& a, int sd, bool asym, int smem, cudaStream_t st) {
    if (sd == ABCQ_F16)
        return asym ? launch_t<XT, YT, __half, true, W>(a, smem, st) : launch_t<XT, YT, __half, false, W>(a, smem, st);
    return asym ? launch_t<XT, YT, float, true, W>(a, smem, st) : launch_t<XT, YT, float, false, W>(a, smem, st);
}

template <typename XT, typename YT>
static int launch_xy(const Args& a, int sd, bool asym, int smem, int W, cudaStream_t st) {
    return W == 16 ? launch_w<XT, YT, 16>(a, sd, asym, smem, st) : launch_w<XT, YT, 8>(a, sd, asym, smem, st);
}

}  // namespace cl

bool cluster_supports(const abcq_model_t* m, int p) {
    if (m->layout != ABCQ_LAYOUT_TILED || p < 1 || p > ABCQ_MAX_PLANES || g_dbg_mode == 23) return false;
    // dispatch (tools/cl_probe.py, tools/per_shape_ab.py, back-to-back single
    // launches, B200): the cluster kernel wins while a GEMV is latency-bound --
    // up to 32 MiB of plane bytes (14336 x 4096 at p = 4: 12.0 vs 13.4 us;
    // the decode step's 28672 x 4096 gate/up at p = 2) and <= 2 slices per CTA
    // at C = 16; larger GEMVs stream better through the persistent batch
    // kernel (the decode step's gate/up at p = 3 / 4)
    // (27: every single GEMV through the cluster kernel -- test coverage;
    //  28: any size up to 32 slices -- experiments)
    if (g_dbg_mode != 27) {
        const int64_t plane_bytes = (int64_t)p * tiled_plane_bytes(m->rows, m->cols);
        if (n_slices(m->cols) > 32 || (g_dbg_mode != 28 && plane_bytes > (int64_t)32 * 1024 * 1024)) return false;
    }
    cl::Geom g;
    return cl::plan(m, p, g);
}

int launch_gemv_cluster(const abcq_model_t* m, int p, const void* x, int x_dtype, void* y, int y_dtype,
                        cudaStream_t st) {
    cl::Geom g;
    if (!cl::plan(m, p, g)) return (int)cudaErrorInvalidConfiguration;
    cl::Args a;
    a.planes = static_cast<const char*>(m->planes);
    a.pst = m->plane_stride_bytes;
    a.alpha = m->alpha[p];
    a.offset = m->asymmetric ? m->offset[p] : nullptr;
    a.x = x;
    a.y = y;
    a.rows = m->rows;
    a.cols = m->cols;
    a.NRT = n_row_tiles(m->rows);
    a.NS = n_slices(m->cols);
    a.items = a.NRT * a.NS;
    a.p = p;
    a.glu = x_dtype == ABCQ_F16_SILU_GLU;
    a.C = g.C;
    a.M = g.M;
    a.tc = g.tc;
    a.ring = g.ring;
    a.stage_bytes = g.stage_bytes;
    a.part_off = g.part_off;
    a.xs_off = g.xs_off;
    a.recv_off = g.recv_off;
    a.ring_off = g.ring_off;
    a.smem = g.smem;
    a.dbg = (g_dbg_mode == 1 ? 1 : 0) | (g_dbg_mode >= 100 && g_dbg_mode < 200 ? (g_dbg_mode - 100) & ~2 : 0);
    static unsigned trace_seq = 0;
    a.trace = g_trace ? g_trace + (size_t)(trace_seq++ % 16) * 168 * 16 : nullptr;
    const bool asym = m->asymmetric != 0;
    const int sd = m->scale_dtype;
    if (x_dtype == ABCQ_F32)
        return y_dtype == ABCQ_F16 ? cl::launch_xy<float, __half>(a, sd, asym, g.smem, g.W, st)
                                   : cl::launch_xy<float, float>(a, sd, asym, g.smem, g.W, st);
    return y_dtype == ABCQ_F16 ? cl::launch_xy<__half, __half>(a, sd, asym, g.smem, g.W, st)
                               : cl::launch_xy<__half, float>(a, sd, asym, g.smem, g.W, st);
}

// geometry report for tools / tests: {C, M, slots, tc, ring, W (consumer warps), smem}
int gemv_cluster_geometry(const abcq_model_t* m, int p, int* out7) {
    cl::Geom g;
    if (!cl::plan(m, p, g)) return -1;
    const int v[7] = {g.C, g.M, g.slots, g.tc, g.ring, g.W, g.smem};
    for (int i = 0; i < 7; ++i) out7[i] = v[i];
    return 0;
}

}  // namespace abcq
