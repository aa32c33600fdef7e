// abcq_capi.cu -- extern "C" entry points of libanybcq_b200.so (include/anybcq_b200.h).
//
// Argument checking happens here, before anything is queued, mirroring the
// reference's validate-then-work order (gemv.py:148-156: UsageError for p
// outside [p_lo, p_hi] or a wrong input length).
#include <cstdarg>
#include <cstdio>

#include "abcq_common.cuh"
#include "abcq_internal.h"

namespace {
thread_local char g_err[512] = "";

int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return code;
}

int cuda_ret(int e, const char* what) {
    if (e == 0) return 0;
    return fail(e, "%s: CUDA error %d (%s)", what, e, cudaGetErrorString((cudaError_t)e));
}

bool dtype_ok(int d) { return d == ABCQ_F32 || d == ABCQ_F16; }

int check_model(const abcq_model_t* m) {
    if (!m) return fail(ABCQ_E_ARG, "model is NULL");
    if (m->rows < 1 || m->cols < 1) return fail(ABCQ_E_ARG, "bad shape %dx%d", m->rows, m->cols);
    if (m->group_size < 1) return fail(ABCQ_E_ARG, "group_size must be >= 1");
    if (!(1 <= m->p_lo && m->p_lo <= m->p_hi && m->p_hi <= ABCQ_MAX_PLANES))
        return fail(ABCQ_E_ARG, "invalid precision range [%d, %d]", m->p_lo, m->p_hi);
    if (!dtype_ok(m->scale_dtype)) return fail(ABCQ_E_ARG, "bad scale dtype %d", m->scale_dtype);
    if (m->layout != ABCQ_LAYOUT_ROWMAJOR && m->layout != ABCQ_LAYOUT_TILED)
        return fail(ABCQ_E_ARG, "bad layout %d", m->layout);
    if (m->layout == ABCQ_LAYOUT_TILED && m->group_size != abcq::kGroup)
        return fail(ABCQ_E_LAYOUT, "tiled layout requires group_size 128, got %d", m->group_size);
    if (!m->planes) return fail(ABCQ_E_ARG, "planes pointer is NULL");
    return 0;
}

int check_call(const abcq_model_t* m, int p, const void* x, int xd, const void* y, int yd) {
    if (int rc = check_model(m)) return rc;
    if (p < m->p_lo || p > m->p_hi)
        return fail(ABCQ_E_PRECISION, "precision %d outside [%d, %d]", p, m->p_lo, m->p_hi);
    if (!m->alpha[p]) return fail(ABCQ_E_ARG, "scale set %d missing", p);
    if (m->asymmetric && !m->offset[p]) return fail(ABCQ_E_ARG, "offset set %d missing", p);
    if (!x || !y) return fail(ABCQ_E_ARG, "x / y pointer is NULL");
    if (!(dtype_ok(xd) || xd == ABCQ_F16_SILU_GLU) || !dtype_ok(yd)) return fail(ABCQ_E_ARG, "bad x/y dtype");
    if (m->layout == ABCQ_LAYOUT_TILED && ((uintptr_t)x & 15u))
        return fail(ABCQ_E_ARG, "x must be 16-byte aligned for the tiled-layout kernels (got %p)", x);
    if (xd == ABCQ_F16_SILU_GLU && !abcq::lut_supports(m, p))
        return fail(ABCQ_E_LAYOUT, "the SiLU-gated x dtype needs the tiled layout (group 128)");
    return 0;
}
}  // namespace

namespace abcq {
int num_sms() {
    static int cached = -1;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 148;
    if (cached < 0) {
        int v = 0;
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
        cached = v;
    }
    return cached;
}
}  // namespace abcq

extern "C" {

int abcq_abi_version(void) { return ABCQ_ABI_VERSION; }

int abcq_set_reserved_sms(int32_t n, int32_t* prev_out) {
    if (n < 0 || n >= abcq::num_sms()) return fail(ABCQ_E_ARG, "reserved SMs %d outside [0, %d)", n, abcq::num_sms());
    if (prev_out) *prev_out = abcq::g_reserved_sms;
    abcq::g_reserved_sms = n;
    return 0;
}

int abcq_debug_set_mode(int32_t mode) {
    if (mode >= 7000 && mode < 7000 + 1 + 255) {  // batch kernel round trace of CTA mode - 7001 (7000 = off)
        abcq::g_rtrace_cta = mode - 7001;
        return 0;
    }
    if (mode >= 6000 && mode < 6100) {  // cluster GEMV consumer warps: 6000 + W (8 / 16; 6000 = automatic)
        abcq::g_cl_warps = mode - 6000;
        return 0;
    }
    if (mode >= 5000 && mode < 6000) {  // cluster GEMV geometry: 5000 + 100*slots + 10*C + tiles/warp (5000 = auto; C digit 6 = 16)
        abcq::g_cl_force = mode - 5000;
        return 0;
    }
    if (mode >= 3000) {  // CTA partition strategy
        abcq::g_partition = mode - 3000;
        return 0;
    }
    if (mode >= 2000) {  // ring slots issued before the PDL wait
        abcq::g_prefill = mode - 2000;
        return 0;
    }
    if (mode >= 1000) {  // load-balance model knob, not a mode
        abcq::g_piece_blocks = mode - 1000;
        return 0;
    }
    abcq::g_dbg_mode = mode;
    return 0;
}

int abcq_debug_set_trace(void* d_buf) {
    abcq::g_trace = static_cast<unsigned long long*>(d_buf);
    return 0;
}

const char* abcq_last_error(void) { return g_err; }

int abcq_debug_gemv_geometry(const abcq_model_t* m, int32_t p, int32_t* out7) {
    if (int rc = check_model(m)) return rc;
    if (!out7) return fail(ABCQ_E_ARG, "out is NULL");
    if (abcq::gemv_cluster_geometry(m, p, out7) != 0)
        return fail(ABCQ_E_LAYOUT, "no cluster geometry for this model / precision");
    return 0;
}

int abcq_device_check(int32_t dev) {
    cudaDeviceProp prop;
    cudaError_t e = cudaGetDeviceProperties(&prop, dev);
    if (e != cudaSuccess) return fail(ABCQ_E_DEVICE, "no CUDA device %d: %s", dev, cudaGetErrorString(e));
    if (prop.major != 10 || prop.minor != 0)
        return fail(ABCQ_E_DEVICE, "device %d is sm_%d%d; this library is built for sm_100a only",
                    dev, prop.major, prop.minor);
    e = (cudaError_t)abcq::probe_kernel_image();
    if (e != cudaSuccess) return fail(ABCQ_E_DEVICE, "sm_100a kernel image unusable: %s", cudaGetErrorString(e));
    return 0;
}

int abcq_tiled_plane_bytes(int32_t rows, int32_t cols, int64_t* out_bytes) {
    if (rows < 1 || cols < 1 || !out_bytes) return fail(ABCQ_E_ARG, "bad arguments");
    *out_bytes = abcq::tiled_plane_bytes(rows, cols);
    return 0;
}

int abcq_tiled_scale_elems(int32_t rows, int32_t cols, int32_t p, int64_t* out_alpha, int64_t* out_offset) {
    if (rows < 1 || cols < 1 || p < 1 || p > ABCQ_MAX_PLANES || !out_alpha || !out_offset)
        return fail(ABCQ_E_ARG, "bad arguments");
    *out_alpha = abcq::tiled_alpha_elems(rows, cols, p);
    *out_offset = abcq::tiled_offset_elems(rows, cols);
    return 0;
}

int abcq_pack_planes(const uint32_t* d_words, int32_t planes, int32_t rows, int32_t cols, void* d_tiled,
                     void* stream) {
    if (!d_words || !d_tiled || planes < 1 || planes > ABCQ_MAX_PLANES || rows < 1 || cols < 1)
        return fail(ABCQ_E_ARG, "abcq_pack_planes: bad arguments");
    return cuda_ret(abcq::launch_pack_planes(d_words, planes, rows, cols, d_tiled, (cudaStream_t)stream),
                    "abcq_pack_planes");
}

int abcq_unpack_planes(const void* d_tiled, int32_t planes, int32_t rows, int32_t cols, uint32_t* d_words,
                       void* stream) {
    if (!d_words || !d_tiled || planes < 1 || planes > ABCQ_MAX_PLANES || rows < 1 || cols < 1)
        return fail(ABCQ_E_ARG, "abcq_unpack_planes: bad arguments");
    return cuda_ret(abcq::launch_unpack_planes(d_tiled, planes, rows, cols, d_words, (cudaStream_t)stream),
                    "abcq_unpack_planes");
}

int abcq_pack_scales(const float* d_alpha, const float* d_offset, int32_t p, int32_t rows, int32_t cols,
                     int32_t group_size, int32_t scale_dtype, void* d_alpha_out, void* d_offset_out,
                     void* stream) {
    if (!d_alpha || !d_alpha_out || p < 1 || p > ABCQ_MAX_PLANES || rows < 1 || cols < 1)
        return fail(ABCQ_E_ARG, "abcq_pack_scales: bad arguments");
    if (group_size != abcq::kGroup)
        return fail(ABCQ_E_LAYOUT, "abcq_pack_scales: tiled scales need group_size 128, got %d", group_size);
    if (!dtype_ok(scale_dtype)) return fail(ABCQ_E_ARG, "abcq_pack_scales: bad dtype");
    if (d_offset && !d_offset_out) return fail(ABCQ_E_ARG, "abcq_pack_scales: offset output missing");
    return cuda_ret(abcq::launch_pack_scales(d_alpha, d_offset, p, rows, cols, scale_dtype, d_alpha_out,
                                             d_offset_out, (cudaStream_t)stream),
                    "abcq_pack_scales");
}

int abcq_lut_build(const void* d_x, int32_t x_dtype, int32_t cols, int32_t chunk_width, float* d_table,
                   void* stream) {
    if (chunk_width < 1 || chunk_width > 8)
        return fail(ABCQ_E_ARG, "chunk width must be in [1, 8], got %d", chunk_width);
    if (!d_x || !d_table || cols < 1 || !dtype_ok(x_dtype)) return fail(ABCQ_E_ARG, "abcq_lut_build: bad arguments");
    return cuda_ret(abcq::launch_lut_build(d_x, x_dtype, cols, chunk_width, d_table, (cudaStream_t)stream),
                    "abcq_lut_build");
}

int abcq_gemv_workspace_bytes(const abcq_model_t* m, size_t* out_bytes) {
    if (int rc = check_model(m)) return rc;
    if (!out_bytes) return fail(ABCQ_E_ARG, "out_bytes is NULL");
    *out_bytes = m->layout == ABCQ_LAYOUT_TILED ? abcq::lut_workspace_bytes(m) : 0;
    return 0;
}

int abcq_gemv(const abcq_model_t* m, int32_t p, const void* d_x, int32_t x_dtype, void* d_y, int32_t y_dtype,
              void* d_workspace, size_t workspace_bytes, void* stream) {
    if (int rc = check_call(m, p, d_x, x_dtype, d_y, y_dtype)) return rc;
    if (abcq::cluster_supports(m, p))  // single GEMV: no workspace
        return cuda_ret(abcq::launch_gemv_cluster(m, p, d_x, x_dtype, d_y, y_dtype, (cudaStream_t)stream),
                        "abcq_gemv");
    if (abcq::lut_supports(m, p)) {
        const size_t need = abcq::lut_workspace_bytes(m);
        if (need && (!d_workspace || workspace_bytes < need))
            return fail(ABCQ_E_WORKSPACE, "workspace %zu bytes < required %zu", workspace_bytes, need);
        return cuda_ret(abcq::launch_gemv_lut(m, p, d_x, x_dtype, d_y, y_dtype, d_workspace, (cudaStream_t)stream),
                        "abcq_gemv");
    }
    return cuda_ret(abcq::launch_gemv_generic(m, p, d_x, x_dtype, d_y, y_dtype, 0, (cudaStream_t)stream),
                    "abcq_gemv");
}

int abcq_gemv_add_rmsnorm(const abcq_model_t* m, int32_t p, const void* d_x, const void* d_residual,
                          const void* d_norm_w, float eps, void* d_x_out, void* d_y, int32_t y_dtype,
                          void* d_workspace, size_t workspace_bytes, void* stream) {
    if (int rc = check_call(m, p, d_x, ABCQ_F16, d_y, y_dtype)) return rc;
    if (!abcq::lut_supports(m, p)) return fail(ABCQ_E_LAYOUT, "abcq_gemv_add_rmsnorm needs the tiled layout (group 128)");
    if (!d_norm_w) return fail(ABCQ_E_ARG, "abcq_gemv_add_rmsnorm: norm weight is NULL");
    if (m->cols > abcq::kRmsMaxN) return fail(ABCQ_E_ARG, "abcq_gemv_add_rmsnorm: cols %d > %d", m->cols, abcq::kRmsMaxN);
    if (d_x_out && (d_x_out == d_x || d_x_out == d_residual))
        return fail(ABCQ_E_ARG, "abcq_gemv_add_rmsnorm: x_out must not alias x or residual (every CTA reads them)");
    const size_t need = abcq::lut_workspace_bytes(m);
    if (need && (!d_workspace || workspace_bytes < need))
        return fail(ABCQ_E_WORKSPACE, "workspace %zu bytes < required %zu", workspace_bytes, need);
    abcq::NormIn nin{d_x, d_residual, d_norm_w, d_x_out, eps};
    return cuda_ret(abcq::launch_gemv_add_rmsnorm(m, p, nin, d_y, y_dtype, d_workspace, (cudaStream_t)stream),
                    "abcq_gemv_add_rmsnorm");
}

int abcq_gemv_rmsnorm_out(const abcq_model_t* m, int32_t p, const void* d_x, int32_t x_dtype, void* d_y,
                          void* d_stream, const void* d_norm_w, float eps, void* d_h, void* d_workspace,
                          size_t workspace_bytes, void* stream) {
    if (int rc = check_call(m, p, d_x, x_dtype, d_y, ABCQ_F16)) return rc;
    if (!abcq::lut_supports(m, p)) return fail(ABCQ_E_LAYOUT, "abcq_gemv_rmsnorm_out needs the tiled layout (group 128)");
    if (x_dtype == ABCQ_F32) return fail(ABCQ_E_ARG, "abcq_gemv_rmsnorm_out: x must be f16 (or f16 SiLU-gated)");
    if (!d_stream || !d_norm_w || !d_h) return fail(ABCQ_E_ARG, "abcq_gemv_rmsnorm_out: stream / norm_w / h is NULL");
    if (m->rows > abcq::kRmsMaxN) return fail(ABCQ_E_ARG, "abcq_gemv_rmsnorm_out: rows %d > %d", m->rows, abcq::kRmsMaxN);
    if (m->cols <= 256) return fail(ABCQ_E_ARG, "abcq_gemv_rmsnorm_out: cols %d <= 256 (no split-K completion)", m->cols);
    if (d_h == d_stream || d_h == d_y || d_stream == d_y)
        return fail(ABCQ_E_ARG, "abcq_gemv_rmsnorm_out: y, stream and h must be distinct buffers");
    const size_t need = abcq::lut_workspace_bytes(m);
    if (need && (!d_workspace || workspace_bytes < need))
        return fail(ABCQ_E_WORKSPACE, "workspace %zu bytes < required %zu", workspace_bytes, need);
    abcq::NormOut nout{d_stream, d_norm_w, d_h, eps};
    return cuda_ret(abcq::launch_gemv_rmsnorm_out(m, p, d_x, x_dtype, d_y, nout, d_workspace, (cudaStream_t)stream),
                    "abcq_gemv_rmsnorm_out");
}

int abcq_gemv_batch_max_jobs(void) { return abcq::lut_max_jobs(); }

static int check_jobs(const abcq_gemv_job_t* jobs, int32_t n) {
    if (!jobs || n < 1) return fail(ABCQ_E_ARG, "empty job list");
    if (n > abcq::lut_max_jobs()) return fail(ABCQ_E_ARG, "%d jobs > max %d", n, abcq::lut_max_jobs());
    const abcq_model_t* m0 = jobs[0].model;
    for (int j = 0; j < n; ++j) {
        const abcq_gemv_job_t& J = jobs[j];
        if (int rc = check_call(J.model, J.p, J.x, J.x_dtype, J.y, J.y_dtype)) return rc;
        if (!abcq::lut_supports(J.model, J.p))
            return fail(ABCQ_E_LAYOUT, "job %d: batched GEMV needs the tiled layout (group 128)", j);
        const int xb = J.x_dtype == ABCQ_F16_SILU_GLU ? ABCQ_F16 : J.x_dtype;
        const int xb0 = jobs[0].x_dtype == ABCQ_F16_SILU_GLU ? ABCQ_F16 : jobs[0].x_dtype;
        if (xb != xb0 || J.y_dtype != jobs[0].y_dtype ||
            J.model->scale_dtype != m0->scale_dtype || J.model->asymmetric != m0->asymmetric)
            return fail(ABCQ_E_ARG, "job %d: dtypes / mode differ from job 0", j);
    }
    return 0;
}

int abcq_gemv_batch_workspace_bytes(const abcq_gemv_job_t* jobs, int32_t n, size_t* out_bytes) {
    if (int rc = check_jobs(jobs, n)) return rc;
    if (!out_bytes) return fail(ABCQ_E_ARG, "out_bytes is NULL");
    const abcq_model_t* models[abcq::kMaxBatchJobs];
    for (int j = 0; j < n; ++j) models[j] = jobs[j].model;
    *out_bytes = abcq::lut_jobs_workspace_bytes(models, n);
    return 0;
}

static int batch_launch(const abcq_gemv_job_t* jobs, int32_t n, void* d_ws, size_t ws_bytes, void* stream,
                        const abcq::PeerOut* pout, const char* what) {
    size_t need = 0;
    if (int rc = abcq_gemv_batch_workspace_bytes(jobs, n, &need)) return rc;
    if (need && (!d_ws || ws_bytes < need))
        return fail(ABCQ_E_WORKSPACE, "workspace %zu bytes < required %zu", ws_bytes, need);
    const abcq_model_t* models[abcq::kMaxBatchJobs];
    int ps[abcq::kMaxBatchJobs];
    const void* xs[abcq::kMaxBatchJobs];
    void* ys[abcq::kMaxBatchJobs];
    int xds[abcq::kMaxBatchJobs];
    for (int j = 0; j < n; ++j) {
        xds[j] = jobs[j].x_dtype;
        models[j] = jobs[j].model;
        ps[j] = jobs[j].p;
        xs[j] = jobs[j].x;
        ys[j] = jobs[j].y;
    }
    return cuda_ret(abcq::launch_gemv_jobs(models, ps, xs, ys, n, xds, jobs[0].y_dtype, d_ws, (cudaStream_t)stream,
                                           nullptr, nullptr, pout),
                    what);
}

size_t abcq_peer_state_bytes(void) { return 256; }

static int peer_out(void* const* peer_bases, uint32_t* const* peer_signals, int32_t world, int32_t rank,
                    const void* d_local_base, uint32_t* d_state, abcq::PeerOut& po) {
    if (world < 1 || world > abcq::kMaxPeerRanks || rank < 0 || rank >= world)
        return fail(ABCQ_E_ARG, "world %d / rank %d outside 1..%d", world, rank, abcq::kMaxPeerRanks);
    if (!d_local_base || !peer_bases || !peer_signals || !d_state) return fail(ABCQ_E_ARG, "fused all-gather: NULL buffer");
    if (peer_bases[rank] != d_local_base)
        return fail(ABCQ_E_ARG, "fused all-gather: peer_bases[rank] must be the local buffer");
    po = abcq::PeerOut{};
    po.n = world;
    po.rank = rank;
    po.local_base = d_local_base;
    po.state = d_state;
    for (int k = 0; k < world; ++k) {
        if (!peer_bases[k] || !peer_signals[k]) return fail(ABCQ_E_ARG, "fused all-gather: rank %d NULL", k);
        po.base[k] = peer_bases[k];
        po.sig[k] = peer_signals[k];
    }
    return 0;
}

int abcq_gemv_batch_peer(const abcq_gemv_job_t* jobs, int32_t n, const void* d_local_base, size_t local_bytes,
                         void* const* peer_bases, uint32_t* const* peer_signals, int32_t world, int32_t rank,
                         uint32_t* d_state, void* d_ws, size_t ws_bytes, void* stream) {
    abcq::PeerOut po;
    if (int rc = peer_out(peer_bases, peer_signals, world, rank, d_local_base, d_state, po)) return rc;
    const char* lo = static_cast<const char*>(d_local_base);
    for (int j = 0; j < n && jobs; ++j) {  // every output inside the symmetric buffer, split jobs
        const char* y = static_cast<const char*>(jobs[j].y);
        const size_t ysz = (size_t)(jobs[j].model ? jobs[j].model->rows : 0) * (jobs[j].y_dtype == ABCQ_F32 ? 4 : 2);
        if (y < lo || y + ysz > lo + local_bytes)
            return fail(ABCQ_E_ARG, "abcq_gemv_batch_peer: job %d's y is outside the gathered buffer", j);
        if (jobs[j].model && jobs[j].model->cols <= 256)
            return fail(ABCQ_E_ARG, "abcq_gemv_batch_peer: job %d has one slice (cols <= 256): no completion pass", j);
    }
    return batch_launch(jobs, n, d_ws, ws_bytes, stream, &po, "abcq_gemv_batch_peer");
}

int abcq_peer_wait(void* const* peer_bases, uint32_t* const* peer_signals, int32_t world, int32_t rank,
                   uint32_t* d_state, uint32_t* d_err, int64_t timeout_ns, void* stream) {
    abcq::PeerOut po;
    if (int rc = peer_out(peer_bases, peer_signals, world, rank, peer_bases ? peer_bases[rank >= 0 && rank < world ? rank : 0] : nullptr,
                          d_state, po))
        return rc;
    if (!d_err) return fail(ABCQ_E_ARG, "abcq_peer_wait: err is NULL");
    return cuda_ret(abcq::launch_peer_wait(po, d_err, timeout_ns, (cudaStream_t)stream), "abcq_peer_wait");
}

int abcq_gemv_batch(const abcq_gemv_job_t* jobs, int32_t n, void* d_ws, size_t ws_bytes, void* stream) {
    return batch_launch(jobs, n, d_ws, ws_bytes, stream, nullptr, "abcq_gemv_batch");
}


int abcq_gemm_mixedp_max_batch(void) { return 16; }

static int check_gemm(const abcq_model_t* m, int32_t B, const int32_t* p_host) {
    if (int rc = check_model(m)) return rc;
    if (m->layout != ABCQ_LAYOUT_TILED) return fail(ABCQ_E_LAYOUT, "mixed-p GEMM needs the tiled layout (group 128)");
    if (B < 1 || B > 16) return fail(ABCQ_E_ARG, "batch %d outside [1, 16]", B);
    if (!p_host) return fail(ABCQ_E_ARG, "p_host is NULL");
    for (int b = 0; b < B; ++b) {
        const int p = p_host[b];
        if (p < m->p_lo || p > m->p_hi)
            return fail(ABCQ_E_PRECISION, "request %d: precision %d outside [%d, %d]", b, p, m->p_lo, m->p_hi);
        if (!m->alpha[p] || (m->asymmetric && !m->offset[p])) return fail(ABCQ_E_ARG, "scale set %d missing", p);
    }
    return 0;
}

int abcq_gemm_mixedp_workspace_bytes(const abcq_model_t* m, int32_t B, size_t* out_bytes) {
    if (int rc = check_model(m)) return rc;
    if (B < 1 || B > 16 || !out_bytes) return fail(ABCQ_E_ARG, "bad batch / out pointer");
    *out_bytes = abcq::gemm_workspace_bytes(m, B);
    return 0;
}

int abcq_gemm_mixedp(const abcq_model_t* m, int32_t B, const int32_t* p_host, const void* d_x, void* d_y,
                     int32_t y_dtype, void* d_ws, size_t ws_bytes, void* stream) {
    if (int rc = check_gemm(m, B, p_host)) return rc;
    if (!d_x || !d_y || !dtype_ok(y_dtype)) return fail(ABCQ_E_ARG, "bad x / y");
    const size_t need = abcq::gemm_workspace_bytes(m, B);
    if (!d_ws || ws_bytes < need) return fail(ABCQ_E_WORKSPACE, "workspace %zu bytes < required %zu", ws_bytes, need);
    return cuda_ret(abcq::launch_gemm_mixedp(m, B, p_host, d_x, d_y, y_dtype, d_ws, (cudaStream_t)stream),
                    "abcq_gemm_mixedp");
}

int abcq_gemv_naive(const abcq_model_t* m, int32_t p, const void* d_x, int32_t x_dtype, void* d_y,
                    int32_t y_dtype, void* stream) {
    if (x_dtype == ABCQ_F16_SILU_GLU) return fail(ABCQ_E_ARG, "abcq_gemv_naive: x must be f16 or f32");
    if (int rc = check_call(m, p, d_x, x_dtype, d_y, y_dtype)) return rc;
    return cuda_ret(abcq::launch_gemv_generic(m, p, d_x, x_dtype, d_y, y_dtype, 1, (cudaStream_t)stream),
                    "abcq_gemv_naive");
}

int abcq_dequantize(const abcq_model_t* m, int32_t p, void* d_w, int32_t w_dtype, void* stream) {
    if (int rc = check_model(m)) return rc;
    if (p < m->p_lo || p > m->p_hi)
        return fail(ABCQ_E_PRECISION, "precision %d outside [%d, %d]", p, m->p_lo, m->p_hi);
    if (!m->alpha[p] || (m->asymmetric && !m->offset[p])) return fail(ABCQ_E_ARG, "scale set %d missing", p);
    if (!d_w || !dtype_ok(w_dtype)) return fail(ABCQ_E_ARG, "abcq_dequantize: bad output");
    return cuda_ret(abcq::launch_dequantize(m, p, d_w, w_dtype, (cudaStream_t)stream), "abcq_dequantize");
}

// ---- decode-step harness ops -------------------------------------------------
static int check_fit(int rows, int cols, int g, int q, const void* w) {
    if (!w || rows < 1 || cols < 1) return fail(ABCQ_E_ARG, "fit: bad matrix");
    if (g < 1 || g > 1024) return fail(ABCQ_E_ARG, "fit: group_size %d outside [1, 1024]", g);
    if (q < 1 || q > ABCQ_MAX_PLANES) return fail(ABCQ_E_PRECISION, "fit: plane count %d outside [1, %d]", q, ABCQ_MAX_PLANES);
    return 0;
}

int abcq_fit_greedy(const double* d_w, int32_t rows, int32_t cols, int32_t group_size, int32_t q, int32_t asymmetric,
                    int8_t* d_codes, double* d_alpha, double* d_offset, double* d_scratch, void* stream) {
    if (int rc = check_fit(rows, cols, group_size, q, d_w)) return rc;
    if (!d_codes || !d_alpha || !d_scratch || (asymmetric && !d_offset)) return fail(ABCQ_E_ARG, "abcq_fit_greedy: bad outputs");
    return cuda_ret(abcq::launch_fit_greedy(d_w, rows, cols, group_size, q, asymmetric != 0, d_codes, d_alpha, d_offset,
                                            d_scratch, (cudaStream_t)stream),
                    "abcq_fit_greedy");
}

int abcq_fit_ls(const double* d_w, const int8_t* d_codes, int32_t q, int32_t rows, int32_t cols, int32_t group_size,
                int32_t asymmetric, double* d_alpha, double* d_offset, int32_t* d_ridged, void* stream) {
    if (int rc = check_fit(rows, cols, group_size, q, d_w)) return rc;
    if (!d_codes || !d_alpha || !d_ridged || (asymmetric && !d_offset)) return fail(ABCQ_E_ARG, "abcq_fit_ls: bad buffers");
    return cuda_ret(abcq::launch_fit_ls(d_w, d_codes, q, rows, cols, group_size, asymmetric != 0, d_alpha, d_offset,
                                        d_ridged, (cudaStream_t)stream),
                    "abcq_fit_ls");
}

int abcq_fit_bs(const double* d_w, const double* d_alpha, const double* d_offset, int32_t q, int32_t rows, int32_t cols,
                int32_t group_size, int8_t* d_codes, void* stream) {
    if (int rc = check_fit(rows, cols, group_size, q, d_w)) return rc;
    if (!d_alpha || !d_codes) return fail(ABCQ_E_ARG, "abcq_fit_bs: bad buffers");
    return cuda_ret(abcq::launch_fit_bs(d_w, d_alpha, d_offset, q, rows, cols, group_size, d_codes, (cudaStream_t)stream),
                    "abcq_fit_bs");
}

int abcq_fit_residual_sign(const double* d_w, const int8_t* d_codes, const double* d_alpha, const double* d_offset,
                           int32_t q, int32_t rows, int32_t cols, int32_t group_size, int8_t* d_plane, void* stream) {
    if (int rc = check_fit(rows, cols, group_size, q, d_w)) return rc;
    if (!d_codes || !d_alpha || !d_plane) return fail(ABCQ_E_ARG, "abcq_fit_residual_sign: bad buffers");
    return cuda_ret(abcq::launch_fit_residual_sign(d_w, d_codes, d_alpha, d_offset, q, rows, cols, group_size, d_plane,
                                                   (cudaStream_t)stream),
                    "abcq_fit_residual_sign");
}

int abcq_argmax_workspace_bytes(size_t* out_bytes) {
    if (!out_bytes) return fail(ABCQ_E_ARG, "out_bytes is NULL");
    *out_bytes = abcq::argmax_workspace_bytes();
    return 0;
}

int abcq_argmax_f16(const void* d_x, int32_t n, int64_t* d_out, void* d_workspace, size_t workspace_bytes,
                    void* stream) {
    if (!d_x || !d_out || n < 1) return fail(ABCQ_E_ARG, "abcq_argmax_f16: bad arguments");
    if (!d_workspace || workspace_bytes < abcq::argmax_workspace_bytes())
        return fail(ABCQ_E_WORKSPACE, "abcq_argmax_f16: workspace too small");
    return cuda_ret(abcq::launch_argmax(d_x, n, reinterpret_cast<long long*>(d_out), d_workspace, (cudaStream_t)stream),
                    "abcq_argmax_f16");
}

int abcq_add_rmsnorm_f16(void* d_x, const void* d_residual, const void* d_w, void* d_y, int32_t n, float eps,
                         void* stream) {
    if (!d_x || !d_w || !d_y || n < 1 || n > 8192) return fail(ABCQ_E_ARG, "abcq_add_rmsnorm_f16: bad arguments");
    return cuda_ret(abcq::launch_add_rmsnorm(d_x, d_residual, d_w, d_y, n, eps, (cudaStream_t)stream),
                    "abcq_add_rmsnorm_f16");
}

int abcq_rope_append_f16(void* d_q, void* d_k, const void* d_v, const float* d_cos, const float* d_sin,
                         void* d_kcache, void* d_vcache, int32_t heads, int32_t kv_heads, int32_t head_dim,
                         int32_t max_ctx, int32_t pos, void* stream) {
    if (!d_q || !d_k || !d_v || !d_cos || !d_sin || !d_kcache || !d_vcache || heads < 1 || kv_heads < 1 ||
        head_dim < 2 || head_dim % 2 || head_dim > 2048 || pos < 0 || pos >= max_ctx)
        return fail(ABCQ_E_ARG, "abcq_rope_append_f16: bad arguments");
    return cuda_ret(abcq::launch_rope_append(d_q, d_k, d_v, d_cos, d_sin, d_kcache, d_vcache, heads, kv_heads,
                                             head_dim, max_ctx, pos, (cudaStream_t)stream),
                    "abcq_rope_append_f16");
}

int abcq_attn_decode_workspace_bytes(int32_t heads, int32_t ctx, size_t* out_bytes) {
    if (!out_bytes || heads < 1 || ctx < 1) return fail(ABCQ_E_ARG, "abcq_attn_decode_workspace_bytes: bad arguments");
    *out_bytes = abcq::attn_decode_workspace_bytes(heads, ctx);
    return 0;
}

int abcq_attn_decode_f16(const void* d_q, const void* d_kcache, const void* d_vcache, int32_t heads,
                         int32_t kv_heads, int32_t max_ctx, int32_t ctx, float scale, void* d_out, void* d_workspace,
                         size_t workspace_bytes, void* stream) {
    if (!d_q || !d_kcache || !d_vcache || !d_out || kv_heads < 1 || heads % kv_heads || heads / kv_heads > 8 ||
        ctx < 1 || ctx > max_ctx)
        return fail(ABCQ_E_ARG, "abcq_attn_decode_f16: bad arguments (head_dim must be 128, heads/kv_heads <= 8)");
    if (!d_workspace || workspace_bytes < abcq::attn_decode_workspace_bytes(heads, ctx))
        return fail(ABCQ_E_WORKSPACE, "abcq_attn_decode_f16: workspace too small");
    return cuda_ret(abcq::launch_attn_decode(d_q, d_kcache, d_vcache, heads, kv_heads, max_ctx, ctx, scale, d_out,
                                             d_workspace, (cudaStream_t)stream),
                    "abcq_attn_decode_f16");
}

int abcq_rope_attn_decode_f16(const void* d_q, const void* d_k, const void* d_v, const float* d_cos,
                              const float* d_sin, void* d_kcache, void* d_vcache, int32_t heads, int32_t kv_heads,
                              int32_t max_ctx, int32_t pos, float scale, void* d_out, void* d_workspace,
                              size_t workspace_bytes, void* stream) {
    if (!d_q || !d_k || !d_v || !d_cos || !d_sin || !d_kcache || !d_vcache || !d_out || kv_heads < 1 ||
        heads % kv_heads || heads / kv_heads > 8 || pos < 0 || pos >= max_ctx)
        return fail(ABCQ_E_ARG, "abcq_rope_attn_decode_f16: bad arguments (head_dim must be 128, heads/kv_heads <= 8)");
    if (!d_workspace || workspace_bytes < abcq::attn_decode_workspace_bytes(heads, pos + 1))
        return fail(ABCQ_E_WORKSPACE, "abcq_rope_attn_decode_f16: workspace too small");
    return cuda_ret(abcq::launch_rope_attn_decode(d_q, d_k, d_v, d_cos, d_sin, d_kcache, d_vcache, heads, kv_heads,
                                                  max_ctx, pos, scale, d_out, d_workspace, (cudaStream_t)stream),
                    "abcq_rope_attn_decode_f16");
}

int abcq_silu_mul_f16(const void* d_g, const void* d_u, void* d_a, int32_t n, void* stream) {
    if (!d_g || !d_u || !d_a || n < 1) return fail(ABCQ_E_ARG, "abcq_silu_mul_f16: bad arguments");
    return cuda_ret(abcq::launch_silu_mul(d_g, d_u, d_a, n, (cudaStream_t)stream), "abcq_silu_mul_f16");
}

}  // extern "C"
