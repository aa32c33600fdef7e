/*
 * anybcq_b200.h -- C ABI of the B200-native AnyBCQ bit-plane matmul.
 *
 * Drop-in boundary for the reference's GEMV engine. The reference
 * (/root/reference/pkg/src/anybcq) is pure Python + one numba kernel and has
 * no FFI of its own; its innermost compiled boundary is
 *
 *     _lut_kernel(idx, table, alpha, chunk_lo, chunk_hi, p_use,
 *                 row_lo, row_hi, out)                    gemv.py:84-95
 *
 * driven by GemvEngine.lut / GemvEngine.naive (gemv.py:170-222) over a
 * MultiPrecisionModel (progressive.py:32-79) whose planes use the packing of
 * packing.py:1-37 and whose scale sets are bcq.ScaleTensor (bcq.py:50-96).
 * Every entry point below states which reference interface it replaces.
 *
 * Conventions (all functions):
 *   - plain pointers and sizes only; every `d_*` pointer is DEVICE memory
 *     owned by the caller; `stream` is a cudaStream_t passed as void*
 *     (NULL = legacy default stream); launches are asynchronous;
 *   - return 0 on success, a NEGATIVE ABCQ_E* code for an invalid argument
 *     (the Python layer raises anybcq's UsageError, gemv.py:148-156,
 *     before any work is queued), a POSITIVE cudaError_t value for a CUDA
 *     failure (Python raises RuntimeError);
 *   - abcq_last_error() returns a thread-local message for the last failure.
 */
#ifndef ANYBCQ_B200_H
#define ANYBCQ_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ABCQ_ABI_VERSION 1
#define ABCQ_MAX_PLANES 16 /* bcq.py:22 MAX_PLANES */

/* element dtypes */
#define ABCQ_F32 0
#define ABCQ_F16 1
/* x dtype of the tiled GEMV only (abcq_gemv / abcq_gemv_batch): x points at
 * 2*cols f16 values [g ; u] and the GEMV input is x_k = f16(silu(g_k) * u_k),
 * computed exactly as abcq_silu_mul_f16 (bitwise) while the tables are built --
 * a decoder's SiLU-gated MLP input without the separate elementwise launch */
#define ABCQ_F16_SILU_GLU 2

/* plane layouts */
#define ABCQ_LAYOUT_ROWMAJOR 0 /* reference layout verbatim: (p_hi, rows, ceil(cols/32)) u32 */
#define ABCQ_LAYOUT_TILED 1    /* B200 tiled layout (group_size == 128) */

/* argument errors (negative) */
#define ABCQ_OK 0
#define ABCQ_E_ARG -1       /* bad pointer / shape / dtype */
#define ABCQ_E_PRECISION -2 /* p outside [p_lo, p_hi] (gemv.py:149-152) */
#define ABCQ_E_LAYOUT -3    /* layout cannot serve this call */
#define ABCQ_E_WORKSPACE -4 /* workspace too small */
#define ABCQ_E_DEVICE -5    /* no sm_100 device / kernel image */

/*
 * A device-resident multi-precision model: ONE stack of p_hi planes shared by
 * every precision plus an independent scale set (and offset set in
 * asymmetric mode) per p in [p_lo, p_hi] -- progressive.py:32-79.
 * alpha[p] / offset[p] are indexed by precision p (entries outside
 * [p_lo, p_hi] are ignored). Layout of each buffer:
 *   ROWMAJOR: planes (p_hi, rows, ceil(cols/32)) u32 as packing.py:1-7;
 *             alpha[p] (p, rows, G) and offset[p] (rows, G), scale_dtype.
 *   TILED:    as produced by abcq_pack_planes / abcq_pack_scales.
 */
typedef struct abcq_model {
    int32_t rows;
    int32_t cols;
    int32_t group_size;
    int32_t p_lo;
    int32_t p_hi;
    int32_t asymmetric;  /* 1: offsets present (bcq.py:31-47 mode) */
    int32_t layout;      /* ABCQ_LAYOUT_* */
    int32_t scale_dtype; /* ABCQ_F32 | ABCQ_F16 */
    int64_t plane_stride_bytes; /* bytes between consecutive planes */
    const void* planes;
    const void* alpha[ABCQ_MAX_PLANES + 1];
    const void* offset[ABCQ_MAX_PLANES + 1];
} abcq_model_t;

/* ---- library ------------------------------------------------------------ */
int abcq_abi_version(void);
const char* abcq_last_error(void);
/* 0 if device `dev` is sm_100 and the sm_100a kernels load, else ABCQ_E_DEVICE */
int abcq_device_check(int32_t dev);

/* The persistent GEMV grid takes one CTA per SM (whole SMs: 227 KB of shared
 * memory, all registers). A kernel running BESIDE it on another stream (an
 * NCCL collective overlapping the GEMV) would hold SMs that some of its CTAs
 * then wait for; n > 0 sizes later persistent grids to (SMs - n), leaving n
 * SMs free. Process-wide (all devices); default 0; *prev_out (if not NULL)
 * receives the previous value. ABCQ_E_ARG for n outside [0, SMs).          */
int abcq_set_reserved_sms(int32_t n, int32_t* prev_out);

/* profiling aid: when d_buf != NULL, every later LUT GEMV launch writes 8
 * u64 %globaltimer stamps per CTA (phases: start, prefetch issued, PDL wait
 * done, table built, stream done, reduction done) to d_buf[cta*8 + k].    */
int abcq_debug_set_trace(void* d_buf);
/* profiling experiments only (results are WRONG when mode is 1 or 2): 1 =
 * skip the table lookups, 2 = skip the weight loads; 22 = split-K completion
 * as the separate kernel for every batch; 23 = route single GEMVs through
 * the batch kernel instead of the cluster kernel; 29 = the separate
 * completion kernel's blocks in plain job order (default: jobs of more than
 * 16 slices first); 32 = the batch
 * kernel's round-1 warp split (cost split of every round instead of slot-sized
 * chunks); 33 = batch CTAs take the schedule in reverse (placement
 * experiment); 7001 + c = per-warp round stamps of batch CTA c after the 16
 * launch slots of the trace buffer (7000 = off); 27 = route every
 * single GEMV through the cluster kernel; 5000 + 100*slots + 10*C + t = force
 * the cluster kernel's geometry (C digit 6 = 16; 5000 = automatic); 6000 + W =
 * force its consumer warps (8 / 16; 6000 = automatic); 1000 + b / 2000 + s /
 * 3000 + v = the batch schedule's piece cost in blocks / ring slots issued
 * before the PDL wait / partition strategy. Default 0. */
int abcq_debug_set_mode(int32_t mode);
/* profiling aid: the launch geometry a single GEMV (abcq_gemv, or a batch of
 * one job) uses for this model and precision -- out7 = {cluster size C,
 * clusters M, CTAs per SM, tiles per stage, ring slots, consumer warps,
 * dynamic shared-memory bytes}; ABCQ_E_LAYOUT when the call takes another kernel. */
int abcq_debug_gemv_geometry(const abcq_model_t* m, int32_t p, int32_t* out7);

/* ---- layout sizes (host-only arithmetic) ---------------------------------
 * Tiled layout: 16-row tiles x 256-column slices; see DESIGN.md §Layout.  */
int abcq_tiled_plane_bytes(int32_t rows, int32_t cols, int64_t* out_bytes);
int abcq_tiled_scale_elems(int32_t rows, int32_t cols, int32_t p,
                           int64_t* out_alpha_elems, int64_t* out_offset_elems);

/* ---- packing: replaces BitPlaneSet.words as the kernel's view ------------
 * abcq_pack_planes: reference words (planes, rows, ceil(cols/32)) u32
 * (packing.py:22-30, BitPlaneSet.words packing.py:40-52) -> tiled planes.
 * A bijection on the code bits; abcq_unpack_planes is its inverse
 * (padding bits come back zero, packing.py:6-7).                          */
int abcq_pack_planes(const uint32_t* d_words, int32_t planes, int32_t rows, int32_t cols,
                     void* d_tiled, void* stream);
int abcq_unpack_planes(const void* d_tiled, int32_t planes, int32_t rows, int32_t cols,
                       uint32_t* d_words, void* stream);
/* ScaleTensor (bcq.py:50-96) of ONE precision p: alpha (p, rows, G) f32,
 * offset (rows, G) f32 or NULL -> tiled scale set in `scale_dtype`
 * (f16 = round-to-nearest-even, the container's scale_width=2 rounding,
 * model_format.py:43-52). group_size must be 128.                          */
int abcq_pack_scales(const float* d_alpha, const float* d_offset, int32_t p, int32_t rows,
                     int32_t cols, int32_t group_size, int32_t scale_dtype,
                     void* d_alpha_out, void* d_offset_out, void* stream);

/* ---- lookup table: replaces LookupTable.build (gemv.py:67-81) -----------
 * d_table (ceil(cols/mu), 2^mu) f32, bit-identical to the reference's
 * doubling construction. Exposed for parity; the GEMV kernels build the
 * same table in shared memory.                                            */
int abcq_lut_build(const void* d_x, int32_t x_dtype, int32_t cols, int32_t chunk_width,
                   float* d_table, void* stream);

/* ---- GEMV: replaces GemvEngine.lut (gemv.py:188-222) ---------------------
 * y = sum_{i<p} alpha^(p)_{i,g} (B_i x) [+ offset^(p) . groupsum(x)]
 * for one request at precision p (runtime argument, no recompile).
 * x: (cols) in x_dtype, 16-byte aligned (TILED); y: (rows) in y_dtype.
 * TILED layout -> an sm_100a LUT kernel: the cluster kernel (split-K through
 * distributed shared memory, one launch, no workspace use) for latency-bound
 * GEMVs (<= 32 MiB of planes and <= 32 column slices), else the persistent
 * streaming kernel; ROWMAJOR layout (any group size) -> the generic kernel.
 * Workspace: >= abcq_gemv_workspace_bytes() (self-resetting completion
 * counters at offset 0, then the split-K partials): zero-filled once before
 * first use; ONE workspace (of the largest size needed) may serve every
 * model's abcq_gemv / abcq_gemv_batch launched in order on a stream -- and
 * should: the partials then stay L2-resident instead of spreading over many
 * buffers -- but not calls running concurrently (one workspace per stream). */
int abcq_gemv_workspace_bytes(const abcq_model_t* m, size_t* out_bytes);
int abcq_gemv(const abcq_model_t* m, int32_t p, const void* d_x, int32_t x_dtype, void* d_y,
              int32_t y_dtype, void* d_workspace, size_t workspace_bytes, void* stream);

/* ---- GEMV with a fused add + RMSNorm input (decoder step) -----------------
 * y = W_p * h, h = f16(f16(x + residual) * rsqrt(mean(f16(x + residual)^2)
 * + eps) * norm_w) -- exactly abcq_add_rmsnorm_f16's output (bitwise), formed
 * by every CTA of the persistent kernel while it builds its tables (one
 * launch instead of two); x + residual is written to d_x_out (if not NULL;
 * must not alias d_x / d_residual). f16 x / residual / norm_w / x_out,
 * cols <= 8192, TILED layout; workspace as abcq_gemv.                       */
int abcq_gemv_add_rmsnorm(const abcq_model_t* m, int32_t p, const void* d_x, const void* d_residual,
                          const void* d_norm_w, float eps, void* d_x_out, void* d_y, int32_t y_dtype,
                          void* d_workspace, size_t workspace_bytes, void* stream);

/* Decoder output fusion (the Llama-3 decode harness): y = W x
 * at precision p (f16 y; x f16 or ABCQ_F16_SILU_GLU), then -- in the block
 * that completes the split-K sums last -- stream += y and
 * h = rmsnorm(stream) * norm_w with abcq_add_rmsnorm_f16's arithmetic
 * (bitwise equal to y = abcq_gemv; abcq_add_rmsnorm_f16(stream, y, norm_w, h)),
 * one launch instead of two. The persistent kernel always (never the cluster
 * kernel); rows <= 8192, cols > 256, y / stream / h distinct; workspace as
 * abcq_gemv. */
int abcq_gemv_rmsnorm_out(const abcq_model_t* m, int32_t p, const void* d_x, int32_t x_dtype, void* d_y,
                          void* d_stream, const void* d_norm_w, float eps, void* d_h, void* d_workspace,
                          size_t workspace_bytes, void* stream);

/* ---- batches of independent GEMVs ----------------------------------------
 * One persistent launch runs n_jobs GemvEngine.lut calls back to back (the
 * TMA stream never drains between them) -- e.g. q/k/v or gate/up of a
 * decoder layer, or several requests' precisions. Always the persistent
 * streaming kernel, also for n_jobs == 1 (abcq_gemv instead takes the
 * latency-path cluster kernel for small GEMVs). All jobs: TILED layout,
 * the same x/y/scale dtypes and mode; n_jobs <= abcq_gemv_batch_max_jobs().
 * Workspace: abcq_gemv_batch_workspace_bytes (per-job self-resetting
 * counters at offset 0, then the jobs' split-K partials): as for abcq_gemv,
 * one zero-filled workspace per stream serves every job list.               */
typedef struct abcq_gemv_job {
    const abcq_model_t* model;
    int32_t p;
    int32_t x_dtype;
    int32_t y_dtype;
    const void* x; /* device (cols) */
    void* y;       /* device (rows) */
} abcq_gemv_job_t;
int abcq_gemv_batch_max_jobs(void);
int abcq_gemv_batch_workspace_bytes(const abcq_gemv_job_t* jobs, int32_t n_jobs, size_t* out_bytes);
int abcq_gemv_batch(const abcq_gemv_job_t* jobs, int32_t n_jobs, void* d_workspace, size_t workspace_bytes,
                    void* stream);

/* Fused all-gather (SURVEY §8e, row-sharded GEMV over `world` ranks, one
 * process per GPU): abcq_gemv_batch whose split-K completion also stores every
 * y row into each rank's gathered buffer over peer memory (NVLink), at the
 * offset the row has in this rank's buffer -- the buffers are symmetric
 * (the same layout on every rank: e.g. torch symmetric memory), and every
 * job's y lies inside [local_base, local_base + local_bytes). Publication is
 * deferred by one launch: the next abcq_gemv_batch_peer (or abcq_peer_wait)
 * on this rank, once past its PDL wait, fences at system scope, increments
 * this rank's epoch (d_state[0]) and writes it to slot [rank] of every rank's
 * signal array -- from the GEMV grid's last CTA, so the fence is off the
 * critical path. peer_bases / peer_signals: HOST arrays of `world` device
 * pointers valid on this device (peer_bases[rank] == local_base; rank k's
 * signals: u32[world]); d_state: abcq_peer_state_bytes() zero-filled once per
 * gathered buffer. Every job must be split (cols > 256).
 * abcq_peer_wait: a one-warp kernel that publishes this rank's pending launch
 * and waits until every rank's slot in this rank's signal array reached this
 * rank's epoch (all ranks' rows of the latest launch have landed); gives up
 * after timeout_ns, setting *d_err to 1 + the first late rank, rather than
 * hang. Every rank calls it after the same launch (SPMD).                   */
size_t abcq_peer_state_bytes(void);
int abcq_gemv_batch_peer(const abcq_gemv_job_t* jobs, int32_t n_jobs, const void* d_local_base, size_t local_bytes,
                         void* const* peer_bases, uint32_t* const* peer_signals, int32_t world, int32_t rank,
                         uint32_t* d_state, void* d_workspace, size_t workspace_bytes, void* stream);
int abcq_peer_wait(void* const* peer_bases, uint32_t* const* peer_signals, int32_t world, int32_t rank,
                   uint32_t* d_state, uint32_t* d_err, int64_t timeout_ns, void* stream);


/* ---- small-batch GEMM with per-request precision --------------------------
 * Replaces the reference's per-request loop (cli.py:122-126 loops
 * GemvEngine.lut over the rows of x; service/server.py:188-206 serves one
 * precision per request): Y[b] = W_{p_b} X[b] for B <= 16 requests in ONE pass
 * over planes 0..max(p_b)-1 (tensor cores, f16 x, f32 accumulate).
 * d_x: (B, cols) fp16; d_y: (B, rows) in y_dtype; p_host: B precisions
 * (host array). TILED layout only.                                          */
int abcq_gemm_mixedp_max_batch(void);
int abcq_gemm_mixedp_workspace_bytes(const abcq_model_t* m, int32_t batch, size_t* out_bytes);
int abcq_gemm_mixedp(const abcq_model_t* m, int32_t batch, const int32_t* p_host, const void* d_x, void* d_y,
                     int32_t y_dtype, void* d_workspace, size_t workspace_bytes, void* stream);

/* ---- naive path: replaces GemvEngine.naive (gemv.py:170-186) ------------
 * Column-by-column decode of the planes (either layout, any group size).   */
int abcq_gemv_naive(const abcq_model_t* m, int32_t p, const void* d_x, int32_t x_dtype,
                    void* d_y, int32_t y_dtype, void* stream);

/* ---- dense reconstruction: replaces bcq.dequantize (bcq.py:372-378) -----
 * d_w (rows, cols) in w_dtype = f32(sum_{i<p} alpha_i b_i [+ offset]) with
 * the sum in f64 (bcq.py:137-152). Used for the dequant oracle and for the
 * half-precision (cuBLAS) comparison weights.                              */
int abcq_dequantize(const abcq_model_t* m, int32_t p, void* d_w, int32_t w_dtype, void* stream);

/* ---- BCQ fitting: replaces the reference's f64 fitting internals ----------
 * (the producer of the planes and scale sets above). All
 * device buffers; w (rows, cols) f64; codes (q, rows, cols) int8 of -1/+1
 * (plane-major, the reference's internal form before pack_signs); alpha
 * (q, rows, G) and offset (rows, G) f64, G = ceil(cols / group_size);
 * group_size <= 1024, 1 <= q <= ABCQ_MAX_PLANES.
 *   abcq_fit_greedy   _greedy64 (bcq.py:160-180): asymmetric offset = group
 *                     mean; plane i = sign(residual) (0 -> +1), alpha_i = mean
 *                     |residual| per group. d_scratch: rows*cols f64.
 *   abcq_fit_ls       _ls64 + _solve_psd_batch (bcq.py:183-230): per-group
 *                     least squares over alpha (+ offset), planes fixed, with
 *                     the reference's eigenvalue ridge rule (RANK_CUTOFF
 *                     1e-10, RIDGE_SCALE 1e-8); *d_ridged |= 1 if any group
 *                     was ridged.
 *   abcq_fit_bs       _bs_codes64 (bcq.py:269-295): each code set to the
 *                     nearest of the 2^q levels (ties to the larger level).
 *   abcq_fit_residual_sign  expand_step's new plane (progressive.py:124-127):
 *                     sign(w - dequant(codes[:q], alpha[:q], offset)).      */
int abcq_fit_greedy(const double* d_w, int32_t rows, int32_t cols, int32_t group_size, int32_t q,
                    int32_t asymmetric, int8_t* d_codes, double* d_alpha, double* d_offset, double* d_scratch,
                    void* stream);
int abcq_fit_ls(const double* d_w, const int8_t* d_codes, int32_t q, int32_t rows, int32_t cols,
                int32_t group_size, int32_t asymmetric, double* d_alpha, double* d_offset, int32_t* d_ridged,
                void* stream);
int abcq_fit_bs(const double* d_w, const double* d_alpha, const double* d_offset, int32_t q, int32_t rows,
                int32_t cols, int32_t group_size, int8_t* d_codes, void* stream);
int abcq_fit_residual_sign(const double* d_w, const int8_t* d_codes, const double* d_alpha, const double* d_offset,
                           int32_t q, int32_t rows, int32_t cols, int32_t group_size, int8_t* d_plane,
                           void* stream);

/* ---- decode-step harness ops (not part of the reference boundary) --------
 * The non-GEMV ops of the Llama-3 decode step (paper_2510_10467_b200/decode.py,
 * SURVEY §8f rank 3), fused, all fp16 tensors with f32 math:
 *   add_rmsnorm: x += residual (if non-NULL); y = x*rsqrt(mean(x^2)+eps)*w (n <= 8192)
 *   rope_append: rotate-half RoPE of q (heads x d) and k (kv_heads x d) in place;
 *                k, v written to the caches (kv_heads, max_ctx, d) at position pos
 *   attn_decode: one query token over positions [0, ctx) of the caches, GQA,
 *                head_dim 128, heads/kv_heads <= 8; out (heads x 128)
 *   rope_attn_decode: rope_append + attn_decode over [0, pos] in ONE launch,
 *                bitwise equal to that pair; q and k are left unrotated (only
 *                the cache row pos receives the rotated k). The workspace
 *                (abcq_attn_decode_workspace_bytes(heads, ctx) with ctx >= pos + 1,
 *                e.g. sized once for max_ctx) must be zero-filled once before
 *                first use: it starts with self-resetting per-head counters
 *                (the last split block combines) at a fixed offset, so one
 *                workspace serves every pos, in any order, and the separate
 *                attn_decode path
 *   silu_mul:    a = silu(g) * u
 *   argmax:      *out = index of the largest of n f16 values (first on ties,
 *                as torch.argmax); the workspace (abcq_argmax_workspace_bytes)
 *                is zero-filled once (a self-resetting completion counter) */
int abcq_add_rmsnorm_f16(void* d_x, const void* d_residual, const void* d_w, void* d_y, int32_t n, float eps,
                         void* stream);
int abcq_rope_append_f16(void* d_q, void* d_k, const void* d_v, const float* d_cos, const float* d_sin,
                         void* d_kcache, void* d_vcache, int32_t heads, int32_t kv_heads, int32_t head_dim,
                         int32_t max_ctx, int32_t pos, void* stream);
int abcq_attn_decode_workspace_bytes(int32_t heads, int32_t ctx, size_t* out_bytes);
int abcq_attn_decode_f16(const void* d_q, const void* d_kcache, const void* d_vcache, int32_t heads,
                         int32_t kv_heads, int32_t max_ctx, int32_t ctx, float scale, void* d_out, void* d_workspace,
                         size_t workspace_bytes, void* stream);
int abcq_rope_attn_decode_f16(const void* d_q, const void* d_k, const void* d_v, const float* d_cos,
                              const float* d_sin, void* d_kcache, void* d_vcache, int32_t heads, int32_t kv_heads,
                              int32_t max_ctx, int32_t pos, float scale, void* d_out, void* d_workspace,
                              size_t workspace_bytes, void* stream);
int abcq_silu_mul_f16(const void* d_g, const void* d_u, void* d_a, int32_t n, void* stream);
int abcq_argmax_workspace_bytes(size_t* out_bytes);
int abcq_argmax_f16(const void* d_x, int32_t n, int64_t* d_out, void* d_workspace, size_t workspace_bytes,
                    void* stream);

#ifdef __cplusplus
}
#endif
#endif /* ANYBCQ_B200_H */
