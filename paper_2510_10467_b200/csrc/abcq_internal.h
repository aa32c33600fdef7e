// abcq_internal.h -- launcher declarations shared between the .cu files.
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/anybcq_b200.h"

namespace abcq {

constexpr int kMaxBatchJobs = 32;  // jobs per abcq_gemv_batch launch (abcq_gemv_batch_max_jobs)

int launch_pack_planes(const uint32_t* words, int planes, int rows, int cols, void* out, cudaStream_t st);
int launch_unpack_planes(const void* tiled, int planes, int rows, int cols, uint32_t* words, cudaStream_t st);
int launch_pack_scales(const float* alpha, const float* offset, int p, int rows, int cols, int scale_dtype,
                       void* alpha_out, void* offset_out, cudaStream_t st);
int launch_lut_build(const void* x, int x_dtype, int cols, int mu, float* table, cudaStream_t st);

// fast path: TILED layout, group 128
size_t lut_workspace_bytes(const abcq_model_t* m);
size_t lut_jobs_workspace_bytes(const abcq_model_t* const* models, int n);
bool lut_supports(const abcq_model_t* m, int p);  // tiled layout and p <= 8
int launch_gemv_lut(const abcq_model_t* m, int p, const void* x, int x_dtype, void* y, int y_dtype,
                    void* ws, cudaStream_t st);
// batch of n independent GEMVs (same dtypes / mode), workspaces concatenated
// in job order (lut_workspace_bytes each)
struct NormIn;
struct NormOut;
struct PeerOut;
int launch_gemv_jobs(const abcq_model_t* const* models, const int* ps, const void* const* xs, void* const* ys,
                     int n, const int* x_dtypes, int y_dtype, void* ws, cudaStream_t st, const NormIn* nin = nullptr,
                     const NormOut* nout = nullptr, const PeerOut* pout = nullptr);
// fused all-gather (abcq_gemv_batch_peer): see Peers in abcq_gemv_batch.cuh
constexpr int kMaxPeerRanks = 8;
struct PeerOut {
    int n, rank;
    const void* local_base;
    void* base[kMaxPeerRanks];
    uint32_t* sig[kMaxPeerRanks];
    uint32_t* state;
};
int launch_peer_wait(const PeerOut& po, uint32_t* err, long long timeout_ns, cudaStream_t st);
int lut_max_jobs();

// fused input mode of the persistent GEMV: input = f16(f16(x + residual) * inv_rms * norm_w),
// x + residual written to x_out (add_rmsnorm_kernel's arithmetic, bitwise)
struct NormIn {
    const void* x;
    const void* residual;
    const void* norm_w;
    void* x_out;
    float eps;
};
int launch_gemv_add_rmsnorm(const abcq_model_t* m, int p, const NormIn& nin, void* y, int y_dtype, void* ws,
                            cudaStream_t st);
// fused output mode (norm epilogue): after y = W x (f16), the last split-K
// completion CTA does stream += y; h = rmsnorm(stream) * norm_w
// (add_rmsnorm_kernel's arithmetic, bitwise)
struct NormOut {
    void* stream;  // residual stream (f16, updated in place)
    const void* norm_w;
    void* h;
    float eps;
};
int launch_gemv_rmsnorm_out(const abcq_model_t* m, int p, const void* x, int x_dtype, void* y, const NormOut& nout,
                            void* ws, cudaStream_t st);

// single GEMV through the cluster kernel (abcq_gemv_cluster.cu): no workspace
bool cluster_supports(const abcq_model_t* m, int p);
int launch_gemv_cluster(const abcq_model_t* m, int p, const void* x, int x_dtype, void* y, int y_dtype,
                        cudaStream_t st);
int gemv_cluster_geometry(const abcq_model_t* m, int p, int* out7);
extern int g_cl_force;
extern int g_cl_warps;

// small-batch mixed-precision GEMM (tensor cores), B <= 16
size_t gemm_workspace_bytes(const abcq_model_t* m, int B);
int launch_gemm_mixedp(const abcq_model_t* m, int B, const int* p_host, const void* x, void* y, int y_dtype,
                       void* ws, cudaStream_t st);

// generic path: either layout, any group size. naive=1 -> f64 per-column
// accumulation (GemvEngine.naive), naive=0 -> f32 group sums (GemvEngine.lut)
int launch_gemv_generic(const abcq_model_t* m, int p, const void* x, int x_dtype, void* y, int y_dtype,
                        int naive, cudaStream_t st);

int launch_dequantize(const abcq_model_t* m, int p, void* w, int w_dtype, cudaStream_t st);

// decode-step harness ops (abcq_decode_ops.cu), f16
int launch_add_rmsnorm(void* x, const void* r, const void* w, void* y, int n, float eps, cudaStream_t st);
int launch_rope_append(void* q, void* k, const void* v, const float* cosv, const float* sinv, void* kc, void* vc,
                       int heads, int kv_heads, int d, int lmax, int pos, cudaStream_t st);
size_t attn_decode_workspace_bytes(int heads, int L);
int launch_rope_attn_decode(const void* q, const void* k, const void* v, const float* cosv, const float* sinv,
                            void* kc, void* vc, int heads, int kv_heads, int lmax, int pos, float scale, void* out,
                            void* ws, cudaStream_t st);
int launch_attn_decode(const void* q, const void* kc, const void* vc, int heads, int kv_heads, int lmax, int L,
                       float scale, void* out, void* ws, cudaStream_t st);
int launch_silu_mul(const void* g, const void* u, void* a, int n, cudaStream_t st);
size_t argmax_workspace_bytes();
int launch_argmax(const void* x, int n, long long* out, void* ws, cudaStream_t st);

// BCQ fitting (abcq_quantize.cu), f64, codes int8 (q, rows, cols)
int launch_fit_greedy(const double* w, int rows, int cols, int g, int q, int asym, int8_t* codes, double* alpha,
                      double* offset, double* scratch, cudaStream_t st);
int launch_fit_ls(const double* w, const int8_t* codes, int q, int rows, int cols, int g, int asym, double* alpha,
                  double* offset, int* ridged, cudaStream_t st);
int launch_fit_bs(const double* w, const double* alpha, const double* offset, int q, int rows, int cols, int g,
                  int8_t* codes, cudaStream_t st);
int launch_fit_residual_sign(const double* w, const int8_t* codes, const double* alpha, const double* offset, int q,
                             int rows, int cols, int g, int8_t* plane, cudaStream_t st);

extern unsigned long long* g_trace;
extern int g_rtrace_cta;  // abcq_debug_set_mode(7001 + cta): per-warp round stamps of one batch-kernel CTA
extern int g_dbg_mode;
extern int g_piece_blocks;
extern int g_prefill;
extern int g_partition;
extern int g_reserved_sms;
int num_sms();
int probe_kernel_image();  // cudaFuncGetAttributes on a packing kernel

}  // namespace abcq
