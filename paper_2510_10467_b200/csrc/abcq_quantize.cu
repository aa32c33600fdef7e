// abcq_quantize.cu -- the BCQ fitting internals on the GPU:
// the producer of the hot path's planes and scale sets. f64 throughout, as the
// reference (/root/reference/pkg/src/anybcq/bcq.py:160-369,
// progressive.py:105-145); one warp per (row, group).
//
//   fit_greedy   = _greedy64      (bcq.py:160-180): residual-sign planes, scale = mean |r|
//   fit_ls       = _ls64 + _solve_psd_batch (bcq.py:183-230): per-group least squares
//                  over the scales (+ offset) with the planes fixed, eigendecomposition
//                  with the reference's ridge rule for rank-deficient groups
//   fit_bs       = _bs_codes64    (bcq.py:269-295): every code to the nearest of the
//                  2^q signed scale combinations (ties -> the larger level)
//   residual_sign = the residual-sign step of expand_step (progressive.py:124-127)
//
// Codes are int8 (q, rows, cols) of -1/+1 (the reference's internal form);
// alpha (q, rows, G) and offset (rows, G) f64.
#include <cstdint>

#include "abcq_common.cuh"
#include "abcq_internal.h"

namespace abcq {
namespace qz {

constexpr int kWarps = 4;  // warps (groups) per block
constexpr int kMaxDim = ABCQ_MAX_PLANES + 1;
constexpr double kRankCutoff = 1e-10;  // bcq.py:27 RANK_CUTOFF
constexpr double kRidgeScale = 1e-8;   // bcq.py:28 RIDGE_SCALE

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// asymmetric offset = group mean of w; residual = w - offset (symmetric: w)
__global__ void greedy_kernel(const double* __restrict__ w, int rows, int cols, int g, int q, int asym,
                              int8_t* __restrict__ codes, double* __restrict__ alpha, double* __restrict__ offset,
                              double* __restrict__ r) {
    const int lane = threadIdx.x & 31;
    const int G = (cols + g - 1) / g;
    const int64_t task = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
    if (task >= (int64_t)rows * G) return;
    const int row = (int)(task / G), gi = (int)(task % G);
    const int lo = gi * g, hi = min(lo + g, cols), n = hi - lo;
    const double* wr = w + (int64_t)row * cols;
    double* rr = r + (int64_t)row * cols;
    double off = 0.0;
    if (asym) {
        double s = 0.0;
        for (int k = lo + lane; k < hi; k += 32) s += wr[k];
        off = warp_sum(s) / n;
        if (lane == 0) offset[(int64_t)row * G + gi] = off;
    }
    for (int k = lo + lane; k < hi; k += 32) rr[k] = wr[k] - off;
    __syncwarp();
    for (int i = 0; i < q; ++i) {
        double s = 0.0;
        for (int k = lo + lane; k < hi; k += 32) s += fabs(rr[k]);
        const double scale = warp_sum(s) / n;  // <r, sign(r)> / ||sign(r)||^2 = mean |r|
        if (lane == 0) alpha[((int64_t)i * rows + row) * G + gi] = scale;
        int8_t* cr = codes + ((int64_t)i * rows + row) * cols;
        for (int k = lo + lane; k < hi; k += 32) {
            const double v = rr[k];
            const int8_t c = v >= 0.0 ? 1 : -1;
            cr[k] = c;
            rr[k] = v - scale * (double)c;
        }
        __syncwarp();
    }
}

// symmetric eigendecomposition (cyclic Jacobi) of a dim x dim matrix in
// shared memory by one thread: A -> diag(evals), V = eigenvectors (columns)
__device__ void jacobi_eigh(double* A, double* V, int dim) {
    for (int i = 0; i < dim; ++i)
        for (int j = 0; j < dim; ++j) V[i * dim + j] = i == j ? 1.0 : 0.0;
    for (int sweep = 0; sweep < 64; ++sweep) {
        double off = 0.0, diag = 0.0;
        for (int i = 0; i < dim; ++i) {
            diag += A[i * dim + i] * A[i * dim + i];
            for (int j = i + 1; j < dim; ++j) off += A[i * dim + j] * A[i * dim + j];
        }
        if (off <= 1e-34 * diag || off == 0.0) break;
        for (int p = 0; p < dim; ++p)
            for (int qq = p + 1; qq < dim; ++qq) {
                const double apq = A[p * dim + qq];
                if (apq == 0.0) continue;
                const double app = A[p * dim + p], aqq = A[qq * dim + qq];
                const double theta = (aqq - app) / (2.0 * apq);
                const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
                const double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
                for (int k = 0; k < dim; ++k) {  // A <- J^T A J
                    const double akp = A[k * dim + p], akq = A[k * dim + qq];
                    A[k * dim + p] = c * akp - s * akq;
                    A[k * dim + qq] = s * akp + c * akq;
                }
                for (int k = 0; k < dim; ++k) {
                    const double apk = A[p * dim + k], aqk = A[qq * dim + k];
                    A[p * dim + k] = c * apk - s * aqk;
                    A[qq * dim + k] = s * apk + c * aqk;
                }
                for (int k = 0; k < dim; ++k) {
                    const double vkp = V[k * dim + p], vkq = V[k * dim + qq];
                    V[k * dim + p] = c * vkp - s * vkq;
                    V[k * dim + qq] = s * vkp + c * vkq;
                }
            }
    }
}

// per-group least squares (bcq.py:207-230): design = planes (+ ones), gram /
// rhs reduced by the warp, solved by lane 0 with the reference's ridge rule
__global__ void ls_kernel(const double* __restrict__ w, const int8_t* __restrict__ codes, int q, int rows, int cols,
                          int g, int asym, double* __restrict__ alpha, double* __restrict__ offset,
                          int* __restrict__ ridged_any) {
    __shared__ double sA[kWarps][kMaxDim * kMaxDim];
    __shared__ double sV[kWarps][kMaxDim * kMaxDim];
    __shared__ double sb[kWarps][kMaxDim];
    const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
    const int G = (cols + g - 1) / g;
    const int64_t task = (int64_t)blockIdx.x * kWarps + wi;
    if (task >= (int64_t)rows * G) return;
    const int row = (int)(task / G), gi = (int)(task % G);
    const int lo = gi * g, hi = min(lo + g, cols);
    const int dim = q + (asym ? 1 : 0);
    const double* wr = w + (int64_t)row * cols;
    auto d = [&](int i, int k) -> double {  // design entry (plane i or the ones row)
        return i < q ? (double)codes[((int64_t)i * rows + row) * cols + k] : 1.0;
    };
    for (int i = 0; i < dim; ++i) {
        for (int j = i; j < dim; ++j) {
            double s = 0.0;
            for (int k = lo + lane; k < hi; k += 32) s += d(i, k) * d(j, k);
            s = warp_sum(s);
            if (lane == 0) sA[wi][i * dim + j] = sA[wi][j * dim + i] = s;
        }
        double s = 0.0;
        for (int k = lo + lane; k < hi; k += 32) s += d(i, k) * wr[k];
        s = warp_sum(s);
        if (lane == 0) sb[wi][i] = s;
    }
    __syncwarp();
    if (lane == 0) {
        double* A = sA[wi];
        double* V = sV[wi];
        double* b = sb[wi];
        double tr = 0.0;
        for (int i = 0; i < dim; ++i) tr += A[i * dim + i];
        jacobi_eigh(A, V, dim);
        double emin = A[0];
        for (int i = 1; i < dim; ++i) emin = fmin(emin, A[i * dim + i]);
        const double cutoff = kRankCutoff * tr / dim;
        const bool ridged = emin <= cutoff;
        const double lam = ridged ? kRidgeScale * tr / dim : 0.0;
        if (ridged) atomicOr(ridged_any, 1);
        double proj[kMaxDim];
        for (int e = 0; e < dim; ++e) {  // proj = V^T b / (evals + lam), zero denominators pinned to 1
            double s = 0.0;
            for (int k = 0; k < dim; ++k) s += V[k * dim + e] * b[k];
            double den = A[e * dim + e] + lam;
            den = den > 0.0 ? den : 1.0;
            proj[e] = s / den;
        }
        for (int i = 0; i < dim; ++i) {
            double s = 0.0;
            for (int e = 0; e < dim; ++e) s += V[i * dim + e] * proj[e];
            if (i < q) alpha[((int64_t)i * rows + row) * G + gi] = s;
            else offset[(int64_t)row * G + gi] = s;
        }
    }
}

// nearest representable level (bcq.py:269-295): levels accumulated in
// ascending plane order (offset first), nearest by |w - level|, ties to the
// larger level (then the larger pattern). q <= 12: the 2^q levels of the group
// in shared memory; q = 13..16: every level recomputed per weight (same
// accumulation order, exact, slow -- the reference's limit is 16 planes)
__global__ void bs_kernel(const double* __restrict__ w, const double* __restrict__ alpha,
                          const double* __restrict__ offset, int q, int rows, int cols, int g,
                          int8_t* __restrict__ codes) {
    extern __shared__ double lv[];  // [kWarps][2^q]
    const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
    const int G = (cols + g - 1) / g;
    const int nl = 1 << q;
    const int64_t task = (int64_t)blockIdx.x * kWarps + wi;
    if (task >= (int64_t)rows * G) return;
    const int row = (int)(task / G), gi = (int)(task % G);
    const int lo = gi * g, hi = min(lo + g, cols);
    const bool in_smem = q <= 12;
    double* L = lv + (size_t)wi * (in_smem ? nl : 0);
    const double off = offset ? offset[(int64_t)row * G + gi] : 0.0;
    auto level = [&](int pat) -> double {
        double v = 0.0;
        if (offset) v += off;
        for (int i = 0; i < q; ++i) v += alpha[((int64_t)i * rows + row) * G + gi] * (((pat >> i) & 1) ? 1.0 : -1.0);
        return v;
    };
    if (in_smem) {
        for (int pat = lane; pat < nl; pat += 32) L[pat] = level(pat);
    }
    __syncwarp();
    const double* wr = w + (int64_t)row * cols;
    for (int k = lo + lane; k < hi; k += 32) {
        const double x = wr[k];
        double bd = INFINITY, bl = -INFINITY;
        int bp = 0;
        for (int pat = 0; pat < nl; ++pat) {
            const double l = in_smem ? L[pat] : level(pat);
            const double dd = fabs(x - l);
            if (dd < bd || (dd == bd && (l > bl || (l == bl && pat > bp)))) {
                bd = dd;
                bl = l;
                bp = pat;
            }
        }
        for (int i = 0; i < q; ++i) codes[((int64_t)i * rows + row) * cols + k] = ((bp >> i) & 1) ? 1 : -1;
    }
}

// expand_step's new plane: sign of w - (sum_i code_i alpha_i + offset) over
// the frozen q planes (the _dequant64 order: planes ascending, offset last)
__global__ void residual_sign_kernel(const double* __restrict__ w, const int8_t* __restrict__ codes,
                                     const double* __restrict__ alpha, const double* __restrict__ offset, int q,
                                     int rows, int cols, int g, int8_t* __restrict__ plane) {
    const int64_t n = (int64_t)rows * cols;
    const int G = (cols + g - 1) / g;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const int row = (int)(e / cols), k = (int)(e % cols), gi = k / g;
        double rec = 0.0;
        for (int i = 0; i < q; ++i)
            rec += (double)codes[(int64_t)i * n + e] * alpha[((int64_t)i * rows + row) * G + gi];
        if (offset) rec += offset[(int64_t)row * G + gi];
        plane[e] = (w[e] - rec) >= 0.0 ? 1 : -1;
    }
}

int blocks_for(int rows, int cols, int g) {
    const int64_t tasks = (int64_t)rows * ((cols + g - 1) / g);
    return (int)((tasks + kWarps - 1) / kWarps);
}

}  // namespace qz

int launch_fit_greedy(const double* w, int rows, int cols, int g, int q, int asym, int8_t* codes, double* alpha,
                      double* offset, double* scratch, cudaStream_t st) {
    qz::greedy_kernel<<<qz::blocks_for(rows, cols, g), qz::kWarps * 32, 0, st>>>(w, rows, cols, g, q, asym, codes,
                                                                               alpha, offset, scratch);
    return (int)cudaGetLastError();
}

int launch_fit_ls(const double* w, const int8_t* codes, int q, int rows, int cols, int g, int asym, double* alpha,
                  double* offset, int* ridged, cudaStream_t st) {
    qz::ls_kernel<<<qz::blocks_for(rows, cols, g), qz::kWarps * 32, 0, st>>>(w, codes, q, rows, cols, g, asym, alpha,
                                                                           offset, ridged);
    return (int)cudaGetLastError();
}

int launch_fit_bs(const double* w, const double* alpha, const double* offset, int q, int rows, int cols, int g,
                  int8_t* codes, cudaStream_t st) {
    const size_t smem = q <= 12 ? (size_t)qz::kWarps * (size_t(1) << q) * sizeof(double) : 0;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(qz::bs_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return (int)e;
    }
    qz::bs_kernel<<<qz::blocks_for(rows, cols, g), qz::kWarps * 32, smem, st>>>(w, alpha, offset, q, rows, cols, g,
                                                                              codes);
    return (int)cudaGetLastError();
}

int launch_fit_residual_sign(const double* w, const int8_t* codes, const double* alpha, const double* offset, int q,
                             int rows, int cols, int g, int8_t* plane, cudaStream_t st) {
    const int64_t n = (int64_t)rows * cols;
    const int blocks = (int)((n + 255) / 256 < 148 * 16 ? (n + 255) / 256 : 148 * 16);
    qz::residual_sign_kernel<<<blocks, 256, 0, st>>>(w, codes, alpha, offset, q, rows, cols, g, plane);
    return (int)cudaGetLastError();
}

}  // namespace abcq
