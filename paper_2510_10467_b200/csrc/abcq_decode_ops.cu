// abcq_decode_ops.cu -- the non-GEMV ops of the Llama-3 decode-step harness
// (paper_2510_10467_b200/decode.py), fused so that one
// decoder layer is ~12 launches instead of ~45 PyTorch elementwise kernels:
//   add_rmsnorm : x += r (optional); y = x * rsqrt(mean(x^2) + eps) * w      (f16 io, f32 math)
//   rope_append : RoPE (rotate-half) of q and k in place, k/v written to the KV cache at pos
//   attn_decode : one query token, GQA, over L cached positions: split-L partial softmax
//                 (max, sum, weighted V) per (kv head, split) + a combine kernel
//   silu_mul    : a = silu(g) * u
// Not part of the reference's operator boundary; the harness's plumbing.
#include <cuda_fp16.h>

#include "abcq_common.cuh"
#include "abcq_internal.h"

namespace abcq {

// Every op here is launched with programmatic stream serialization (PDL): it
// waits for its producer with griddepcontrol.wait before touching inputs, and
// releases its consumer early -- in a CUDA-graphed decode step each launch's
// ramp overlaps the previous kernel's tail (one decoder layer is ~13 kernels).
__device__ __forceinline__ void pdl_enter() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" :::);
}

template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// one block of 1024 threads; n <= 8192 (4 values per thread, half2 loads)
__global__ void __launch_bounds__(1024) add_rmsnorm_kernel(__half* __restrict__ x, const __half* __restrict__ r,
                                                           const __half* __restrict__ w, __half* __restrict__ y,
                                                           int n, float eps) {
    pdl_enter();
    __shared__ float red[32];
    float v[8];
    float ss = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const int i = threadIdx.x + k * 1024;
        float xv = 0.f;
        if (i < n) {
            xv = __half2float(x[i]);
            if (r) {
                xv = __half2float(__float2half_rn(xv + __half2float(r[i])));  // residual stream kept in f16
                x[i] = __float2half_rn(xv);
            }
        }
        v[k] = xv;
        ss += xv * xv;
    }
    ss = warp_sum(ss);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
    __syncthreads();
    if (threadIdx.x < 32) {
        float t = warp_sum(red[threadIdx.x]);
        if (threadIdx.x == 0) red[0] = rsqrtf(t / n + eps);
    }
    __syncthreads();
    const float inv = red[0];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const int i = threadIdx.x + k * 1024;
        if (i < n) y[i] = __float2half_rn(v[k] * inv * __half2float(w[i]));
    }
}

// grid: heads + kv_heads blocks of d/2 threads; block b < heads rotates q head b,
// else k head (b - heads) and also stores k, v to the cache at position pos
__global__ void rope_append_kernel(__half* __restrict__ q, __half* __restrict__ k, const __half* __restrict__ v,
                                   const float* __restrict__ cosv, const float* __restrict__ sinv,
                                   __half* __restrict__ kc, __half* __restrict__ vc, int heads, int kv_heads,
                                   int d, int lmax, int pos) {
    pdl_enter();
    const int b = blockIdx.x, t = threadIdx.x, h2 = d / 2;
    const bool isq = b < heads;
    __half* vec = isq ? q + (size_t)b * d : k + (size_t)(b - heads) * d;
    const float x1 = __half2float(vec[t]), x2 = __half2float(vec[t + h2]);
    const float c = cosv[t], s = sinv[t];
    const __half o1 = __float2half_rn(x1 * c - x2 * s), o2 = __float2half_rn(x2 * c + x1 * s);
    vec[t] = o1;
    vec[t + h2] = o2;
    if (!isq) {
        const int kh = b - heads;
        __half* kdst = kc + ((size_t)kh * lmax + pos) * d;
        __half* vdst = vc + ((size_t)kh * lmax + pos) * d;
        kdst[t] = o1;
        kdst[t + h2] = o2;
        vdst[t] = v[(size_t)kh * d + t];
        vdst[t + h2] = v[(size_t)kh * d + t + h2];
    }
}

// split-L decode attention, d == 128, group g = heads / kv_heads <= 8.
// grid (kv_heads, splits); block = 32 * g threads: warp w owns query head
// kh*g + w; lane l owns positions l, l+32 of the split (scores) and dims
// 4l..4l+3 (output). Partials: m, l and acc[128] per (head, split).
constexpr int kAttnSplit = 64;
constexpr int kPartStride = 4 + 128;  // m, l, pad, pad, acc[128] (16-byte aligned acc)
__global__ void attn_decode_partial(const __half* __restrict__ q, const __half* __restrict__ kc,
                                    const __half* __restrict__ vc, int heads, int kv_heads, int lmax, int L,
                                    float scale, float* __restrict__ part) {
    pdl_enter();
    constexpr int d = 128;
    __shared__ __half ks[kAttnSplit][d + 2];  // odd word stride: lane-per-row dots are conflict-free
    __shared__ __half vs[kAttnSplit][d];
    const int kh = blockIdx.x, sp = blockIdx.y, g = heads / kv_heads;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int p0 = sp * kAttnSplit, n = min(kAttnSplit, L - p0);
    for (int i = threadIdx.x; i < kAttnSplit * d / 2; i += blockDim.x) {  // 4-byte copies
        const int r = i / (d / 2), c2 = (i % (d / 2)) * 2;
        __half2 kv = __floats2half2_rn(0.f, 0.f), vv = kv;
        if (r < n) {
            kv = *reinterpret_cast<const __half2*>(kc + ((size_t)kh * lmax + p0 + r) * d + c2);
            vv = *reinterpret_cast<const __half2*>(vc + ((size_t)kh * lmax + p0 + r) * d + c2);
        }
        *reinterpret_cast<__half2*>(&ks[r][c2]) = kv;
        *reinterpret_cast<__half2*>(&vs[r][c2]) = vv;
    }
    __syncthreads();
    const int h = kh * g + warp;
    const __half* qh = q + (size_t)h * d;
    float s[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        const int r = lane + 32 * j;
        float acc = 0.f;
        for (int c = 0; c < d; c += 2) {
            const float2 qq = __half22float2(*reinterpret_cast<const __half2*>(qh + c));
            const float2 kk = __half22float2(*reinterpret_cast<const __half2*>(&ks[r][c]));
            acc = fmaf(qq.x, kk.x, fmaf(qq.y, kk.y, acc));
        }
        s[j] = r < n ? acc * scale : -INFINITY;
    }
    const float m = warp_max(fmaxf(s[0], s[1]));
    const float e0 = __expf(s[0] - m), e1 = __expf(s[1] - m);
    const float l = warp_sum(e0 + e1);
    float o[4] = {0.f, 0.f, 0.f, 0.f};
    for (int r = 0; r < n; ++r) {
        const float pr = __shfl_sync(0xffffffffu, r < 32 ? e0 : e1, r & 31);
        const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&vs[r][4 * lane]));
        const float2 b = __half22float2(*reinterpret_cast<const __half2*>(&vs[r][4 * lane + 2]));
        o[0] = fmaf(pr, a.x, o[0]);
        o[1] = fmaf(pr, a.y, o[1]);
        o[2] = fmaf(pr, b.x, o[2]);
        o[3] = fmaf(pr, b.y, o[3]);
    }
    float* pp = part + ((size_t)h * gridDim.y + sp) * kPartStride;
    if (lane == 0) {
        pp[0] = m;
        pp[1] = l;
    }
    *reinterpret_cast<float4*>(pp + 4 + 4 * lane) = make_float4(o[0], o[1], o[2], o[3]);
}

// one block of 128 threads per head: out[h] = sum_s e^{m_s - M} acc_s / sum_s e^{m_s - M} l_s
__global__ void attn_decode_combine(const float* __restrict__ part, int splits, __half* __restrict__ out) {
    pdl_enter();
    constexpr int d = 128;
    const int h = blockIdx.x, t = threadIdx.x;
    const float* ph = part + (size_t)h * splits * kPartStride;
    float M = -INFINITY;
    for (int s = 0; s < splits; ++s) M = fmaxf(M, ph[s * kPartStride]);
    float num = 0.f, den = 0.f;
    for (int s = 0; s < splits; ++s) {
        const float w = __expf(ph[s * kPartStride] - M);
        den = fmaf(w, ph[s * kPartStride + 1], den);
        num = fmaf(w, ph[s * kPartStride + 4 + t], num);
    }
    out[(size_t)h * d + t] = __float2half_rn(num / den);
}

__global__ void silu_mul_kernel(const __half* __restrict__ g, const __half* __restrict__ u, __half* __restrict__ a,
                                int n) {
    pdl_enter();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        const float gv = __half2float(g[i]);
        a[i] = __float2half_rn(gv / (1.f + __expf(-gv)) * __half2float(u[i]));
    }
}

int launch_add_rmsnorm(void* x, const void* r, const void* w, void* y, int n, float eps, cudaStream_t st) {
    return (int)launch_pdl(add_rmsnorm_kernel, dim3(1), dim3(1024), st, static_cast<__half*>(x),
                           static_cast<const __half*>(r), static_cast<const __half*>(w), static_cast<__half*>(y), n,
                           eps);
}

int launch_rope_append(void* q, void* k, const void* v, const float* cosv, const float* sinv, void* kc, void* vc,
                       int heads, int kv_heads, int d, int lmax, int pos, cudaStream_t st) {
    return (int)launch_pdl(rope_append_kernel, dim3(heads + kv_heads), dim3(d / 2), st, static_cast<__half*>(q),
                           static_cast<__half*>(k), static_cast<const __half*>(v), cosv, sinv,
                           static_cast<__half*>(kc), static_cast<__half*>(vc), heads, kv_heads, d, lmax, pos);
}

size_t attn_decode_workspace_bytes(int heads, int L) {
    return (size_t)heads * ((L + kAttnSplit - 1) / kAttnSplit) * kPartStride * sizeof(float);
}

int launch_attn_decode(const void* q, const void* kc, const void* vc, int heads, int kv_heads, int lmax, int L,
                       float scale, void* out, void* ws, cudaStream_t st) {
    const int splits = (L + kAttnSplit - 1) / kAttnSplit;
    cudaError_t e = launch_pdl(attn_decode_partial, dim3(kv_heads, splits), dim3(32 * (heads / kv_heads)), st,
                               static_cast<const __half*>(q), static_cast<const __half*>(kc),
                               static_cast<const __half*>(vc), heads, kv_heads, lmax, L, scale,
                               static_cast<float*>(ws));
    if (e != cudaSuccess) return (int)e;
    return (int)launch_pdl(attn_decode_combine, dim3(heads), dim3(128), st, static_cast<const float*>(ws), splits,
                           static_cast<__half*>(out));
}

int launch_silu_mul(const void* g, const void* u, void* a, int n, cudaStream_t st) {
    return (int)launch_pdl(silu_mul_kernel, dim3((n + 255) / 256), dim3(256), st, static_cast<const __half*>(g),
                           static_cast<const __half*>(u), static_cast<__half*>(a), n);
}

}  // namespace abcq
