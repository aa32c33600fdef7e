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
__global__ void __launch_bounds__(kRmsThreads) add_rmsnorm_kernel(__half* __restrict__ x,
                                                                  const __half* __restrict__ r,
                                                                  const __half* __restrict__ w,
                                                                  __half* __restrict__ y, int n, float eps) {
    pdl_enter();
    __shared__ float red[17];
    float v[16];
    const int t = threadIdx.x;
    const float ss = rms_load(x, r, n, t, v);  // (the statistics the fused GEMV input recomputes bitwise)
    const float inv = rms_inv(ss, n, eps, red);
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        const int i = (k < 8 ? 8 * t + k : 4096 + 8 * t + (k - 8));
        if (i < n) {
            if (r) x[i] = __float2half_rn(v[k]);
            y[i] = __float2half_rn(v[k] * inv * __half2float(w[i]));
        }
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
constexpr int kAttnSplit = 64;  // positions per block
constexpr int kPartStride = 4 + 128;  // m, l, pad, pad, acc[128] (16-byte aligned acc)
// stage rows [p0, p0 + n) of one kv head's K and V (d = 128) in shared memory,
// zero-filling rows >= n and skipping row `skip`: 16-byte loads, all of a
// thread's loads issued before its stores (a split is 32 KB; 4-byte copies
// left the loads latency-bound at ~0.4 TB/s)
template <int NR>
__device__ __forceinline__ void stage_kv(const __half* __restrict__ kc, const __half* __restrict__ vc, int kh,
                                         int lmax, int p0, int n, int skip, __half (*ks)[128 + 2],
                                         __half (*vs)[128]) {
    constexpr int d = 128, kVec = NR * d / 8;
    for (int base = 0; base < kVec; base += 8 * (int)blockDim.x) {
        uint4 kr[8], vr[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int i = base + threadIdx.x + j * blockDim.x, r = i >> 4, c8 = (i & 15) * 8;
            kr[j] = vr[j] = make_uint4(0u, 0u, 0u, 0u);
            if (i < kVec && r < n && r != skip) {
                kr[j] = __ldg(reinterpret_cast<const uint4*>(kc + ((size_t)kh * lmax + p0 + r) * d + c8));
                vr[j] = __ldg(reinterpret_cast<const uint4*>(vc + ((size_t)kh * lmax + p0 + r) * d + c8));
            }
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int i = base + threadIdx.x + j * blockDim.x, r = i >> 4, c8 = (i & 15) * 8;
            if (i < kVec && r != skip) {  // (row `skip` is the caller's)
                uint32_t* kd = reinterpret_cast<uint32_t*>(&ks[r][c8]);  // odd-word row stride: 4-byte stores
                kd[0] = kr[j].x;
                kd[1] = kr[j].y;
                kd[2] = kr[j].z;
                kd[3] = kr[j].w;
                *reinterpret_cast<uint4*>(&vs[r][c8]) = vr[j];
            }
        }
    }
}

// one warp = one query head over the staged split: scores (lane = row), the
// split's max / sum of exponentials, and the exp-weighted V rows (lane = dims
// 4l..4l+3) -> part = {m, l, -, -, acc[128]}. Independent partial chains
// (4 per dot product, 2 over the V rows) keep the FMA latency off the
// critical path.
__device__ __forceinline__ void split_attend(const __half* qh, const __half (*ks)[128 + 2],
                                             const __half (*vs)[128], int n, float scale, int lane, float* pp) {
    constexpr int d = 128, RPL = kAttnSplit / 32;
    float s[RPL];
#pragma unroll
    for (int j = 0; j < RPL; ++j) {
        const int r = lane + 32 * j;
        float a4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 4
        for (int c = 0; c < d; c += 8) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const float2 qq = __half22float2(*reinterpret_cast<const __half2*>(qh + c + 2 * u));
                const float2 kk = __half22float2(*reinterpret_cast<const __half2*>(&ks[r][c + 2 * u]));
                a4[u] = fmaf(qq.x, kk.x, fmaf(qq.y, kk.y, a4[u]));
            }
        }
        s[j] = r < n ? ((a4[0] + a4[1]) + (a4[2] + a4[3])) * scale : -INFINITY;
    }
    float mx = s[0];
#pragma unroll
    for (int j = 1; j < RPL; ++j) mx = fmaxf(mx, s[j]);
    const float m = warp_max(mx);
    float e[RPL], es = 0.f;
#pragma unroll
    for (int j = 0; j < RPL; ++j) {
        e[j] = __expf(s[j] - m);
        es += e[j];
    }
    const float l = warp_sum(es);
    float o0[4] = {0.f, 0.f, 0.f, 0.f}, o1[4] = {0.f, 0.f, 0.f, 0.f};
    auto pick = [&](int r) {
        float ej = e[0];
#pragma unroll
        for (int j = 1; j < RPL; ++j) ej = (r >> 5) == j ? e[j] : ej;
        return __shfl_sync(0xffffffffu, ej, r & 31);
    };
    auto row = [&](int r, float pr, float (&oo)[4]) {
        const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&vs[r][4 * lane]));
        const float2 b = __half22float2(*reinterpret_cast<const __half2*>(&vs[r][4 * lane + 2]));
        oo[0] = fmaf(pr, a.x, oo[0]);
        oo[1] = fmaf(pr, a.y, oo[1]);
        oo[2] = fmaf(pr, b.x, oo[2]);
        oo[3] = fmaf(pr, b.y, oo[3]);
    };
    int r = 0;
#pragma unroll 4
    for (; r + 1 < n; r += 2) {  // rows r, r+1 into two independent chains
        const float p0 = pick(r), p1 = pick(r + 1);
        row(r, p0, o0);
        row(r + 1, p1, o1);
    }
    if (r < n) row(r, pick(r), o0);
    if (lane == 0) {
        pp[0] = m;
        pp[1] = l;
    }
    *reinterpret_cast<float4*>(pp + 4 + 4 * lane) =
        make_float4(o0[0] + o1[0], o0[1] + o1[1], o0[2] + o1[2], o0[3] + o1[3]);
}

__global__ void attn_decode_partial(const __half* __restrict__ q, const __half* __restrict__ kc,
                                    const __half* __restrict__ vc, int heads, int kv_heads, int lmax, int L,
                                    float scale, float* __restrict__ part) {
    pdl_enter();
    constexpr int d = 128;
    __shared__ __half ks[kAttnSplit][d + 2];  // odd word stride: lane-per-row dots are conflict-free
    __shared__ __align__(16) __half vs[kAttnSplit][d];
    const int kh = blockIdx.x, sp = blockIdx.y, g = heads / kv_heads;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int p0 = sp * kAttnSplit, n = min(kAttnSplit, L - p0);
    stage_kv<kAttnSplit>(kc, vc, kh, lmax, p0, n, -1, ks, vs);
    __syncthreads();
    const int h = kh * g + warp;
    split_attend(q + (size_t)h * d, ks, vs, n, scale, lane, part + ((size_t)h * gridDim.y + sp) * kPartStride);
}

// RoPE + KV append + split-L partials + combine in ONE launch (the decode
// step's attention; replaces rope_append_kernel -> attn_decode_partial ->
// attn_decode_combine, bitwise equal to that sequence). grid (kv_heads,
// splits) over positions [0, pos]; block = 32 * g threads. Each warp rotates
// its own query head into shared memory (q itself is left untouched); the
// block whose split holds `pos` rotates the new key, writes k and v to the
// caches and uses them from shared memory (no other split reads `pos`). The
// last block of a kv head to finish (a per-head counter, zero-filled once,
// self-resetting) combines that head group's partials.
__global__ void rope_attn_decode_fused(const __half* __restrict__ q, const __half* __restrict__ k,
                                       const __half* __restrict__ v, const float* __restrict__ cosv,
                                       const float* __restrict__ sinv, __half* __restrict__ kc,
                                       __half* __restrict__ vc, int heads, int kv_heads, int lmax, int pos,
                                       float scale, float* __restrict__ part, unsigned* __restrict__ cnt,
                                       __half* __restrict__ out) {
    constexpr int d = 128, h2 = d / 2;
    __shared__ __half ks[kAttnSplit][d + 2];
    __shared__ __align__(16) __half vs[kAttnSplit][d];
    __shared__ __align__(16) __half qs[8][d];
    __shared__ int last;
    const int kh = blockIdx.x, sp = blockIdx.y, g = heads / kv_heads, splits = gridDim.y;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int L = pos + 1, p0 = sp * kAttnSplit, n = min(kAttnSplit, L - p0);
    const int h = kh * g + warp;
    const int rnew = pos - p0;  // the new token's row, if it lies in this split
    // cache rows < pos are not the producer's output (q/k/v are): staged BEFORE
    // the PDL wait, so on the SMs the previous grid's early CTAs free the KV
    // reads overlap its tail
    stage_kv<kAttnSplit>(kc, vc, kh, lmax, p0, n, rnew, ks, vs);
    pdl_enter();
    for (int t = lane; t < h2; t += 32) {  // rope_append_kernel's expression, per query head
        const float x1 = __half2float(q[(size_t)h * d + t]), x2 = __half2float(q[(size_t)h * d + t + h2]);
        const float c = cosv[t], s = sinv[t];
        qs[warp][t] = __float2half_rn(x1 * c - x2 * s);
        qs[warp][t + h2] = __float2half_rn(x2 * c + x1 * s);
    }
    if (rnew >= 0 && rnew < n) {
        for (int t = threadIdx.x; t < h2; t += blockDim.x) {
            const float x1 = __half2float(k[(size_t)kh * d + t]), x2 = __half2float(k[(size_t)kh * d + t + h2]);
            const float c = cosv[t], s = sinv[t];
            const __half o1 = __float2half_rn(x1 * c - x2 * s), o2 = __float2half_rn(x2 * c + x1 * s);
            const __half v1 = v[(size_t)kh * d + t], v2 = v[(size_t)kh * d + t + h2];
            ks[rnew][t] = o1;
            ks[rnew][t + h2] = o2;
            vs[rnew][t] = v1;
            vs[rnew][t + h2] = v2;
            __half* kdst = kc + ((size_t)kh * lmax + pos) * d;
            __half* vdst = vc + ((size_t)kh * lmax + pos) * d;
            kdst[t] = o1;
            kdst[t + h2] = o2;
            vdst[t] = v1;
            vdst[t + h2] = v2;
        }
    }
    __syncthreads();
    split_attend(qs[warp], ks, vs, n, scale, lane, part + ((size_t)h * splits + sp) * kPartStride);
    __syncthreads();  // the block's partial stores, then one gpu-scope fence (cumulative) + arrival
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned prev = atomicAdd(&cnt[kh * 32], 1u);
        last = prev == (unsigned)splits - 1;
        if (last) cnt[kh * 32] = 0;  // self-reset for the next launch
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    // attn_decode_combine's arithmetic for the g heads of this kv head: warp w, dims 4l..4l+3
    const float* ph = part + (size_t)h * splits * kPartStride;
    float M = -INFINITY;
    float num[4] = {0.f, 0.f, 0.f, 0.f}, den = 0.f;
    if (splits <= 32) {
        // every split's (m, l) in flight at once (lane t holds split t), the max
        // by shuffles (exact, order-free), then the same ascending fmaf chains
        // as below with the acc rows loaded 8 splits at a time: a few L2 round
        // trips instead of one per split -- bitwise the same result
        const float mt = lane < splits ? __ldcg(ph + lane * kPartStride) : -INFINITY;
        const float lt = lane < splits ? __ldcg(ph + lane * kPartStride + 1) : 0.f;
        M = warp_max(mt);
        const float wt = lane < splits ? __expf(mt - M) : 0.f;
        for (int t0 = 0; t0 < splits; t0 += 8) {
            float4 a[8];
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (t0 + u < splits)
                    a[u] = __ldcg(reinterpret_cast<const float4*>(ph + (t0 + u) * kPartStride + 4 + 4 * lane));
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                if (t0 + u >= splits) break;
                const float w = __shfl_sync(0xffffffffu, wt, t0 + u);
                den = fmaf(w, __shfl_sync(0xffffffffu, lt, t0 + u), den);
                num[0] = fmaf(w, a[u].x, num[0]);
                num[1] = fmaf(w, a[u].y, num[1]);
                num[2] = fmaf(w, a[u].z, num[2]);
                num[3] = fmaf(w, a[u].w, num[3]);
            }
        }
    } else {
        for (int t = 0; t < splits; ++t) M = fmaxf(M, __ldcg(ph + t * kPartStride));
        for (int t = 0; t < splits; ++t) {
            const float w = __expf(__ldcg(ph + t * kPartStride) - M);
            den = fmaf(w, __ldcg(ph + t * kPartStride + 1), den);
            const float4 a = __ldcg(reinterpret_cast<const float4*>(ph + t * kPartStride + 4 + 4 * lane));
            num[0] = fmaf(w, a.x, num[0]);
            num[1] = fmaf(w, a.y, num[1]);
            num[2] = fmaf(w, a.z, num[2]);
            num[3] = fmaf(w, a.w, num[3]);
        }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) out[(size_t)h * d + 4 * lane + j] = __float2half_rn(num[j] / den);
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
        a[i] = __float2half_rn(__fdividef(gv, 1.f + __expf(-gv)) * __half2float(u[i]));
    }
}

int launch_add_rmsnorm(void* x, const void* r, const void* w, void* y, int n, float eps, cudaStream_t st) {
    return (int)launch_pdl(add_rmsnorm_kernel, dim3(1), dim3(kRmsThreads), st, static_cast<__half*>(x),
                           static_cast<const __half*>(r), static_cast<const __half*>(w), static_cast<__half*>(y), n,
                           eps);
}

int launch_rope_append(void* q, void* k, const void* v, const float* cosv, const float* sinv, void* kc, void* vc,
                       int heads, int kv_heads, int d, int lmax, int pos, cudaStream_t st) {
    return (int)launch_pdl(rope_append_kernel, dim3(heads + kv_heads), dim3(d / 2), st, static_cast<__half*>(q),
                           static_cast<__half*>(k), static_cast<const __half*>(v), cosv, sinv,
                           static_cast<__half*>(kc), static_cast<__half*>(vc), heads, kv_heads, d, lmax, pos);
}

// workspace: one counter per head on its own 128-byte line (fused kernel;
// zero-filled once, self-resetting) at a FIXED offset 0 -- independent of the
// position, so one workspace serves every pos / ctx -- then the partials
size_t attn_decode_counter_bytes(int heads) { return (size_t)heads * 32 * sizeof(unsigned); }
size_t attn_decode_part_bytes(int heads, int L) {
    return (size_t)heads * ((L + kAttnSplit - 1) / kAttnSplit) * kPartStride * sizeof(float);
}
size_t attn_decode_workspace_bytes(int heads, int L) {
    return attn_decode_counter_bytes(heads) + attn_decode_part_bytes(heads, L);
}

int launch_rope_attn_decode(const void* q, const void* k, const void* v, const float* cosv, const float* sinv,
                            void* kc, void* vc, int heads, int kv_heads, int lmax, int pos, float scale, void* out,
                            void* ws, cudaStream_t st) {
    const int splits = (pos + 1 + kAttnSplit - 1) / kAttnSplit;
    unsigned* cnt = static_cast<unsigned*>(ws);
    float* part = reinterpret_cast<float*>(static_cast<char*>(ws) + attn_decode_counter_bytes(heads));
    return (int)launch_pdl(rope_attn_decode_fused, dim3(kv_heads, splits), dim3(32 * (heads / kv_heads)), st,
                           static_cast<const __half*>(q), static_cast<const __half*>(k),
                           static_cast<const __half*>(v), cosv, sinv, static_cast<__half*>(kc),
                           static_cast<__half*>(vc), heads, kv_heads, lmax, pos, scale, part, cnt,
                           static_cast<__half*>(out));
}

int launch_attn_decode(const void* q, const void* kc, const void* vc, int heads, int kv_heads, int lmax, int L,
                       float scale, void* out, void* ws, cudaStream_t st) {
    const int splits = (L + kAttnSplit - 1) / kAttnSplit;
    cudaError_t e = launch_pdl(attn_decode_partial, dim3(kv_heads, splits), dim3(32 * (heads / kv_heads)), st,
                               static_cast<const __half*>(q), static_cast<const __half*>(kc),
                               static_cast<const __half*>(vc), heads, kv_heads, lmax, L, scale,
                               reinterpret_cast<float*>(static_cast<char*>(ws) + attn_decode_counter_bytes(heads)));
    if (e != cudaSuccess) return (int)e;
    return (int)launch_pdl(attn_decode_combine, dim3(heads), dim3(128), st,
                           reinterpret_cast<const float*>(static_cast<const char*>(ws) + attn_decode_counter_bytes(heads)),
                           splits, static_cast<__half*>(out));
}

// argmax over n f16 values (the decode step's greedy token): every block
// reduces a grid-stride share to (max, first index), the last block to finish
// (a self-resetting counter in the workspace) reduces the block results; ties
// resolve to the smallest index, as torch.argmax
constexpr int kArgmaxBlocks = 128;
__device__ __forceinline__ void argmax_pair(float& v, int& i, float v2, int i2) {
    if (v2 > v || (v2 == v && i2 < i)) {
        v = v2;
        i = i2;
    }
}
__global__ void __launch_bounds__(256) argmax_kernel(const __half* __restrict__ x, int n, long long* __restrict__ out,
                                                     float* __restrict__ bv, int* __restrict__ bi,
                                                     unsigned* __restrict__ cnt) {
    pdl_enter();
    __shared__ float sv[8];
    __shared__ int si[8];
    __shared__ bool last;
    float v = -INFINITY;
    int i = 0x7fffffff;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x)
        argmax_pair(v, i, __half2float(x[k]), k);
    auto block_reduce = [&]() {
#pragma unroll
        for (int o = 16; o; o >>= 1) argmax_pair(v, i, __shfl_xor_sync(0xffffffffu, v, o), __shfl_xor_sync(0xffffffffu, i, o));
        if ((threadIdx.x & 31) == 0) {
            sv[threadIdx.x >> 5] = v;
            si[threadIdx.x >> 5] = i;
        }
        __syncthreads();
        if (threadIdx.x == 0)
            for (int w = 1; w < (int)(blockDim.x >> 5); ++w) argmax_pair(v, i, sv[w], si[w]);
    };
    block_reduce();
    if (threadIdx.x == 0) {
        bv[blockIdx.x] = v;
        bi[blockIdx.x] = i;
        __threadfence();
        last = atomicAdd(cnt, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    v = -INFINITY;
    i = 0x7fffffff;
    for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) argmax_pair(v, i, __ldcg(bv + b), __ldcg(bi + b));
    __syncthreads();
    block_reduce();
    if (threadIdx.x == 0) {
        *out = i;
        *cnt = 0u;  // self-reset for the next launch
    }
}

size_t argmax_workspace_bytes() { return kArgmaxBlocks * (sizeof(float) + sizeof(int)) + 128; }

int launch_argmax(const void* x, int n, long long* out, void* ws, cudaStream_t st) {
    char* w = static_cast<char*>(ws);
    unsigned* cnt = reinterpret_cast<unsigned*>(w);
    float* bv = reinterpret_cast<float*>(w + 128);
    int* bi = reinterpret_cast<int*>(w + 128 + kArgmaxBlocks * sizeof(float));
    const int blocks = n < kArgmaxBlocks * 256 ? (n + 255) / 256 : kArgmaxBlocks;
    return (int)launch_pdl(argmax_kernel, dim3(blocks), dim3(256), st, static_cast<const __half*>(x), n, out, bv, bi,
                           cnt);
}

int launch_silu_mul(const void* g, const void* u, void* a, int n, cudaStream_t st) {
    return (int)launch_pdl(silu_mul_kernel, dim3((n + 255) / 256), dim3(256), st, static_cast<const __half*>(g),
                           static_cast<const __half*>(u), static_cast<__half*>(a), n);
}

}  // namespace abcq
