// abcq_common.cuh -- shared constants and device helpers for the sm_100a kernels.
#pragma once

#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "../../include/anybcq_b200.h"

namespace abcq {

// ---------------------------------------------------------------------------
// Tiled plane layout. group_size must be 128.
//   tile  = 16 rows, slice = 256 columns (2 groups of 128 = 32 byte-chunks)
//   block = one (slice, tile) pair of one plane = 32 lanes x 16 B = 512 B
//   plane i, block (s, rt) at byte offset (s * NRT + rt) * 512
//   lane l = half * 16 + r holds the 16 reference bytes of
//       (row rt*16 + r, group 2*s + half)  -- words[i][row][4g .. 4g+3]
//   rotated left by r: stored byte j = reference byte (j + r) & 15.
// The rotation makes the 32 lanes of a warp touch 32 distinct table
// columns (= 32 distinct smem banks) at every lookup step.
// ---------------------------------------------------------------------------
constexpr int kTileRows = 16;
constexpr int kSliceCols = 256;
constexpr int kGroup = 128;
constexpr int kBlockBytes = 512;
constexpr int kChunksPerSlice = kSliceCols / 8;  // 32

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ inline int n_row_tiles(int rows) { return (int)ceil_div(rows, kTileRows); }
__host__ __device__ inline int n_slices(int cols) { return (int)ceil_div(cols, kSliceCols); }
__host__ __device__ inline int words_per_row(int cols) { return (int)ceil_div(cols, 32); }
__host__ __device__ inline int group_count(int cols, int g) { return (int)ceil_div(cols, g); }

__host__ __device__ inline int64_t tiled_plane_bytes(int rows, int cols) {
    return (int64_t)n_slices(cols) * n_row_tiles(rows) * kBlockBytes;
}
// scale set p: element (i*items + item)*32 + lane, item = s*NRT + rt, items = NS*NRT;
// offsets: item*32 + lane
__host__ __device__ inline int64_t tiled_alpha_elems(int rows, int cols, int p) {
    return (int64_t)n_slices(cols) * n_row_tiles(rows) * p * 32;
}
__host__ __device__ inline int64_t tiled_offset_elems(int rows, int cols) {
    return (int64_t)n_slices(cols) * n_row_tiles(rows) * 32;
}

// ---------------------------------------------------------------------------
// element load/store helpers
// ---------------------------------------------------------------------------
template <typename T> __device__ __forceinline__ float to_f32(T v);
template <> __device__ __forceinline__ float to_f32<float>(float v) { return v; }
template <> __device__ __forceinline__ float to_f32<__half>(__half v) { return __half2float(v); }

template <typename T> __device__ __forceinline__ T from_f32(float v);
template <> __device__ __forceinline__ float from_f32<float>(float v) { return v; }
template <> __device__ __forceinline__ __half from_f32<__half>(float v) { return __float2half_rn(v); }

__device__ __forceinline__ float load_any(const void* p, int dtype, int64_t i) {
    return dtype == ABCQ_F16 ? __half2float(static_cast<const __half*>(p)[i])
                             : static_cast<const float*>(p)[i];
}
__device__ __forceinline__ void store_any(void* p, int dtype, int64_t i, float v) {
    if (dtype == ABCQ_F16)
        static_cast<__half*>(p)[i] = __float2half_rn(v);
    else
        static_cast<float*>(p)[i] = v;
}

// ---------------------------------------------------------------------------
// 16 entries of one mu=8 chunk of the reference lookup table (gemv.py:67-81),
// bit-exact: the doubling concatenation gives every entry the f32 rounding
// sequence T[t] = ((((0 -/+ x0) -/+ x1) ...) -/+ x7) in ascending j, which is
// evaluated here directly. Entry t = hi*16 + u, u = 0..15.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void lut_chunk_entries16(const float (&xs)[8], int hi, float (&out)[16]) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
        float v = 0.f;
#pragma unroll
        for (int j = 0; j < 4; ++j) v = ((u >> j) & 1) ? v + xs[j] : v - xs[j];
#pragma unroll
        for (int j = 4; j < 8; ++j) v = ((hi >> (j - 4)) & 1) ? v + xs[j] : v - xs[j];
        out[u] = v;
    }
}

// ---------------------------------------------------------------------------
// inline PTX helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
    uint32_t r;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
    return r;
}

// packed fp32x2 add (sm_100+: FADD2) -- two independent partial sums per op
__device__ __forceinline__ unsigned long long pack2(float a, float b) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ unsigned long long fadd2(unsigned long long a, unsigned long long b) {
    unsigned long long r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ float2 unpack2(unsigned long long v) {
    float2 r;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
    return r;
}

// 16-byte global -> shared async copy; bytes past src_bytes are zero-filled
__device__ __forceinline__ void cp_async16_zfill(void* smem_dst, const void* src, uint32_t src_bytes) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(smem_dst)),
                 "l"(src), "r"(src_bytes)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// streaming 128-bit weight load: read once, keep out of L1
__device__ __forceinline__ uint4 ldg_stream(const uint4* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

// ... with an L2 cache-policy hint (e.g. evict-first after the read)
__device__ __forceinline__ uint4 ldg_stream_hint(const uint4* p, uint64_t pol) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p), "l"(pol));
    return r;
}

}  // namespace abcq

namespace abcq {
// ---------------------------------------------------------------------------
// mbarrier + bulk async copy (TMA engine, cp.async.bulk) helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}\n" ::"r"(smem_addr(bar)),
        "r"(phase)
        : "memory");
}
// L2 policy for data read exactly once per launch (weights, scales): evict
// first, so the streamed bytes do not push x and the split-K partials out of L2
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
// ... and evict-last for the split-K partials, read back by the reduce kernel
__device__ __forceinline__ uint64_t l2_evict_last_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void st_f32_hint(float* p, float v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(p), "f"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                              uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], "
        "%4;" ::"r"(smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(pol)
        : "memory");
}
// global -> shared bulk copy through the TMA engine; completes on `bar`
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}
}  // namespace abcq

namespace abcq {
// TMA-engine prefetch of a contiguous global range into L2 (no smem, no regs)
__device__ __forceinline__ void prefetch_l2_bulk(const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
// prefetch [src, src + bytes) in <= 64 KiB pieces; src and bytes multiples of 16
__device__ __forceinline__ void prefetch_l2_range(const void* src, int64_t bytes) {
    const char* p = static_cast<const char*>(src);
    while (bytes > 0) {
        const uint32_t n = bytes > 65536 ? 65536u : (uint32_t)bytes;
        prefetch_l2_bulk(p, n);
        p += n;
        bytes -= n;
    }
}
}  // namespace abcq

namespace abcq {
// ---------------------------------------------------------------------------
// add + RMSNorm statistics shared bitwise by add_rmsnorm_kernel and the GEMV's
// fused input mode (ABCQ add_rmsnorm GEMV): a 512-thread block; thread t owns
// elements 8t..8t+7 and 4096+8t..4096+8t+7 (n <= 8192); v = f16(x + r) (the
// residual stream is kept in f16); ss summed per thread in element order, then
// an xor-butterfly per warp, then the 16 warp sums in warp order.
// ---------------------------------------------------------------------------
constexpr int kRmsThreads = 512;
constexpr int kRmsMaxN = 8192;

__device__ __forceinline__ float rms_warp_sum(float v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// v[16] = f16(x + r) of the thread's elements (0 beyond n); returns the
// thread's partial sum of squares
__device__ __forceinline__ float rms_load(const __half* x, const __half* r, int n, int t, float (&v)[16]) {
    float ss = 0.f;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        const int i = (k < 8 ? 8 * t + k : 4096 + 8 * t + (k - 8));
        float xv = 0.f;
        if (i < n) {
            xv = __half2float(x[i]);
            if (r) xv = __half2float(__float2half_rn(xv + __half2float(r[i])));
        }
        v[k] = xv;
        ss += xv * xv;
    }
    return ss;
}

// block-wide inverse RMS (all 512 threads call; red: 17 floats of shared memory)
__device__ __forceinline__ float rms_inv(float ss, int n, float eps, float* red) {
    ss = rms_warp_sum(ss);
    const int t = threadIdx.x;
    if ((t & 31) == 0) red[t >> 5] = ss;
    __syncthreads();
    if (t == 0) {
        float tot = 0.f;
        for (int w = 0; w < kRmsThreads / 32; ++w) tot += red[w];
        red[16] = rsqrtf(tot / n + eps);
    }
    __syncthreads();
    return red[16];
}
}  // namespace abcq
