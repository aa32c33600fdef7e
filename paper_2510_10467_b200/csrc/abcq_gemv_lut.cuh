// abcq_gemv_lut.cuh -- building blocks of the sm_100a batch-1 bit-plane GEMV
// (the kernel itself: abcq_gemv_batch.cuh).
//
// Replaces GemvEngine.lut + LookupTable.build + _lut_kernel
// (/root/reference/pkg/src/anybcq/gemv.py:67-95,188-222):
//
//   y[n] = sum_{i<p} sum_g alpha^(p)[i,n,g] * s(i,n,g)   (+ offset^(p)[n,g] * gx[g])
//   s(i,n,g) = sum_{c in g} T[c][byte(i,n,c)]             (mu = 8 chunk table)
//
// Design:
//  * work item = (256-column slice s, 16-row tile rt) = one 512-byte block per
//    plane; items are ordered slice-major and split evenly over a one-wave
//    grid; a CTA owns a contiguous item range spanning at most two slices
//    ("segments"). For every plane that range is ONE contiguous byte range.
//  * TMA bulk-copy pipeline: a producer warp streams stages of
//    (kChunk items x one plane) -- weights, that plane's scales, and (plane 0,
//    asymmetric) the offsets -- global -> shared through the TMA engine into a
//    kStages-deep ring (mbarrier full/empty). ~100 KB per SM stay in flight
//    continuously, independent of the consumers' issue; weights are static
//    model data, so the producer never waits on the previous kernel (PDL).
//  * consumers (16 warps) build the reference lookup table of the CTA's
//    slices in shared memory -- 32 chunks x 256 entries x f32 per slice in a
//    [t][col] slab with a 256-byte t-row, segment k = columns 32k..32k+31 --
//    so that smem address = PRMT(weight word, lane column bytes) = t<<8|col*4
//    costs ONE instruction per looked-up byte; the pack-time byte rotation
//    (abcq_pack.cu) puts the 32 lanes on 32 distinct banks.
//  * p is a runtime kernel argument: stages run chunk-major, plane-minor; a
//    warp owns 2 items of every chunk and keeps their accumulators across the
//    p plane stages. Per element: 16 lookups summed with packed FADD2, one
//    FFMA by alpha; asymmetric offsets: one FFMA with the group sum of x.
//  * split over slices: each item writes a 16-row partial to an L2-resident
//    workspace; a small PDL-chained kernel sums the partials in a fixed
//    order (deterministic) and writes y.
#pragma once
#include <type_traits>

#include "abcq_common.cuh"
#include "abcq_internal.h"

namespace abcq {

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
constexpr int kTraceCtas = 168;  // per launch trace slot: 8 stamps per CTA

constexpr int kMaxFastP = ABCQ_MAX_PLANES;
constexpr int kTableBytes = 256 * 256;  // 256 t-rows x 64 cols x 4 B: two 32-col segments
constexpr int kXBytes = 2 * kSliceCols * 4;



// The lookup table lives at shared-window address kTableWindow (64 KiB), so a
// PRMT of (weight word, lane column register) yields the ABSOLUTE smem address
// 0x1_tt_cc: byte0 = column*4 (rb byte), byte1 = weight byte t, byte2 = rb
// byte 3 (= 0x01), byte3 = sign of rb byte 3 (= 0) -- no base-register add.
constexpr uint32_t kTableWindow = 0x10000;

__device__ __forceinline__ float lds_f32(uint32_t addr) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
    return v;
}

// 16 lookups of one 16-byte lane block. rb[k] holds the column bytes of steps
// 3k..3k+2 in bytes 0..2 and 0x01 in byte 3. SEG selects the table segment
// (+32 columns = +128 B) through the load's immediate offset. Four packed
// FADD2 chains keep the dependent-add depth at 2.
template <int SEG>
__device__ __forceinline__ float lut16(const uint4 w, const uint32_t (&rb)[6]) {
    const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
    unsigned long long acc[4];
#pragma unroll
    for (int j = 0; j < 16; j += 2) {
        const uint32_t a0 = prmt(ww[j >> 2], rb[j / 3], 0xF700u | ((j & 3) << 4) | (4 + j % 3));
        const uint32_t a1 =
            prmt(ww[(j + 1) >> 2], rb[(j + 1) / 3], 0xF700u | (((j + 1) & 3) << 4) | (4 + (j + 1) % 3));
        const float v0 = lds_f32(a0 + SEG * 128);
        const float v1 = lds_f32(a1 + SEG * 128);
        const int ch = (j >> 1) & 3;
        acc[ch] = j < 8 ? pack2(v0, v1) : fadd2(acc[ch], pack2(v0, v1));
    }
    const float2 f = unpack2(fadd2(fadd2(acc[0], acc[1]), fadd2(acc[2], acc[3])));
    return f.x + f.y;
}

template <typename XT>
__device__ __forceinline__ void load_x8(const XT* x, int k0, int cols, float (&xs)[8]) {
    if (k0 + 8 <= cols) {
        if constexpr (sizeof(XT) == 2) {
            const uint4 v = __ldg(reinterpret_cast<const uint4*>(x + k0));
            const __half2* h = reinterpret_cast<const __half2*>(&v);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const float2 f = __half22float2(h[j]);
                xs[2 * j] = f.x;
                xs[2 * j + 1] = f.y;
            }
        } else {
            const float4 a = __ldg(reinterpret_cast<const float4*>(x + k0));
            const float4 b = __ldg(reinterpret_cast<const float4*>(x + k0 + 4));
            xs[0] = a.x; xs[1] = a.y; xs[2] = a.z; xs[3] = a.w;
            xs[4] = b.x; xs[5] = b.y; xs[6] = b.z; xs[7] = b.w;
        }
    } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) xs[j] = (k0 + j < cols) ? to_f32<XT>(x[k0 + j]) : 0.f;
    }
}

// x = [g ; u] (2*cols f16, ABCQ_F16_SILU_GLU): the input is f16(silu(g) * u),
// the same expression as silu_mul_kernel (abcq_decode_ops.cu) -> bitwise equal
__device__ __forceinline__ float silu_glu(__half g, __half u) {
    const float gv = __half2float(g);
    return __half2float(__float2half_rn(__fdividef(gv, 1.f + __expf(-gv)) * __half2float(u)));
}

template <typename XT>
__device__ __forceinline__ void load_x8_glu(const XT* x, int k0, int cols, float (&xs)[8]) {
    if constexpr (sizeof(XT) == 2) {
        const __half* g = reinterpret_cast<const __half*>(x);
        const __half* u = g + cols;
        if (k0 + 8 <= cols && (cols & 7) == 0) {
            const uint4 gv = __ldg(reinterpret_cast<const uint4*>(g + k0));
            const uint4 uv = __ldg(reinterpret_cast<const uint4*>(u + k0));
            const __half* gh = reinterpret_cast<const __half*>(&gv);
            const __half* uh = reinterpret_cast<const __half*>(&uv);
#pragma unroll
            for (int j = 0; j < 8; ++j) xs[j] = silu_glu(gh[j], uh[j]);
        } else {
#pragma unroll
            for (int j = 0; j < 8; ++j) xs[j] = (k0 + j < cols) ? silu_glu(g[k0 + j], u[k0 + j]) : 0.f;
        }
    } else {
        load_x8<XT>(x, k0, cols, xs);  // (f32 x has no gated form; the host rejects it)
    }
}

template <typename XT>
__device__ __forceinline__ void load_x8_any(const XT* x, int k0, int cols, int glu, float (&xs)[8]) {
    if (glu) load_x8_glu<XT>(x, k0, cols, xs);
    else load_x8<XT>(x, k0, cols, xs);
}

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" :::); }
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}



}  // namespace abcq
