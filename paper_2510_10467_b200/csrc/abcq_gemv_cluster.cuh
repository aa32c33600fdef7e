// abcq_gemv_cluster.cuh -- low-latency single bit-plane GEMV for sm_100a: the
// split-K reduction happens inside a thread-block cluster through distributed
// shared memory, so a GEMV is ONE launch with no global partials, no workspace,
// no grid-wide arrival counters and no trailing reduce pass.
//
// Replaces GemvEngine.lut (/root/reference/pkg/src/anybcq/gemv.py:188-222) for
// one request: y = sum_{i<p} alpha^(p)_{i,g} (B_i x) [+ offset^(p) . gsum(x)],
// with the reference's mu = 8 chunk table (LookupTable.build, gemv.py:67-81,
// bit-identical f32 entries) and _lut_kernel's per-(plane, row, group) f32 sums
// of 16 table entries scaled by alpha (gemv.py:84-95).
//
// Decomposition (tiled layout, abcq_common.cuh): the (row tile x 256-column
// slice) plane is cut into M x C rectangles. Cluster m (C CTAs) owns row tiles
// [t0, t1); its CTA of rank c owns slices [c*NS/C, (c+1)*NS/C) of those tiles.
// Per (plane, slice) a CTA's blocks are ONE contiguous byte range, so the
// weights arrive by a handful of large TMA bulk copies.
//
// CTA = W consumer warps (8 when two CTAs share an SM, 16 for one CTA per SM)
// + 1 producer warp:
//  * producer (one lane): streams stages (slice, tile chunk, plane) of weights,
//    that plane's scales and (plane 0, asymmetric) offsets into a ring of
//    shared-memory slots (cp.async.bulk ... mbarrier::complete_tx, full/empty
//    mbarriers). Weights are static model data: it never waits on the previous
//    kernel, so with programmatic dependent launch the ring fills while the
//    previous kernel is still running (the CTA triggers its own dependents at
//    entry, so when the kernel fits two CTAs per SM the NEXT GEMV's CTAs prefetch
//    during this one).
//  * consumers: griddepcontrol.wait, then build the slices' lookup tables from x
//    (packed f32x2 adds over two chunk columns at a time, 16-byte stores) into a
//    64 KiB [t][64 col] table at a fixed shared-window address, two slices
//    resident (double-buffered across the CTA's slices), and look up: ONE PRMT
//    of (weight word, lane column register) forms the smem address, the table
//    base is the load's immediate offset. Accumulators over the p planes of a
//    (slice, tile) live in registers; per-slice row partials add into a
//    shared-memory [tile][16] buffer owned by one lane each (no races).
//  * completion: cluster barrier (release/acquire), then rank c sums its share
//    of the cluster's rows over the C ranks' partial buffers through DSMEM
//    (ld.shared::cluster) in ascending rank order -- a fixed order, so results
//    are bitwise reproducible for a given shape -- and writes y; a second
//    cluster barrier keeps every CTA's shared memory alive until read.
#pragma once
#include "abcq_gemv_lut.cuh"

namespace abcq {
namespace cl {

constexpr int kMaxTCW = 2;                  // tiles per consumer warp per stage
template <int W>
constexpr int threads_of() { return (W + 1) * 32; }  // W consumer warps + one producer warp
constexpr int kMaxRing = 32;                // ring slots (barrier space)
constexpr uint32_t kTBase = 0x800;          // table window address (low 16 bits)
constexpr uint32_t kHdrBytes = 0x400;       // [dyn base, kTBase): barriers, chunk sums
constexpr int kTblBytes = 256 * 256;        // 256 t-rows x 64 columns x f32
constexpr int kDynBase = 0x400;             // expected window address of dynamic smem
constexpr int kSmem2 = 113 * 1024;          // two CTAs per SM
constexpr int kSmem1 = 227 * 1024;          // one CTA per SM

struct Args {
    const char* planes;
    int64_t pst;          // plane stride (bytes)
    const void* alpha;    // scale set p, tiled [i][item][lane]
    const void* offset;   // offsets of set p, tiled [item][lane] (asymmetric)
    const void* x;
    void* y;
    int rows, cols, NRT, NS, items, p, glu;
    int C, M;             // cluster size, clusters
    int tc;               // max tiles per stage (<= W * kMaxTCW)
    int ring;             // ring slots
    int stage_bytes;      // bytes per slot
    int part_off;         // dynamic-smem offset of the [tile][16] partials
    int xs_off;           // dynamic-smem offset of the staged x (f32) of the CTA's slices
    int recv_off;         // dynamic-smem offset of the DSMEM receive buffer [rank][rows per rank]
    int ring_off;         // dynamic-smem offset of slot 0
    int smem;             // dynamic smem bytes (checked)
    int dbg;              // 1 = skip the lookups (profiling experiment)
    unsigned long long* trace;  // optional: 8 stamps per CTA
};

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ float ld_dsmem_f32(uint32_t local_addr, uint32_t rank) {
    uint32_t ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(local_addr), "r"(rank));
    float v;
    asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(ra) : "memory");
    return v;
}
template <int W>
__device__ __forceinline__ void bar_consumers() { asm volatile("bar.sync 1, %0;" ::"n"(W * 32) : "memory"); }
__device__ __forceinline__ void mbar_arrive_cta(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ float lds_f32_at(uint32_t addr) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ uint4 lds_v4(uint32_t addr) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
    return v;
}
__device__ __forceinline__ float4 lds_v4f(uint32_t addr) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
    return v;
}
template <typename ST>
__device__ __forceinline__ float lds_scale(uint32_t addr) {
    if constexpr (sizeof(ST) == 2) {
        unsigned short h;
        asm volatile("ld.shared.u16 %0, [%1];" : "=h"(h) : "r"(addr));
        return __half2float(__ushort_as_half(h));
    } else {
        return lds_f32_at(addr);
    }
}
__device__ __forceinline__ void sts_f32(uint32_t addr, float v) {
    asm volatile("st.shared.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}
__device__ __forceinline__ void sts_v2(uint32_t addr, float a, float b) {
    asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(addr), "f"(a), "f"(b) : "memory");
}

// 16 lookups of one 16-byte lane block. rb[k] = column bytes of steps 2k, 2k+1
// in bytes 0..1 and the high half of the table's window address in bytes 2..3;
// the low half of the table base (kTBase) and the segment (+32 columns) are the
// load's immediate offset. Four packed FADD2 chains.
template <int SEG>
__device__ __forceinline__ float lut16c(const uint4 w, const uint32_t (&rb)[8]) {
    const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
    unsigned long long acc[4];
#pragma unroll
    for (int j = 0; j < 16; j += 2) {
        const uint32_t a0 = prmt(ww[j >> 2], rb[j >> 1], 0x7604u | ((j & 3) << 4));
        const uint32_t a1 = prmt(ww[(j + 1) >> 2], rb[j >> 1], 0x7605u | (((j + 1) & 3) << 4));
        const float v0 = lds_f32_at(a0 + kTBase + SEG * 128);
        const float v1 = lds_f32_at(a1 + kTBase + SEG * 128);
        const int ch = (j >> 1) & 3;
        acc[ch] = j < 8 ? pack2(v0, v1) : fadd2(acc[ch], pack2(v0, v1));
    }
    const float2 f = unpack2(fadd2(fadd2(acc[0], acc[1]), fadd2(acc[2], acc[3])));
    return f.x + f.y;
}

// Table build of one slice into segment `seg` by one consumer thread: chunk
// columns 2cp, 2cp+1 (packed f32x2), entries t = u + 16h, h = 0..15. Every entry
// keeps the reference's f32 rounding sequence ((((0 -/+ x0) -/+ x1) ...) -/+ x7)
// (gemv.py:67-81): the prefix over x0..x3 (bits of u), then the binary tree over
// x4..x7 -- 34 packed adds and 16 8-byte stores per 32 entries.
__device__ __forceinline__ void build_cols2(const float (&xa)[8], const float (&xb)[8], int u, int cp,
                                            uint32_t tbl_lo, int seg, uint32_t csum_lo) {
    unsigned long long v = 0ull;  // (+0, +0)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const unsigned long long xv = ((u >> j) & 1) ? pack2(xa[j], xb[j]) : pack2(-xa[j], -xb[j]);
        v = fadd2(v, xv);
    }
    unsigned long long leaf[16];
    leaf[0] = v;
#pragma unroll
    for (int j = 4; j < 8; ++j) {
        const int n = 1 << (j - 4);
        const unsigned long long px = pack2(xa[j], xb[j]), nx = pack2(-xa[j], -xb[j]);
#pragma unroll
        for (int k = n - 1; k >= 0; --k) {
            leaf[k + n] = fadd2(leaf[k], px);
            leaf[k] = fadd2(leaf[k], nx);
        }
    }
#pragma unroll
    for (int h = 0; h < 16; ++h) {
        const float2 e = unpack2(leaf[h]);
        sts_v2(tbl_lo + (uint32_t)((u + 16 * h) * 256 + seg * 128 + cp * 8), e.x, e.y);
    }
    if (u == 15 && csum_lo) {  // T[255] = chunk sum (asymmetric group sums)
        const float2 e = unpack2(leaf[15]);
        sts_v2(csum_lo + (uint32_t)((seg * 32 + 2 * cp) * 4), e.x, e.y);
    }
}

// the same build split over two threads (W = 16: 512 builders): entries
// t = u + 16h for h in [8hb, 8hb + 8) -- the tree over x4..x6, then -/+ x7
// (h bit 3 = hb): the reference's rounding sequence unchanged
__device__ __forceinline__ void build_cols2_half(const float (&xa)[8], const float (&xb)[8], int u, int hb, int cp,
                                                 uint32_t tbl_lo, int seg, uint32_t csum_lo) {
    unsigned long long v = 0ull;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const unsigned long long xv = ((u >> j) & 1) ? pack2(xa[j], xb[j]) : pack2(-xa[j], -xb[j]);
        v = fadd2(v, xv);
    }
    unsigned long long leaf[8];
    leaf[0] = v;
#pragma unroll
    for (int j = 4; j < 7; ++j) {
        const int n = 1 << (j - 4);
        const unsigned long long px = pack2(xa[j], xb[j]), nx = pack2(-xa[j], -xb[j]);
#pragma unroll
        for (int k = n - 1; k >= 0; --k) {
            leaf[k + n] = fadd2(leaf[k], px);
            leaf[k] = fadd2(leaf[k], nx);
        }
    }
    const unsigned long long x7 = hb ? pack2(xa[7], xb[7]) : pack2(-xa[7], -xb[7]);
#pragma unroll
    for (int h = 0; h < 8; ++h) {
        const float2 e = unpack2(fadd2(leaf[h], x7));
        sts_v2(tbl_lo + (uint32_t)((u + 16 * (h + 8 * hb)) * 256 + seg * 128 + cp * 8), e.x, e.y);
        if (h == 7 && hb && u == 15 && csum_lo) sts_v2(csum_lo + (uint32_t)((seg * 32 + 2 * cp) * 4), e.x, e.y);
    }
}

// x values of chunk columns 2cp, 2cp+1 of slice s (16 consecutive inputs)
template <typename XT>
__device__ __forceinline__ void slice_x16(const Args& a, int s, int cp, float (&xa)[8], float (&xb)[8]) {
    const XT* x = static_cast<const XT*>(a.x);
    const int k0 = s * kSliceCols + 16 * cp;
    load_x8_any<XT>(x, k0, a.cols, a.glu, xa);
    load_x8_any<XT>(x, k0 + 8, a.cols, a.glu, xb);
}

#define ABCQ_CTRACE(k)                                                                        \
    do {                                                                                      \
        if (a.trace) a.trace[(size_t)blockIdx.x * 16 + (k)] = globaltimer();                   \
    } while (0)

template <typename XT, typename YT, typename ST, bool ASYM, int W>
__global__ void __launch_bounds__(threads_of<W>(), (W == 8 ? 2 : 1)) gemv_cluster_kernel(const __grid_constant__ Args a) {
    extern __shared__ __align__(1024) char smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t base = smem_addr(smem);
    // the table sits at window address hi | kTBase; the header below it
    if ((base & 0xFFFFu) + 768u > kTBase || (int)(kTBase - (base & 0xFFFFu)) + kTblBytes > a.part_off) {
        if (tid == 0) __trap();
    }
    // shared-memory accesses by explicit window address: in a cluster launch
    // the CTA's own window carries its rank in bits 24..31 (an address with
    // the rank bits stripped faults with an illegal-instruction error)
    const uint32_t lo_base = base;
    const uint32_t tbl_lo = lo_base + (kTBase - (base & 0xFFFFu));  // low 16 bits == kTBase
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* empty = full + kMaxRing;
    const uint32_t csum_lo = lo_base + 2 * kMaxRing * 8;  // [2][32] f32
    const uint32_t part_lo = lo_base + a.part_off;       // [tile][16] f32
    const uint32_t xs_lo = lo_base + a.xs_off;
    const uint32_t ring_lo = lo_base + a.ring_off;
    char* ring = smem + a.ring_off;

    const int C = a.C;
    const int rank = C > 1 ? (int)cluster_rank() : 0;
    const int m = blockIdx.x / C;
    const int t0 = (int)((int64_t)m * a.NRT / a.M), t1 = (int)((int64_t)(m + 1) * a.NRT / a.M);
    const int s0 = (int)((int64_t)rank * a.NS / C), s1 = (int)((int64_t)(rank + 1) * a.NS / C);
    const int T = t1 - t0, S = s1 - s0;
    const int nch = T > 0 ? (T + a.tc - 1) / a.tc : 0;
    const int R = a.ring, p = a.p;
    const int nst = S * nch;

    if (tid == 0) {
        ABCQ_CTRACE(0);
        if (a.trace) {
            uint32_t smid;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
            a.trace[(size_t)blockIdx.x * 16 + 6] = smid;
        }
        for (int s = 0; s < R; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], W);
        }
        fence_mbar_init();
    }
    __syncthreads();
    // the next kernel may launch now: with two CTAs per SM its producers fill
    // their rings while this grid runs (dbg 64: only once past the PDL wait)
    if (!(a.dbg & 64)) pdl_launch_dependents();

    if (warp == W) {
        // ---------------- producer: weights/scales never depend on the previous kernel
        if (lane == 0 && nst > 0) {
            ABCQ_CTRACE(11);
            const uint64_t pol = l2_evict_first_policy();
            const int esz = (int)sizeof(ST);
            int sl = 0, k = 0, slot = 0;
            uint32_t ph = 0;
            const uint32_t wsz = (uint32_t)(a.tc * kBlockBytes), ssz = (uint32_t)(a.tc * 32 * esz);
            for (int e = 0; e < nst; ++e) {
                if (e == 1) ABCQ_CTRACE(12);
                if (e >= R) mbar_wait(&empty[slot], ph ^ 1u);
                const int s = s0 + sl;
                const int ta = t0 + k * T / nch, tb = t0 + (k + 1) * T / nch;
                const int n = tb - ta;
                const int64_t item0 = (int64_t)s * a.NRT + ta;
                char* st = ring + (size_t)slot * a.stage_bytes;
                const uint32_t wb = (uint32_t)n * kBlockBytes, ab = (uint32_t)(n * 32 * esz);
                mbar_arrive_expect_tx(&full[slot], (uint32_t)p * (wb + ab) + (ASYM ? ab : 0u));
                const char* wsrc = a.planes + item0 * kBlockBytes;
                const char* asrc = static_cast<const char*>(a.alpha) + item0 * 32 * esz;
                for (int i = 0; i < p; ++i) {  // plane i: weights [i][tile], scales [i][tile][lane]
                    bulk_g2s_hint(st + i * wsz, wsrc + (int64_t)i * a.pst, wb, &full[slot], pol);
                    bulk_g2s_hint(st + p * wsz + i * ssz, asrc + (int64_t)i * a.items * 32 * esz, ab, &full[slot], pol);
                }
                if (ASYM)
                    bulk_g2s_hint(st + p * (wsz + ssz), static_cast<const char*>(a.offset) + item0 * 32 * esz, ab,
                                  &full[slot], pol);
                if (++k == nch) {
                    k = 0;
                    ++sl;
                }
                if (++slot == R) {
                    slot = 0;
                    ph ^= 1u;
                }
            }
            ABCQ_CTRACE(8);
        }
        __syncwarp();
    } else {
        // ---------------- consumers
        const int half = lane >> 4, r = lane & 15;
        uint32_t rb0[8];  // column bytes of segment 0 (+ the window's high bits)
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const uint32_t c0 = (uint32_t)((half * 16 + ((2 * k + r) & 15)) * 4);
            const uint32_t c1 = (uint32_t)((half * 16 + ((2 * k + 1 + r) & 15)) * 4);
            rb0[k] = c0 | (c1 << 8) | (tbl_lo & 0xFFFF0000u);
        }
        for (int q = tid; q < T * 16; q += W * 32) sts_f32(part_lo + q * 4, 0.f);
        const int cp = tid & 15, u = (tid >> 4) & 15, hb = tid >> 8;  // build role: column pair, entry bits
        const uint32_t cs = ASYM ? csum_lo : 0u;
        // build slice sl's table into segment sl & 1 from the staged x
        auto build = [&](int sl) {
            const uint32_t xv = xs_lo + (uint32_t)((sl * kSliceCols + cp * 16) * 4);
            const float4 v0 = lds_v4f(xv), v1 = lds_v4f(xv + 16), v2 = lds_v4f(xv + 32), v3 = lds_v4f(xv + 48);
            const float pa[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
            const float pb[8] = {v2.x, v2.y, v2.z, v2.w, v3.x, v3.y, v3.z, v3.w};
            if constexpr (W == 8) build_cols2(pa, pb, u, cp, tbl_lo, sl & 1, cs);
            else build_cols2_half(pa, pb, u, hb, cp, tbl_lo, sl & 1, cs);
        };

        pdl_wait();  // x (and y) belong to the previous kernel
        if (a.dbg & 64) pdl_launch_dependents();
        if (tid == 0) ABCQ_CTRACE(1);
        {
            // x of the CTA's slices -> shared memory (f32): one loop (one copy
            // of the f16 / f32 / SiLU-gated load code), every load in flight
            const int nq = S * kChunksPerSlice;
            const XT* xg = static_cast<const XT*>(a.x);
#pragma unroll 1
            for (int q = tid; q < ((a.dbg & 32) ? 0 : nq); q += W * 32) {
                float xq[8];
                load_x8_any<XT>(xg, s0 * kSliceCols + q * 8, a.cols, a.glu, xq);
                const uint32_t d = xs_lo + (uint32_t)(q * 32);
                sts_v2(d, xq[0], xq[1]);
                sts_v2(d + 8, xq[2], xq[3]);
                sts_v2(d + 16, xq[4], xq[5]);
                sts_v2(d + 24, xq[6], xq[7]);
            }
        }
        bar_consumers<W>();
        if (tid == 0) ABCQ_CTRACE(9);
#pragma unroll 1
        for (int sl = 0; sl < S && sl < 2 && !(a.dbg & 4); ++sl) build(sl);
        bar_consumers<W>();
        if (tid == 0) ABCQ_CTRACE(2);

        int slot = 0;
        uint32_t ph = 0;
        const uint32_t wsz = (uint32_t)(a.tc * kBlockBytes);                  // one plane's weights in a slot
        const uint32_t ssz = (uint32_t)(a.tc * 32 * (int)sizeof(ST));        // one plane's scales in a slot
        const uint32_t soff = (uint32_t)p * wsz, zoff = (uint32_t)p * (wsz + ssz);
#pragma unroll 1
        for (int sl = 0; sl < S; ++sl) {
            uint32_t rb[8];
            const uint32_t segadd = (sl & 1) ? 0x8080u : 0u;  // +32 columns in both column bytes
#pragma unroll
            for (int k = 0; k < 8; ++k) rb[k] = rb0[k] + segadd;
            float gx = 0.f;
            if constexpr (ASYM) {
#pragma unroll
                for (int c = 0; c < 16; ++c) gx += lds_f32_at(csum_lo + ((sl & 1) * 32 + half * 16 + c) * 4);
            }
            // four independent blocks (tile slot q, plane i) of the slot: loads first, then the lookups
            auto group4 = [&](uint32_t st, const uint32_t (&qq)[4], const uint32_t (&ii)[4], const bool (&vv)[4],
                              const bool (&to1)[4], float& acc0, float& acc1) {
                uint4 w[4];
                float sc[4];
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    w[b] = lds_v4(st + ii[b] * wsz + qq[b] * kBlockBytes + lane * 16);
                    sc[b] = lds_scale<ST>(st + soff + ii[b] * ssz + (qq[b] * 32 + lane) * (uint32_t)sizeof(ST));
                }
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    const float l = lut16c<0>(w[b], rb);
                    if (vv[b]) {
                        if (to1[b]) acc1 = fmaf(sc[b], l, acc1);
                        else acc0 = fmaf(sc[b], l, acc0);
                    }
                }
            };
#pragma unroll 1
            for (int k = 0; k < nch; ++k) {
                const int ta = k * T / nch, tb = (k + 1) * T / nch;
                const int nt = tb - ta;  // chunk tiles; this warp takes q = warp (and warp + W)
                const bool v0 = warp < nt, v1 = warp + W < nt;
                const uint32_t q0 = (uint32_t)(v0 ? warp : 0), q1 = (uint32_t)(v1 ? warp + W : 0);
                float acc0 = 0.f, acc1 = 0.f;
                mbar_wait(&full[slot], ph);
                if (tid == 0 && sl == 0 && k == 0) ABCQ_CTRACE(13);
                const uint32_t st = ring_lo + (uint32_t)(slot * a.stage_bytes);
                if ((a.dbg & 1) == 0 && v0) {
                    // two tiles x two planes per group (one code path: a warp
                    // without a second tile looks up a duplicate, discarded)
#pragma unroll 1
                    for (int i = 0; i < p; i += 2) {
                        const bool pv = i + 1 < p;
                        const uint32_t i1 = pv ? i + 1 : i;
                        const uint32_t qq[4] = {q0, q1, q0, q1}, ii[4] = {(uint32_t)i, (uint32_t)i, i1, i1};
                        const bool vv[4] = {true, v1, pv, v1 && pv}, t1[4] = {false, true, false, true};
                        group4(st, qq, ii, vv, t1, acc0, acc1);
                    }
                    if constexpr (ASYM) {  // + offset . group sum of x, after the planes
                        acc0 = fmaf(lds_scale<ST>(st + zoff + (q0 * 32 + lane) * (uint32_t)sizeof(ST)), gx, acc0);
                        if (v1) acc1 = fmaf(lds_scale<ST>(st + zoff + (q1 * 32 + lane) * (uint32_t)sizeof(ST)), gx, acc1);
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive_cta(&empty[slot]);
                if (++slot == R) {
                    slot = 0;
                    ph ^= 1u;
                }
                // the slice's two groups (lanes l, l+16) -> row partials of this slice
                const float r0v = acc0 + __shfl_down_sync(0xffffffffu, acc0, 16);
                const float r1v = acc1 + __shfl_down_sync(0xffffffffu, acc1, 16);
                if (lane < 16) {
                    if (v0) {
                        const uint32_t pa = part_lo + ((ta + warp) * 16 + lane) * 4;
                        sts_f32(pa, lds_f32_at(pa) + r0v);
                    }
                    if (v1) {
                        const uint32_t pa = part_lo + ((ta + warp + W) * 16 + lane) * 4;
                        sts_f32(pa, lds_f32_at(pa) + r1v);
                    }
                }
            }
            if (sl + 1 < S && S > 2) {
                bar_consumers<W>();  // all warps done with segment sl&1; publishes the build of slice sl+1
                if (sl + 2 < S) build(sl + 2);
            }
        }
        bar_consumers<W>();  // all row partials of this CTA written
        if (tid == 0) ABCQ_CTRACE(3);
        if (C == 1) {
            YT* y = static_cast<YT*>(a.y);
            const int r0 = t0 * kTileRows, r1 = min(t1 * kTileRows, a.rows);
            for (int row = r0 + tid; row < r1; row += W * 32) y[row] = from_f32<YT>(lds_f32_at(part_lo + (row - r0) * 4));
        }
    }
    if (C > 1 && !(a.dbg & 8)) {
        // push: the cluster's rows are split over the ranks; every rank stores
        // its partial of rank c's rows into c's receive buffer (DSMEM), one
        // cluster barrier, then each rank sums its rows over the ranks in
        // ascending order (fixed: bitwise reproducible) and writes y
        const int r0 = t0 * kTileRows, nr = min(t1 * kTileRows, a.rows) - r0;
        const int rpr = (nr + C - 1) / C;  // rows per rank
        const uint32_t recv_lo = lo_base + a.recv_off;
        if (warp < W) {
            for (int q = tid; q < nr; q += W * 32) {
                const int c = q / rpr;
                uint32_t ra;
                asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
                             : "=r"(ra)
                             : "r"(recv_lo + (uint32_t)((rank * rpr + q - c * rpr) * 4)), "r"((uint32_t)c));
                asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(ra), "f"(lds_f32_at(part_lo + q * 4)) : "memory");
            }
        }
        cluster_sync_all();  // every rank's pushes landed
        if (tid == 0) ABCQ_CTRACE(10);
        if (warp < W) {
            YT* y = static_cast<YT*>(a.y);
            const int lo = rank * rpr, hi_r = min(nr, lo + rpr);
            for (int q = lo + tid; q < hi_r; q += W * 32) {
                float sum = lds_f32_at(recv_lo + (uint32_t)((q - lo) * 4));
                for (int c = 1; c < C; ++c) sum += lds_f32_at(recv_lo + (uint32_t)((c * rpr + q - lo) * 4));
                y[r0 + q] = from_f32<YT>(sum);
            }
        }
    }
    if (tid == 0) ABCQ_CTRACE(4);
}

}  // namespace cl
}  // namespace abcq
