// imf_count.cu -- K1 for 8/16-bit tiles whose histogram and omega fit shared
// memory: the paper's bucket (counting) sort (PAPER.md:262-276,
// ordinal.py:62-79 _rank_by_bucket) with the tile held in registers.
#include <type_traits>

#include "imf_k1.cuh"

namespace imf {

// k1_count with the tile held in registers: warp w owns input rows w + 32j,
// lane l owns columns l + 32k (j, k < NK = ceil(S/32)), so every value is read
// from global memory ONCE, with all NK*NK loads of a thread in flight together
// (the two-pass k1_count re-reads the tile and exposes the L2 latency per row).
// 1024 threads; same histogram / scan / scatter as k1_count.
// ---- TMA tile load (planar layouts: s_x == 1) ------------------------------
// One elected thread arms an mbarrier with the box's byte count and issues a
// 4D cp.async.bulk.tensor (dims W, H, C, B) for the tile's whole input box;
// the box may hang off the image (TMA fills zeros there) and every thread then
// reads its pixels at CLAMPED box coordinates -- the replicate padding of
// tiling.py:134-140 without a padded copy.  Interleaved (HWC) images keep the
// per-lane __ldg path: TMA cannot stride the innermost dimension, and a box of
// all channels would not fit next to the 128 KB histogram.
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(bar),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void tma_load_4d(uint32_t dst, const CUtensorMap* tm, int c0, int c1, int c2, int c3,
                                            uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
        "%5}], [%6];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar)
        : "memory");
}

template <int DT, int NK, bool TMA>
__global__ void __launch_bounds__(1024) k1_count_reg(Geom g, uint16_t* __restrict__ omega_out,
                                                     const __grid_constant__ CUtensorMap tmap) {
    extern __shared__ __align__(128) unsigned char smem[];
    constexpr int NB = DT == DT_U8 ? 256 : 65536;
    constexpr int NW = NB / 2;
    using T = typename std::conditional<DT == DT_U8, uint8_t, uint16_t>::type;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const TileCoord tc = tile_coord_cta(g, g.tile_begin + blockIdx.x);
    const int S = g.Sw, SH = g.Sh;
    uint32_t* hw = reinterpret_cast<uint32_t*>(smem);
    uint32_t* dummy = hw + NW;  // 32 words: per-lane sink for the atomics of unranked slots
    // hw + NW + 32: the TMA mbarrier (8 B); omega (and the TMA box) 128-B aligned after it
    uint16_t* om = reinterpret_cast<uint16_t*>(hw + NW + 64);
    uint32_t v[NK][NK];
    if (TMA) {
        // the box lands where omega will be built (omega is written only after
        // every value has moved into registers)
        const T* box = reinterpret_cast<const T*>(om);
        const uint32_t bar = (uint32_t)__cvta_generic_to_shared(hw + NW + 32);
        // the box's first column must sit on a 16-byte boundary (TMA tile mode):
        // start at the aligned column at or left of the tile's first input column
        constexpr int Q = 16 / (int)sizeof(T);
        const int xin = tc.ox0 - g.r + g.vshift, by0 = tc.oy0 - g.r + g.vshift;
        const int bx0 = xin - (((xin % Q) + Q) % Q);
        if (tid == 0) {
            mbar_init(bar, 1);
            mbar_expect_tx(bar, (uint32_t)(g.tma_bw * SH * (int)sizeof(T)));
            tma_load_4d((uint32_t)__cvta_generic_to_shared(om), &tmap, bx0, by0, tc.c, tc.b, bar);
        }
        int xb[NK];
#pragma unroll
        for (int k = 0; k < NK; k++) {
            const int x = xin + lane + 32 * k;
            xb[k] = (x < 0 ? 0 : (x >= g.W ? g.W - 1 : x)) - bx0;
        }
        __syncthreads();  // barrier initialized before anyone waits on it
        mbar_wait(bar, 0);
#pragma unroll
        for (int j = 0; j < NK; j++) {
            const int y = wid + 32 * j;
            const int yy = by0 + y;
            const T* row = box + ((yy < 0 ? 0 : (yy >= g.H ? g.H - 1 : yy)) - by0) * g.tma_bw;
            uint32_t lohi = (uint32_t)(S - 1) << 16;
            if (g.fprow) lohi = y < SH ? __ldg(g.fprow + y) : 0xffffffffu;
            else if (y >= SH) lohi = 0xffffffffu;
            const int lo = (int)(lohi & 0xffffu), span = (int)(lohi >> 16) - lo;
#pragma unroll
            for (int k = 0; k < NK; k++) {
                const bool ok = (unsigned)(lane + 32 * k - lo) <= (unsigned)span;
                v[j][k] = ok ? (uint32_t)row[xb[k]] : 0xffffffffu;
            }
        }
    } else {
        // element offsets within one (image, channel) plane fit 32 bits
        int xo[NK];
#pragma unroll
        for (int k = 0; k < NK; k++) {
            int x = tc.ox0 + lane + 32 * k - g.r + g.vshift;
            x = x < 0 ? 0 : (x >= g.W ? g.W - 1 : x);
            xo[k] = x * (int)g.s_x;
        }
        const T* plane = reinterpret_cast<const T*>(tc.src);
#pragma unroll
        for (int j = 0; j < NK; j++) {
            const int y = wid + 32 * j;
            int yy = tc.oy0 + y - g.r + g.vshift;
            yy = yy < 0 ? 0 : (yy >= g.H ? g.H - 1 : yy);
            const T* row = plane + yy * (int)g.s_y;
            // ranked columns of this row: [lo, hi] (footprint table, else the whole row)
            // (lo = hi = 0xffff: no pixel -- x < 256 never matches)
            uint32_t lohi = (uint32_t)(S - 1) << 16;
            if (g.fprow) lohi = y < SH ? __ldg(g.fprow + y) : 0xffffffffu;
            else if (y >= SH) lohi = 0xffffffffu;
            const int lo = (int)(lohi & 0xffffu), span = (int)(lohi >> 16) - lo;
#pragma unroll
            for (int k = 0; k < NK; k++) {
                const bool ok = (unsigned)(lane + 32 * k - lo) <= (unsigned)span;
                v[j][k] = ok ? (uint32_t)__ldg(row + xo[k]) : 0xffffffffu;
            }
        }
    }
    {
        uint4* h4 = reinterpret_cast<uint4*>(hw);
        for (int i = tid; i < NW / 4; i += blockDim.x) h4[i] = make_uint4(0, 0, 0, 0);
    }
    __syncthreads();  // (TMA: every value is in registers; the box may be overwritten)
    // counting pass: the count a pixel's atomic returns is its index among the
    // tile's equal values, kept in the key's high half, so rank = prefix(value)
    // + that index -- the scatter needs a load, not a second atomic.  Unranked
    // slots count into a per-lane sink word (no branch, no same-address
    // serialization).
#pragma unroll
    for (int j = 0; j < NK; j++)
#pragma unroll
        for (int k = 0; k < NK; k++) {
            const uint32_t val = v[j][k];
            const bool ok = val != 0xffffffffu;
            const uint32_t sh = (val & 1) << 4;
            uint32_t* w = ok ? hw + (val >> 1) : dummy + lane;
            const uint32_t old = atomicAdd(w, 1u << sh);
            v[j][k] = ok ? val | (((old >> sh) & 0xffffu) << 16) : val;
        }
    __syncthreads();
    if (NW == 32768 && blockDim.x == 1024)
        hist16_scan_lanes(hw);
    else
        hist16_exclusive_scan(hw, NW);
    __syncthreads();
    // scatter, one register row at a time: the row's NK prefix words are all
    // loaded before any omega store (a load after a store to omega could
    // alias it, so the compiler would otherwise wait out every load's latency)
#pragma unroll
    for (int j = 0; j < NK; j++) {
        uint32_t hv[NK];
#pragma unroll
        for (int k = 0; k < NK; k++) hv[k] = hw[(v[j][k] >> 1) & (NW - 1)];  // unranked: a valid word, unused
#pragma unroll
        for (int k = 0; k < NK; k++) {
            const uint32_t val = v[j][k];
            if (val != 0xffffffffu) {
                const uint32_t rank = ((hv[k] >> ((val & 1) << 4)) & 0xffffu) + (val >> 16);
                om[rank] = (uint16_t)((lane + 32 * k) | ((wid + 32 * j) << 8));
            }
        }
    }
    for (int i = g.N + tid; i < g.Npad; i += blockDim.x) om[i] = 0xffffu;
    __syncthreads();
    if (g.k1_bulk)
        store_omega_bulk(g, om, omega_slot(g, omega_out));
    else
        store_omega(g, om, omega_slot(g, omega_out));
}

#define IMF_K1R(DT, TMA)                                                                     \
    template __global__ void k1_count_reg<DT, 1, TMA>(Geom, uint16_t*, const __grid_constant__ CUtensorMap); \
    template __global__ void k1_count_reg<DT, 2, TMA>(Geom, uint16_t*, const __grid_constant__ CUtensorMap); \
    template __global__ void k1_count_reg<DT, 3, TMA>(Geom, uint16_t*, const __grid_constant__ CUtensorMap); \
    template __global__ void k1_count_reg<DT, 4, TMA>(Geom, uint16_t*, const __grid_constant__ CUtensorMap); \
    template __global__ void k1_count_reg<DT, 5, TMA>(Geom, uint16_t*, const __grid_constant__ CUtensorMap); \
    template __global__ void k1_count_reg<DT, 6, TMA>(Geom, uint16_t*, const __grid_constant__ CUtensorMap);
IMF_K1R(DT_U8, false)
IMF_K1R(DT_U16, false)
IMF_K1R(DT_U8, true)
IMF_K1R(DT_U16, true)

}  // namespace imf
