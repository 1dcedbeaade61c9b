// imf_sort.cu -- K1: per-tile rank ordering (ordinal transform) on sm_100a.
//
// Replaces the reference's per-tile ordinal_transform (ordinal.py:126-172:
// _rank_by_bucket :62-79 for u8/u16, float_order_key + _rank_by_radix16
// :82-123 for f32).  One CTA sorts one input tile of N <= 65536 pixels by key
// and writes the rank -> position map omega (u16, x | y << 8) to a global
// scratch slot; K2 (imf_select.cu) rebuilds the ordinal image from it.
//
// Ties: the reference breaks ties by row-major position (stable sort), which
// only matters for its tile-to-tile forwarding.  The output of
// a selection is a multiset quantile and does not depend on the tie order
// (oracle.py:8-13), and K2 never forwards, so the FIRST counting pass here is
// unstable (warp-aggregated shared atomics); later LSD passes are stable
// (warp match_any ranking + per-warp digit counters scanned digit-major).
//
//   u8 : 1 counting pass (256 bins)                       smem ~2N bytes
//   u16: low byte unstable, high byte stable              smem ~5N bytes
//   f32: 4 byte passes on the u32 order key (1 unstable)  smem ~8N bytes
// When the tile does not fit shared memory, the large arrays live in a
// per-CTA global scratch slot (L2-resident) -- same code, GMEM=true.
#include "imf_common.cuh"

namespace imf {

constexpr unsigned FULL = 0xffffffffu;

// Exclusive scan of a[0..n) in place by the whole CTA.
__device__ void block_exclusive_scan(uint32_t* a, int n) {
    __shared__ uint32_t warp_tot[32];
    const int nt = blockDim.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int per = (n + nt - 1) / nt;
    const int b0 = tid * per, b1 = min(n, b0 + per);
    uint32_t s = 0;
    for (int i = b0; i < b1; i++) s += a[i];
    uint32_t incl = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t v = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += v;
    }
    if (lane == 31) warp_tot[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        const int nw = nt >> 5;
        uint32_t v = lane < nw ? warp_tot[lane] : 0, x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(FULL, x, o);
            if (lane >= o) x += y;
        }
        if (lane < nw) warp_tot[lane] = x - v;
    }
    __syncthreads();
    uint32_t run = warp_tot[wid] + incl - s;
    for (int i = b0; i < b1; i++) {
        uint32_t v = a[i];
        a[i] = run;
        run += v;
    }
    __syncthreads();
}

// Unstable counting pass: digit(i) for i in [0, N) -> emit(i, destination).
template <typename DigitFn, typename EmitFn>
__device__ void unstable_pass(int N, uint32_t* hist, DigitFn digit, EmitFn emit) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    for (int base = wid * 32; base < N; base += nw * 32) {
        int i = base + lane;
        uint32_t d = i < N ? digit(i) : 0xffffffffu;
        unsigned peers = __match_any_sync(FULL, d);
        int leader = __ffs(peers) - 1;
        if (i < N && lane == leader) atomicAdd(&hist[d], (uint32_t)__popc(peers));
    }
    __syncthreads();
    block_exclusive_scan(hist, 256);
    for (int base = wid * 32; base < N; base += nw * 32) {
        int i = base + lane;
        uint32_t d = i < N ? digit(i) : 0xffffffffu;
        unsigned peers = __match_any_sync(FULL, d);
        int leader = __ffs(peers) - 1;
        uint32_t b = 0;
        if (i < N && lane == leader) b = atomicAdd(&hist[d], (uint32_t)__popc(peers));
        b = __shfl_sync(FULL, b, leader);
        if (i < N) emit(i, (int)(b + __popc(peers & lanemask_lt())));
    }
    __syncthreads();
}

// Stable counting pass over k in [0, N): destination order of equal digits
// follows k.  Warp w owns the contiguous chunk [w*CH, (w+1)*CH).
template <typename DigitFn, typename EmitFn>
__device__ void stable_pass(int N, uint32_t* cnt, DigitFn digit, EmitFn emit) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int CH = ((N + nw * 32 - 1) / (nw * 32)) * 32;
    const int k0 = wid * CH, k1 = min(N, k0 + CH);
    for (int i = threadIdx.x; i < 256 * nw; i += blockDim.x) cnt[i] = 0;
    __syncthreads();
    for (int it = 0; it < CH; it += 32) {
        int k = k0 + it + lane;
        bool valid = k < k1;
        uint32_t d = valid ? digit(k) : 0xffffffffu;
        unsigned peers = __match_any_sync(FULL, d);
        if (valid && lane == __ffs(peers) - 1) cnt[d * nw + wid] += __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    block_exclusive_scan(cnt, 256 * nw);
    for (int it = 0; it < CH; it += 32) {
        int k = k0 + it + lane;
        bool valid = k < k1;
        uint32_t d = valid ? digit(k) : 0xffffffffu;
        unsigned peers = __match_any_sync(FULL, d);
        uint32_t base = valid ? cnt[d * nw + wid] : 0;
        __syncwarp();
        if (valid && lane == __ffs(peers) - 1) cnt[d * nw + wid] = base + __popc(peers);
        __syncwarp();
        if (valid) emit(k, (int)(base + __popc(peers & lanemask_lt())));
    }
    __syncthreads();
}

__device__ __forceinline__ uint16_t pack_pos(int i, int Sw, float invS) {
    int x, y;
    lin_to_xy(i, Sw, invS, x, y);
    return (uint16_t)(x | (y << 8));
}

// Copy the finished omega (smem, N entries) to its global slot, 16 B at a time.
__device__ __forceinline__ void store_omega(const Geom& g, const uint16_t* om_s, uint16_t* om_g) {
    const int n16 = g.Npad >> 3;  // uint4 count
    const uint4* s = reinterpret_cast<const uint4*>(om_s);
    uint4* d = reinterpret_cast<uint4*>(om_g);
    for (int i = threadIdx.x; i < n16; i += blockDim.x) d[i] = s[i];
}

template <int DT, bool GMEM>
__global__ void __launch_bounds__(512) k1_sort(Geom g, uint16_t* __restrict__ omega_out,
                                               unsigned char* __restrict__ gscratch,
                                               long long gscratch_stride) {
    extern __shared__ __align__(16) unsigned char smem[];
    const long long t = g.tile_begin + blockIdx.x;
    const TileCoord tc = tile_coord(g, t);
    const int N = g.N, Sw = g.Sw;
    const float invS = 1.0f / (float)Sw;
    const int nw = blockDim.x >> 5;
    uint32_t* hist = reinterpret_cast<uint32_t*>(smem);
    uint32_t* cnt = hist + 256;
    uint16_t* om = reinterpret_cast<uint16_t*>(cnt + (DT == DT_U8 ? 0 : 256 * nw));
    unsigned char* big = GMEM ? gscratch + blockIdx.x * gscratch_stride
                              : reinterpret_cast<unsigned char*>(om + g.Npad);
    uint16_t* om_g = omega_out + (long long)blockIdx.x * g.Npad;

    if (DT == DT_U8) {
        auto digit = [&](int i) {
            int x, y;
            lin_to_xy(i, Sw, invS, x, y);
            return load_key(g, tc, y, x);
        };
        auto emit = [&](int i, int dst) { om[dst] = pack_pos(i, Sw, invS); };
        unstable_pass(N, hist, digit, emit);
    } else if (DT == DT_U16) {
        uint16_t* tpos = reinterpret_cast<uint16_t*>(big);
        uint8_t* thi = reinterpret_cast<uint8_t*>(tpos + g.Npad);
        auto d0 = [&](int i) {
            int x, y;
            lin_to_xy(i, Sw, invS, x, y);
            return load_key(g, tc, y, x) & 0xffu;
        };
        auto e0 = [&](int i, int dst) {
            int x, y;
            lin_to_xy(i, Sw, invS, x, y);
            tpos[dst] = (uint16_t)(x | (y << 8));
            thi[dst] = (uint8_t)(load_key(g, tc, y, x) >> 8);
        };
        unstable_pass(N, hist, d0, e0);
        auto d1 = [&](int k) { return (uint32_t)thi[k]; };
        auto e1 = [&](int k, int dst) { om[dst] = tpos[k]; };
        stable_pass(N, cnt, d1, e1);
    } else {
        uint32_t* keys = reinterpret_cast<uint32_t*>(big);
        uint16_t* posA = reinterpret_cast<uint16_t*>(keys + g.Npad);
        for (int i = threadIdx.x; i < N; i += blockDim.x) {
            int x, y;
            lin_to_xy(i, Sw, invS, x, y);
            keys[i] = load_key(g, tc, y, x);
        }
        __syncthreads();
        auto d0 = [&](int i) { return keys[i] & 0xffu; };
        auto e0 = [&](int i, int dst) { posA[dst] = (uint16_t)i; };
        unstable_pass(N, hist, d0, e0);
        auto d1 = [&](int k) { return (keys[posA[k]] >> 8) & 0xffu; };
        auto e1 = [&](int k, int dst) { om[dst] = posA[k]; };  // om used as posB
        stable_pass(N, cnt, d1, e1);
        auto d2 = [&](int k) { return (keys[om[k]] >> 16) & 0xffu; };
        auto e2 = [&](int k, int dst) { posA[dst] = om[k]; };
        stable_pass(N, cnt, d2, e2);
        auto d3 = [&](int k) { return keys[posA[k]] >> 24; };
        auto e3 = [&](int k, int dst) { om[dst] = pack_pos(posA[k], Sw, invS); };
        stable_pass(N, cnt, d3, e3);
    }
    for (int i = N + threadIdx.x; i < g.Npad; i += blockDim.x) om[i] = 0;
    __syncthreads();
    store_omega(g, om, om_g);
}

template __global__ void k1_sort<DT_U8, false>(Geom, uint16_t*, unsigned char*, long long);
template __global__ void k1_sort<DT_U16, false>(Geom, uint16_t*, unsigned char*, long long);
template __global__ void k1_sort<DT_U16, true>(Geom, uint16_t*, unsigned char*, long long);
template __global__ void k1_sort<DT_F32, false>(Geom, uint16_t*, unsigned char*, long long);
template __global__ void k1_sort<DT_F32, true>(Geom, uint16_t*, unsigned char*, long long);

// Shared-memory bytes K1 needs for a tile (GMEM: large arrays in global scratch).
size_t k1_smem_bytes(int dtype, int Npad, int nwarps, bool gmem) {
    size_t b = 256 * 4 + (dtype == DT_U8 ? 0 : 256 * 4 * (size_t)nwarps) + 2 * (size_t)Npad;
    if (gmem || dtype == DT_U8) return b;
    if (dtype == DT_U16) return b + 3 * (size_t)Npad;
    return b + 6 * (size_t)Npad;
}

size_t k1_gscratch_bytes(int dtype, int Npad) {
    if (dtype == DT_U16) return 3 * (size_t)Npad;
    if (dtype == DT_F32) return 6 * (size_t)Npad;
    return 0;
}

}  // namespace imf
