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
#include <algorithm>
#include <type_traits>

#include "imf_k1.cuh"

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
    // counters digit-major with a padded row (nw + 1 per digit): the lanes of a
    // warp touch cnt[d * (nw + 1) + wid] for different digits d, which a row of
    // exactly nw (= 16) words would fold onto 2 banks; the pad slot stays 0 and
    // the digit-major exclusive scan is unchanged
    const int row = nw + 1;
    for (int i = threadIdx.x; i < 256 * row; i += blockDim.x) cnt[i] = 0;
    __syncthreads();
    for (int it = 0; it < CH; it += 32) {
        int k = k0 + it + lane;
        bool valid = k < k1;
        uint32_t d = valid ? digit(k) : 0xffffffffu;
        unsigned peers = __match_any_sync(FULL, d);
        if (valid && lane == __ffs(peers) - 1) cnt[d * row + wid] += __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    block_exclusive_scan(cnt, 256 * row);
    for (int it = 0; it < CH; it += 32) {
        int k = k0 + it + lane;
        bool valid = k < k1;
        uint32_t d = valid ? digit(k) : 0xffffffffu;
        unsigned peers = __match_any_sync(FULL, d);
        uint32_t base = valid ? cnt[d * row + wid] : 0;
        __syncwarp();
        if (valid && lane == __ffs(peers) - 1) cnt[d * row + wid] = base + __popc(peers);
        __syncwarp();
        if (valid) emit(k, (int)(base + __popc(peers & lanemask_lt())));
    }
    __syncthreads();
}

template <int DT, bool GMEM>
__device__ void k1_sort_tile(const Geom& g, uint16_t* __restrict__ omega_out, unsigned char* __restrict__ gscratch,
                             long long gscratch_stride, const int bt) {
    extern __shared__ __align__(16) unsigned char smem[];
    const long long t = g.tile_begin + bt;
    const TileCoord tc = tile_coord(g, t);
    const int N = g.N, Sw = g.Sw;
    const float invS = 1.0f / (float)Sw;
    const int nw = blockDim.x >> 5;
    // footprint tiles (g.fprow): index i < N is the i-th footprint pixel in
    // row-major order; s_fpre[y] = footprint pixels in rows < y
    __shared__ uint32_t s_fpre[256];
    if (g.fprow) {
        for (int y = threadIdx.x; y < 256; y += blockDim.x) {
            const uint32_t v = y < g.Sh ? __ldg(g.fprow + y) : 0xffffffffu;
            const int lo = (int)(v & 0xffffu), hi = (int)(v >> 16);
            s_fpre[y] = lo > 255 ? 0u : (uint32_t)(hi - lo + 1);  // empty row: lo = hi = 0xffff
        }
        __syncthreads();
        block_exclusive_scan(s_fpre, 256);
    }
    auto xy_of = [&](int i, int& x, int& y) {
        if (!g.fprow) {
            lin_to_xy(i, Sw, invS, x, y);
            return;
        }
        int lo = 0, hi = g.Sh - 1;  // the last row whose prefix is <= i
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if ((int)s_fpre[mid] <= i) lo = mid; else hi = mid - 1;
        }
        y = lo;
        x = (int)(__ldg(g.fprow + lo) & 0xffffu) + i - (int)s_fpre[lo];
    };
    auto pos_of = [&](int i) {
        int x, y;
        xy_of(i, x, y);
        return (uint16_t)(x | (y << 8));
    };
    uint32_t* hist = reinterpret_cast<uint32_t*>(smem);
    uint32_t* cnt = hist + 256;
    uint16_t* om = reinterpret_cast<uint16_t*>(cnt + (DT == DT_U8 ? 0 : 256 * (nw + 1)));
    unsigned char* big = GMEM ? gscratch + bt * gscratch_stride
                              : reinterpret_cast<unsigned char*>(om + g.Npad);
    uint16_t* om_g = omega_slot(g, omega_out, bt);

    if (DT == DT_U8) {
        auto digit = [&](int i) {
            int x, y;
            xy_of(i, x, y);
            return load_key(g, tc, y, x);
        };
        auto emit = [&](int i, int dst) { om[dst] = pos_of(i); };
        unstable_pass(N, hist, digit, emit);
    } else if (DT == DT_U16) {
        uint16_t* tpos = reinterpret_cast<uint16_t*>(big);
        uint8_t* thi = reinterpret_cast<uint8_t*>(tpos + g.Npad);
        auto d0 = [&](int i) {
            int x, y;
            xy_of(i, x, y);
            return load_key(g, tc, y, x) & 0xffu;
        };
        auto e0 = [&](int i, int dst) {
            int x, y;
            xy_of(i, x, y);
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
            xy_of(i, x, y);
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
        auto e3 = [&](int k, int dst) { om[dst] = pos_of(posA[k]); };
        stable_pass(N, cnt, d3, e3);
    }
    for (int i = N + threadIdx.x; i < g.Npad; i += blockDim.x) om[i] = 0xffffu;
    __syncthreads();
    store_omega(g, om, om_g);
}

// One CTA per tile; or, with `only` (the f32 bucket kernel's fallback list:
// only[0] = count, only[1..] = chunk tile indices), a small grid looping over
// the listed tiles.
template <int DT, bool GMEM>
__global__ void __launch_bounds__(1024) k1_sort(Geom g, uint16_t* __restrict__ omega_out,
                                               unsigned char* __restrict__ gscratch,
                                               long long gscratch_stride, const int* __restrict__ only) {
    if (!only) {
        k1_sort_tile<DT, GMEM>(g, omega_out, gscratch, gscratch_stride, blockIdx.x);
        return;
    }
    const int n = only[0];
    for (int i = blockIdx.x; i < n; i += gridDim.x) {
        k1_sort_tile<DT, GMEM>(g, omega_out, gscratch, gscratch_stride, only[1 + i]);
        __syncthreads();
    }
}

// Direct counting sort for 8/16-bit tiles (ordinal.py:62-79 _rank_by_bucket,
// the paper's 16-bit bucket sort): one 2^bits-bin histogram
// of u16 counters packed two per 32-bit word in shared memory (65536 bins =
// 128 KB for u16), shared atomics for the histogram and for the scatter
// (ties unordered -- output-neutral, see above).  Input tile rows are read
// straight from global memory twice (L2-resident), with the clamped column
// offsets of every lane precomputed once.  Requires N <= 65535 (S <= 255).
template <int DT>
__global__ void __launch_bounds__(1024) k1_count(Geom g, uint16_t* __restrict__ omega_out) {
    extern __shared__ __align__(16) unsigned char smem[];
    constexpr int NB = DT == DT_U8 ? 256 : 65536;
    constexpr int NW = NB / 2;  // histogram words
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
    const TileCoord tc = tile_coord(g, g.tile_begin + blockIdx.x);
    const int S = g.Sw, Sh = g.Sh;
    uint32_t* hw = reinterpret_cast<uint32_t*>(smem);
    uint16_t* om = reinterpret_cast<uint16_t*>(hw + NW);
    {
        uint4* h4 = reinterpret_cast<uint4*>(hw);
        for (int i = tid; i < NW / 4; i += blockDim.x) h4[i] = make_uint4(0, 0, 0, 0);
    }
    // clamped column offsets of this lane's columns x = lane + 32k
    long long xo[8];
#pragma unroll
    for (int k = 0; k < 8; k++) {
        int x = tc.ox0 + lane + 32 * k - g.r + g.vshift;
        x = x < 0 ? 0 : (x >= g.W ? g.W - 1 : x);
        xo[k] = (long long)x * g.s_x;
    }
    const int nk = (S + 31) >> 5;
    __syncthreads();
    auto row_ptr = [&](int y) {
        int yy = tc.oy0 + y - g.r + g.vshift;
        yy = yy < 0 ? 0 : (yy >= g.H ? g.H - 1 : yy);
        return tc.src + (long long)yy * g.s_y * (DT == DT_U8 ? 1 : 2);
    };
    for (int y = wid; y < Sh; y += nw) {
        const char* rp = row_ptr(y);
#pragma unroll
        for (int k = 0; k < 8; k++) {
            if (k < nk && lane + 32 * k < S) {
                uint32_t v = DT == DT_U8 ? (uint32_t)__ldg((const uint8_t*)rp + xo[k])
                                         : (uint32_t)__ldg((const uint16_t*)rp + xo[k]);
                atomicAdd(&hw[v >> 1], 1u << ((v & 1) << 4));
            }
        }
    }
    __syncthreads();
    if (NW == 32768 && blockDim.x == 1024)
        hist16_scan_lanes(hw);
    else
        hist16_exclusive_scan(hw, NW);
    __syncthreads();
    for (int y = wid; y < Sh; y += nw) {
        const char* rp = row_ptr(y);
#pragma unroll
        for (int k = 0; k < 8; k++) {
            const int x = lane + 32 * k;
            if (k < nk && x < S) {
                uint32_t v = DT == DT_U8 ? (uint32_t)__ldg((const uint8_t*)rp + xo[k])
                                         : (uint32_t)__ldg((const uint16_t*)rp + xo[k]);
                const uint32_t sh = (v & 1) << 4;
                const uint32_t old = atomicAdd(&hw[v >> 1], 1u << sh);
                om[(old >> sh) & 0xffffu] = (uint16_t)(x | (y << 8));
            }
        }
    }
    for (int i = g.N + tid; i < g.Npad; i += blockDim.x) om[i] = 0xffffu;
    __syncthreads();
    store_omega(g, om, omega_slot(g, omega_out));
}

#undef IMF_K1R


// f32 ordinal transform by buckets: count-sort the u32 order keys (ordinal.py:
// 109-123) by their HIGH 16 bits with the u16 machinery (register-resident tile,
// 64K-bin packed histogram, packed scan), scatter entries (low16 << 16 | pos)
// into bucket order, then rank each entry inside its bucket by counting the
// smaller entries (buckets are contiguous; a bitmap marks their starts).  Ties
// break by position (output-neutral).  Cost ~ sum of squared bucket sizes: a
// tile whose largest bucket exceeds kMaxBucket (narrow value range, flat
// regions) writes flag 1 and no omega; a k1_sort launch redoes those tiles.
// Ranking cost is sum(n_b^2) entry compares per tile; above this (about 60K per
// thread of a 1024-thread CTA) the tile goes to the LSD radix sort instead.

// Adaptive buckets for f32 keys.  Bucketing on the key's top 16 bits
// (sign, exponent, 7 mantissa bits) leaves a tile's values in a few hundred
// buckets of tens of entries each, and the in-bucket ranking costs the sum of
// squared bucket sizes.  Instead: 4096 coarse bins on key >> 20 are counted
// first; populated bin c (n_c keys, P populated) gets f_c = 2^l_c fine
// buckets, f_c = pow2floor(16 + n_c (65536 - 16 P) / N) (>= 16, total <=
// 65536), splitting it on the next l_c key bits.  A fine bucket then spans
// <= 2^16 keys (l_c >= 4), so the entry's low 16 key bits still order it, and
// holds ~2 N / 65536 keys.  tab[c]: coarse count in, base | l_c << 16 out.
// Below this many tile pixels the top-16-bit buckets are already small and the
// coarse pass (4096-bin atomics, allocation scan) costs more than it saves.

__device__ void coarse_alloc(uint32_t* tab, int N) {
    __shared__ int s_pop;
    const int tid = threadIdx.x, per = kCoarse / 1024;  // 1024-thread CTAs: 4 bins per thread
    if (tid == 0) s_pop = 0;
    __syncthreads();
    int pop = 0;
    for (int i = 0; i < per; i++) pop += tab[tid * per + i] ? 1 : 0;
    pop = (int)__reduce_add_sync(0xffffffffu, (unsigned)pop);
    if ((tid & 31) == 0 && pop) atomicAdd(&s_pop, pop);
    __syncthreads();
    const unsigned long long room = 65536ull - 16ull * (unsigned long long)s_pop;
    uint32_t fv[kCoarse / 1024];
    for (int i = 0; i < per; i++) {
        const uint32_t n = tab[tid * per + i];
        fv[i] = n ? 1u << (31 - __clz(16u + (uint32_t)(n * room / (unsigned long long)N))) : 0u;
    }
    __syncthreads();
    for (int i = 0; i < per; i++) tab[tid * per + i] = fv[i];
    __syncthreads();
    block_exclusive_scan(tab, kCoarse);  // ends with a barrier
    for (int i = 0; i < per; i++) {
        const int c = tid * per + i;
        tab[c] = fv[i] ? (tab[c] | ((uint32_t)(31 - __clz(fv[i])) << 16)) : 0u;
    }
    __syncthreads();
}

// Call-wide fine-bucket table (f32): the coarse histogram of every pixel the
// call reads (rows [y0, y1) of every plane), allocated once by coarse_alloc;
// tiles then skip their own coarse pass.  Every key of every tile lies in a
// populated coarse bin of this superset, so the table is valid for each tile
// (f_c >= 16: fine buckets still span <= 2^16 keys); a tile whose values
// cluster differently only sees larger buckets (sum-of-squares check).
__global__ void __launch_bounds__(1024) k_coarse_hist(Geom g, int y0, int y1, uint32_t* __restrict__ counts) {
    __shared__ uint32_t h[kCoarse];
    for (int i = threadIdx.x; i < kCoarse; i += blockDim.x) h[i] = 0;
    __syncthreads();
    const long long rows = (long long)(y1 - y0) * g.B * g.C;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (long long rr = (long long)blockIdx.x * nw + wid; rr < rows; rr += (long long)gridDim.x * nw) {
        const int y = y0 + (int)(rr % (y1 - y0));
        const long long pc = rr / (y1 - y0);
        TileCoord tc;
        tc.b = (int)(pc / g.C);
        tc.c = (int)(pc % g.C);
        tc.src = (const char*)g.src + (tc.b * g.s_b + tc.c * g.s_c) * 4;
        for (int x = lane; x < g.W; x += 32) atomicAdd(&h[f32_key(g, tc, y, x) >> 20], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kCoarse; i += blockDim.x)
        if (h[i]) atomicAdd(&counts[i], h[i]);
}

__global__ void __launch_bounds__(1024) k_coarse_alloc(uint32_t* __restrict__ tab) {
    __shared__ uint32_t t[kCoarse];
    __shared__ unsigned long long s_n;
    if (threadIdx.x == 0) s_n = 0;
    __syncthreads();
    unsigned long long n = 0;
    for (int i = threadIdx.x; i < kCoarse; i += blockDim.x) {
        t[i] = tab[i];
        n += t[i];
    }
    atomicAdd(&s_n, n);
    __syncthreads();
    // counts above 2^32 / 65536 would overflow coarse_alloc's 32-bit products
    // only through n * room; it divides in 64 bits, but N is an int
    coarse_alloc(t, (int)min(s_n, (unsigned long long)0x7fffffff));
    for (int i = threadIdx.x; i < kCoarse; i += blockDim.x) tab[i] = t[i];
}

__device__ __forceinline__ uint32_t fine_bucket(const uint32_t* tab, uint32_t key) {
    const uint32_t t = tab[key >> 20], l = t >> 16;
    return (t & 0xffffu) + ((key & 0xfffffu) >> (20 - l));
}

// Replicate-boundary copies.  Tile column x reads image column clamp(X0 + x);
// the columns reading one clamped image column are a contiguous range
// [first, first + cnt).  (Same for rows.)
__device__ __forceinline__ void rep_axis(int X0, int x, int S, int W, int& cnt, bool& first) {
    const int X = X0 + x;
    if (W == 1) {
        cnt = S;
        first = x == 0;
    } else if (X <= 0) {
        cnt = min(S, 1 - X0);
        first = x == 0;
    } else if (X >= W - 1) {
        const int f = max(0, W - 1 - X0);
        cnt = S - f;
        first = x == f;
    } else {
        cnt = 1;
        first = true;
    }
}

// Weight of a tile pixel in the bucket transform: the copies of one image
// pixel (replicate boundary, >= run_min of them) are ranked once, as a RUN of
// consecutive ranks held by the first copy (weight = copy count, the others
// 0); ties order arbitrarily (imf_sort.cu header), so the run's internal
// order is free.  A run of w copies starting at slot s:
//   ent[s]            = key16 << 16 | 0xffff   (head)
//   ent[s+1 .. s+w)   = key16 << 16 | 0xfffe   (interior)
// and a descriptor: first copy x | y << 8 and copy rectangle cx | cy << 8, in
// the side array d16[s], d16[s+1] (global-entry kernels) or in the CTA's run
// list (shared-memory entries; a tile with more runs goes to the radix sort).  Plain entries are key16 << 16 | pos, pos <= 0xfefe (x, y <
// 255).  Ranking orders slots by (entry | 1, slot): the interior of a run then
// compares exactly like its head, so a bucket scan counts a whole run with
// plain compares (no data-dependent skip), and only the head's thread ranks it.
constexpr int kRunList = 64;   // runs per tile without a side array
// Runs longer than kMarkSelf are LONG: listed (RunList::mark), their interior
// written by the CTA, and skipped whole by bucket scans (a corner run of
// (r+1)^2 slots would otherwise be scanned by every entry sharing its bucket).
constexpr int kMarkSelf = 128;
constexpr int kBigRuns = 32;   // queued long runs (interior marks, omega fill)

struct RunList {
    int n, nbig, nmark, abort;
    uint2 run[kRunList];   // list mode: (slot, pos | cx << 16 | cy << 24)
    uint2 mark[kBigRuns];  // (slot, key16 << 16 | 0xfffe) of the long runs (kMarkSelf)
    uint2 mlen[kBigRuns];  // (w, 0)
    uint4 big[kBigRuns];   // (rank, pos, cx, cy) of heads with more than 256 copies
};

// Largest copy group of a tile (columns [X0, X0 + S) of an image W wide).
__device__ __forceinline__ int max_copies(int X0, int S, int W) {
    if (W == 1) return S;
    const int l = X0 < 0 ? min(S, 1 - X0) : 1;
    const int r = X0 + S > W ? S - max(0, W - 1 - X0) : 1;
    return max(l, r);
}

__device__ __forceinline__ bool has_runs(const Geom& g, const TileCoord& tc) {
    const int X0 = tc.ox0 - g.r + g.vshift, Y0 = tc.oy0 - g.r + g.vshift;
    return max_copies(X0, g.Sw, g.W) * max_copies(Y0, g.Sh, g.H) >= g.run_min;
}

// Weight code of tile pixel (x, y) with copy counts cx, cy (fx, fy: it is the
// first copy on that axis): the slots it takes in bits [0, 20) -- 1 for a
// plain ranked pixel, the copies inside the tile footprint for the head of a
// run, 0 otherwise -- plus kRunBit for a run head.  A run the footprint clips
// to one slot stays a run: that slot is not the head's own position.
constexpr int kRunBit = 1 << 20;
__device__ __forceinline__ int wt_of(int code) { return code & (kRunBit - 1); }

__device__ __forceinline__ int pixel_weight(const Geom& g, const uint32_t* fprow, int x, int cx, bool fx, int y,
                                            int cy, bool fy) {
    if (cx * cy < g.run_min) return in_footprint(fprow, x, y) ? 1 : 0;
    if (!(fx && fy)) return 0;
    const int w = fp_rect_count(fprow, x, cx, y, cy);
    return w ? (w | kRunBit) : 0;
}

// The omega entries of a run ranked from rk: its copy rectangle (first copy
// pos, cx x cy) row by row, each row clipped to the footprint; thread t0 of a
// group of `step` writes every step-th position of a row.
__device__ __forceinline__ void fill_run(const uint32_t* fprow, uint16_t* om, int rk, uint32_t pos, int cx, int cy,
                                         int t0, int step) {
    const int x0 = (int)(pos & 0xffu), y0 = (int)(pos >> 8);
    for (int yy = y0; yy < y0 + cy; yy++) {
        int lo = x0, hi = x0 + cx - 1;
        if (fprow) {
            const uint32_t v = __ldg(fprow + yy);
            lo = max(lo, (int)(v & 0xffffu));
            hi = min(hi, (int)(v >> 16));
        }
        for (int x = lo + t0; x <= hi; x += step) om[rk + x - lo] = (uint16_t)(x | (yy << 8));
        rk += max(0, hi - lo + 1);
    }
}

__device__ __forceinline__ void put_entry(uint32_t* ent, uint16_t* d16, int slot, uint32_t key16, int x, int y,
                                          int code, int cx, int cy, RunList* rl, const uint32_t* fprow) {
    const uint32_t pos = (uint32_t)(x | (y << 8));
    const int w = wt_of(code);
    if (!(code & kRunBit)) {
        ent[slot] = (key16 << 16) | pos;
        return;
    }
    if (w == 1 && fprow) {  // a run the footprint clips to one copy: a plain entry at that copy
        for (int yy = y; yy < y + cy; yy++) {
            const uint32_t v = __ldg(fprow + yy);
            const int lo = max(x, (int)(v & 0xffffu));
            if (lo <= min(x + cx - 1, (int)(v >> 16))) {
                ent[slot] = (key16 << 16) | (uint32_t)(lo | (yy << 8));
                return;
            }
        }
    }
    ent[slot] = (key16 << 16) | 0xffffu;
    if (d16) {
        d16[slot] = (uint16_t)pos;
        d16[slot + 1] = (uint16_t)(cx | (cy << 8));
    } else {
        const int k = atomicAdd(&rl->n, 1);
        if (k >= kRunList) {
            rl->abort = 1;
            return;
        }
        rl->run[k] = make_uint2((uint32_t)slot, pos | ((uint32_t)cx << 16) | ((uint32_t)cy << 24));
    }
    const uint32_t mv = (key16 << 16) | 0xfffeu;
    if (w > kMarkSelf) {
        const int k = atomicAdd(&rl->nmark, 1);
        if (k < kBigRuns) {
            rl->mark[k] = make_uint2((uint32_t)slot, mv);
            rl->mlen[k] = make_uint2((uint32_t)w, 0u);
            return;
        }
    }
    for (int i = 1; i < w; i++) ent[slot + i] = mv;
}

// After the scatter barrier: the interiors of the long runs, by the CTA, then
// a barrier (block-uniform: rl->nmark is read after one).
__device__ __forceinline__ void mark_runs(uint32_t* ent, const RunList* rl) {
    const int n = min(rl->nmark, kBigRuns);
    if (!n) return;
    for (int k = 0; k < n; k++) {
        const uint2 d = rl->mark[k];
        const int w = (int)rl->mlen[k].x;
        for (int i = 1 + (int)threadIdx.x; i < w; i += blockDim.x) ent[d.x + i] = d.y;
    }
    __syncthreads();
}

// Rank every entry within its bucket (starts: bucket-start bitmap) and write
// omega.  RUNS: the (entry | 1, slot) order above; the head of a run writes
// its w ranks (long runs: queued for fill_big_runs).
#ifdef IMF_STATS
__device__ unsigned long long g_rstats[128];  // [64 + 2k], k < 12: phase cycles  // [0, 64): bucket span per ranked entry (dev aid)
// [64 + 2k]: sum, [65 + 2k]: max over CTAs of phase k's clock cycles (thread 0)
#define PHASE_T0 long long _t0 = clock64()
#define PHASE(k)                                                              \
    if (threadIdx.x == 0) {                                                   \
        const long long _t = clock64();                                       \
        atomicAdd(&g_rstats[64 + 2 * (k)], (unsigned long long)(_t - _t0));   \
        atomicMax(&g_rstats[65 + 2 * (k)], (unsigned long long)(_t - _t0));   \
        _t0 = _t;                                                             \
    }
#else
#define PHASE_T0
#define PHASE(k)
#endif

// Tiles with runs skip the sum-of-squares estimate (run weights inflate it):
// their scans are bounded by a per-thread budget of scanned slots instead; a
// thread past it sets rl->abort and the tile goes to the radix sort.
constexpr int kScanBudget = 32768;

template <bool RUNS>
__device__ void rank_buckets(const uint32_t* ent, const uint16_t* d16, const uint32_t* starts, int N, uint16_t* om,
                             RunList* rl, const uint32_t* fprow) {
    const int nsw = (N + 31) >> 5;
    const int nlong = RUNS ? min(rl->nmark, kBigRuns) : 0;
    int work = 0;
    for (int sp = threadIdx.x; sp < N; sp += blockDim.x) {
        const uint32_t e = ent[sp];
        const uint32_t lo = e & 0xffffu;
        if (RUNS && lo == 0xfffeu) continue;  // inside a run
        int w = sp >> 5;
        uint32_t m = starts[w] & (0xffffffffu >> (31 - (sp & 31)));  // start bits <= sp
        while (!m) m = starts[--w];
        const int b0 = (w << 5) + 31 - __clz(m);
        w = sp >> 5;
        m = (sp & 31) == 31 ? 0u : starts[w] & (0xfffffffeu << (sp & 31));  // start bits > sp
        while (!m && ++w < nsw) m = starts[w];
        const int b1 = m ? (w << 5) + __ffs(m) - 1 : N;
        int rk = b0;
#ifdef IMF_RSTATS
        atomicAdd(&g_rstats[min(b1 - b0, 63)], 1ull);
#endif
        if (!RUNS) {
            for (int q = b0; q < b1; q++) rk += ent[q] < e ? 1 : 0;
            om[rk] = (uint16_t)lo;
            continue;
        }
        const uint32_t e1 = e | 1u;
        auto scan = [&](int q0, int q1) {
            work += q1 - q0;
            if (work > kScanBudget) {
                rl->abort = 1;
                return;
            }
            for (int q = q0; q < q1; q++) {
                const uint32_t v1 = ent[q] | 1u;
                rk += (v1 < e1 || (v1 == e1 && q < sp)) ? 1 : 0;
            }
        };
        // long runs inside [b0, b1), in slot order: counted whole, not scanned
        int qa = b0;
        for (;;) {
            int kn = -1;
            uint32_t sn = 0xffffffffu;
            for (int k = 0; k < nlong; k++) {
                const uint32_t sk = rl->mark[k].x;
                if (sk >= (uint32_t)qa && sk < (uint32_t)b1 && sk < sn) {
                    sn = sk;
                    kn = k;
                }
            }
            if (kn < 0) break;
            scan(qa, (int)sn);
            const uint32_t v1 = rl->mark[kn].y | 1u;  // the run's value (| 1: as its head)
            if (v1 < e1 || (v1 == e1 && (int)sn < sp)) rk += (int)rl->mlen[kn].x;
            qa = (int)sn + (int)rl->mlen[kn].x;
        }
        scan(qa, b1);
        if (work > kScanBudget) break;
        if (lo != 0xffffu) {
            om[rk] = (uint16_t)lo;
            continue;
        }
        uint32_t d = 0;  // this head's descriptor: pos | cx << 16 | cy << 24
        if (d16) {
            d = (uint32_t)d16[sp] | ((uint32_t)d16[sp + 1] << 16);
        } else {
            for (int k = 0; k < min(rl->n, kRunList); k++)
                if (rl->run[k].x == (uint32_t)sp) d = rl->run[k].y;
        }
        const int cx = (int)((d >> 16) & 0xffu), len = cx * (int)(d >> 24);
        const uint32_t pos = d & 0xffffu;
        if (len > 256) {  // the CTA fills it (fill_big_runs)
            const int k = atomicAdd(&rl->nbig, 1);
            if (k < kBigRuns) {
                rl->big[k] = make_uint4((uint32_t)rk, pos, (uint32_t)cx, (uint32_t)(d >> 24));
                continue;
            }
        }
        fill_run(fprow, om, rk, pos, cx, (int)(d >> 24), 0, 1);
    }
}

// After the barrier closing rank_buckets: fill the long runs with the CTA.
__device__ void fill_big_runs(uint16_t* om, const RunList* rl, const uint32_t* fprow) {
    for (int k = 0; k < min(rl->nbig, kBigRuns); k++) {
        const uint4 b = rl->big[k];
        fill_run(fprow, om, (int)b.x, b.y, (int)b.z, (int)b.w, (int)threadIdx.x, (int)blockDim.x);
    }
}

// GENT: the entries live in the tile's global scratch slot (tiles too large
// for shared-memory entries); the keys stay in registers either way.
// EDGE: the tile reads clamped (replicated) image pixels; the copies of one
// pixel are ranked as a run (pixel_weight).  Interior tiles take the EDGE =
// false instance, which carries none of that.
template <int NK, bool GENT, bool EDGE, bool FP>
__device__ __forceinline__ void f32_bucket_tile(const Geom& g, const TileCoord& tc, const int bt,
                                                uint16_t* __restrict__ omega_out,
                                                int* __restrict__ fallback, uint32_t* __restrict__ gent,
                                                long long gent_stride, unsigned long long max_sumsq) {
    extern __shared__ __align__(16) unsigned char smem[];
    constexpr int NW = 32768;  // histogram words (65536 16-bit counters)
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int S = g.Sw, SH = g.Sh, N = g.N;
    const uint32_t* fpr = FP ? g.fprow : nullptr;  // footprint rows (FP: the plan ranks a footprint)
    uint32_t* hw = reinterpret_cast<uint32_t*>(smem);
    uint32_t* ent = GENT ? gent + bt * gent_stride : hw + NW;  // N entries
    // bucket starts, ceil(N/32) words; the coarse table (f32) aliases the
    // shared entries (dead until the scatter) or follows the starts
    uint32_t* starts = GENT ? hw + NW : ent + max((N + 3) & ~3, kCoarse);
    const int nsw = (N + 31) >> 5;
    uint32_t* ctab = GENT ? starts + ((nsw + 3) & ~3) : ent;
    uint16_t* d16 = GENT ? reinterpret_cast<uint16_t*>(ent + N) : nullptr;  // run descriptors (2 B / slot)
    const bool adaptive = g.dtype == DT_F32 && N > kAdaptiveMinN;
    // OWN16 (interior tiles too large for 4-byte shared entries, N > ~23.7K):
    // each slot keeps only its entry's low 16 key bits, in SHARED memory after
    // the coarse table (2 B per pixel, S <= 192: 221 KB in all); a thread
    // holds (bucket << 16 | slot) per pixel and ranks its own pixels against
    // the bucket's slots (ties by slot), so the bucket entries never go
    // through the global scratch slot (whose scattered stores and dependent
    // L2 reads bound this kernel: profiles/ncu_k1_f32_c3r64_r2*).
    constexpr bool OWN16 = GENT && !EDGE;
    uint16_t* l16 = reinterpret_cast<uint16_t*>(ctab + kCoarse);
    // interior tiles with adaptive (~2-key) buckets rank their own register
    // pixels (lanes in different buckets: fine while buckets are that small);
    // others rank slot-parallel over a start bitmap
    const bool own_rank = !EDGE && (NK <= 5 || OWN16) && adaptive;
    __shared__ unsigned long long s_sumsq;
    __shared__ int s_runs;
    __shared__ RunList s_rl;
    uint32_t v[NK][NK];
    // which of this thread's pixels are ranked (inside the tile and its
    // footprint, weight > 0): a mask on edge tiles (weights are costly to
    // recompute); on interior tiles an unranked slot holds the key kSent
    // instead (no register held, one compare per test: the 1024-thread budget
    // is 64 registers).  A ranked key equal to kSent -- the NaN 0x7fffffff, or
    // a fine-bucket entry 0xffff'ffff -- sends the tile to the LSD fallback.
    constexpr uint32_t kSent = 0xffffffffu;
    __shared__ int s_collide;
    bool coll = false;
    unsigned long long okm = 0;
    // replicate copies (rep_axis), edge tiles only, recomputed where used
    // (keeps the 1024-thread register budget for the keys)
    const int X0 = tc.ox0 - g.r + g.vshift, Y0 = tc.oy0 - g.r + g.vshift;
    PHASE_T0;
    auto weight = [&](int j, int k) {
        if (!EDGE) return 1;
        int cx, cy;
        bool fx, fy;
        rep_axis(X0, lane + 32 * k, S, g.W, cx, fx);
        rep_axis(Y0, wid + 32 * j, SH, g.H, cy, fy);
        return pixel_weight(g, fpr, lane + 32 * k, cx, fx, wid + 32 * j, cy, fy);
    };
    auto cnt_x = [&](int k) {
        int c;
        bool f;
        rep_axis(X0, lane + 32 * k, S, g.W, c, f);
        return c;
    };
    auto cnt_y = [&](int j) {
        int c;
        bool f;
        rep_axis(Y0, wid + 32 * j, SH, g.H, c, f);
        return c;
    };
    {
        int xc[NK];
#pragma unroll
        for (int k = 0; k < NK; k++) {
            int x = X0 + lane + 32 * k;
            xc[k] = x < 0 ? 0 : (x >= g.W ? g.W - 1 : x);
        }
#pragma unroll
        for (int j = 0; j < NK; j++) {
            const int y = wid + 32 * j;
            int yy = Y0 + y;
            yy = yy < 0 ? 0 : (yy >= g.H ? g.H - 1 : yy);
#pragma unroll
            for (int k = 0; k < NK; k++) {
                const bool ok = y < SH && lane + 32 * k < S &&
                                (EDGE ? weight(j, k) != 0 : in_footprint(fpr, lane + 32 * k, y));
                if (EDGE) {
                    v[j][k] = ok ? f32_key(g, tc, yy, xc[k]) : 0u;
                    okm |= (ok ? 1ull : 0ull) << (j * NK + k);
                } else {
                    v[j][k] = ok ? f32_key(g, tc, yy, xc[k]) : kSent;
                    coll |= ok && v[j][k] == kSent;
                }
            }
        }
    }
    auto okf = [&](int j, int k) -> bool {
        if (EDGE) return (okm >> (j * NK + k)) & 1ull;
        return v[j][k] != kSent;
    };
    {
        uint4* h4 = reinterpret_cast<uint4*>(hw);
        for (int i = tid; i < NW / 4; i += blockDim.x) h4[i] = make_uint4(0, 0, 0, 0);
        if (!own_rank)
            for (int i = tid; i < nsw; i += blockDim.x) starts[i] = 0;
        if (adaptive)
            for (int i = tid; i < kCoarse; i += blockDim.x) ctab[i] = g.ctab_g ? g.ctab_g[i] : 0u;
        if (tid == 0) {
            s_sumsq = 0;
            s_runs = s_rl.n = s_rl.nbig = s_rl.nmark = s_rl.abort = s_collide = 0;
        }
    }
    __syncthreads();
    PHASE(6);
    if (adaptive) {  // keys -> fine bucket << 16 | low 16 key bits
        if (!g.ctab_g) {  // no call-wide table: this tile's own coarse pass
#pragma unroll
            for (int j = 0; j < NK; j++)
#pragma unroll
                for (int k = 0; k < NK; k++)
                    if (okf(j, k)) atomicAdd(&ctab[v[j][k] >> 20], (uint32_t)wt_of(weight(j, k)));
            coarse_alloc(ctab, N);
        }
#pragma unroll
        for (int j = 0; j < NK; j++)
#pragma unroll
            for (int k = 0; k < NK; k++)
                if (okf(j, k)) {
                    v[j][k] = (fine_bucket(ctab, v[j][k]) << 16) | (v[j][k] & 0xffffu);
                    if (!EDGE) coll |= v[j][k] == kSent;
                }
    }
    bool runs = false;
#pragma unroll
    for (int j = 0; j < NK; j++)
#pragma unroll
        for (int k = 0; k < NK; k++)
            if (okf(j, k)) {
                const uint32_t h = v[j][k] >> 16, sh = (h & 1) << 4;
                const int wc = weight(j, k);
                runs |= (wc & kRunBit) != 0;
                atomicAdd(&hw[h >> 1], (uint32_t)wt_of(wc) << sh);
            }
    if (runs) s_runs = 1;
    if (coll) s_collide = 1;
    __syncthreads();
    PHASE(7);
    hist16_exclusive_scan(hw, NW, own_rank ? nullptr : starts, &s_sumsq);
    __syncthreads();
    PHASE(8);
    // tiles with runs skip the estimate (run weights inflate it); their scans
    // are budgeted instead (rank_buckets)
    if ((!s_runs && s_sumsq > max_sumsq) || s_collide) {  // block-uniform: hand the tile to the radix sort
        if (tid == 0) fallback[1 + atomicAdd(fallback, 1)] = bt;
        return;
    }
#pragma unroll
    for (int j = 0; j < NK; j++)
#pragma unroll
        for (int k = 0; k < NK; k++)
            if (okf(j, k)) {
                const uint32_t key = v[j][k], h = key >> 16, sh = (h & 1) << 4;
                const int wc = weight(j, k);
                const uint32_t old = atomicAdd(&hw[h >> 1], (uint32_t)wt_of(wc) << sh);
                if (OWN16 && own_rank) {
                    const uint32_t slot = (old >> sh) & 0xffffu;
                    l16[slot] = (uint16_t)(key & 0xffffu);
                    v[j][k] = (h << 16) | slot;
                } else {
                    put_entry(ent, d16, (old >> sh) & 0xffffu, key & 0xffffu, lane + 32 * k, wid + 32 * j, wc,
                              cnt_x(k), cnt_y(j), &s_rl, fpr);
                }
            }
    __syncthreads();
    PHASE(9);
    uint16_t* om = reinterpret_cast<uint16_t*>(hw);  // the histogram is dead: omega goes here
    if (own_rank) {
        // each thread ranks its own pixels: the counters now hold every bucket's
        // end, so bucket id spans [end(id - 1), end(id)) -- no start bitmap
#pragma unroll
        for (int j = 0; j < NK; j++)
#pragma unroll
            for (int k = 0; k < NK; k++)
                if (okf(j, k)) {
                    const uint32_t id = v[j][k] >> 16;
                    const int b1 = (int)((hw[id >> 1] >> ((id & 1u) << 4)) & 0xffffu);
                    const int b0 = id ? (int)((hw[(id - 1) >> 1] >> (((id - 1) & 1u) << 4)) & 0xffffu) : 0;
                    int rk = b0;
                    if (OWN16) {
                        const int slot = (int)(v[j][k] & 0xffffu);
                        const uint32_t my = l16[slot];
                        for (int q = b0; q < b1; q++) {
                            const uint32_t l = l16[q];
                            rk += (l < my || (l == my && q < slot)) ? 1 : 0;
                        }
                    } else {
                        const uint32_t e = (v[j][k] << 16) | (uint32_t)((lane + 32 * k) | ((wid + 32 * j) << 8));
                        for (int q = b0; q < b1; q++) rk += ent[q] < e ? 1 : 0;
                    }
                    v[j][k] = (uint32_t)rk;
                }
        __syncthreads();
        PHASE(10);
#pragma unroll
        for (int j = 0; j < NK; j++)
#pragma unroll
            for (int k = 0; k < NK; k++)
                if (okf(j, k)) om[v[j][k]] = (uint16_t)((lane + 32 * k) | ((wid + 32 * j) << 8));
        for (int i = N + tid; i < g.Npad; i += blockDim.x) om[i] = 0xffffu;
        __syncthreads();
        store_omega(g, om, omega_slot(g, omega_out, bt));
        PHASE(11);
        return;
    }
    mark_runs(ent, &s_rl);
    if (s_rl.abort) {  // run list overflow (block-uniform after the scatter barrier)
        if (tid == 0) fallback[1 + atomicAdd(fallback, 1)] = bt;
        return;
    }
    if (s_runs)
        rank_buckets<true>(ent, d16, starts, N, om, &s_rl, fpr);
    else
        rank_buckets<false>(ent, d16, starts, N, om, &s_rl, fpr);
    __syncthreads();
    if (s_rl.abort) {  // a scan over budget (block-uniform after the barrier)
        if (tid == 0) fallback[1 + atomicAdd(fallback, 1)] = bt;
        return;
    }
    fill_big_runs(om, &s_rl, fpr);
    for (int i = N + tid; i < g.Npad; i += blockDim.x) om[i] = 0xffffu;
    __syncthreads();
    store_omega(g, om, omega_slot(g, omega_out, bt));
}

// FP: the plan ranks a tile footprint (g.fprow); a separate instance, so the
// footprint tests cost the usual (whole-tile) instance no registers.
template <int NK, bool GENT, bool FP>
__global__ void __launch_bounds__(1024) k1_f32_bucket(Geom g, uint16_t* __restrict__ omega_out,
                                                     int* __restrict__ fallback, uint32_t* __restrict__ gent,
                                                     long long gent_stride, unsigned long long max_sumsq) {
    const int bt = chunk_tile(g);  // costly (replicate-run) tiles start first
    const TileCoord tc = tile_coord(g, g.tile_begin + bt);
    if (has_runs(g, tc))
        f32_bucket_tile<NK, GENT, true, FP>(g, tc, bt, omega_out, fallback, gent, gent_stride, max_sumsq);
    else
        f32_bucket_tile<NK, GENT, false, FP>(g, tc, bt, omega_out, fallback, gent, gent_stride, max_sumsq);
}

// k1_f32_bucket for tiles too large for shared-memory entries (N > ~23.7K,
// e.g. r >= 54): the bucket-ordered entries live in the tile's global scratch
// slot (L2-resident: written once, read bucket by bucket), the keys are read
// from the image twice instead of held in registers, and only the 128 KB
// histogram (later omega) and the bucket-start bitmap stay in shared memory.
__global__ void __launch_bounds__(1024) k1_f32_bucket_g(Geom g, uint16_t* __restrict__ omega_out,
                                                       int* __restrict__ fallback,
                                                       uint32_t* __restrict__ gent, long long gent_stride,
                                                       unsigned long long max_sumsq) {
    extern __shared__ __align__(16) unsigned char smem[];
    constexpr int NW = 32768;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
    const int bt = chunk_tile(g);  // costly (replicate-run) tiles start first
    const TileCoord tc = tile_coord(g, g.tile_begin + bt);
    PHASE_T0;
    const int S = g.Sw, SH = g.Sh, N = g.N;
    uint32_t* hw = reinterpret_cast<uint32_t*>(smem);
    uint32_t* starts = hw + NW;
    const int nsw = (N + 31) >> 5;
    uint32_t* ctab = starts + ((nsw + 3) & ~3);  // coarse bins / fine-bucket table (f32)
    const bool adaptive = g.dtype == DT_F32 && N > kAdaptiveMinN;
    uint32_t* ent = gent + bt * gent_stride;
    uint16_t* d16 = reinterpret_cast<uint16_t*>(ent + N);  // run descriptors (2 B / slot)
    __shared__ unsigned long long s_sumsq;
    __shared__ int s_runs;
    __shared__ RunList s_rl;
    const int X0 = tc.ox0 - g.r + g.vshift, Y0 = tc.oy0 - g.r + g.vshift;
    const bool edge = has_runs(g, tc);
    {
        uint4* h4 = reinterpret_cast<uint4*>(hw);
        for (int i = tid; i < NW / 4; i += blockDim.x) h4[i] = make_uint4(0, 0, 0, 0);
        for (int i = tid; i < nsw; i += blockDim.x) starts[i] = 0;
        if (tid == 0) {
            s_sumsq = 0;
            s_runs = s_rl.n = s_rl.nbig = s_rl.nmark = s_rl.abort = 0;
        }
    }
    __syncthreads();
    const int nk = (S + 31) >> 5;
    PHASE(0);

    // visit every ranked pixel: fn(x, y, key, weight, cx, cy); a row's keys
    // (<= 8 per lane, S <= 255) are loaded before any is used
    auto each_pixel = [&](auto fn) {
        for (int y = wid; y < SH; y += nw) {
            int yy = Y0 + y;
            yy = yy < 0 ? 0 : (yy >= g.H ? g.H - 1 : yy);
            int cy = 1;
            bool fy = true;
            if (edge) rep_axis(Y0, y, SH, g.H, cy, fy);
            // footprint columns of this row (empty: lo = hi = 0xffff)
            const uint32_t fr = g.fprow ? __ldg(g.fprow + y) : (uint32_t)(S - 1) << 16;
            const int flo = (int)(fr & 0xffffu), fspan = (int)(fr >> 16) - flo;
            uint32_t kv[8];
#pragma unroll
            for (int k = 0; k < 8; k++) {
                if (k < nk) {
                    int xx = X0 + min(lane + 32 * k, S - 1);
                    xx = xx < 0 ? 0 : (xx >= g.W ? g.W - 1 : xx);
                    kv[k] = f32_key(g, tc, yy, xx);
                }
            }
#pragma unroll
            for (int k = 0; k < 8; k++) {
                const int x = lane + 32 * k;
                if (k < nk && x < S) {
                    int cx = 1;
                    bool fx = true;
                    int wc = (unsigned)(x - flo) <= (unsigned)fspan ? 1 : 0;
                    if (edge) {
                        rep_axis(X0, x, S, g.W, cx, fx);
                        wc = pixel_weight(g, g.fprow, x, cx, fx, y, cy, fy);
                    }
                    if (wc) fn(x, y, kv[k], wc, cx, cy);
                }
            }
        }
    };
    // f32: fine bucket << 16 | low 16 key bits (coarse_alloc); u16: the key
    auto bucket_key = [&](uint32_t key) {
        return adaptive ? (fine_bucket(ctab, key) << 16) | (key & 0xffffu) : key;
    };
    if (adaptive) {
        for (int i = tid; i < kCoarse; i += blockDim.x) ctab[i] = g.ctab_g ? g.ctab_g[i] : 0u;
        __syncthreads();
        if (!g.ctab_g) {  // no call-wide table: this tile's own coarse pass
            each_pixel([&](int, int, uint32_t key, int wc, int, int) { atomicAdd(&ctab[key >> 20], (uint32_t)wt_of(wc)); });
            coarse_alloc(ctab, N);
        }
        PHASE(1);
    }
    bool runs = false;
    each_pixel([&](int, int, uint32_t key, int wc, int, int) {
        runs |= (wc & kRunBit) != 0;
        const uint32_t h = bucket_key(key) >> 16, sh = (h & 1) << 4;
        atomicAdd(&hw[h >> 1], (uint32_t)wt_of(wc) << sh);
    });
    if (runs) s_runs = 1;
    __syncthreads();
    hist16_exclusive_scan(hw, NW, starts, &s_sumsq);
    __syncthreads();
    PHASE(2);
    if (!s_runs && s_sumsq > max_sumsq) {
        if (tid == 0) fallback[1 + atomicAdd(fallback, 1)] = bt;
        return;
    }
    each_pixel([&](int x, int y, uint32_t key, int wc, int cx, int cy) {
        const uint32_t bk = bucket_key(key), h = bk >> 16, sh = (h & 1) << 4;
        const uint32_t old = atomicAdd(&hw[h >> 1], (uint32_t)wt_of(wc) << sh);
        put_entry(ent, d16, (old >> sh) & 0xffffu, bk & 0xffffu, x, y, wc, cx, cy, &s_rl, g.fprow);
    });
    __syncthreads();  // block-scope ordering of the entry stores (global, same CTA)
    mark_runs(ent, &s_rl);
    PHASE(3);
    uint16_t* om = reinterpret_cast<uint16_t*>(hw);
    if (s_rl.abort) {  // run list overflow (block-uniform after the scatter barrier)
        if (tid == 0) fallback[1 + atomicAdd(fallback, 1)] = bt;
        return;
    }
    if (s_runs)
        rank_buckets<true>(ent, d16, starts, N, om, &s_rl, g.fprow);
    else
        rank_buckets<false>(ent, d16, starts, N, om, &s_rl, g.fprow);
    __syncthreads();
    PHASE(4);
    if (s_rl.abort) {  // a scan over budget (block-uniform after the barrier)
        if (tid == 0) fallback[1 + atomicAdd(fallback, 1)] = bt;
        return;
    }
    fill_big_runs(om, &s_rl, g.fprow);
    for (int i = N + tid; i < g.Npad; i += blockDim.x) om[i] = 0xffffu;
    __syncthreads();
    store_omega(g, om, omega_slot(g, omega_out, bt));
    PHASE(5);

}

size_t k1_f32_bucket_g_smem_bytes(int N) {
    return 32768 * 4 + 4 * (size_t)(((N + 31) >> 5) + 3 & ~3) + 4 * (size_t)kCoarse + 16;
}

#define IMF_K1F1(NK, FP)                                                                             \
    template __global__ void k1_f32_bucket<NK, false, FP>(Geom, uint16_t*, int*, uint32_t*, long long, \
                                                          unsigned long long);                      \
    template __global__ void k1_f32_bucket<NK, true, FP>(Geom, uint16_t*, int*, uint32_t*, long long,  \
                                                         unsigned long long);
#define IMF_K1F(NK) IMF_K1F1(NK, false) IMF_K1F1(NK, true)
IMF_K1F(1)
IMF_K1F(2)
IMF_K1F(3)
IMF_K1F(4)
IMF_K1F(5)
IMF_K1F(6)
#undef IMF_K1F

size_t k1_f32_bucket_smem_bytes(int N) {
    return 32768 * 4 + 4 * (size_t)std::max((N + 3) & ~3, kCoarse) + 4 * (size_t)((N + 31) >> 5) + 16;
}

template __global__ void k1_count<DT_U8>(Geom, uint16_t*);
template __global__ void k1_count<DT_U16>(Geom, uint16_t*);

// u16 tiles too large for the histogram AND omega in shared memory (S > ~180,
// r > ~85): the same counting sort with omega scattered straight to the tile's
// global slot (2-byte stores, L2-resident), keys read twice from the image.
__global__ void __launch_bounds__(1024) k1_count_g(Geom g, uint16_t* __restrict__ omega_out) {
    extern __shared__ __align__(16) unsigned char smem[];
    constexpr int NW = 32768;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
    const TileCoord tc = tile_coord(g, g.tile_begin + blockIdx.x);
    const int S = g.Sw, SH = g.Sh, nk = (S + 31) >> 5;
    uint32_t* hw = reinterpret_cast<uint32_t*>(smem);
    uint16_t* om = omega_slot(g, omega_out);
    {
        uint4* h4 = reinterpret_cast<uint4*>(hw);
        for (int i = tid; i < NW / 4; i += blockDim.x) h4[i] = make_uint4(0, 0, 0, 0);
    }
    __syncthreads();
    auto each_pixel = [&](auto fn) {
        for (int y = wid; y < SH; y += nw) {
            uint32_t kv[8];
#pragma unroll
            for (int k = 0; k < 8; k++)
                if (k < nk) kv[k] = load_key(g, tc, y, min(lane + 32 * k, S - 1));
#pragma unroll
            for (int k = 0; k < 8; k++)
                if (k < nk && lane + 32 * k < S) fn(lane + 32 * k, y, kv[k]);
        }
    };
    each_pixel([&](int, int, uint32_t v) { atomicAdd(&hw[v >> 1], 1u << ((v & 1) << 4)); });
    __syncthreads();
    if (NW == 32768 && blockDim.x == 1024)
        hist16_scan_lanes(hw);
    else
        hist16_exclusive_scan(hw, NW);
    __syncthreads();
    each_pixel([&](int x, int y, uint32_t v) {
        const uint32_t sh = (v & 1) << 4;
        const uint32_t old = atomicAdd(&hw[v >> 1], 1u << sh);
        om[(old >> sh) & 0xffffu] = (uint16_t)(x | (y << 8));
    });
    for (int i = g.N + tid; i < g.Npad; i += blockDim.x) om[i] = 0xffffu;
    if (tid < OMEGA_SLOT_PAD) {
        om[-OMEGA_SLOT_PAD + tid] = 0xffffu;
        om[g.Npad + tid] = 0xffffu;
    }
}

size_t k1_count_g_smem_bytes() { return 32768 * 4 + 16; }

size_t k1_count_smem_bytes(int dtype, int Npad) {
    return (dtype == DT_U8 ? 128 * 4 : 32768 * 4) + 256 + 2 * (size_t)Npad;  // + k1_count_reg's sink words, mbarrier
}

template __global__ void k1_sort<DT_U8, false>(Geom, uint16_t*, unsigned char*, long long, const int*);
template __global__ void k1_sort<DT_U16, false>(Geom, uint16_t*, unsigned char*, long long, const int*);
template __global__ void k1_sort<DT_U16, true>(Geom, uint16_t*, unsigned char*, long long, const int*);
template __global__ void k1_sort<DT_F32, false>(Geom, uint16_t*, unsigned char*, long long, const int*);
template __global__ void k1_sort<DT_F32, true>(Geom, uint16_t*, unsigned char*, long long, const int*);

// Shared-memory bytes K1 needs for a tile (GMEM: large arrays in global scratch).
size_t k1_smem_bytes(int dtype, int Npad, int nwarps, bool gmem) {
    size_t b = 256 * 4 + (dtype == DT_U8 ? 0 : 256 * 4 * (size_t)(nwarps + 1)) + 2 * (size_t)Npad;
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

#ifdef IMF_STATS
extern "C" int imf_rstats(unsigned long long* out, int reset) {
    if (cudaMemcpyFromSymbol(out, imf::g_rstats, sizeof(imf::g_rstats))) return 2;
    if (reset) {
        static const unsigned long long z[128] = {};
        cudaMemcpyToSymbol(imf::g_rstats, z, sizeof(z));
    }
    return 0;
}
#endif
