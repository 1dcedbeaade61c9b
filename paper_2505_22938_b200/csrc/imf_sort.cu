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

__device__ __forceinline__ uint16_t pack_pos(int i, int Sw, float invS) {
    int x, y;
    lin_to_xy(i, Sw, invS, x, y);
    return (uint16_t)(x | (y << 8));
}

// Copy the finished omega (smem, N entries) to its global slot, 16 B at a time.
// Global omega slot of a tile: OMEGA_SLOT_PAD sentinel entries on both sides
// of Npad ranks, so scans may step a few ranks past either end.
__device__ __forceinline__ uint16_t* omega_slot(const Geom& g, uint16_t* base, int bt = -1) {
    if (bt < 0) bt = blockIdx.x;
    return base + (long long)bt * (g.Npad + 2 * OMEGA_SLOT_PAD) + OMEGA_SLOT_PAD;
}

__device__ __forceinline__ void store_omega(const Geom& g, const uint16_t* om_s, uint16_t* om_g) {
    const int n16 = g.Npad >> 3;  // uint4 count
    const uint4* s = reinterpret_cast<const uint4*>(om_s);
    uint4* d = reinterpret_cast<uint4*>(om_g);
    for (int i = threadIdx.x; i < n16; i += blockDim.x) d[i] = s[i];
    if (threadIdx.x < OMEGA_SLOT_PAD) {
        om_g[-OMEGA_SLOT_PAD + (int)threadIdx.x] = 0xffffu;
        om_g[g.Npad + threadIdx.x] = 0xffffu;
    }
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
    uint32_t* hist = reinterpret_cast<uint32_t*>(smem);
    uint32_t* cnt = hist + 256;
    uint16_t* om = reinterpret_cast<uint16_t*>(cnt + (DT == DT_U8 ? 0 : 256 * (nw + 1)));
    unsigned char* big = GMEM ? gscratch + bt * gscratch_stride
                              : reinterpret_cast<unsigned char*>(om + g.Npad);
    uint16_t* om_g = omega_slot(g, omega_out, bt);

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

// Exclusive scan, in place, of the 2*NW 16-bit counters packed two per word
// in hw[0..NW).  Warp w owns words [w*NW/nw, (w+1)*NW/nw); lanes stride by one
// word, so every shared access is bank-conflict free.  Ends with the counters
// replaced by their exclusive prefix (no trailing barrier).
__device__ __forceinline__ void hist16_exclusive_scan(uint32_t* hw, const int NW,
                                                      uint32_t* starts = nullptr,
                                                      unsigned long long* sumsq = nullptr) {
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
    __shared__ uint32_t wt[32];
    const int per = NW / nw;  // words per warp (NW and nw are powers of two)
    if (per >= 128) {
        // 16-byte chunks: lane l of the warp handles chunk i*32 + l of the warp's
        // range (conflict-free), 8 counters per lane per step.  Every prefix of a
        // tile's counters is < 65536, so the scan runs on PACKED words: adding
        // words adds both 16-bit halves independently (no carry can cross), and
        // counter 2i's exclusive prefix is lo + hi of the packed word prefix.
        uint4* wb = reinterpret_cast<uint4*>(hw + wid * per);
        const int nch = per >> 2;  // chunks per warp, multiple of 32
        uint32_t sum = 0;
        for (int i = lane; i < nch; i += 32) {
            const uint4 q = wb[i];
            sum += q.x + q.y + q.z + q.w;
        }
        sum = __reduce_add_sync(0xffffffffu, sum);
        sum = (sum & 0xffffu) + (sum >> 16);
        if (lane == 0) wt[wid] = sum;
        __syncthreads();
        if (wid == 0) {
            uint32_t v = lane < nw ? wt[lane] : 0, x = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                uint32_t t = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += t;
            }
            if (lane < nw) wt[lane] = x - v;
        }
        __syncthreads();
        uint32_t carry = wt[wid];  // plain (unpacked) count before this chunk row
        for (int i0 = 0; i0 < nch; i0 += 32) {
            uint4 q = wb[i0 + lane];
            const uint32_t p1 = q.x, p2 = p1 + q.y, p3 = p2 + q.z, tot = p3 + q.w;  // packed prefixes
            uint32_t incl = tot;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += t;
            }
            const uint32_t ex = incl - tot;  // packed exclusive prefix of this lane's chunk
            const uint32_t base = carry + (ex & 0xffffu) + (ex >> 16);
            // counters before word k: base + flat(packed prefix of words < k)
            const uint32_t b0 = base, b1 = base + (p1 & 0xffffu) + (p1 >> 16);
            const uint32_t b2 = base + (p2 & 0xffffu) + (p2 >> 16), b3 = base + (p3 & 0xffffu) + (p3 >> 16);
            if (starts) {  // bit at every non-empty counter's first position (bucket starts)
                const uint32_t cw[4] = {q.x, q.y, q.z, q.w}, bw[4] = {b0, b1, b2, b3};
                unsigned long long sq = 0;
#pragma unroll
                for (int k = 0; k < 4; k++) {
                    const uint32_t lo = cw[k] & 0xffffu, hi = cw[k] >> 16, e0 = bw[k], e1 = bw[k] + lo;
                    if (lo) atomicOr(&starts[e0 >> 5], 1u << (e0 & 31));
                    if (hi) atomicOr(&starts[e1 >> 5], 1u << (e1 & 31));
                    sq += (unsigned long long)(lo * lo) + (unsigned long long)(hi * hi);
                }
                // clamp per lane at 2^26 (> kMaxSumSq: the tile falls back anyway) so
                // the 32-bit warp sum cannot wrap
                const unsigned wsq = __reduce_add_sync(0xffffffffu, (unsigned)min(sq, 1ull << 26));
                if (lane == 0 && wsq) atomicAdd(sumsq, (unsigned long long)wsq);
            }
            q.x = b0 | ((b0 + (q.x & 0xffffu)) << 16);
            q.y = b1 | ((b1 + (q.y & 0xffffu)) << 16);
            q.z = b2 | ((b2 + (q.z & 0xffffu)) << 16);
            q.w = b3 | ((b3 + (q.w & 0xffffu)) << 16);
            wb[i0 + lane] = q;
            const uint32_t last = __shfl_sync(0xffffffffu, incl, 31);
            carry += (last & 0xffffu) + (last >> 16);
        }
        return;
    }
    // small histograms (u8: 128 words): one word per lane per step
    const uint32_t* wbase = hw + wid * per;
    uint32_t sum = 0;
    for (int i = lane; i < per; i += 32) {
        const uint32_t w = wbase[i];
        sum += (w & 0xffffu) + (w >> 16);
    }
    sum = __reduce_add_sync(0xffffffffu, sum);
    if (lane == 0) wt[wid] = sum;
    __syncthreads();
    if (wid == 0) {
        uint32_t v = lane < nw ? wt[lane] : 0, x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t t = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += t;
        }
        if (lane < nw) wt[lane] = x - v;
    }
    __syncthreads();
    uint32_t carry = wt[wid];
    uint32_t* wb = hw + wid * per;
    for (int i0 = 0; i0 < per; i0 += 32) {
        const bool ok = i0 + lane < per;
        const uint32_t w = ok ? wb[i0 + lane] : 0u;
        const uint32_t lo = w & 0xffffu, tot = lo + (w >> 16);
        uint32_t incl = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        const uint32_t ex = carry + incl - tot;
        if (ok) wb[i0 + lane] = ex | ((ex + lo) << 16);
        if (starts && ok) {  // bucket starts, as in the chunked branch
            const uint32_t hi = w >> 16;
            if (lo) atomicOr(&starts[ex >> 5], 1u << (ex & 31));
            if (hi) atomicOr(&starts[(ex + lo) >> 5], 1u << ((ex + lo) & 31));
            if (sumsq) {
                const unsigned long long sq = (unsigned long long)lo * lo + (unsigned long long)hi * hi;
                atomicAdd(sumsq, sq);
            }
        }
        carry += __shfl_sync(0xffffffffu, incl, 31);
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

// k1_count with the tile held in registers: warp w owns input rows w + 32j,
// lane l owns columns l + 32k (j, k < NK = ceil(S/32)), so every value is read
// from global memory ONCE, with all NK*NK loads of a thread in flight together
// (the two-pass k1_count re-reads the tile and exposes the L2 latency per row).
// 1024 threads; same histogram / scan / scatter as k1_count.
template <int DT, int NK>
__global__ void __launch_bounds__(1024) k1_count_reg(Geom g, uint16_t* __restrict__ omega_out) {
    extern __shared__ __align__(16) unsigned char smem[];
    constexpr int NB = DT == DT_U8 ? 256 : 65536;
    constexpr int NW = NB / 2;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const TileCoord tc = tile_coord(g, g.tile_begin + blockIdx.x);
    const int S = g.Sw, SH = g.Sh;
    uint32_t* hw = reinterpret_cast<uint32_t*>(smem);
    uint16_t* om = reinterpret_cast<uint16_t*>(hw + NW);
    uint32_t v[NK][NK];
    {
        // element offsets within one (image, channel) plane fit 32 bits
        int xo[NK];
#pragma unroll
        for (int k = 0; k < NK; k++) {
            int x = tc.ox0 + lane + 32 * k - g.r + g.vshift;
            x = x < 0 ? 0 : (x >= g.W ? g.W - 1 : x);
            xo[k] = x * (int)g.s_x;
        }
#pragma unroll
        for (int j = 0; j < NK; j++) {
            const int y = wid + 32 * j;
            int yy = tc.oy0 + y - g.r + g.vshift;
            yy = yy < 0 ? 0 : (yy >= g.H ? g.H - 1 : yy);
            const int ro = yy * (int)g.s_y;
            // footprint columns of this row: [flo, fhi] (all columns without one)
            int flo = 0, fhi = S - 1;
            if (g.fp) {
                const int ey = max(0, max(g.r - y, y - (g.r + g.Th - 1)));
                const int D = g.fpR2 - ey * ey;
                int w = D < 0 ? -1 : (int)sqrtf((float)D);
                if (w >= 0) {
                    while (w * w > D) w--;
                    while ((w + 1) * (w + 1) <= D) w++;
                }
                flo = w < 0 ? S : g.r - w;
                fhi = g.r + g.Tw - 1 + w;
            }
#pragma unroll
            for (int k = 0; k < NK; k++) {
                const int x = lane + 32 * k;
                const bool ok = y < SH && x < S && x >= flo && x <= fhi;
                uint32_t val = 0xffffffffu;
                if (ok) {
                    val = DT == DT_U8 ? (uint32_t)__ldg((const uint8_t*)tc.src + (ro + xo[k]))
                                      : (uint32_t)__ldg((const uint16_t*)tc.src + (ro + xo[k]));
                }
                v[j][k] = val;
            }
        }
    }
    {
        uint4* h4 = reinterpret_cast<uint4*>(hw);
        for (int i = tid; i < NW / 4; i += blockDim.x) h4[i] = make_uint4(0, 0, 0, 0);
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < NK; j++)
#pragma unroll
        for (int k = 0; k < NK; k++)
            if (v[j][k] != 0xffffffffu) atomicAdd(&hw[v[j][k] >> 1], 1u << ((v[j][k] & 1) << 4));
    __syncthreads();
    hist16_exclusive_scan(hw, NW);
    __syncthreads();
#pragma unroll
    for (int j = 0; j < NK; j++)
#pragma unroll
        for (int k = 0; k < NK; k++) {
            const uint32_t val = v[j][k];
            if (val != 0xffffffffu) {
                const uint32_t sh = (val & 1) << 4;
                const uint32_t old = atomicAdd(&hw[val >> 1], 1u << sh);
                om[(old >> sh) & 0xffffu] = (uint16_t)((lane + 32 * k) | ((wid + 32 * j) << 8));
            }
        }
    for (int i = g.N + tid; i < g.Npad; i += blockDim.x) om[i] = 0xffffu;
    __syncthreads();
    store_omega(g, om, omega_slot(g, omega_out));
}

#define IMF_K1R(DT) \
    template __global__ void k1_count_reg<DT, 1>(Geom, uint16_t*); \
    template __global__ void k1_count_reg<DT, 2>(Geom, uint16_t*); \
    template __global__ void k1_count_reg<DT, 3>(Geom, uint16_t*); \
    template __global__ void k1_count_reg<DT, 4>(Geom, uint16_t*); \
    template __global__ void k1_count_reg<DT, 5>(Geom, uint16_t*); \
    template __global__ void k1_count_reg<DT, 6>(Geom, uint16_t*);
IMF_K1R(DT_U8)
IMF_K1R(DT_U16)
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
constexpr unsigned long long kMaxSumSq = 64ull << 20;

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
// pixel (replicate boundary, >= kRunMin of them: tile corners and edges) are
// ranked once, as a RUN of consecutive ranks held by the first copy (weight =
// copy count, the others 0); ties order arbitrarily (imf_sort.cu header), so
// the run's internal order is free.  Entries of a run starting at slot s:
//   ent[s]     = key16 << 16 | 0xffff                  (run head)
//   ent[s + 1] = pos << 16 | 0xfffe                     (first copy x | y << 8)
//   ent[s + 2] = (cnt_x | cnt_y << 8) << 16 | 0xfffe    (copy rectangle)
//   ent[s + 3 ..] = 0xfffe                               (interior)
// Plain entries are key16 << 16 | pos with pos <= 0xfefe (x, y < 255).
// Only groups of >= kRunMin copies become runs: ranking a group of m plain
// copies costs m^2 compares (~1 per thread at m = 32 for a 1024-thread CTA),
// which only the tile-corner groups, (r+1)^2 copies, make worth the run
// bookkeeping (measured: edges, r+1 copies, gain nothing even at r = 100).
constexpr int kRunMin = 1024;

// Largest copy group of a tile (columns [X0, X0 + S) of an image W wide).
__device__ __forceinline__ int max_copies(int X0, int S, int W) {
    if (W == 1) return S;
    const int l = X0 < 0 ? min(S, 1 - X0) : 1;
    const int r = X0 + S > W ? S - max(0, W - 1 - X0) : 1;
    return max(l, r);
}

__device__ __forceinline__ bool has_runs(const Geom& g, const TileCoord& tc) {
    const int X0 = tc.ox0 - g.r + g.vshift, Y0 = tc.oy0 - g.r + g.vshift;
    return !g.fp && max_copies(X0, g.Sw, g.W) * max_copies(Y0, g.Sh, g.H) >= kRunMin;
}

__device__ __forceinline__ int pixel_weight(int cx, bool fx, int cy, bool fy) {
    const int m = cx * cy;
    if (m < kRunMin) return 1;
    return (fx && fy) ? m : 0;
}

__device__ __forceinline__ void put_entry(uint32_t* ent, int slot, uint32_t key16, int x, int y, int w, int cx,
                                          int cy) {
    const uint32_t pos = (uint32_t)(x | (y << 8));
    if (w == 1) {
        ent[slot] = (key16 << 16) | pos;
        return;
    }
    ent[slot] = (key16 << 16) | 0xffffu;
    ent[slot + 1] = (pos << 16) | 0xfffeu;
    ent[slot + 2] = ((uint32_t)(cx | (cy << 8)) << 16) | 0xfffeu;
    for (int i = 3; i < w; i++) ent[slot + i] = 0xfffeu;
}

// Rank every entry within its bucket (starts: bucket-start bitmap) and write
// omega.  Each scan is bounded (kScanMax steps); a thread past its budget sets
// *abort and the caller hands the tile to the radix sort (block-uniform after
// the closing barrier).  Long runs are filled by the whole CTA.
constexpr int kScanMax = 4096;
constexpr int kScanBudget = 16384;
constexpr int kBigRuns = 16;

// RUNS = false (tiles without runs, already bounded by the sum-of-squares
// estimate): the plain unrolled compare loop.
template <bool RUNS>
__device__ void rank_buckets(const uint32_t* ent, const uint32_t* starts, int N, uint16_t* om, int* abort_flag,
                             int* nbig, uint4* big) {
    const int nsw = (N + 31) >> 5;
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
        if (!RUNS) {
            for (int q = b0; q < b1; q++) rk += ent[q] < e ? 1 : 0;
            om[rk] = (uint16_t)lo;
            continue;
        }
        int q = b0, it = 0;
        for (; q < b1 && it < kScanMax; it++) {
            if (q + 4 <= b1) {  // four plain entries at once (no run head among them)
                const uint32_t v0 = ent[q], v1 = ent[q + 1], v2 = ent[q + 2], v3 = ent[q + 3];
                const bool h = (v0 & 0xffffu) == 0xffffu || (v1 & 0xffffu) == 0xffffu ||
                               (v2 & 0xffffu) == 0xffffu || (v3 & 0xffffu) == 0xffffu;
                if (!h) {
                    rk += (v0 < e ? 1 : 0) + (v1 < e ? 1 : 0) + (v2 < e ? 1 : 0) + (v3 < e ? 1 : 0);
                    q += 4;
                    continue;
                }
            }
            const uint32_t v = ent[q];
            if ((v & 0xffffu) == 0xffffu) {  // run head: the run orders as a whole
                const uint32_t d = ent[q + 2] >> 16;
                const int len = (int)(d & 0xffu) * (int)(d >> 8);
                rk += (v < e || (v == e && q < sp)) ? len : 0;
                q += len;
            } else {
                rk += v < e ? 1 : 0;
                q++;
            }
        }
        work += it;
        if (q < b1 || work > kScanBudget) {
            *abort_flag = 1;
            break;
        }
        if (lo != 0xffffu) {
            om[rk] = (uint16_t)lo;
            continue;
        }
        const uint32_t pos = ent[sp + 1] >> 16, d = ent[sp + 2] >> 16;
        const int cx = (int)(d & 0xffu), cy = (int)(d >> 8), len = cx * cy;
        if (len > 256) {
            const int k = atomicAdd(nbig, 1);
            if (k < kBigRuns) {
                big[k] = make_uint4((uint32_t)rk, pos, (uint32_t)cx, (uint32_t)cy);
                continue;
            }
        }
        for (int i = 0; i < len; i++) {
            const int yy = i / cx, xx = i - yy * cx;
            om[rk + i] = (uint16_t)(pos + (uint32_t)(xx | (yy << 8)));
        }
    }
}

// After the barrier closing rank_buckets: fill the long runs with the CTA.
__device__ void fill_big_runs(uint16_t* om, int nbig, const uint4* big) {
    for (int k = 0; k < min(nbig, kBigRuns); k++) {
        const uint4 b = big[k];
        const int cx = (int)b.z, len = cx * (int)b.w;
        for (int i = threadIdx.x; i < len; i += blockDim.x) {
            const int yy = i / cx, xx = i - yy * cx;
            om[b.x + i] = (uint16_t)(b.y + (uint32_t)(xx | (yy << 8)));
        }
    }
}

// GENT: the entries live in the tile's global scratch slot (tiles too large
// for shared-memory entries); the keys stay in registers either way.
// EDGE: the tile reads clamped (replicated) image pixels; the copies of one
// pixel are ranked as a run (pixel_weight).  Interior tiles take the EDGE =
// false instance, which carries none of that.
template <int NK, bool GENT, bool EDGE>
__device__ __forceinline__ void f32_bucket_tile(const Geom& g, const TileCoord& tc, uint16_t* __restrict__ omega_out,
                                                int* __restrict__ fallback, uint32_t* __restrict__ gent,
                                                long long gent_stride, unsigned long long max_sumsq) {
    extern __shared__ __align__(16) unsigned char smem[];
    constexpr int NW = 32768;  // histogram words (65536 16-bit counters)
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int S = g.Sw, SH = g.Sh, N = g.N;
    uint32_t* hw = reinterpret_cast<uint32_t*>(smem);
    uint32_t* ent = GENT ? gent + blockIdx.x * gent_stride : hw + NW;  // N entries
    uint32_t* starts = GENT ? hw + NW : ent + ((N + 3) & ~3);        // bucket starts, ceil(N/32) words
    const int nsw = (N + 31) >> 5;
    __shared__ unsigned long long s_sumsq;
    __shared__ int s_runs, s_abort, s_nbig;
    __shared__ uint4 s_big[kBigRuns];
    uint32_t v[NK][NK];
    unsigned long long okm = 0;  // which of this thread's pixels are ranked (weight > 0)
    // replicate copies (rep_axis), edge tiles only, recomputed where used
    // (keeps the 1024-thread register budget for the keys)
    const int X0 = tc.ox0 - g.r + g.vshift, Y0 = tc.oy0 - g.r + g.vshift;
    auto weight = [&](int j, int k) {
        if (!EDGE) return 1;
        int cx, cy;
        bool fx, fy;
        rep_axis(X0, lane + 32 * k, S, g.W, cx, fx);
        rep_axis(Y0, wid + 32 * j, SH, g.H, cy, fy);
        return pixel_weight(cx, fx, cy, fy);
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
                const bool ok = y < SH && lane + 32 * k < S && in_footprint(g, lane + 32 * k, y) && weight(j, k) > 0;
                v[j][k] = ok ? f32_key(g, tc, yy, xc[k]) : 0u;
                okm |= (ok ? 1ull : 0ull) << (j * NK + k);
            }
        }
    }
    {
        uint4* h4 = reinterpret_cast<uint4*>(hw);
        for (int i = tid; i < NW / 4; i += blockDim.x) h4[i] = make_uint4(0, 0, 0, 0);
        for (int i = tid; i < nsw; i += blockDim.x) starts[i] = 0;
        if (tid == 0) {
            s_sumsq = 0;
            s_runs = s_abort = s_nbig = 0;
        }
    }
    __syncthreads();
    bool runs = false;
#pragma unroll
    for (int j = 0; j < NK; j++)
#pragma unroll
        for (int k = 0; k < NK; k++)
            if ((okm >> (j * NK + k)) & 1ull) {
                const uint32_t h = v[j][k] >> 16, sh = (h & 1) << 4;
                const int wt = weight(j, k);
                runs |= wt > 1;
                atomicAdd(&hw[h >> 1], (uint32_t)wt << sh);
            }
    if (runs) s_runs = 1;
    __syncthreads();
    hist16_exclusive_scan(hw, NW, starts, &s_sumsq);
    __syncthreads();
    // tiles with runs skip the estimate (run weights inflate it); their scans
    // are bounded instead (rank_buckets)
    if (!s_runs && s_sumsq > max_sumsq) {  // block-uniform: hand the tile to the radix sort
        if (tid == 0) fallback[1 + atomicAdd(fallback, 1)] = blockIdx.x;
        return;
    }
#pragma unroll
    for (int j = 0; j < NK; j++)
#pragma unroll
        for (int k = 0; k < NK; k++)
            if ((okm >> (j * NK + k)) & 1ull) {
                const uint32_t key = v[j][k], h = key >> 16, sh = (h & 1) << 4;
                const int wt = weight(j, k);
                const uint32_t old = atomicAdd(&hw[h >> 1], (uint32_t)wt << sh);
                put_entry(ent, (old >> sh) & 0xffffu, key & 0xffffu, lane + 32 * k, wid + 32 * j, wt, cnt_x(k),
                          cnt_y(j));
            }
    __syncthreads();
    uint16_t* om = reinterpret_cast<uint16_t*>(hw);  // the histogram is dead: omega goes here
    if (s_runs)
        rank_buckets<true>(ent, starts, N, om, &s_abort, &s_nbig, s_big);
    else
        rank_buckets<false>(ent, starts, N, om, &s_abort, &s_nbig, s_big);
    __syncthreads();
    if (s_abort) {
        if (tid == 0) fallback[1 + atomicAdd(fallback, 1)] = blockIdx.x;
        return;
    }
    fill_big_runs(om, s_nbig, s_big);
    for (int i = N + tid; i < g.Npad; i += blockDim.x) om[i] = 0xffffu;
    __syncthreads();
    store_omega(g, om, omega_slot(g, omega_out));
}

template <int NK, bool GENT>
__global__ void __launch_bounds__(1024) k1_f32_bucket(Geom g, uint16_t* __restrict__ omega_out,
                                                     int* __restrict__ fallback, uint32_t* __restrict__ gent,
                                                     long long gent_stride, unsigned long long max_sumsq) {
    const TileCoord tc = tile_coord(g, g.tile_begin + blockIdx.x);
    if (has_runs(g, tc))
        f32_bucket_tile<NK, GENT, true>(g, tc, omega_out, fallback, gent, gent_stride, max_sumsq);
    else
        f32_bucket_tile<NK, GENT, false>(g, tc, omega_out, fallback, gent, gent_stride, max_sumsq);
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
    const TileCoord tc = tile_coord(g, g.tile_begin + blockIdx.x);
    const int S = g.Sw, SH = g.Sh, N = g.N;
    uint32_t* hw = reinterpret_cast<uint32_t*>(smem);
    uint32_t* starts = hw + NW;
    const int nsw = (N + 31) >> 5;
    uint32_t* ent = gent + blockIdx.x * gent_stride;
    __shared__ unsigned long long s_sumsq;
    __shared__ int s_runs, s_abort, s_nbig;
    __shared__ uint4 s_big[kBigRuns];
    const int X0 = tc.ox0 - g.r + g.vshift, Y0 = tc.oy0 - g.r + g.vshift;
    const bool edge = has_runs(g, tc);
    {
        uint4* h4 = reinterpret_cast<uint4*>(hw);
        for (int i = tid; i < NW / 4; i += blockDim.x) h4[i] = make_uint4(0, 0, 0, 0);
        for (int i = tid; i < nsw; i += blockDim.x) starts[i] = 0;
        if (tid == 0) {
            s_sumsq = 0;
            s_runs = s_abort = s_nbig = 0;
        }
    }
    __syncthreads();
    const int nk = (S + 31) >> 5;
    bool runs = false;
    for (int y = wid; y < SH; y += nw) {
        int yy = Y0 + y;
        yy = yy < 0 ? 0 : (yy >= g.H ? g.H - 1 : yy);
        int cy = 1;
        bool fy = true;
        if (edge) rep_axis(Y0, y, SH, g.H, cy, fy);
        for (int k = 0; k < nk; k++) {
            const int x = lane + 32 * k;
            if (x < S) {
                int xx = X0 + x;
                xx = xx < 0 ? 0 : (xx >= g.W ? g.W - 1 : xx);
                int cx = 1;
                bool fx = true;
                if (edge) rep_axis(X0, x, S, g.W, cx, fx);
                const int wt = pixel_weight(cx, fx, cy, fy);
                if (wt) {
                    runs |= wt > 1;
                    const uint32_t h = f32_key(g, tc, yy, xx) >> 16;
                    const uint32_t sh = (h & 1) << 4;
                    atomicAdd(&hw[h >> 1], (uint32_t)wt << sh);
                }
            }
        }
    }
    if (runs) s_runs = 1;
    __syncthreads();
    hist16_exclusive_scan(hw, NW, starts, &s_sumsq);
    __syncthreads();
    if (!s_runs && s_sumsq > max_sumsq) {
        if (tid == 0) fallback[1 + atomicAdd(fallback, 1)] = blockIdx.x;
        return;
    }
    for (int y = wid; y < SH; y += nw) {
        int yy = Y0 + y;
        yy = yy < 0 ? 0 : (yy >= g.H ? g.H - 1 : yy);
        int cy = 1;
        bool fy = true;
        if (edge) rep_axis(Y0, y, SH, g.H, cy, fy);
        for (int k = 0; k < nk; k++) {
            const int x = lane + 32 * k;
            if (x < S) {
                int xx = X0 + x;
                xx = xx < 0 ? 0 : (xx >= g.W ? g.W - 1 : xx);
                int cx = 1;
                bool fx = true;
                if (edge) rep_axis(X0, x, S, g.W, cx, fx);
                const int wt = pixel_weight(cx, fx, cy, fy);
                if (wt) {
                    const uint32_t key = f32_key(g, tc, yy, xx);
                    const uint32_t h = key >> 16, sh = (h & 1) << 4;
                    const uint32_t old = atomicAdd(&hw[h >> 1], (uint32_t)wt << sh);
                    put_entry(ent, (old >> sh) & 0xffffu, key & 0xffffu, x, y, wt, cx, cy);
                }
            }
        }
    }
    __syncthreads();  // block-scope ordering of the entry stores (global, same CTA)
    uint16_t* om = reinterpret_cast<uint16_t*>(hw);
    if (s_runs)
        rank_buckets<true>(ent, starts, N, om, &s_abort, &s_nbig, s_big);
    else
        rank_buckets<false>(ent, starts, N, om, &s_abort, &s_nbig, s_big);
    __syncthreads();
    if (s_abort) {
        if (tid == 0) fallback[1 + atomicAdd(fallback, 1)] = blockIdx.x;
        return;
    }
    fill_big_runs(om, s_nbig, s_big);
    for (int i = N + tid; i < g.Npad; i += blockDim.x) om[i] = 0xffffu;
    __syncthreads();
    store_omega(g, om, omega_slot(g, omega_out));
}

size_t k1_f32_bucket_g_smem_bytes(int N) { return 32768 * 4 + 4 * (size_t)((N + 31) >> 5) + 16; }

#define IMF_K1F(NK)                                                                                  \
    template __global__ void k1_f32_bucket<NK, false>(Geom, uint16_t*, int*, uint32_t*, long long,  \
                                                      unsigned long long);                          \
    template __global__ void k1_f32_bucket<NK, true>(Geom, uint16_t*, int*, uint32_t*, long long,   \
                                                     unsigned long long);
IMF_K1F(1)
IMF_K1F(2)
IMF_K1F(3)
IMF_K1F(4)
IMF_K1F(5)
IMF_K1F(6)
#undef IMF_K1F

size_t k1_f32_bucket_smem_bytes(int N) {
    return 32768 * 4 + 4 * (size_t)((N + 3) & ~3) + 4 * (size_t)((N + 31) >> 5) + 16;
}

template __global__ void k1_count<DT_U8>(Geom, uint16_t*);
template __global__ void k1_count<DT_U16>(Geom, uint16_t*);

size_t k1_count_smem_bytes(int dtype, int Npad) {
    return (dtype == DT_U8 ? 128 * 4 : 32768 * 4) + 2 * (size_t)Npad;
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
