// imf_grank.cu -- image-wide ranks of f32 order keys (sm_100a).
//
// A float tile's keys spread over the u32 key space so unevenly (exponent +
// top mantissa bits) that a tile-local bucket sort on the high 16 key bits
// meets buckets of hundreds of pixels at large radii.  Ranking every pixel of
// the plane once -- an LSD radix sort of (key, index) pairs over the rows the
// launch reads, 4 passes of 8-bit digits (stable block scatter: warp
// match_any + per-warp digit counters) -- replaces each key by its unique
// image rank; a tile's pixels then occupy distinct ranks and the bucket
// transform on the high 16 bits of (rank << shift) sees buckets of at most
// 2^(bits-16) pixels (<= 64 for a 4 Mpixel plane, ~1 per bucket per tile).
// Ties are broken by position; the order of equal keys is output-neutral.
#include "imf_common.cuh"

namespace imf {

constexpr int GR_THREADS = 1024;
constexpr int GR_ITEMS = 4;                                  // elements per thread
constexpr int GR_CH = GR_THREADS * GR_ITEMS;                 // elements per block
constexpr int GR_PER_WARP = GR_CH / (GR_THREADS / 32);       // 128 consecutive elements per warp

// keys / indices of rows [y0, y1) of plane (b, c), row-major, index = position in that range
__global__ void k_gr_keys(Geom g, int b, int c, int y0, int y1, uint32_t* __restrict__ keys,
                          uint32_t* __restrict__ idx) {
    const long long n = (long long)(y1 - y0) * g.W;
    const char* base = (const char*)g.src + (b * g.s_b + c * g.s_c) * 4;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
        const int y = y0 + (int)(e / g.W), x = (int)(e % g.W);
        keys[e] = float_key(__ldg((const uint32_t*)base + (long long)y * g.s_y + (long long)x * g.s_x));
        idx[e] = (uint32_t)e;
    }
}

// per-block digit histograms, digit-major: hist[d * nb + block]
__global__ void __launch_bounds__(GR_THREADS) k_gr_hist(const uint32_t* __restrict__ keys, int n, int shift,
                                                        uint32_t* __restrict__ hist) {
    __shared__ uint32_t h[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) h[i] = 0;
    __syncthreads();
    const int e0 = blockIdx.x * GR_CH;
    for (int i = threadIdx.x; i < GR_CH; i += blockDim.x)
        if (e0 + i < n) atomicAdd(&h[(keys[e0 + i] >> shift) & 0xffu], 1u);
    __syncthreads();
    for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[(long long)i * gridDim.x + blockIdx.x] = h[i];
}

// Exclusive scan of the digit-major block histograms in two levels: one CTA
// per digit scans that digit's row over the nb blocks (and writes the row
// total), then one CTA turns the 256 totals into digit bases.
__device__ __forceinline__ uint32_t block_excl_scan_1024(uint32_t v, uint32_t* wt, uint32_t& total) {
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += t;
    }
    if (lane == 31) wt[wid] = x;
    __syncthreads();
    if (wid == 0) {
        const uint32_t w = wt[lane];
        uint32_t y = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, y, o);
            if (lane >= o) y += t;
        }
        wt[lane] = y - w;
        if (lane == 31) wt[32] = y;
    }
    __syncthreads();
    total = wt[32];
    const uint32_t r = wt[wid] + x - v;
    __syncthreads();
    return r;
}

__global__ void __launch_bounds__(1024) k_gr_scan_rows(uint32_t* __restrict__ hist, int nb,
                                                       uint32_t* __restrict__ totals) {
    __shared__ uint32_t wt[33];
    uint32_t* row = hist + (long long)blockIdx.x * nb;
    uint32_t carry = 0;
    for (int base = 0; base < nb; base += 1024) {
        const int i = base + threadIdx.x;
        const uint32_t v = i < nb ? row[i] : 0u;
        uint32_t tot;
        const uint32_t ex = block_excl_scan_1024(v, wt, tot);
        if (i < nb) row[i] = carry + ex;
        carry += tot;
    }
    if (threadIdx.x == 0) totals[blockIdx.x] = carry;
}

__global__ void __launch_bounds__(1024) k_gr_scan_totals(uint32_t* __restrict__ totals) {
    __shared__ uint32_t wt[33];
    const uint32_t v = threadIdx.x < 256 ? totals[threadIdx.x] : 0u;
    uint32_t tot;
    const uint32_t ex = block_excl_scan_1024(v, wt, tot);
    if (threadIdx.x < 256) totals[threadIdx.x] = ex;
}

// stable scatter of one block's elements by digit
__global__ void __launch_bounds__(GR_THREADS) k_gr_scatter(const uint32_t* __restrict__ kin,
                                                           const uint32_t* __restrict__ iin,
                                                           uint32_t* __restrict__ kout, uint32_t* __restrict__ iout,
                                                           int n, int shift, const uint32_t* __restrict__ hist,
                                                           const uint32_t* __restrict__ dbase) {
    __shared__ uint32_t cnt[256][33];  // [digit][warp], padded row
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const unsigned lt = lanemask_lt();
    for (int i = tid; i < 256 * 33; i += blockDim.x) (&cnt[0][0])[i] = 0;
    __syncthreads();
    const int w0 = blockIdx.x * GR_CH + wid * GR_PER_WARP;
    // 1. per-warp digit counts
    for (int j = 0; j < GR_PER_WARP; j += 32) {
        const int e = w0 + j + lane;
        const bool ok = e < n;
        const uint32_t d = ok ? (kin[e] >> shift) & 0xffu : 0x100u + lane;
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        if (ok && lane == __ffs(peers) - 1) cnt[d][wid] += __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    // 2. per digit: global offset of this block + prefix over warps
    if (tid < 256) {
        uint32_t run = dbase[tid] + hist[(long long)tid * gridDim.x + blockIdx.x];
        for (int w = 0; w < 32; w++) {
            const uint32_t c = cnt[tid][w];
            cnt[tid][w] = run;
            run += c;
        }
    }
    __syncthreads();
    // 3. scatter in element order
    for (int j = 0; j < GR_PER_WARP; j += 32) {
        const int e = w0 + j + lane;
        const bool ok = e < n;
        const uint32_t key = ok ? kin[e] : 0u;
        const uint32_t d = ok ? (key >> shift) & 0xffu : 0x100u + lane;
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        uint32_t base = ok ? cnt[d][wid] : 0u;
        __syncwarp();
        if (ok) {
            const uint32_t pos = base + __popc(peers & lt);
            kout[pos] = key;
            iout[pos] = iin[e];
            if (lane == __ffs(peers) - 1) cnt[d][wid] = base + __popc(peers);
        }
        __syncwarp();
    }
}

__global__ void k_gr_final(const uint32_t* __restrict__ idx_sorted, int n, uint32_t* __restrict__ grank) {
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) grank[idx_sorted[p]] = (uint32_t)p;
}

// Host: ranks of plane (b, c) rows [y0, y1) into grank (n = (y1-y0)*W entries);
// scratch: 4 arrays of n u32 + 256 * ceil(n / GR_CH) u32.
inline size_t gr_scratch_words(long long n) { return 4 * (size_t)n + 256 * (size_t)((n + GR_CH - 1) / GR_CH) + 512; }

inline cudaError_t gr_rank_plane(const Geom& g, int b, int c, int y0, int y1, uint32_t* grank, uint32_t* scratch,
                                 cudaStream_t s) {
    const long long nl = (long long)(y1 - y0) * g.W;
    if (nl <= 0) return cudaSuccess;
    const int n = (int)nl;
    const int nb = (n + GR_CH - 1) / GR_CH;
    uint32_t* kA = scratch;
    uint32_t* kB = kA + n;
    uint32_t* iA = kB + n;
    uint32_t* iB = iA + n;
    uint32_t* hist = iB + n;
    uint32_t* dbase = hist + 256 * (size_t)nb;
    k_gr_keys<<<std::min(nb * 4, 4096), 1024, 0, s>>>(g, b, c, y0, y1, kA, iA);
    for (int pass = 0; pass < 4; pass++) {
        k_gr_hist<<<nb, GR_THREADS, 0, s>>>(kA, n, 8 * pass, hist);
        k_gr_scan_rows<<<256, 1024, 0, s>>>(hist, nb, dbase);
        k_gr_scan_totals<<<1, 1024, 0, s>>>(dbase);
        k_gr_scatter<<<nb, GR_THREADS, 0, s>>>(kA, iA, kB, iB, n, 8 * pass, hist, dbase);
        std::swap(kA, kB);
        std::swap(iA, iB);
    }
    k_gr_final<<<std::min(nb * 4, 4096), 1024, 0, s>>>(iA, n, grank);
    return cudaGetLastError();
}

}  // namespace imf
