// imf_common.cuh -- shared device definitions for the B200 rank-order filter.
//
// Layout vocabulary:
//   tile      one T_w x T_h block of output pixels of one channel of one image;
//             it reads an input tile of S_w x S_h = (T_w+2r) x (T_h+2r) pixels,
//             coordinates clamped to the image (replicate == np.pad "edge",
//             tiling.py:134-140) or shifted by r (valid mode, tiling.py:102-105).
//   key       u32 order key of a pixel: the value for u8/u16, the float order key
//             for f32 (ordinal.py:109-123) -- no float compare ever runs on device.
//   omega     the rank -> position map (the paper's omnigram), u16 per rank,
//             packed x | y << 8 (ordinal.py:56-59); S_w, S_h <= 255.
//   I         the ordinal image: I[y*S_w + x] = rank of input-tile pixel (x, y)
//             (rank >> 1 in the pair kernel's halved mode, compared only
//             against even pivots).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace imf {

enum Dtype : int { DT_U8 = 0, DT_U16 = 1, DT_F32 = 2 };

constexpr int OMEGA_SLOT_PAD = 8;  // sentinel (0xffff) entries around each tile's omega

struct Geom {
    const void* src;
    void* dst;
    int dtype;
    int B, H, W, C;
    long long s_b, s_y, s_x, s_c;  // source strides, elements
    long long d_b, d_y, d_x, d_c;  // destination strides, elements
    int out_h, out_w;              // out_h: exclusive end of the output rows this launch writes
    int oy_base;                   // first output row of this launch (row stripe)
    int vshift;                    // r in valid mode, 0 in replicate mode
    int r;
    int Tw, Th, Sw, Sh, N, Npad;   // N: ranked pixels per tile; Npad: N rounded up to a multiple of 64
    int fp;                        // only footprint pixels are ranked (fprow)
    const uint32_t* fprow;         // footprint rows: input-tile row y ranks columns [lo, hi], lo | hi << 16
                                   // (lo > hi: none); device memory (workspace), nullptr = whole tile
    int tma_bw;                    // K1 TMA box width (elements per box row) when the launch uses TMA
    int k1_bulk;                   // k1_count_reg copies omega out with one bulk async copy (IMF_K1_BULK)
    int nrt;                       // f32 bucket K1: chunk tiles with replicate runs (the costly ones),
    int rt[16];                    //   run first: chunk-relative indices, ascending (chunk_tile)
    int nrr;                       // K2: chunk-relative tile ranges to run first (bottom image-border
    int rr_lo[4], rr_len[4];       //   tile rows: clamped margins make their walks long), ascending
    int run_min;                   // bucket K1: copy groups (replicate boundary) this large rank as one run
    const uint32_t* ctab_g;        // f32 bucket K1: call-wide fine-bucket table (k_coarse_*), or nullptr
    int tiles_x, tiles_y;
    long long tile_begin;          // first tile of this launch (chunking)
    unsigned mx, my, mc;           // division magics: n / d == (n * m) >> s for n < 2^31 (host: set_magic)
    int sx, sy, sc;
};

// Kernel offset tables, passed by value as a __grid_constant__ kernel parameter
// (constant bank): every thread of a warp reads the same entry in the same
// iteration, so the tables are uniform-datapath loads, not shared-memory traffic.
constexpr int KTAB_MAX = 249;  // 2*124 + 1 rows / columns
struct KTab {
    int2 v[KTAB_MAX];    // per kernel column: ((ybot+1)*Sw + dx, ytop*Sw + dx)  (down-slide enter, exit)
    int2 h[KTAB_MAX];    // per kernel row:    (dy*Sw + xhi, dy*Sw + xlo)          (right-slide enter, exit)
    int span[KTAB_MAX];  // per dy + r: (xlo & 0xffff) | (xhi - xlo) << 16
};

struct TileCoord {
    int b, c, ty, tx;
    int oy0, ox0;                  // output origin of the tile
    const char* src;               // image (b, c) base
};

struct SelParams {
    int circle;          // 1: arithmetic circle test (kernels.py:70-71); 0: span table
    int R2;              // r*(r+1): 4(dx^2+dy^2) <= (2r+1)^2  <=>  dx^2+dy^2 <= r(r+1)
    int ncols, nrows;
    int target;          // scalar target rank (tiling.py:176-177 / kernels.py:191-192)
    const int* tmap;     // per-pixel target ranks [out_h*out_w] or nullptr
    int G;               // seed rows per tile
    int* status;         // device status word (1 = scan defect)
    int debug_defect;    // test hook (IMF_FLAG_DEBUG_DEFECT): corrupt one slide count in tile 0
};

// Chunk-relative tile of this CTA: the listed costly tiles (g.rt) first, then
// the rest in order (the b-th unlisted index: step over each listed index <= it).
__device__ __forceinline__ int chunk_tile(const Geom& g) {
    int b = blockIdx.x;
    if (b < g.nrt) return g.rt[b];
    b -= g.nrt;
    for (int i = 0; i < g.nrt; i++)
        if (g.rt[i] <= b) b++;
    return b;
}

// K2's chunk-relative tile of this CTA: the listed ranges first (in order),
// then the remaining tiles in order.
__device__ __forceinline__ int chunk_tile_ranges(const Geom& g) {
    int b = blockIdx.x;
    for (int i = 0; i < g.nrr; i++) {
        if (b < g.rr_len[i]) return g.rr_lo[i] + b;
        b -= g.rr_len[i];
    }
    for (int i = 0; i < g.nrr; i++)
        if (g.rr_lo[i] <= b) b += g.rr_len[i];
    return b;
}

__device__ __forceinline__ TileCoord tile_coord(const Geom& g, long long t64) {
    TileCoord tc;
    // tile indices fit 32 bits (<= 2^31 tiles per call); 32-bit unsigned
    // division is a few instructions, the 64-bit one a ~100-instruction call
    // Enumeration: channel fastest, then tile column, tile row, image -- the
    // channels of one (interleaved) tile are neighbours (they read the same
    // bytes), and consecutive tile indices walk DOWN the image, which lets the
    // host pipeline gate chunks on the input rows uploaded so far.
    unsigned t = (unsigned)t64;
    const unsigned tx = (unsigned)g.tiles_x, ty = (unsigned)g.tiles_y, C = (unsigned)g.C;
    unsigned q = (unsigned)(((unsigned long long)t * g.mc) >> g.sc);  // t / C (exact for t < 2^31)
    tc.c = (int)(t - q * C);
    t = q;
    q = (unsigned)(((unsigned long long)t * g.mx) >> g.sx);
    tc.tx = (int)(t - q * tx);
    t = q;
    q = (unsigned)(((unsigned long long)t * g.my) >> g.sy);
    tc.ty = (int)(t - q * ty);
    tc.b = (int)q;
    // The last tile of a row / column is shifted back to end at the image edge
    // (overlapping its neighbour; both write identical values) instead of
    // hanging past it: windows far into the clamped margin are all ties and
    // cost the refine far more than the overlap does.
    tc.oy0 = g.oy_base + min(tc.ty * g.Th, max(g.out_h - g.oy_base - g.Th, 0));
    tc.ox0 = min(tc.tx * g.Tw, max(g.out_w - g.Tw, 0));
    int esz = g.dtype == DT_U8 ? 1 : (g.dtype == DT_U16 ? 2 : 4);
    tc.src = (const char*)g.src + (tc.b * g.s_b + tc.c * g.s_c) * esz;
    return tc;
}

// tile_coord computed once per CTA (thread 0) and broadcast through shared
// memory: its magic-number divisions cost every warp ~40 instructions
// otherwise.  Block-wide barrier: call from every thread, before any other
// barrier-dependent work.
__device__ __forceinline__ TileCoord tile_coord_cta(const Geom& g, long long t64) {
    __shared__ TileCoord s_tc;
    if (threadIdx.x == 0) s_tc = tile_coord(g, t64);
    __syncthreads();
    return s_tc;
}

// Image coordinates of input-tile pixel (ly, lx), clamped to the image.
__device__ __forceinline__ long long src_offset(const Geom& g, const TileCoord& tc, int ly, int lx) {
    int y = tc.oy0 + ly - g.r + g.vshift;
    int x = tc.ox0 + lx - g.r + g.vshift;
    y = y < 0 ? 0 : (y >= g.H ? g.H - 1 : y);
    x = x < 0 ? 0 : (x >= g.W ? g.W - 1 : x);
    return (long long)y * g.s_y + (long long)x * g.s_x;
}

// Tile footprint (tiling.py:148-162 _footprint_mask is the
// CPU analog): the input-tile pixels some window of the tile contains, i.e. the
// Minkowski sum of the output rectangle and the kernel.  Convex kernels give
// one column interval per input-tile row, the host's g.fprow table.  Pixels
// outside are never ranked: omega is shorter and denser (output-neutral: they
// belong to no window).
__device__ __forceinline__ bool in_footprint(const uint32_t* fprow, int x, int y) {
    if (!fprow) return true;
    const uint32_t v = __ldg(fprow + y);  // empty row: lo = hi = 0xffff (no x < 256 matches)
    const int lo = (int)(v & 0xffffu);
    return (unsigned)(x - lo) <= (unsigned)((int)(v >> 16) - lo);
}

// Footprint pixels of the rectangle [x0, x0 + cx) x [y0, y0 + cy).
__device__ __forceinline__ int fp_rect_count(const uint32_t* fprow, int x0, int cx, int y0, int cy) {
    if (!fprow) return cx * cy;
    int n = 0;
    for (int y = y0; y < y0 + cy; y++) {
        const uint32_t v = __ldg(fprow + y);
        n += max(0, min((int)(v >> 16), x0 + cx - 1) - max((int)(v & 0xffffu), x0) + 1);
    }
    return n;
}

__device__ __forceinline__ uint32_t float_key(uint32_t u) {
    // ordinal.py:120: (u >> 31) ? ~u : u | 0x80000000
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// u32 order key of f32 image pixel (yy, xx) (clamped image coordinates): the
// float key (ordinal.py:109-123).
__device__ __forceinline__ uint32_t f32_key(const Geom& g, const TileCoord& tc, int yy, int xx) {
    if (g.dtype == DT_U16)  // bucket transform on u16 tiles: the value in the high half
        return (uint32_t)__ldg((const uint16_t*)tc.src + (long long)yy * g.s_y + (long long)xx * g.s_x) << 16;
    return float_key(__ldg((const uint32_t*)tc.src + (long long)yy * g.s_y + (long long)xx * g.s_x));
}

__device__ __forceinline__ uint32_t load_key(const Geom& g, const TileCoord& tc, int ly, int lx) {
    if (g.dtype == DT_F32) {
        int y = tc.oy0 + ly - g.r + g.vshift, x = tc.ox0 + lx - g.r + g.vshift;
        y = y < 0 ? 0 : (y >= g.H ? g.H - 1 : y);
        x = x < 0 ? 0 : (x >= g.W ? g.W - 1 : x);
        return f32_key(g, tc, y, x);
    }
    long long o = src_offset(g, tc, ly, lx);
    if (g.dtype == DT_U8) return __ldg((const uint8_t*)tc.src + o);
    return __ldg((const uint16_t*)tc.src + o);
}

// y = i / Sw, x = i % Sw for i < 65536, Sw <= 256, via an exact float reciprocal
// ((i + 0.5)/Sw sits >= 1/512 away from an integer; float error < 2^-15).
__device__ __forceinline__ void lin_to_xy(int i, int Sw, float invS, int& x, int& y) {
    y = __float2int_rz(((float)i + 0.5f) * invS);
    x = i - y * Sw;
}

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

}  // namespace imf
