// imf_api.cu -- extern "C" entry points (include/isomedian_b200.h) and the
// launch planner: tile geometry, quantization of the ordinal image, chunking
// of the tile stream through an L2-sized omega scratch, K1/K2 launches.
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <mutex>
#include <cstdlib>
#include <cstring>
#include <string>
#include <utility>
#include <vector>

#include "../../include/isomedian_b200.h"
#include "imf_kernels.cuh"


using namespace imf;

static std::atomic<uint64_t> g_launches{0};
static thread_local char g_err[256];

struct ProfileRec {
    float sort_ms = 0.f, select_ms = 0.f;
    int launches = 0;
    long long tiles = 0, chunk = 0;
    int tile = 0, qs = 0;
};
static thread_local ProfileRec g_prof;
static thread_local bool g_last_tma = false;  // the last call's K1 loaded its tiles with TMA (diagnostic)

static int cuda_fail(cudaError_t e, const char* where) {
    snprintf(g_err, sizeof(g_err), "%s: %s", where, cudaGetErrorString(e));
    return IMF_ERR_CUDA;
}

namespace {

constexpr size_t kOptinSmem = 227 * 1024;       // B200 opt-in shared memory per block (232448 B)
constexpr size_t kSmemMax = kOptinSmem - 1024;  // dynamic budget of kernels with <= 1 KB static smem
// Static shared memory each K1 family declares (the kernel's own __shared__
// variables; cuobjdump's SHARED also counts the 1 KB system reserve), rounded
// up: a launch needs dynamic + static <= kOptinSmem.  tests/test_plan.py checks
// the built kernels stay within these.
constexpr size_t kStaticK1Sort = 2048, kStaticK1Bucket = 4096;
constexpr int kK1Threads = 1024;      // k1_count (latency-bound: more warps)
constexpr int kK1SortThreads = 512;   // k1_sort (per-warp digit counters)
constexpr size_t kStatusBytes = 2048;    // status word at 0, footprint row table at kFpOffset
constexpr size_t kFpOffset = 256;        // 256 rows x 4 B
constexpr size_t kOmegaScratchTarget = 96ull << 20;  // stays mostly L2-resident

struct Plan {
    Geom g;
    int G, k2_threads, k1_threads;
    bool k1_gmem, k1_count, omg;
    bool k1_f32b;         // f32 bucket ordinal transform (+ k1_sort fallback on flagged tiles)
    bool k1_f32b_g;       // ... with the bucket entries in a global scratch slot per tile
    size_t k1b_smem;
    bool k1_count_g;  // u16, S > ~180: counting sort scattering omega to global memory
    int full_out_h;
    bool direct;  // k_direct: per-pixel register sort (window area <= 32)
    int hs;     // k2_pair: ordinal image holds rank >> hs
    bool pair;  // K2 fast path (imf_pair.cu): two windows per thread, 15-bit ranks
    size_t k1_smem, k2_smem, k1_gs_per_tile;
    long long total_tiles, chunk_tiles;
    size_t ws_omega, ws_k1g, ws_flags, ws_lane, ws_ctab, ws_total;
    int ct_y0, ct_y1;  // rows of every plane the call reads (call-wide coarse table)
    int lanes;  // chunk streams (1 or 2)
    uint32_t fprow[256];  // footprint rows (g.fp): lo | hi << 16 per input-tile row
    bool k1_tma;          // k1_count_reg loads its tile box with TMA (planar layouts)
};

int env_int(const char* name, int dflt) {
    const char* v = getenv(name);
    return v && *v ? atoi(v) : dflt;
}

int dtype_size(int dt) { return dt == IMF_DTYPE_U8 ? 1 : (dt == IMF_DTYPE_U16 ? 2 : 4); }

// Round-up multiplicative inverse for unsigned division by d of n < 2^31:
// n / d == (n * m) >> (31 + l) with l = ceil(log2 d), m = ceil(2^(31+l) / d)
// (m <= 2^32 - 1 for d >= 2; m = 2^31 for d = 1; the error term stays < 1/d).
void set_magic(unsigned d, unsigned& m, int& s) {
    int l = 0;
    while ((1ull << l) < d) l++;
    s = 31 + l;
    m = (unsigned)(((1ull << (31 + l)) + d - 1) / d);
}

// Tile geometry: output tile side T (input side S = T + 2r <= 255 so ranks,
// positions and 16-bit histogram counters fit), seed rows G, and whether omega
// stays in global memory (OMG).  Among feasible shapes pick the one with the
// most output pixels per sorted input pixel (T^2 / S^2, the sort amortization,
// SURVEY.md App. C), slightly preferring omega in shared memory.
int make_plan(const imf_image* src, const imf_kernel* k, const imf_options* opt, Plan* pl) {
    if (!src || !k || !opt) return IMF_ERR_INVALID;
    if (src->dtype < 0 || src->dtype > 2) return IMF_ERR_INVALID;
    const int r = k->radius;
    if (r < 0 || r > 124) return IMF_ERR_UNSUPPORTED;
    if (k->nrows < 1 || k->ncols < 1 || k->area < 1) return IMF_ERR_INVALID;
    const int H = src->height, W = src->width;
    if (src->batch < 1 || src->channels < 1 || H < 1 || W < 1) return IMF_ERR_INVALID;
    const int valid = opt->boundary == IMF_BOUNDARY_VALID;
    const int out_h = valid ? H - 2 * r : H, out_w = valid ? W - 2 * r : W;
    if (out_h < 1 || out_w < 1) return IMF_ERR_INVALID;
    const int row0 = opt->row_end > 0 ? opt->row_begin : 0;
    const int row1 = opt->row_end > 0 ? opt->row_end : out_h;
    if (row0 < 0 || row1 > out_h || row0 >= row1) return IMF_ERR_INVALID;

    Plan& p = *pl;
    memset(&p, 0, sizeof(p));
    // Default output tile 64 (sort amortization vs shared memory); 32 when the
    // window is tiny (r <= 4: walks through a 68^2 rank space are long) or when
    // 64-tiles would not give the GPU two CTAs per SM (small images).
    int tdef = env_int("IMF_TILE", 0);
    if (tdef <= 0) {
        const long long planes = (long long)src->batch * src->channels;
        const long long t64 = planes * ((out_h + 63) / 64) * ((out_w + 63) / 64);
        tdef = (r <= 4 || t64 < 2 * 148) ? 32 : 64;
    }
    const int Tmax0 = std::max(1, std::min(opt->tile_size > 0 ? opt->tile_size : tdef, 255 - 2 * r));
    const int G0 = opt->seed_rows > 0 ? opt->seed_rows : env_int("IMF_SEED_ROWS", 4);
    // f32 tiles use the bucket ordinal transform when N <= 23,716 (S <= 154):
    // cap the tile at 154 - 2r while that keeps it >= 48 (r <= 53)
    int Tmax = Tmax0;
    if (src->dtype == IMF_DTYPE_F32 && env_int("IMF_F32_BUCKET", 1) && opt->tile_size <= 0) {
        const int tb = (154 - 2 * r) & ~1;  // S <= 154: hist + 4.125 N bytes fit
        if (tb >= 48) Tmax = std::min(Tmax, tb);
    }
    double best = -1.0;
    // Tiny windows (area <= 32, e.g. r <= 2): direct per-pixel selection, no ranks.
    if (k->area <= 32 && env_int("IMF_DIRECT", 1)) {
        p.direct = true;
        best = 1.0;
        p.g.Tw = p.g.Th = 32;
        p.g.Sw = p.g.Sh = 32 + 2 * r;
        p.g.N = p.g.Sw * p.g.Sh;
        p.g.Npad = (p.g.N + 63) & ~63;
        p.k2_threads = 1024;
        p.k2_smem = 4 * (size_t)p.g.N;
    }
    // K2 fast path: tile ranks < 2^15 (S <= 181), even T, and T + r <= 128 for
    // the packed circle test.  Largest such tile.
    // circles and squares have packed membership tests; other shapes (span
    // table per rank) are faster on the general path
    const bool packed_shape = k->shape_code == IMF_SHAPE_CIRCLE || k->shape_code == IMF_SHAPE_SQUARE ||
                              (k->shape_code == IMF_SHAPE_POLYGON && env_int("IMF_PAIR_POLY", 1));
    if (!p.direct && env_int("IMF_PAIR", 1) && (packed_shape || env_int("IMF_PAIR_ANY", 0))) {
        // columns: even, <= Tmax, packed circle test needs Tw + r <= 128; rows: the
        // tallest tile keeping N = Sw * Sh <= 32768 (ranks < 2^15), at most Tw
        // the packed byte tests need T + r <= 128; circles whose T would drop
        // below the default take a full tile with the wide test (SH_CIRCLEW)
        const bool wide = k->shape_code == IMF_SHAPE_CIRCLE && 128 - r < std::min(Tmax, 64) &&
                          env_int("IMF_PAIR_WIDE", 1);
        const bool packed_fit = packed_shape && !wide;
        int Tw = std::min(Tmax, 255 - 2 * r);
        if (packed_fit) Tw = std::min(Tw, 128 - r);
        Tw &= ~1;
        const int Sw = Tw + 2 * r;
        int Th = std::min(Tw, 65536 / std::max(Sw, 1) - 2 * r);
        if (packed_fit) Th = std::min(Th, 128 - r);
        // rectangular tiles (Th < Tw) measured slower than the generic path
        // (short sweeps, more seed rows per output row): square tiles only, and
        // no smaller than the default 64 (small tiles sort too much per output)
        const bool shape_ok = Tw >= (std::min(Tmax, 64) & ~1) &&
                              Th >= (env_int("IMF_PAIR_RECT", 0) ? std::max(2, Tw / 4) : Tw);
        if (Tw >= 2 && shape_ok) {
            const int Sh = Th + 2 * r;
            const int N = Sw * Sh, Npad = (N + 63) & ~63;
            int G = std::max(1, std::min(opt->seed_rows > 0 ? opt->seed_rows : env_int("IMF_SEED_ROWS", 8), Th));
            const int tpg = 2 * (((Tw >> 1) + 31) & ~31);  // threads per seed-row group: 2 dirs x pairs (whole warps)
            while (G > 1 && ((G * tpg + 31) & ~31) > 512) G--;
            // omega in L2 when omega + I would leave room for only one CTA per SM
            const int forced = env_int("IMF_PAIR_OMG", -1);
            bool pomg = forced >= 0 ? forced != 0
                                    : k2_pair_smem_bytes(N, Npad, N, r, G, Tw, Th, false) > 113 * 1024;
            const size_t ks = k2_pair_smem_bytes(N, Npad, N, r, G, Tw, Th, pomg);
            if (N <= 65536 && ((G * tpg + 31) & ~31) <= 512 && ks <= kSmemMax && k->ncols <= PT_MAX &&
                k->nrows <= PT_MAX) {
                best = 1.0;
                p.pair = true;
                p.hs = N > 32768 ? 1 : 0;  // ranks >= 2^15: halved ordinal image, even pivots
                p.g.Tw = Tw;
                p.g.Th = Th;
                p.g.Sw = Sw;
                p.g.Sh = Sh;
                p.g.N = N;
                p.g.Npad = Npad;
                p.G = G;
                p.k2_threads = std::max((G * tpg + 31) & ~31, 64);  // whole warps (phase A/B ballots)
                p.k2_smem = ks;
                p.omg = pomg;
            }
        }
    }
    for (int T = Tmax; T >= 1 && !p.pair && !p.direct; T--) {
        const int S = T + 2 * r;
        const int N = S * S, Npad = (N + 63) & ~63;
        const int G = std::max(1, std::min(G0, T));
        const int thr = std::min(((T * G * 2 + 31) / 32) * 32, 512);
        for (int omg = 0; omg < 2; omg++) {
            const size_t k2s = k2_smem_bytes(N, Npad, k->ncols, k->nrows, r, G, T, T, omg != 0);
            if (k2s > kSmemMax) continue;
            const double score = (double)T * T / ((double)S * S) * (omg ? 0.9 : 1.0);
            if (score > best) {
                best = score;
                p.g.Tw = p.g.Th = T;
                p.g.Sw = p.g.Sh = S;
                p.g.N = N;
                p.g.Npad = Npad;
                p.G = G;
                p.k2_threads = thr;
                p.k2_smem = k2s;
                p.omg = omg != 0;
            }
        }
        if (best > 0 && T * 2 < Tmax) break;  // smaller tiles only lose amortization
    }
    if (best < 0) return IMF_ERR_UNSUPPORTED;
    Geom& g = p.g;
    g.dtype = src->dtype;
    g.B = src->batch;
    g.H = H;
    g.W = W;
    g.C = src->channels;
    g.s_b = src->stride_b;
    g.s_y = src->stride_y;
    g.s_x = src->stride_x;
    g.s_c = src->stride_c;
    g.out_h = row1;
    g.oy_base = row0;
    g.out_w = out_w;
    g.vshift = valid ? r : 0;
    g.r = r;
    g.tiles_x = (out_w + g.Tw - 1) / g.Tw;
    g.tiles_y = (row1 - row0 + g.Th - 1) / g.Th;
    p.full_out_h = out_h;
    p.total_tiles = (long long)g.tiles_x * g.tiles_y * g.C * g.B;
    set_magic((unsigned)g.tiles_x, g.mx, g.sx);
    set_magic((unsigned)g.tiles_y, g.my, g.sy);
    set_magic((unsigned)g.C, g.mc, g.sc);
    if (p.total_tiles >= (1ll << 31)) return IMF_ERR_UNSUPPORTED;  // tile_coord uses 32-bit indices

    g.run_min = std::max(kRunMinFloor, env_int("IMF_RUNMIN", kRunMin));
    // K1 variant and its memory for the ranked pixels per tile g.N (chosen
    // again once a footprint shrinks N)
    auto choose_k1 = [&]() {
        p.k1_f32b_g = false;
        const size_t k1s_max = kOptinSmem - kStaticK1Sort;
        p.k1_count = g.dtype != DT_F32 && k1_count_smem_bytes(g.dtype, g.Npad) <= kSmemMax;
        p.k1b_smem = k1_f32_bucket_smem_bytes(g.N);
        p.k1_f32b = g.dtype == DT_F32 && env_int("IMF_F32_BUCKET", 1) && g.Sw <= 160 &&
                    p.k1b_smem <= kOptinSmem - kStaticK1Bucket;
        // f32 tiles beyond shared-memory entries, and u16 tiles beyond the 64K-bin
        // counting sort (S > ~180): the bucket transform with global entries
        // (u16 keys v << 16: every bucket is one value, ties only)
        // u16 tiles beyond it: the counting sort with omega in global memory
        p.k1_count_g = g.dtype == DT_U16 && !p.k1_count && env_int("IMF_K1_COUNT_G", 1);
        if ((g.dtype == DT_F32 || (g.dtype == DT_U16 && !p.k1_count && !p.k1_count_g)) && !p.k1_f32b &&
            env_int("IMF_F32_BUCKET", 1)) {
            p.k1_f32b = p.k1_f32b_g = true;
            p.k1b_smem = k1_f32_bucket_g_smem_bytes(g.N);
        }
        p.k1_threads = p.k1_count ? kK1Threads : kK1SortThreads;
        p.k1_gmem = !p.k1_count && k1_smem_bytes(g.dtype, g.Npad, p.k1_threads / 32, false) > k1s_max;
        p.k1_smem = p.k1_count ? k1_count_smem_bytes(g.dtype, g.Npad)
                               : k1_smem_bytes(g.dtype, g.Npad, p.k1_threads / 32, p.k1_gmem);
        p.k1_gs_per_tile = (p.k1_gmem && !p.k1_count_g) ? k1_gscratch_bytes(g.dtype, g.Npad) : 0;
        // the global-entries bucket kernels need 6 B per pixel (entries + run
        // descriptors); the LSD fallback reuses the same slot (k1_gscratch_bytes(f32)
        // = 6 B per pixel when it needs one)
        if (p.k1_f32b_g) p.k1_gs_per_tile = std::max(p.k1_gs_per_tile, (size_t)6 * g.Npad);  // + run descriptors
        // k1_f32_bucket<NK <= 6, global entries>: interior tiles keep 16-bit entries
        // in shared memory after the coarse table (imf_sort.cu OWN16)
        if (p.k1_f32b_g && ((g.Sw + 31) >> 5) <= 6) p.k1b_smem += 2 * (size_t)g.Npad + 16;
    };
    choose_k1();

    // Tile footprint (pair path; register-resident u8/u16 K1 or the f32 bucket
    // transform and its LSD fallback): rank only the input
    // pixels some window of the tile contains -- the Minkowski sum of the
    // output rectangle and the kernel (tiling.py:148-162 _footprint_mask,
    // PAPER.md:283,294): per input-tile row y, kernel rows dy whose window
    // centre row y - dy lies in the tile contribute columns [r + xlo, r + Tw - 1
    // + xhi - 1] (convex kernels: the union is one interval).  Circles give the
    // rounded rectangle (c2: 25,600 -> 23,616 pixels); squares the whole tile.
    const bool k1reg = p.k1_count && ((g.Sw + 31) >> 5) <= 6 && env_int("IMF_K1REG", 1) &&
                       (long long)(g.H - 1) * g.s_y + (long long)(g.W - 1) * g.s_x < (1ll << 31);
    // f32: the footprint pays on the shared-entry bucket kernel (S <= 160:
    // c3 r=32 / 48 -2 / -3 %) and the global-entries kernel (S > 192: r=100
    // -7 %), not on the 16-bit-entry kernel in between (161..192, r=64: its
    // register spills cost K1 more than the 10 % fewer pixels save; path
    // +13 %).  IMF_F32_FOOTPRINT: 0 never, 1 auto, 2 always.
    // (decided on the tile size, not on the whole-tile K1 choice above: the
    // footprint can bring a tile back under the shared-entry kernel's limit)
    const int f32fp = env_int("IMF_F32_FOOTPRINT", 1);
    const bool own16 = g.Sw > 160 && ((g.Sw + 31) >> 5) <= 6;
    const bool fp_k1 = k1reg || (g.dtype == DT_F32 && env_int("IMF_F32_BUCKET", 1) &&
                                 (f32fp == 2 || (f32fp == 1 && !own16)));
    if (p.pair && k->shape_code != IMF_SHAPE_SQUARE && fp_k1 && g.Sh <= 256 && env_int("IMF_FOOTPRINT", 1)) {
        // the table depends on the kernel's row spans and the tile geometry only:
        // memoized per thread (the host pipeline plans every stripe of a frame)
        uint64_t h = 1469598103934665603ull;
        auto mix = [&](uint64_t v) { h = (h ^ v) * 1099511628211ull; };
        mix((uint64_t)r | (uint64_t)g.Tw << 16 | (uint64_t)g.Th << 32 | (uint64_t)g.Sw << 48);
        mix((uint64_t)g.Sh | (uint64_t)k->nrows << 16);
        for (int i = 0; i < k->nrows; i++)
            mix((uint64_t)(uint32_t)k->row_dy[i] | (uint64_t)(uint16_t)k->row_xlo[i] << 32 |
                (uint64_t)(uint16_t)k->row_xhi[i] << 48);
        static thread_local uint64_t fp_key = 0;
        static thread_local int fp_n = 0;
        static thread_local uint32_t fp_rows[256];
        int nfp = 0;
        if (fp_key == h && h != 0) {
            memcpy(p.fprow, fp_rows, sizeof(fp_rows));
            nfp = fp_n;
        } else {
            for (int y = 0; y < g.Sh; y++) {
                int lo = 1 << 30, hi = -1;
                for (int i = 0; i < k->nrows; i++) {
                    const int cy = y - k->row_dy[i];  // window centre row (input-tile coordinates)
                    if (cy < r || cy > r + g.Th - 1 || k->row_xhi[i] <= k->row_xlo[i]) continue;
                    lo = std::min(lo, r + k->row_xlo[i]);
                    hi = std::max(hi, r + g.Tw - 1 + k->row_xhi[i] - 1);
                }
                lo = std::max(lo, 0);
                hi = std::min(hi, g.Sw - 1);
                if (lo > hi) {
                    p.fprow[y] = 0xffffffffu;  // lo = hi = 65535: no pixel of this row
                    continue;
                }
                p.fprow[y] = (uint32_t)lo | ((uint32_t)hi << 16);
                nfp += hi - lo + 1;
            }
            memcpy(fp_rows, p.fprow, sizeof(fp_rows));
            fp_n = nfp;
            fp_key = h;
        }
        const int NI = g.Sw * g.Sh;
        g.fp = 1;
        g.N = nfp;
        g.Npad = (nfp + 63) & ~63;
        p.hs = nfp > 32768 ? 1 : 0;
        const int forced = env_int("IMF_PAIR_OMG", -1);
        const bool pomg = forced >= 0 ? forced != 0
                                      : k2_pair_smem_bytes(g.N, g.Npad, NI, r, p.G, g.Tw, g.Th, false) > 113 * 1024;
        p.omg = pomg;
        p.k2_smem = k2_pair_smem_bytes(g.N, g.Npad, NI, r, p.G, g.Tw, g.Th, pomg);
        choose_k1();
    }

    // K1 tile loads through TMA when the plane is pixel-contiguous (s_x == 1):
    // one 2D box (Sw x Sh, width rounded to 16 B) per tile into the omega area
    // (imf_count.cu).  Interleaved channels keep the per-lane loads.
    {
        const int esz = dtype_size(g.dtype);
        p.k1_tma = k1reg && g.dtype != DT_F32 && g.s_x == 1 && env_int("IMF_TMA", 1) &&
                   ((long long)g.s_y * esz) % 16 == 0 && (g.C == 1 || ((long long)g.s_c * esz) % 16 == 0) &&
                   (g.B == 1 || ((long long)g.s_b * esz) % 16 == 0);
        if (p.k1_tma) {
            const int q = 16 / esz;  // box starts 16-byte aligned: up to q - 1 extra columns on the left
            g.tma_bw = (g.Sw + q - 1 + q - 1) / q * q;
            p.k1_smem = std::max(p.k1_smem, k1_count_smem_bytes(g.dtype, 0) + (size_t)g.tma_bw * g.Sh * esz);
        }
    }
    g.k1_bulk = env_int("IMF_K1_BULK", 1);
    const size_t slot = 2 * (size_t)(g.Npad + 2 * OMEGA_SLOT_PAD);
    const size_t per_tile = slot + p.k1_gs_per_tile;
    // Two lanes (streams) alternate chunks when there are enough tiles: each
    // lane's K1 fills the other's K2 tail.  The omega scratch target is split
    // between them; each lane has its own scratch, k1 scratch and flag list.
    // Chunks below ~2 full K2 waves (2 x 296 CTAs) leave the GPU idle, so two
    // lanes only when there are >= 4 such chunks' worth of tiles.
    // (The f32 global-entries transform is K1-bound: its chunks overlap even
    // when small.)
    const long long min_chunk = p.k1_f32b_g ? 296 : 592;
    p.lanes = (p.total_tiles >= (p.k1_f32b_g ? 2 : 3) * min_chunk && env_int("IMF_LANES", 2) > 1) ? 2 : 1;
    // the L2 budget counts the omega slots only (they carry K1's result to K2);
    // K1's private scratch (entries) is written and read back within one CTA
    const size_t l2_per_tile = env_int("IMF_CHUNK_OMEGA_ONLY", 1) ? slot : per_tile;
    const size_t target = (size_t)env_int("IMF_SCRATCH_MB", (int)(kOmegaScratchTarget >> 20)) << 20;
    long long chunk = (long long)(target / p.lanes / l2_per_tile);
    if (p.lanes == 2) {
        const int nch = std::max(2, env_int("IMF_CHUNKS", 4));
        chunk = std::min<long long>(chunk, std::max<long long>(min_chunk, (p.total_tiles + nch - 1) / nch));
        chunk = std::max<long long>(148, chunk / 148 * 148);  // whole waves of one-CTA-per-SM K1
    }
    chunk = std::max<long long>(chunk, 148);
    chunk = std::min<long long>(chunk, p.total_tiles);
    chunk = std::min<long long>(chunk, 65535LL * 1024);
    p.chunk_tiles = chunk;
    p.ws_omega = (((size_t)chunk * slot) + 255) & ~(size_t)255;
    p.ws_k1g = (size_t)chunk * p.k1_gs_per_tile;
    p.ws_flags = p.k1_f32b ? (((size_t)(chunk + 1) * 4 + 255) & ~(size_t)255) : 0;
    p.ws_lane = p.ws_omega + p.ws_k1g + p.ws_flags;
    // f32 adaptive buckets on the largest tiles (global entries, N > 40K):
    // one call-wide coarse table instead of a coarse pass per tile.  The
    // pre-pass over the image is serial; below ~40K-pixel tiles it costs more
    // than the tiles' coarse passes (c3 r64: +6 %, r100: -4 %).  IMF_GCOARSE:
    // 0 off, 1 auto, 2 for every adaptive tile.
    p.ws_ctab = 0;
    const int gco = env_int("IMF_GCOARSE", 1);
    if (g.dtype == DT_F32 && p.k1_f32b && g.N > kAdaptiveMinN && (gco == 2 || (gco == 1 && g.N > 40000))) {
        p.ct_y0 = std::max(0, std::min(H, g.oy_base - r + g.vshift));
        p.ct_y1 = std::max(p.ct_y0, std::min(H, g.out_h + r + g.vshift));
        p.ws_ctab = 4 * (size_t)kCoarse;
    }
    p.ws_total = kStatusBytes + p.lanes * p.ws_lane + p.ws_ctab;
    return IMF_OK;
}

void build_ktab_struct(const imf_kernel* k, int Sw, KTab& t) {
    memset(&t, 0, sizeof(t));
    const int r = k->radius;
    // byte offsets into the 16-bit ordinal image
    for (int i = 0; i < k->ncols; i++)
        t.v[i] = make_int2(2 * ((k->col_ybot[i] + 1) * Sw + k->col_dx[i]),
                           2 * (k->col_ytop[i] * Sw + k->col_dx[i]));
    for (int i = 0; i < k->nrows; i++) {
        t.h[i] = make_int2(2 * (k->row_dy[i] * Sw + k->row_xhi[i]), 2 * (k->row_dy[i] * Sw + k->row_xlo[i]));
        t.span[k->row_dy[i] + r] = (k->row_xlo[i] & 0xffff) | ((k->row_xhi[i] - k->row_xlo[i]) << 16);
    }
}


// cudaFuncSetAttribute (the >48 KB shared-memory opt-in) is per device:
// one bit per device ordinal, set once under a mutex.
constexpr int kMaxDev = 64;
std::atomic<uint64_t> g_attr_mask{0};
std::mutex g_attr_mu;

template <typename F>
cudaError_t allow_smem(F* f, int optin) {
    cudaFuncAttributes a;
    cudaError_t e = cudaFuncGetAttributes(&a, f);
    if (e) return e;
    return cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                optin - (int)a.sharedSizeBytes);
}

// Kernel rows symmetric in x (xlo = -(xhi - 1), xhi exclusive) and in y (rows dy
// and -dy alike): the pair kernel's SH_POLYSYM membership test applies.
bool kernel_symmetric(const imf_kernel* k) {
    const int r = k->radius;
    if (r > 127 || k->nrows > 2 * r + 1) return false;
    std::vector<int> w(2 * r + 1, 0);
    for (int i = 0; i < k->nrows; i++) {
        const int dy = k->row_dy[i];
        if (dy < -r || dy > r || k->row_xlo[i] != 1 - k->row_xhi[i]) return false;
        w[dy + r] = k->row_xhi[i] - k->row_xlo[i];
    }
    for (int dy = 0; dy <= r; dy++)
        if (w[r + dy] != w[r - dy]) return false;
    return true;
}

cudaError_t set_attrs() {
    int dev = 0, optin = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e) return e;
    if (dev >= kMaxDev) return cudaErrorInvalidDevice;
    const uint64_t bit = 1ull << dev;
    if (g_attr_mask.load(std::memory_order_acquire) & bit) return cudaSuccess;
    std::lock_guard<std::mutex> lk(g_attr_mu);
    if (g_attr_mask.load(std::memory_order_relaxed) & bit) return cudaSuccess;
    e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (!e) e = allow_smem(k1_sort<DT_U8, false>, optin);
    if (!e) e = allow_smem(k1_sort<DT_U16, false>, optin);
    if (!e) e = allow_smem(k1_sort<DT_U16, true>, optin);
    if (!e) e = allow_smem(k1_sort<DT_F32, false>, optin);
    if (!e) e = allow_smem(k1_sort<DT_F32, true>, optin);
    if (!e) e = allow_smem(k1_count<DT_U8>, optin);
    if (!e) e = allow_smem(k1_count<DT_U16>, optin);
    if (!e) e = allow_smem(k1_count_g, optin);
#define IMF_K1R_ATTR(DT, TMA)                                                     \
    if (!e) e = allow_smem(k1_count_reg<DT, 1, TMA>, optin);                     \
    if (!e) e = allow_smem(k1_count_reg<DT, 2, TMA>, optin);                     \
    if (!e) e = allow_smem(k1_count_reg<DT, 3, TMA>, optin);                     \
    if (!e) e = allow_smem(k1_count_reg<DT, 4, TMA>, optin);                     \
    if (!e) e = allow_smem(k1_count_reg<DT, 5, TMA>, optin);                     \
    if (!e) e = allow_smem(k1_count_reg<DT, 6, TMA>, optin);
    IMF_K1R_ATTR(DT_U8, false)
    IMF_K1R_ATTR(DT_U16, false)
    IMF_K1R_ATTR(DT_U8, true)
    IMF_K1R_ATTR(DT_U16, true)
#undef IMF_K1R_ATTR
#define IMF_K1F_ATTR(NK)                                               \
    if (!e) e = allow_smem(k1_f32_bucket<NK, false, false>, optin);    \
    if (!e) e = allow_smem(k1_f32_bucket<NK, true, false>, optin);     \
    if (!e) e = allow_smem(k1_f32_bucket<NK, false, true>, optin);     \
    if (!e) e = allow_smem(k1_f32_bucket<NK, true, true>, optin);
    IMF_K1F_ATTR(1)
    IMF_K1F_ATTR(2)
    IMF_K1F_ATTR(3)
    IMF_K1F_ATTR(4)
    IMF_K1F_ATTR(5)
    IMF_K1F_ATTR(6)
#undef IMF_K1F_ATTR
    if (!e) e = allow_smem(k1_f32_bucket_g, optin);
    if (!e) e = allow_smem(k_direct<DT_U8>, optin);
    if (!e) e = allow_smem(k_direct<DT_U16>, optin);
    if (!e) e = allow_smem(k_direct<DT_F32>, optin);
    if (!e) e = allow_smem(k2_select<true, false>, optin);
    if (!e) e = allow_smem(k2_select<false, false>, optin);
    if (!e) e = allow_smem(k2_select<true, true>, optin);
    if (!e) e = allow_smem(k2_select<false, true>, optin);
    if (!e) e = allow_smem(k2_pair<SH_SPAN, false>, optin);
    if (!e) e = allow_smem(k2_pair<SH_CIRCLE, false>, optin);
    if (!e) e = allow_smem(k2_pair<SH_SQUARE, false>, optin);
    if (!e) e = allow_smem(k2_pair<SH_SPAN, true>, optin);
    if (!e) e = allow_smem(k2_pair<SH_CIRCLE, true>, optin);
    if (!e) e = allow_smem(k2_pair<SH_SQUARE, true>, optin);
    if (!e) e = allow_smem(k2_pair<SH_POLY, false>, optin);
    if (!e) e = allow_smem(k2_pair<SH_POLY, true>, optin);
    if (!e) e = allow_smem(k2_pair<SH_POLYSYM, false>, optin);
    if (!e) e = allow_smem(k2_pair<SH_POLYSYM, true>, optin);
    if (!e) e = allow_smem(k2_pair<SH_CIRCLEW, false>, optin);
    if (!e) e = allow_smem(k2_pair<SH_CIRCLEW, true>, optin);
    if (!e) g_attr_mask.fetch_or(bit, std::memory_order_release);
    return e;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_tiled() {
    static EncodeTiledFn fn = []() -> EncodeTiledFn {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &f, 12000, cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return nullptr;
        return reinterpret_cast<EncodeTiledFn>(f);
    }();
    return fn;
}

// 4D tensor map (W, H, C, B) of the source planes, box (tma_bw, Sh, 1, 1) for
// k1_count_reg<.., TMA>.  False when the layout cannot be described (then the
// per-lane loads run).
bool make_k1_tmap(const Geom& g, const void* data, CUtensorMap* tm) {
    EncodeTiledFn enc = encode_tiled();
    const int esz = g.dtype == DT_U8 ? 1 : 2;
    if (!enc || ((uintptr_t)data & 15)) return false;
    const cuuint64_t sy = (cuuint64_t)g.s_y * esz;
    const cuuint64_t sc = g.C > 1 ? (cuuint64_t)g.s_c * esz : sy * (cuuint64_t)g.H;
    const cuuint64_t sb = g.B > 1 ? (cuuint64_t)g.s_b * esz : sc * (cuuint64_t)g.C;
    const cuuint64_t dims[4] = {(cuuint64_t)g.W, (cuuint64_t)g.H, (cuuint64_t)g.C, (cuuint64_t)g.B};
    const cuuint64_t strides[3] = {sy, sc, sb};
    const cuuint32_t box[4] = {(cuuint32_t)g.tma_bw, (cuuint32_t)g.Sh, 1, 1};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    for (cuuint64_t st : strides)
        if (st % 16 || st >= (1ull << 40)) return false;
    return enc(tm, esz == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_UINT16, 4,
               const_cast<void*>(data), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Host mirror of tile_coord (imf_common.cuh): channel fastest, then tile
// column, tile row, image; output origin of the tile (edge tiles shifted in).
void host_tile(const Geom& q, long long t, int& tx, int& ty, int& c, int& b, int& ox0, int& oy0) {
    c = (int)(t % q.C);
    t /= q.C;
    tx = (int)(t % q.tiles_x);
    t /= q.tiles_x;
    ty = (int)(t % q.tiles_y);
    b = (int)(t / q.tiles_y);
    oy0 = q.oy_base + std::min(ty * q.Th, std::max(q.out_h - q.oy_base - q.Th, 0));
    ox0 = std::min(tx * q.Tw, std::max(q.out_w - q.Tw, 0));
}

// Host mirror of the f32 bucket K1's has_runs (imf_sort.cu) for tile t of a
// call: tiles whose replicate-copy groups reach run_min (image corners) are
// the slow ones; the chunk lists them so their CTAs start first.
int host_max_copies(int X0, int S, int W) {
    if (W == 1) return S;
    const int l = X0 < 0 ? std::min(S, 1 - X0) : 1;
    const int r = X0 + S > W ? S - std::max(0, W - 1 - X0) : 1;
    return std::max(l, r);
}

void list_costly_tiles(const Plan& p, Geom& g, long long t0, int nb) {
    g.nrt = 0;
    if (!p.k1_f32b) return;
    const Geom& q = p.g;
    for (int b = 0; b < nb && g.nrt < 16; b++) {
        int tx, ty, c, im, ox0, oy0;
        host_tile(q, t0 + b, tx, ty, c, im, ox0, oy0);
        const int X0 = ox0 - q.r + q.vshift, Y0 = oy0 - q.r + q.vshift;
        if (host_max_copies(X0, q.Sw, q.W) * host_max_copies(Y0, q.Sh, q.H) >= q.run_min) g.rt[g.nrt++] = b;
    }
}

// K2's costly tiles of a chunk: the top and bottom tile rows of each plane
// whose input boxes reach past the image (clamped margins: windows there walk
// long runs of ties) -- as ranges, run first so they do not form the tail.
void list_costly_rows(const Plan& p, Geom& g, long long t0, int nb) {
    g.nrr = 0;
    const Geom& q = p.g;
    const int last_oy0 = q.oy_base + std::min((q.tiles_y - 1) * q.Th, std::max(q.out_h - q.oy_base - q.Th, 0));
    const bool top = q.oy_base - q.r + q.vshift < 0, bottom = last_oy0 - q.r + q.vshift + q.Sh > q.H;
    auto add = [&](long long a, long long b) {  // tiles [a, b) of the call, clipped to the chunk
        a = std::max(a, t0);
        b = std::min(b, t0 + nb);
        if (b <= a || g.nrr >= 4) return;
        if (g.nrr && g.rr_lo[g.nrr - 1] + g.rr_len[g.nrr - 1] == (int)(a - t0)) {  // merge adjacent
            g.rr_len[g.nrr - 1] += (int)(b - a);
            return;
        }
        g.rr_lo[g.nrr] = (int)(a - t0);
        g.rr_len[g.nrr] = (int)(b - a);
        g.nrr++;
    };
    // tiles of tile row ty of image b: [((b * tiles_y + ty) * tiles_x) * C, + tiles_x * C)
    const long long row_tiles = (long long)q.tiles_x * q.C, per_image = row_tiles * q.tiles_y;
    for (long long im = t0 / per_image; im * per_image < t0 + nb; im++) {
        const long long base = im * per_image;
        if (top && q.tiles_y > 1) add(base, base + row_tiles);
        if (bottom) add(base + (long long)(q.tiles_y - 1) * row_tiles, base + per_image);
    }
}

void launch_k1(const Plan& p, const Geom& g, int nblocks, uint16_t* omega, unsigned char* k1g,
               int* flags, cudaStream_t s, const CUtensorMap* tm) {
    const dim3 grid(nblocks), block(p.k1_threads);
    const long long gs = (long long)p.k1_gs_per_tile;
    if (p.k1_f32b) {
        const dim3 b1024(1024);
        cudaMemsetAsync(flags, 0, sizeof(int), s);  // fallback list count
        const unsigned long long mss = (unsigned long long)env_int("IMF_MAXSUMSQ_K", 65536) << 10;
        const int nk = (g.Sw + 31) >> 5;
        if (p.k1_f32b_g && nk > 6) {
            k1_f32_bucket_g<<<grid, b1024, p.k1b_smem, s>>>(g, omega, flags, (uint32_t*)k1g, gs / 4, mss);
        } else {
#define IMF_K1F_LAUNCH2(NK, FP)                                                                              \
    if (p.k1_f32b_g)                                                                                            \
        k1_f32_bucket<NK, true, FP><<<grid, b1024, p.k1b_smem, s>>>(g, omega, flags, (uint32_t*)k1g, gs / 4, mss); \
    else                                                                                                        \
        k1_f32_bucket<NK, false, FP><<<grid, b1024, p.k1b_smem, s>>>(g, omega, flags, nullptr, 0, mss);
#define IMF_K1F_LAUNCH(NK)        \
    if (g.fp) {                   \
        IMF_K1F_LAUNCH2(NK, true) \
    } else {                      \
        IMF_K1F_LAUNCH2(NK, false) \
    }
            switch (nk) {
                case 1: IMF_K1F_LAUNCH(1) break;
                case 2: IMF_K1F_LAUNCH(2) break;
                case 3: IMF_K1F_LAUNCH(3) break;
                case 4: IMF_K1F_LAUNCH(4) break;
                case 5: IMF_K1F_LAUNCH(5) break;
                default: IMF_K1F_LAUNCH(6) break;
            }
#undef IMF_K1F_LAUNCH
#undef IMF_K1F_LAUNCH2
        }
        // tiles whose buckets are too large (sum of squared sizes above the
        // limit): LSD radix sort over the list
        const dim3 fgrid(std::min(nblocks, 148));
        if (g.dtype == DT_U16) {
            if (p.k1_gmem)
                k1_sort<DT_U16, true><<<fgrid, block, p.k1_smem, s>>>(g, omega, k1g, gs, flags);
            else
                k1_sort<DT_U16, false><<<fgrid, block, p.k1_smem, s>>>(g, omega, k1g, gs, flags);
        } else if (p.k1_gmem) {
            k1_sort<DT_F32, true><<<fgrid, block, p.k1_smem, s>>>(g, omega, k1g, gs, flags);
        } else {
            k1_sort<DT_F32, false><<<fgrid, block, p.k1_smem, s>>>(g, omega, k1g, gs, flags);
        }
        return;
    }
    if (p.k1_count_g) {
        k1_count_g<<<grid, dim3(1024), k1_count_g_smem_bytes(), s>>>(g, omega);
        return;
    }
    if (p.k1_count) {
        const int nk = (g.Sw + 31) >> 5;
        // k1_count_reg addresses a plane with 32-bit element offsets
        const bool plane32 = (long long)(g.H - 1) * g.s_y + (long long)(g.W - 1) * g.s_x < (1ll << 31);
        if (nk <= 6 && plane32 && env_int("IMF_K1REG", 1)) {
#define IMF_K1R_CASE(DT, TMA)                                                                      \
    switch (nk) {                                                                                  \
        case 1: k1_count_reg<DT, 1, TMA><<<grid, block, p.k1_smem, s>>>(g, omega, tmap); break;  \
        case 2: k1_count_reg<DT, 2, TMA><<<grid, block, p.k1_smem, s>>>(g, omega, tmap); break;  \
        case 3: k1_count_reg<DT, 3, TMA><<<grid, block, p.k1_smem, s>>>(g, omega, tmap); break;  \
        case 4: k1_count_reg<DT, 4, TMA><<<grid, block, p.k1_smem, s>>>(g, omega, tmap); break;  \
        case 5: k1_count_reg<DT, 5, TMA><<<grid, block, p.k1_smem, s>>>(g, omega, tmap); break;  \
        default: k1_count_reg<DT, 6, TMA><<<grid, block, p.k1_smem, s>>>(g, omega, tmap); break; \
    }
            const bool tma = tm != nullptr;
            const CUtensorMap tmap = tma ? *tm : CUtensorMap{};
            if (g.dtype == DT_U8) {
                if (tma) { IMF_K1R_CASE(DT_U8, true) } else { IMF_K1R_CASE(DT_U8, false) }
            } else {
                if (tma) { IMF_K1R_CASE(DT_U16, true) } else { IMF_K1R_CASE(DT_U16, false) }
            }
#undef IMF_K1R_CASE
            return;
        }
        if (g.dtype == DT_U8)
            k1_count<DT_U8><<<grid, block, p.k1_smem, s>>>(g, omega);
        else
            k1_count<DT_U16><<<grid, block, p.k1_smem, s>>>(g, omega);
        return;
    }
    switch (g.dtype * 2 + (p.k1_gmem ? 1 : 0)) {
        case 0:
        case 1: k1_sort<DT_U8, false><<<grid, block, p.k1_smem, s>>>(g, omega, k1g, gs, nullptr); break;
        case 2: k1_sort<DT_U16, false><<<grid, block, p.k1_smem, s>>>(g, omega, k1g, gs, nullptr); break;
        case 3: k1_sort<DT_U16, true><<<grid, block, p.k1_smem, s>>>(g, omega, k1g, gs, nullptr); break;
        case 4: k1_sort<DT_F32, false><<<grid, block, p.k1_smem, s>>>(g, omega, k1g, gs, nullptr); break;
        default: k1_sort<DT_F32, true><<<grid, block, p.k1_smem, s>>>(g, omega, k1g, gs, nullptr); break;
    }
}

}  // namespace

extern "C" {

size_t imf_workspace_size(const imf_image* src, const imf_kernel* kernel, const imf_options* opt) {
    Plan p;
    if (make_plan(src, kernel, opt, &p) != IMF_OK) return 0;
    return p.ws_total;
}

}  // extern "C"

// Device-side inputs of K1 for a call: the launch geometry, the footprint
// table (uploaded into the workspace), the call-wide f32 coarse bucket table
// (k_coarse_hist / k_coarse_alloc), and the TMA descriptor of planar tiles.
static int prep_k1(const Plan& p, const imf_image* src, unsigned char* ws, cudaStream_t s, Geom& g,
                   CUtensorMap& tmap, bool& use_tma) {
    g = p.g;
    g.src = src->data;
    g.ctab_g = nullptr;
    g.fprow = nullptr;
    if (g.fp) {  // footprint rows into the workspace (the copy is staged at call time)
        uint32_t* d = (uint32_t*)(ws + kFpOffset);
        if (cudaError_t e = cudaMemcpyAsync(d, p.fprow, 4 * (size_t)g.Sh, cudaMemcpyHostToDevice, s))
            return cuda_fail(e, "footprint table upload");
        g.fprow = d;
    }
    if (p.ws_ctab && p.ct_y1 > p.ct_y0) {
        uint32_t* ct = (uint32_t*)(ws + kStatusBytes + p.lanes * p.ws_lane);
        if (cudaError_t e = cudaMemsetAsync(ct, 0, p.ws_ctab, s)) return cuda_fail(e, "coarse table memset");
        const long long rows = (long long)(p.ct_y1 - p.ct_y0) * g.B * g.C;
        const int cgrid = (int)std::min<long long>(296, (rows + 31) / 32);
        k_coarse_hist<<<cgrid, 1024, 0, s>>>(g, p.ct_y0, p.ct_y1, ct);
        k_coarse_alloc<<<1, 1024, 0, s>>>(ct);
        g_launches += 2;
        g.ctab_g = ct;
    }
    use_tma = p.k1_tma && make_k1_tmap(g, src->data, &tmap);
    g_last_tma = use_tma;
    return IMF_OK;
}

// One K1 (ordinal transform) per chunk of tiles, then one K2 (selection) per
// requested output: n scalar targets (the "bracket", core.py:412-426) reuse
// the same omega.  n == 1 with an optional per-pixel target map is imf_filter.
static int filter_impl(const imf_image* src, imf_image* dsts, int n, const int32_t* targets,
                       const int32_t* target_map, int32_t tmin, int32_t tmax, const imf_kernel* kernel,
                       const imf_options* opt, void* workspace, size_t workspace_bytes, void* stream) {
    if (!src || !kernel || !opt || !dsts || n < 1 || !targets || !src->data) return IMF_ERR_INVALID;
    if (target_map && n != 1) return IMF_ERR_INVALID;
    for (int i = 0; i < n; i++) {
        const imf_image* dst = dsts + i;
        if (!dst->data || src->data == dst->data) return IMF_ERR_INVALID;
        if (dst->dtype != src->dtype || dst->batch != src->batch || dst->channels != src->channels)
            return IMF_ERR_INVALID;
        if (targets[i] < 0 || targets[i] >= kernel->area) return IMF_ERR_INVALID;
    }
    if (!target_map) tmin = tmax = targets[0];
    if (tmin < 0 || tmax >= kernel->area || tmin > tmax) return IMF_ERR_INVALID;
    Plan p;
    int st = make_plan(src, kernel, opt, &p);
    if (st) return st;
    for (int i = 0; i < n; i++)
        if (dsts[i].height != p.full_out_h || dsts[i].width != p.g.out_w) return IMF_ERR_INVALID;
    if (!workspace || workspace_bytes < p.ws_total) return IMF_ERR_WORKSPACE;
    cudaStream_t s = (cudaStream_t)stream;
    if (cudaError_t e = set_attrs()) return cuda_fail(e, "cudaFuncSetAttribute");

    unsigned char* ws = (unsigned char*)workspace;
    int* status = (int*)ws;
    unsigned char* lane_base[2] = {ws + kStatusBytes, ws + kStatusBytes + p.ws_lane};

    if (p.direct) {  // tiny windows: one kernel, no ordinal transform
        DirectTab dtab;
        memset(&dtab, 0, sizeof(dtab));
        dtab.area = 0;
        for (int i = 0; i < kernel->nrows; i++)
            for (int x = kernel->row_xlo[i]; x < kernel->row_xhi[i]; x++)
                dtab.off[dtab.area++] = kernel->row_dy[i] * p.g.Sw + x;
        if (!(opt->flags & IMF_FLAG_KEEP_STATUS))
            if (cudaError_t e = cudaMemsetAsync(status, 0, sizeof(int), s)) return cuda_fail(e, "status memset");
        Geom g = p.g;
        g.src = src->data;
        g.tile_begin = 0;
        const unsigned nb = (unsigned)p.total_tiles;
        for (int i = 0; i < n; i++) {
            g.dst = dsts[i].data;
            g.d_b = dsts[i].stride_b;
            g.d_y = dsts[i].stride_y;
            g.d_x = dsts[i].stride_x;
            g.d_c = dsts[i].stride_c;
            if (g.dtype == DT_U8)
                k_direct<DT_U8><<<nb, 1024, p.k2_smem, s>>>(g, dtab, targets[i], target_map);
            else if (g.dtype == DT_U16)
                k_direct<DT_U16><<<nb, 1024, p.k2_smem, s>>>(g, dtab, targets[i], target_map);
            else
                k_direct<DT_F32><<<nb, 1024, p.k2_smem, s>>>(g, dtab, targets[i], target_map);
            g_launches += 1;
        }
        if (cudaError_t e = cudaGetLastError()) return cuda_fail(e, "kernel launch");
        if (opt->flags & IMF_FLAG_PROFILE) {
            cudaStreamSynchronize(s);
            g_prof = ProfileRec{};
            g_prof.tiles = p.total_tiles;
            g_prof.tile = p.g.Tw;
            g_prof.qs = 3;
        }
        return IMF_OK;
    }

    static thread_local KTab kt;
    build_ktab_struct(kernel, p.g.Sw, kt);
    if (!(opt->flags & IMF_FLAG_KEEP_STATUS))
        if (cudaError_t e = cudaMemsetAsync(status, 0, sizeof(int), s)) return cuda_fail(e, "status memset");

    Geom g;
    CUtensorMap k1_tmap;
    bool use_tma = false;
    if (int e = prep_k1(p, src, ws, s, g, k1_tmap, use_tma)) return e;

    SelParams sp;
    memset(&sp, 0, sizeof(sp));
    sp.circle = kernel->shape_code == IMF_SHAPE_CIRCLE;
    sp.R2 = kernel->radius * (kernel->radius + 1);
    sp.ncols = kernel->ncols;
    sp.nrows = kernel->nrows;
    sp.target = targets[0];
    sp.tmap = target_map;
    sp.G = p.G;
    sp.status = status;
    // test hook: IMF_FLAG_DEBUG_DEFECT, or IMF_DEBUG_DEFECT=1 in the environment
    // (reaches the hook through every entry point, the CLI included)
    const int dbg_defect = (opt->flags & IMF_FLAG_DEBUG_DEFECT) || env_int("IMF_DEBUG_DEFECT", 0) ? 1 : 0;
    sp.debug_defect = dbg_defect;

    static thread_local PairTab ptab;
    PairParams pp;
    memset(&pp, 0, sizeof(pp));
    if (p.pair) {
        const int r = kernel->radius;
        if (!build_pair_tab(kernel->row_dy, kernel->row_xlo, kernel->row_xhi, kernel->nrows, kernel->col_dx,
                            kernel->col_ytop, kernel->col_ybot, kernel->ncols, r, p.g.Sw, ptab, pp))
            return IMF_ERR_UNSUPPORTED;
        const bool bytes_ok = p.g.Tw + r <= 128 && p.g.Th + r <= 128;  // |dx|, |dy| <= 127 in a tile
        pp.shape = !bytes_ok ? (kernel->shape_code == IMF_SHAPE_CIRCLE ? SH_CIRCLEW : SH_SPAN)
                   : kernel->shape_code == IMF_SHAPE_CIRCLE ? SH_CIRCLE
                   : kernel->shape_code == IMF_SHAPE_SQUARE ? SH_SQUARE : SH_POLY;
        if (pp.shape == SH_POLY && kernel_symmetric(kernel) && env_int("IMF_POLYSYM", 1)) pp.shape = SH_POLYSYM;
        pp.R2p1 = r * (r + 1) + 1;
        pp.nR2p1 = -pp.R2p1;
        pp.target = targets[0];
        pp.tmap = target_map;
        pp.G = p.G;
        pp.hs = p.hs;
        pp.grouped = p.k2_threads == 64 * p.G && p.g.Tw <= 64 && p.G <= 15 && env_int("IMF_GROUPED", 1);
        pp.status = status;
        pp.debug_defect = dbg_defect;
        pp.refine_mode = env_int("IMF_REFINE", 1);
    }

    // Optional per-kernel timing (opt->reserved[0] & 1): CUDA events recorded on
    // `stream` around every launch; the call then synchronizes and leaves the
    // sums in imf_profile_last().  Used by bench.py for the roofline figure.
    const bool prof = (opt->flags & IMF_FLAG_PROFILE) != 0;
    std::vector<cudaEvent_t> ev;
    // second lane: fork from s, join back into s at the end (stream-ordered API)
    const int lanes = prof ? 1 : p.lanes;
    cudaStream_t ls[2] = {s, nullptr};
    cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
    if (lanes == 2) {
        // one lane-2 stream per (thread, device), created once, destroyed when
        // the thread exits
        struct Lane2 {
            cudaStream_t s[kMaxDev] = {};
            ~Lane2() {
                for (int d = 0; d < kMaxDev; d++)
                    if (s[d] && cudaSetDevice(d) == cudaSuccess) cudaStreamDestroy(s[d]);
            }
        };
        static thread_local Lane2 lane2;
        int dev = 0;
        if (cudaError_t e = cudaGetDevice(&dev)) return cuda_fail(e, "cudaGetDevice");
        if (!lane2.s[dev])
            if (cudaError_t e = cudaStreamCreateWithFlags(&lane2.s[dev], cudaStreamNonBlocking))
                return cuda_fail(e, "lane stream");
        ls[1] = lane2.s[dev];
        cudaEventCreateWithFlags(&fork_ev, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&join_ev, cudaEventDisableTiming);
        cudaEventRecord(fork_ev, s);  // after the status memset
        cudaStreamWaitEvent(ls[1], fork_ev, 0);
    }
    int ci = 0;
    for (long long t0 = 0; t0 < p.total_tiles; t0 += p.chunk_tiles, ci++) {
        const int nb = (int)std::min(p.chunk_tiles, p.total_tiles - t0);
        g.tile_begin = t0;
        const int li = lanes == 2 ? (ci & 1) : 0;
        cudaStream_t s = ls[li];
        uint16_t* omega = (uint16_t*)lane_base[li];
        unsigned char* k1g = lane_base[li] + p.ws_omega;
        int* k1flags = (int*)(lane_base[li] + p.ws_omega + p.ws_k1g);
        cudaEvent_t e0 = nullptr, e1 = nullptr, e2 = nullptr;
        if (prof) {
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventCreate(&e2);
            cudaEventRecord(e0, s);
        }
        if (env_int("IMF_COSTLY_FIRST", 1)) list_costly_tiles(p, g, t0, nb);
        launch_k1(p, g, nb, omega, k1g, k1flags, s, use_tma ? &k1_tmap : nullptr);
        g.nrt = 0;
        if (env_int("IMF_COSTLY_FIRST", 1)) list_costly_rows(p, g, t0, nb);
        if (prof) cudaEventRecord(e1, s);
        for (int i = 0; i < n; i++) {
        g.dst = dsts[i].data;
        g.d_b = dsts[i].stride_b;
        g.d_y = dsts[i].stride_y;
        g.d_x = dsts[i].stride_x;
        g.d_c = dsts[i].stride_c;
        sp.target = pp.target = targets[i];
        if (p.pair) {
#define IMF_K2P_LAUNCH(S, O) k2_pair<S, O><<<nb, p.k2_threads, p.k2_smem, s>>>(g, pp, ptab, omega)
            switch (pp.shape * 2 + (p.omg ? 1 : 0)) {
                case SH_CIRCLE * 2: IMF_K2P_LAUNCH(SH_CIRCLE, false); break;
                case SH_CIRCLE * 2 + 1: IMF_K2P_LAUNCH(SH_CIRCLE, true); break;
                case SH_SQUARE * 2: IMF_K2P_LAUNCH(SH_SQUARE, false); break;
                case SH_SQUARE * 2 + 1: IMF_K2P_LAUNCH(SH_SQUARE, true); break;
                case SH_POLY * 2: IMF_K2P_LAUNCH(SH_POLY, false); break;
                case SH_POLY * 2 + 1: IMF_K2P_LAUNCH(SH_POLY, true); break;
                case SH_POLYSYM * 2: IMF_K2P_LAUNCH(SH_POLYSYM, false); break;
                case SH_POLYSYM * 2 + 1: IMF_K2P_LAUNCH(SH_POLYSYM, true); break;
                case SH_CIRCLEW * 2: IMF_K2P_LAUNCH(SH_CIRCLEW, false); break;
                case SH_CIRCLEW * 2 + 1: IMF_K2P_LAUNCH(SH_CIRCLEW, true); break;
                case SH_SPAN * 2 + 1: IMF_K2P_LAUNCH(SH_SPAN, true); break;
                default: IMF_K2P_LAUNCH(SH_SPAN, false); break;
            }
#undef IMF_K2P_LAUNCH
        } else if (sp.circle && !p.omg)
            k2_select<true, false><<<nb, p.k2_threads, p.k2_smem, s>>>(g, sp, kt, omega);
        else if (!p.omg)
            k2_select<false, false><<<nb, p.k2_threads, p.k2_smem, s>>>(g, sp, kt, omega);
        else if (sp.circle)
            k2_select<true, true><<<nb, p.k2_threads, p.k2_smem, s>>>(g, sp, kt, omega);
        else
            k2_select<false, true><<<nb, p.k2_threads, p.k2_smem, s>>>(g, sp, kt, omega);
        }
        if (prof) {
            cudaEventRecord(e2, s);
            ev.push_back(e0);
            ev.push_back(e1);
            ev.push_back(e2);
        }
        g_launches += 1 + n;
        g.nrr = 0;
    }
    if (lanes == 2) {
        cudaEventRecord(join_ev, ls[1]);
        cudaStreamWaitEvent(s, join_ev, 0);
        cudaEventDestroy(fork_ev);  // released once the recorded work completes
        cudaEventDestroy(join_ev);
    }
    if (cudaError_t e = cudaGetLastError()) return cuda_fail(e, "kernel launch");
    if (prof) {
        g_prof = ProfileRec{};
        if (!ev.empty()) cudaEventSynchronize(ev.back());
        for (size_t i = 0; i + 2 < ev.size(); i += 3) {
            float a = 0.f, b = 0.f;
            cudaEventElapsedTime(&a, ev[i], ev[i + 1]);
            cudaEventElapsedTime(&b, ev[i + 1], ev[i + 2]);
            g_prof.sort_ms += a;
            g_prof.select_ms += b;
            g_prof.launches += 1;
        }
        for (cudaEvent_t e : ev) cudaEventDestroy(e);
        g_prof.tiles = p.total_tiles;
        g_prof.tile = p.g.Tw;
        g_prof.qs = p.pair ? 2 : (p.omg ? 1 : 0);
        g_prof.chunk = p.chunk_tiles;
    }
    return IMF_OK;
}

extern "C" {

int imf_filter(const imf_image* src, imf_image* dst, const imf_kernel* kernel, int32_t target,
               const int32_t* target_map, int32_t tmin, int32_t tmax, const imf_options* opt,
               void* workspace, size_t workspace_bytes, void* stream) {
    if (!dst) return IMF_ERR_INVALID;
    return filter_impl(src, dst, 1, &target, target_map, tmin, tmax, kernel, opt, workspace, workspace_bytes,
                       stream);
}

int imf_filter_bracket(const imf_image* src, imf_image* dsts, int32_t n, const int32_t* targets,
                       const imf_kernel* kernel, const imf_options* opt, void* workspace,
                       size_t workspace_bytes, void* stream) {
    if (n < 1 || !targets) return IMF_ERR_INVALID;
    int32_t tmin = targets[0], tmax = targets[0];
    for (int i = 1; i < n; i++) {
        tmin = std::min(tmin, targets[i]);
        tmax = std::max(tmax, targets[i]);
    }
    return filter_impl(src, dsts, n, targets, nullptr, tmin, tmax, kernel, opt, workspace, workspace_bytes,
                       stream);
}

int imf_profile_last(float* sort_ms, float* select_ms, int32_t* launches, int64_t* tiles,
                     int32_t* tile_side, int32_t* qshift) {
    if (sort_ms) *sort_ms = g_prof.sort_ms;
    if (select_ms) *select_ms = g_prof.select_ms;
    if (launches) *launches = g_prof.launches;
    if (tiles) *tiles = g_prof.tiles;
    if (tile_side) *tile_side = g_prof.tile;
    if (qshift) *qshift = g_prof.qs;
    return IMF_OK;
}

uint32_t imf_last_features(void) { return g_last_tma ? IMF_FEATURE_K1_TMA : 0u; }

int imf_plan_info(const imf_image* src, const imf_kernel* kernel, const imf_options* opt, int64_t* info) {
    if (!info) return IMF_ERR_INVALID;
    Plan p;
    if (int st = make_plan(src, kernel, opt, &p)) return st;
    const Geom& g = p.g;
    const int64_t v[16] = {g.Tw, g.Th, g.Sw, g.Sh, g.N, g.Npad, p.total_tiles, p.chunk_tiles, p.lanes,
                           p.direct ? 0 : (p.pair ? 2 : 1), g.fp, p.k1_tma ? 1 : 0, p.hs, p.G,
                           (int64_t)p.ws_total,
                           p.k1_f32b ? (p.k1_f32b_g ? 2 : 1) : p.k1_count ? 3 : p.k1_count_g ? 4 : 0};
    memcpy(info, v, sizeof(v));
    return IMF_OK;
}

int imf_tile_omega(const imf_image* src, const imf_kernel* kernel, const imf_options* opt, int64_t tile,
                   uint16_t* omega, int32_t capacity, int32_t* info, void* workspace, size_t workspace_bytes,
                   void* stream) {
    if (!src || !kernel || !opt || !src->data || !omega || !info) return IMF_ERR_INVALID;
    Plan p;
    if (int st = make_plan(src, kernel, opt, &p)) return st;
    if (p.direct) return IMF_ERR_UNSUPPORTED;  // tiny windows: no ordinal transform
    if (tile < 0 || tile >= p.total_tiles) return IMF_ERR_INVALID;
    if (!workspace || workspace_bytes < p.ws_total) return IMF_ERR_WORKSPACE;
    if (capacity < p.g.N) return IMF_ERR_INVALID;
    cudaStream_t s = (cudaStream_t)stream;
    if (cudaError_t e = set_attrs()) return cuda_fail(e, "cudaFuncSetAttribute");
    unsigned char* ws = (unsigned char*)workspace;
    Geom g;
    CUtensorMap tmap;
    bool use_tma = false;
    if (int e = prep_k1(p, src, ws, s, g, tmap, use_tma)) return e;
    g.tile_begin = tile;
    unsigned char* lane = ws + kStatusBytes;
    launch_k1(p, g, 1, (uint16_t*)lane, lane + p.ws_omega, (int*)(lane + p.ws_omega + p.ws_k1g), s,
              use_tma ? &tmap : nullptr);
    if (cudaError_t e = cudaGetLastError()) return cuda_fail(e, "K1 launch");
    if (cudaError_t e = cudaMemcpyAsync(omega, (uint16_t*)lane + OMEGA_SLOT_PAD, 2 * (size_t)p.g.N,
                                        cudaMemcpyDeviceToHost, s))
        return cuda_fail(e, "omega download");
    if (cudaError_t e = cudaStreamSynchronize(s)) return cuda_fail(e, "stream synchronize");
    // the tile's input origin (image coordinates of input-tile pixel (0, 0),
    // before clamping; tile_coord on the host) and its input extent
    const Geom& q = p.g;
    int tx, ty, c, b, ox0, oy0;
    host_tile(q, tile, tx, ty, c, b, ox0, oy0);
    info[0] = q.N;
    info[1] = ox0 - q.r + q.vshift;
    info[2] = oy0 - q.r + q.vshift;
    info[3] = q.Sw;
    info[4] = q.Sh;
    info[5] = c;
    info[6] = b;
    info[7] = q.fp;
    return IMF_OK;
}

int imf_workspace_status(void* workspace, void* stream) {
    int h = 0;
    if (!workspace) return IMF_ERR_INVALID;
    if (cudaError_t e = cudaMemcpyAsync(&h, workspace, sizeof(int), cudaMemcpyDeviceToHost, (cudaStream_t)stream))
        return cuda_fail(e, "status read");
    if (cudaError_t e = cudaStreamSynchronize((cudaStream_t)stream)) return cuda_fail(e, "stream synchronize");
    return h ? IMF_ERR_DEFECT : IMF_OK;
}

static size_t extent_bytes(const imf_image* im) {
    const long long last = (long long)(im->batch - 1) * im->stride_b +
                           (long long)(im->height - 1) * im->stride_y +
                           (long long)(im->width - 1) * im->stride_x +
                           (long long)(im->channels - 1) * im->stride_c;
    return (size_t)(last + 1) * dtype_size(im->dtype);
}

// Rows are outermost within an image (HW / HWC / NHWC): rows [a, b) of image
// bi are the contiguous element range [bi*s_b + a*s_y, bi*s_b + b*s_y).
static bool rows_outermost(const imf_image* im) {
    const long long row = (long long)(im->width - 1) * im->stride_x + (long long)(im->channels - 1) * im->stride_c + 1;
    return im->stride_x >= 0 && im->stride_c >= 0 && im->stride_y >= row &&
           (im->batch == 1 || im->stride_b >= (long long)im->height * im->stride_y);
}

namespace {
constexpr int kMaxStripeLanes = 4;
struct HostStreams {
    cudaStream_t up = nullptr, down = nullptr;
    cudaStream_t comp[kMaxStripeLanes] = {};  // comp[0] unused: lane 0 is the caller's stream
    int* status_h = nullptr;                  // pinned: the lanes' status words, read once per call
    std::vector<cudaEvent_t> events;          // reused across calls (timing disabled)
    void release() {  // the thread's resources on the current device
        for (cudaStream_t* p : {&up, &down, &comp[1], &comp[2], &comp[3]})
            if (*p) cudaStreamDestroy(*p), *p = nullptr;
        for (cudaEvent_t e : events) cudaEventDestroy(e);
        events.clear();
        if (status_h) cudaFreeHost(status_h), status_h = nullptr;
    }
};
// per (thread, device), created on first use; released when the thread exits
// (threads that come and go, e.g. one per filter_multi call, leak nothing)
struct HostStreamSet {
    HostStreams dev[kMaxDev];
    ~HostStreamSet() {
        for (int d = 0; d < kMaxDev; d++)
            if (dev[d].up && cudaSetDevice(d) == cudaSuccess) dev[d].release();
    }
};
thread_local HostStreamSet g_hs_set;
}  // namespace

int imf_filter_host(const imf_image* src, imf_image* dst, const imf_kernel* kernel, int32_t target,
                    const int32_t* target_map, int32_t tmin, int32_t tmax, const imf_options* opt,
                    void* stream) {
    if (!src || !dst || !kernel || !opt || !src->data || !dst->data) return IMF_ERR_INVALID;
    cudaStream_t s = (cudaStream_t)stream;
    if (!target_map) tmin = tmax = target;
    Plan p;
    int st = make_plan(src, kernel, opt, &p);
    if (st) return st;
    const int dsz = dtype_size(src->dtype);
    if (src->stride_b < 0 || src->stride_y < 0 || src->stride_x < 0 || src->stride_c < 0 || dst->stride_b < 0 ||
        dst->stride_y < 0 || dst->stride_x < 0 || dst->stride_c < 0)
        return IMF_ERR_INVALID;
    const size_t sb = extent_bytes(src), db = extent_bytes(dst);
    // results come back as whole byte ranges of dst: every byte of dst's extent
    // must belong to one of its elements (dense layout, e.g. C-contiguous), or
    // host bytes between elements would be overwritten
    if ((size_t)dst->batch * dst->height * dst->width * dst->channels * dsz != db) return IMF_ERR_INVALID;
    const size_t tb = target_map ? (size_t)p.full_out_h * p.g.out_w * 4 : 0;
    int dev = 0;
    if (cudaGetDevice(&dev)) return IMF_ERR_CUDA;
    if (dev >= kMaxDev) return IMF_ERR_INVALID;
    HostStreams& g_hs = g_hs_set.dev[dev];
    if (!g_hs.up) {
        if (cudaStreamCreateWithFlags(&g_hs.up, cudaStreamNonBlocking) ||
            cudaStreamCreateWithFlags(&g_hs.down, cudaStreamNonBlocking) ||
            cudaStreamCreateWithFlags(&g_hs.comp[1], cudaStreamNonBlocking) ||
            cudaStreamCreateWithFlags(&g_hs.comp[2], cudaStreamNonBlocking) ||
            cudaStreamCreateWithFlags(&g_hs.comp[3], cudaStreamNonBlocking) ||
            cudaMallocHost(&g_hs.status_h, kMaxStripeLanes * sizeof(int)))
            return cuda_fail(cudaGetLastError(), "stream create");
        // keep freed pool memory cached across calls (default threshold 0 returns
        // it to the driver at every synchronization)
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t thr = 4ull << 30;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
    }
    void *dsrc = nullptr, *ddst = nullptr, *dtm = nullptr;
    void* dws[kMaxStripeLanes] = {};
    std::vector<cudaEvent_t> evs;
    // IMF_HOST_TRACE=1: timed events, and a per-stripe timeline on stderr (dev aid)
    const bool trace = env_int("IMF_HOST_TRACE", 0) != 0;
    std::vector<std::pair<std::string, cudaEvent_t>> tl;
    // events: from the per-(thread, device) pool (recycled: every use below is
    // complete once the call returns), or created with timing for a trace
    size_t ev_used = 0;
    auto event = [&]() {
        cudaEvent_t e = nullptr;
        if (trace) {
            cudaEventCreateWithFlags(&e, cudaEventDefault);
            evs.push_back(e);
            return e;
        }
        if (ev_used == g_hs.events.size()) {
            cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
            g_hs.events.push_back(e);
        }
        return g_hs.events[ev_used++];
    };
    auto mark = [&](const char* what, int i, cudaStream_t st) {
        if (!trace) return;
        cudaEvent_t e = event();
        cudaEventRecord(e, st);
        tl.emplace_back(std::string(what) + " " + std::to_string(i), e);
    };
    mark("start", 0, s);
    int rc = IMF_OK;
    // compute lanes (stripes rotate over them, each with its own
    // workspace) so one stripe's K1 fills the tail of the previous stripe's K2
    const int nl0 = std::max(1, std::min(kMaxStripeLanes, env_int("IMF_STRIPE_LANES", 3)));
    const int OH0 = p.full_out_h;
    // output rows [R0, R1) (opt->row_begin/row_end: one device's stripe of a
    // multi-device job; the other rows of dst are left untouched)
    const bool ranged = opt->row_end > 0;
    const int R0 = ranged ? opt->row_begin : 0, R1 = ranged ? opt->row_end : OH0;
    const bool pipe0 = rows_outermost(src) && rows_outermost(dst) && (ranged || OH0 > 2 * p.g.Th);
    if (ranged && !pipe0) return IMF_ERR_INVALID;  // row ranges need row-outermost layouts
    const int nl = pipe0 ? nl0 : 1;
    // batches stream through a ring of two device image slots (image b in slot
    // b % 2, reused once image b - 2 is downloaded): device memory and the
    // per-call allocation stay two images deep however long the batch
    const bool ring = pipe0 && src->batch > 2 && env_int("IMF_RING", 1);
    const int nslot = ring ? 2 : src->batch;
    const size_t sbA = ring ? (size_t)nslot * src->stride_b * dsz : sb;
    const size_t dbA = ring ? (size_t)nslot * dst->stride_b * dsz : db;
    if (cudaMallocAsync(&dsrc, sbA, s) || cudaMallocAsync(&ddst, dbA, s) || (tb && cudaMallocAsync(&dtm, tb, s)))
        rc = cuda_fail(cudaGetLastError(), "cudaMallocAsync");
    if (!rc && tb && cudaMemcpyAsync(dtm, target_map, tb, cudaMemcpyHostToDevice, s))
        rc = cuda_fail(cudaGetLastError(), "target map upload");
    imf_image ds = *src, dd = *dst;
    ds.data = dsrc;
    dd.data = ddst;
    const int r = kernel->radius, vshift = opt->boundary == IMF_BOUNDARY_VALID ? r : 0;
    const int H = src->height, OH = OH0;
    const bool pipe = pipe0;
    // Stripes of whole tile rows: a two-tile-row first stripe (the filter starts
    // after a small upload), a two-tile-row last stripe (little left to download
    // after the last filter), ramp stripes and 8 middle stripes; consecutive
    // stripes rotate over three compute streams, so each stripe's K1 fills the
    // previous stripes' K2 tails (c2 with the round-2 kernels: 1.87 ms
    // host->host vs 1.94 with two streams and one-tile-row edges; c5 -3 %).
    std::vector<int> cuts{0};  // in tile rows from R0, then output rows
    if (pipe) {
        const int tiles_y = (R1 - R0 + p.g.Th - 1) / p.g.Th;
        const int edge = std::max(1, env_int("IMF_STRIPE_EDGE", 2));
        const int mid = std::max(1, env_int("IMF_STRIPE_MID", 8));
        // ramp (IMF_STRIPE_RAMP=1): after the first (edge) stripe, stripes
        // of 1 and 2 tile rows, so the GPU fills while the larger middle
        // stripes upload; mirrored (2, 1) before the last one-row stripe
        const int ramp = env_int("IMF_STRIPE_RAMP", 1) ? 3 : 0;  // tile rows in the ramp stripes, each end
        if (tiles_y <= 2 * (edge + ramp) + 1) {
            for (int t = 1; t <= tiles_y; t++) cuts.push_back(t);
        } else {
            cuts.push_back(edge);
            if (ramp) {
                cuts.push_back(edge + 1);
                cuts.push_back(edge + 3);
            }
            const int lo = edge + ramp, body = tiles_y - 2 * (edge + ramp);
            for (int i = 1; i <= mid; i++) cuts.push_back(lo + (int)((long long)body * i / mid));
            if (ramp) {
                cuts.push_back(tiles_y - edge - 1);
                cuts.push_back(tiles_y - edge);
            }
            cuts.push_back(tiles_y);
        }
        for (int& c : cuts) c = std::min(R1, R0 + c * p.g.Th);
        cuts.erase(std::unique(cuts.begin(), cuts.end()), cuts.end());
    } else {
        cuts.push_back(OH);
    }
    // The first stripe's input rows go up before the workspace is planned and
    // allocated below (host work that would otherwise delay the first copy).
    int pre_up_hi = -1;  // image 0: input rows [.., pre_up_hi) already uploaded
    if (!rc && pipe) {
        cudaEvent_t e_io = event();
        cudaEventRecord(e_io, s);
        cudaStreamWaitEvent(g_hs.up, e_io, 0);
        const int lo = std::max(0, std::min(H, R0 + vshift - r));
        const int need = std::min(H, cuts[1] - 1 + r + vshift + 1);
        if (need > lo) {
            const size_t off = (size_t)((long long)lo * src->stride_y) * dsz;
            const size_t len = (size_t)((long long)(need - lo) * src->stride_y) * dsz;
            if (cudaMemcpyAsync((char*)dsrc + off, (const char*)src->data + off,
                                std::min(len, std::min(sb - off, sbA - off)), cudaMemcpyHostToDevice, g_hs.up))
                rc = cuda_fail(cudaGetLastError(), "stripe upload");
            pre_up_hi = need;
        }
    }
    // Workspace per compute lane: the largest any stripe's launch plan needs (a
    // one-image stripe plans fewer tiles than the whole call -- one chunk lane,
    // whose single chunk can exceed the call's two-lane chunks); plans depend
    // on the stripe height only, so each distinct height is planned once.
    size_t ws_need = p.ws_total;
    if (pipe) {
        imf_image one = *src;
        one.batch = 1;
        std::vector<int> seen;
        for (size_t si = 0; si + 1 < cuts.size(); si++) {
            const int hgt = cuts[si + 1] - cuts[si];
            if (std::find(seen.begin(), seen.end(), hgt) != seen.end()) continue;
            seen.push_back(hgt);
            imf_options o = *opt;
            o.row_begin = cuts[si];
            o.row_end = cuts[si + 1];
            Plan q;
            if (make_plan(&one, kernel, &o, &q) == IMF_OK) ws_need = std::max(ws_need, q.ws_total);
        }
    }
    for (int i = 0; i < nl && !rc; i++)
        if (cudaMallocAsync(&dws[i], ws_need, s)) rc = cuda_fail(cudaGetLastError(), "cudaMallocAsync");
    cudaEvent_t e_alloc = event();
    if (!rc) cudaEventRecord(e_alloc, s);
    int nstripe = 0;
    if (!rc) {
        cudaStreamWaitEvent(g_hs.up, e_alloc, 0);
        for (int i = 1; i < nl; i++) cudaStreamWaitEvent(g_hs.comp[i], e_alloc, 0);
        std::vector<cudaEvent_t> slot_free(nslot, nullptr);  // ring: last download of the slot's image
        for (int bi = 0; bi < src->batch && !rc; bi++) {
            // host offsets of image bi; device offsets of its slot
            const long long sbase = (long long)bi * src->stride_b, dbase = (long long)bi * dst->stride_b;
            const int slot = ring ? bi % nslot : bi;
            const long long sdev = (long long)slot * src->stride_b, ddev = (long long)slot * dst->stride_b;
            if (ring && slot_free[slot]) cudaStreamWaitEvent(g_hs.up, slot_free[slot], 0);
            // input rows [first row the stripe reads, up_hi) of image bi are uploaded
            int up_hi = (bi == 0 && pre_up_hi >= 0) ? pre_up_hi : std::max(0, std::min(H, R0 + vshift - r));
            for (size_t si = 0; si + 1 < cuts.size() && !rc; si++) {
                const int y0 = cuts[si], y1 = cuts[si + 1];
                if (pipe) {
                    const int need = std::min(H, y1 - 1 + r + vshift + 1);
                    if (need > up_hi) {
                        const size_t off = (size_t)(sbase + (long long)up_hi * src->stride_y) * dsz;
                        const size_t doff = (size_t)(sdev + (long long)up_hi * src->stride_y) * dsz;
                        const size_t len = (size_t)((long long)(need - up_hi) * src->stride_y) * dsz;
                        const size_t cap = std::min(sb - off, sbA - doff);
                        if (cudaMemcpyAsync((char*)dsrc + doff, (const char*)src->data + off, std::min(len, cap),
                                            cudaMemcpyHostToDevice, g_hs.up))
                            rc = cuda_fail(cudaGetLastError(), "stripe upload");
                        up_hi = need;
                    }
                } else if (bi == 0 && y0 == 0) {
                    if (cudaMemcpyAsync(dsrc, src->data, sb, cudaMemcpyHostToDevice, g_hs.up))
                        rc = cuda_fail(cudaGetLastError(), "upload");
                }
                const int lane_i = nstripe % nl;
                cudaStream_t cs = lane_i ? g_hs.comp[lane_i] : s;
                void* wsl = dws[lane_i];
                mark("uploaded", nstripe, g_hs.up);
                cudaEvent_t e_up = event();
                cudaEventRecord(e_up, g_hs.up);
                cudaStreamWaitEvent(cs, e_up, 0);
                imf_options o = *opt;
                o.flags &= ~IMF_FLAG_PROFILE;
                if (nstripe >= nl) o.flags |= IMF_FLAG_KEEP_STATUS;  // earlier defects persist
                nstripe++;
                o.row_begin = y0;
                o.row_end = y1;
                imf_image dsi = ds, ddi = dd;
                if (pipe) {  // one image of the batch per launch sequence
                    dsi.data = (char*)dsrc + (size_t)sdev * dsz;
                    ddi.data = (char*)ddst + (size_t)ddev * dsz;
                    dsi.batch = ddi.batch = 1;
                } else {
                    o.row_begin = o.row_end = 0;
                }
                if (!rc)
                    rc = imf_filter(&dsi, &ddi, kernel, target, (const int32_t*)dtm, tmin, tmax, &o, wsl,
                                    ws_need, cs);
                mark("filtered", nstripe - 1, cs);
                cudaEvent_t e_done = event();
                cudaEventRecord(e_done, cs);
                cudaStreamWaitEvent(g_hs.down, e_done, 0);
                if (!rc) {
                    if (pipe) {
                        const size_t off = (size_t)(dbase + (long long)y0 * dst->stride_y) * dsz;
                        const size_t doff = (size_t)(ddev + (long long)y0 * dst->stride_y) * dsz;
                        const size_t len = std::min({(size_t)((long long)(y1 - y0) * dst->stride_y) * dsz, db - off,
                                                     dbA - doff});
                        if (cudaMemcpyAsync((char*)dst->data + off, (char*)ddst + doff, len, cudaMemcpyDeviceToHost,
                                            g_hs.down))
                            rc = cuda_fail(cudaGetLastError(), "stripe download");
                    } else if (cudaMemcpyAsync(dst->data, ddst, db, cudaMemcpyDeviceToHost, g_hs.down)) {
                        rc = cuda_fail(cudaGetLastError(), "download");
                    }
                }
                mark("downloaded", nstripe - 1, g_hs.down);
                if (!pipe) break;
            }
            if (ring) {
                slot_free[slot] = event();
                cudaEventRecord(slot_free[slot], g_hs.down);
            }
            if (!pipe) break;
        }
    }
    cudaEvent_t e_end = event();
    cudaEventRecord(e_end, g_hs.down);
    cudaStreamWaitEvent(s, e_end, 0);
    for (int i = 1; i < nl; i++) {
        cudaEvent_t e_c = event();
        cudaEventRecord(e_c, g_hs.comp[i]);
        cudaStreamWaitEvent(s, e_c, 0);
    }
    // every lane's status word in one pinned read; one synchronization for the call
    const int nst = rc ? 0 : std::min(nl, std::max(nstripe, 1));
    for (int i = 0; i < nst; i++) {
        g_hs.status_h[i] = 0;
        if (cudaError_t e = cudaMemcpyAsync(g_hs.status_h + i, dws[i], sizeof(int), cudaMemcpyDeviceToHost, s)) {
            rc = cuda_fail(e, "status read");
            break;
        }
    }
    if (dsrc) cudaFreeAsync(dsrc, s);
    if (ddst) cudaFreeAsync(ddst, s);
    for (int i = 0; i < nl; i++)
        if (dws[i]) cudaFreeAsync(dws[i], s);
    if (dtm) cudaFreeAsync(dtm, s);
    if (cudaError_t e = cudaStreamSynchronize(s)) {
        if (!rc) rc = cuda_fail(e, "stream synchronize");
    }
    for (int i = 0; i < nst && !rc; i++)
        if (g_hs.status_h[i]) rc = IMF_ERR_DEFECT;
    if (trace && !tl.empty()) {
        for (auto& kv : tl) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, tl[0].second, kv.second);
            fprintf(stderr, "imf_host_trace %-14s %8.3f ms\n", kv.first.c_str(), ms);
        }
    }
    for (cudaEvent_t e : evs) cudaEventDestroy(e);
    return rc;
}

const char* imf_strerror(int status) {
    switch (status) {
        case IMF_OK: return "ok";
        case IMF_ERR_INVALID: return "invalid argument";
        case IMF_ERR_CUDA: return "CUDA runtime error";
        case IMF_ERR_DEFECT: return "segment scan exhausted; pivot/count state was inconsistent";
        case IMF_ERR_WORKSPACE: return "workspace too small";
        case IMF_ERR_UNSUPPORTED: return "unsupported geometry";
        default: return "unknown status";
    }
}

int imf_version(void) { return 100; }

const char* imf_last_error(void) { return g_err; }

uint64_t imf_launch_count(void) { return g_launches.load(); }

}  // extern "C"
