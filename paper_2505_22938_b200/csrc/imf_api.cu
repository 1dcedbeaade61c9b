// imf_api.cu -- extern "C" entry points (include/isomedian_b200.h) and the
// launch planner: tile geometry, quantization of the ordinal image, chunking
// of the tile stream through an L2-sized omega scratch, K1/K2 launches.
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../../include/isomedian_b200.h"
#include "imf_common.cuh"


using namespace imf;

static std::atomic<uint64_t> g_launches{0};
static thread_local char g_err[256];

static int cuda_fail(cudaError_t e, const char* where) {
    snprintf(g_err, sizeof(g_err), "%s: %s", where, cudaGetErrorString(e));
    return IMF_ERR_CUDA;
}

namespace {

constexpr size_t kSmemMax = 227 * 1024 - 1024;  // B200 opt-in 232448 B minus static smem headroom
constexpr int kK1Threads = 512;
constexpr size_t kStatusBytes = 256;
constexpr size_t kOmegaScratchTarget = 96ull << 20;  // stays mostly L2-resident

struct Plan {
    Geom g;
    int G, K, k2_threads, k1_threads;
    bool k1_gmem;
    size_t k1_smem, k2_smem, k1_gs_per_tile;
    long long total_tiles, chunk_tiles;
    int qs, qb, P_lo, P_hi;
    size_t ws_ktab, ws_omega, ws_k1g, ws_total;
    int ktab_n;
};

int env_int(const char* name, int dflt) {
    const char* v = getenv(name);
    return v && *v ? atoi(v) : dflt;
}

int dtype_size(int dt) { return dt == IMF_DTYPE_U8 ? 1 : (dt == IMF_DTYPE_U16 ? 2 : 4); }

int make_plan(const imf_image* src, const imf_kernel* k, const imf_options* opt, int tmin, int tmax,
              Plan* pl) {
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
    if (tmin < 0 || tmax >= k->area || tmin > tmax) return IMF_ERR_INVALID;

    Plan& p = *pl;
    memset(&p, 0, sizeof(p));
    int T = opt->tile_size > 0 ? opt->tile_size : env_int("IMF_TILE", 64);
    T = std::min(T, 256 - 2 * r);
    T = std::max(T, 1);
    const int G0 = opt->seed_rows > 0 ? opt->seed_rows : env_int("IMF_SEED_ROWS", 4);
    for (;; T = T > 8 ? T - 4 : T - 1) {
        if (T < 1) return IMF_ERR_UNSUPPORTED;
        const int S = T + 2 * r;
        const int N = S * S, Npad = (N + 63) & ~63;
        const int G = std::max(1, std::min(G0, T));
        int K = opt->seeds_per_row > 0 ? opt->seeds_per_row : env_int("IMF_SEEDS", std::max(1, T / 16));
        K = std::max(1, std::min(K, T));
        const int thr = ((T * G * 2 + 31) / 32) * 32;
        const int k2thr = std::min(thr, 512);
        const size_t k2s = k2_smem_bytes(N, Npad, k->ncols, k->nrows, r, G, K, T, k2thr / 32);
        if (k2s > kSmemMax) continue;
        p.g.Tw = p.g.Th = T;
        p.g.Sw = p.g.Sh = S;
        p.g.N = N;
        p.g.Npad = Npad;
        p.G = G;
        p.K = K;
        p.k2_threads = k2thr;
        p.k2_smem = k2s;
        break;
    }
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
    g.out_h = out_h;
    g.out_w = out_w;
    g.vshift = valid ? r : 0;
    g.r = r;
    g.tiles_x = (out_w + g.Tw - 1) / g.Tw;
    g.tiles_y = (out_h + g.Th - 1) / g.Th;
    p.total_tiles = (long long)g.tiles_x * g.tiles_y * g.C * g.B;

    p.k1_threads = kK1Threads;
    p.k1_gmem = k1_smem_bytes(g.dtype, g.Npad, p.k1_threads / 32, false) > kSmemMax;
    p.k1_smem = k1_smem_bytes(g.dtype, g.Npad, p.k1_threads / 32, p.k1_gmem);
    p.k1_gs_per_tile = p.k1_gmem ? k1_gscratch_bytes(g.dtype, g.Npad) : 0;

    // Quantization of the ordinal image: smallest qs >= 6 such that
    // every pivot nearest a possible solution rank in [tmin, N - area + tmax] has
    // (P >> qs) - qb within [1, 255].  Pivots are clamped to [P_lo, P_hi] anyway,
    // so exactness never depends on this choice -- only the refine distance does.
    const int lo = tmin, hi = g.N - k->area + tmax;
    int qs = 6, qb = 0;
    for (; qs < 16; qs++) {
        qb = std::max(0, (lo >> qs) - 1);
        const int pmax = ((hi + (1 << (qs - 1))) >> qs) - qb;
        if (pmax <= 255) break;
    }
    p.qs = qs;
    p.qb = qb;
    p.P_lo = (qb + 1) << qs;
    const int ncap = ((g.N + (1 << qs) - 1) >> qs) << qs;
    p.P_hi = std::max(p.P_lo, std::min((qb + 255) << qs, ncap));

    p.ktab_n = 2 * k->ncols + 2 * k->nrows + 2 * r + 1;
    const size_t per_tile = 2 * (size_t)g.Npad + p.k1_gs_per_tile;
    long long chunk = (long long)(kOmegaScratchTarget / per_tile);
    chunk = std::max<long long>(chunk, 148);
    chunk = std::min<long long>(chunk, p.total_tiles);
    chunk = std::min<long long>(chunk, 65535LL * 1024);
    p.chunk_tiles = chunk;
    p.ws_ktab = ((size_t)p.ktab_n * 4 + 255) & ~(size_t)255;
    p.ws_omega = (size_t)chunk * 2 * g.Npad;
    p.ws_k1g = (size_t)chunk * p.k1_gs_per_tile;
    p.ws_total = kStatusBytes + p.ws_ktab + p.ws_omega + p.ws_k1g;
    return IMF_OK;
}

void build_ktab(const imf_kernel* k, int Sw, std::vector<int>& t) {
    const int r = k->radius;
    t.assign(2 * k->ncols + 2 * k->nrows + 2 * r + 1, 0);
    int o = 0;
    for (int i = 0; i < k->ncols; i++) {
        t[o++] = (k->col_ybot[i] + 1) * Sw + k->col_dx[i];  // VE: entering on a down slide
        t[o++] = k->col_ytop[i] * Sw + k->col_dx[i];        // VX: exiting on a down slide
    }
    for (int i = 0; i < k->nrows; i++) {
        t[o++] = k->row_dy[i] * Sw + k->row_xhi[i];  // HP: entering on a right slide
        t[o++] = k->row_dy[i] * Sw + k->row_xlo[i];  // HM: exiting on a right slide
    }
    for (int i = 0; i < k->nrows; i++) {
        const int dy = k->row_dy[i];
        const int w = k->row_xhi[i] - k->row_xlo[i];
        t[o + dy + r] = (k->row_xlo[i] & 0xffff) | (w << 16);
    }
}

bool g_attr_done = false;

template <typename F>
cudaError_t allow_smem(F* f, int optin) {
    cudaFuncAttributes a;
    cudaError_t e = cudaFuncGetAttributes(&a, f);
    if (e) return e;
    return cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                optin - (int)a.sharedSizeBytes);
}

cudaError_t set_attrs() {
    if (g_attr_done) return cudaSuccess;
    int dev = 0, optin = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (!e) e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (!e) e = allow_smem(k1_sort<DT_U8, false>, optin);
    if (!e) e = allow_smem(k1_sort<DT_U16, false>, optin);
    if (!e) e = allow_smem(k1_sort<DT_U16, true>, optin);
    if (!e) e = allow_smem(k1_sort<DT_F32, false>, optin);
    if (!e) e = allow_smem(k1_sort<DT_F32, true>, optin);
    if (!e) e = allow_smem(k2_select<true>, optin);
    if (!e) e = allow_smem(k2_select<false>, optin);
    if (!e) g_attr_done = true;
    return e;
}

void launch_k1(const Plan& p, const Geom& g, int nblocks, uint16_t* omega, unsigned char* k1g,
               cudaStream_t s) {
    const dim3 grid(nblocks), block(p.k1_threads);
    const long long gs = (long long)p.k1_gs_per_tile;
    switch (g.dtype * 2 + (p.k1_gmem ? 1 : 0)) {
        case 0:
        case 1: k1_sort<DT_U8, false><<<grid, block, p.k1_smem, s>>>(g, omega, k1g, gs); break;
        case 2: k1_sort<DT_U16, false><<<grid, block, p.k1_smem, s>>>(g, omega, k1g, gs); break;
        case 3: k1_sort<DT_U16, true><<<grid, block, p.k1_smem, s>>>(g, omega, k1g, gs); break;
        case 4: k1_sort<DT_F32, false><<<grid, block, p.k1_smem, s>>>(g, omega, k1g, gs); break;
        default: k1_sort<DT_F32, true><<<grid, block, p.k1_smem, s>>>(g, omega, k1g, gs); break;
    }
}

}  // namespace

extern "C" {

size_t imf_workspace_size(const imf_image* src, const imf_kernel* kernel, const imf_options* opt) {
    Plan p;
    if (make_plan(src, kernel, opt, 0, kernel ? kernel->area - 1 : 0, &p) != IMF_OK) return 0;
    return p.ws_total;
}

int imf_filter(const imf_image* src, imf_image* dst, const imf_kernel* kernel, int32_t target,
               const int32_t* target_map, int32_t tmin, int32_t tmax, const imf_options* opt,
               void* workspace, size_t workspace_bytes, void* stream) {
    if (!dst || !src || !src->data || !dst->data || src->data == dst->data) return IMF_ERR_INVALID;
    if (dst->dtype != src->dtype || dst->batch != src->batch || dst->channels != src->channels)
        return IMF_ERR_INVALID;
    if (!target_map) tmin = tmax = target;
    Plan p;
    int st = make_plan(src, kernel, opt, tmin, tmax, &p);
    if (st) return st;
    if (dst->height != p.g.out_h || dst->width != p.g.out_w) return IMF_ERR_INVALID;
    if (!workspace || workspace_bytes < p.ws_total) return IMF_ERR_WORKSPACE;
    cudaStream_t s = (cudaStream_t)stream;
    if (cudaError_t e = set_attrs()) return cuda_fail(e, "cudaFuncSetAttribute");

    unsigned char* ws = (unsigned char*)workspace;
    int* status = (int*)ws;
    int* ktab_d = (int*)(ws + kStatusBytes);
    uint16_t* omega = (uint16_t*)(ws + kStatusBytes + p.ws_ktab);
    unsigned char* k1g = ws + kStatusBytes + p.ws_ktab + p.ws_omega;

    std::vector<int> ktab;
    build_ktab(kernel, p.g.Sw, ktab);
    if (cudaError_t e = cudaMemsetAsync(status, 0, sizeof(int), s)) return cuda_fail(e, "status memset");
    if (cudaError_t e = cudaMemcpyAsync(ktab_d, ktab.data(), ktab.size() * 4, cudaMemcpyHostToDevice, s))
        return cuda_fail(e, "kernel table upload");

    Geom g = p.g;
    g.src = src->data;
    g.dst = dst->data;
    g.d_b = dst->stride_b;
    g.d_y = dst->stride_y;
    g.d_x = dst->stride_x;
    g.d_c = dst->stride_c;

    SelParams sp;
    memset(&sp, 0, sizeof(sp));
    sp.circle = kernel->shape_code == IMF_SHAPE_CIRCLE;
    sp.R2 = kernel->radius * (kernel->radius + 1);
    sp.ncols = kernel->ncols;
    sp.nrows = kernel->nrows;
    sp.target = target;
    sp.tmap = target_map;
    sp.qs = p.qs;
    sp.qb = p.qb;
    sp.P_lo = p.P_lo;
    sp.P_hi = p.P_hi;
    sp.G = p.G;
    sp.K = p.K;
    sp.ktab = ktab_d;
    sp.status = status;

    for (long long t0 = 0; t0 < p.total_tiles; t0 += p.chunk_tiles) {
        const int nb = (int)std::min(p.chunk_tiles, p.total_tiles - t0);
        g.tile_begin = t0;
        launch_k1(p, g, nb, omega, k1g, s);
        if (sp.circle)
            k2_select<true><<<nb, p.k2_threads, p.k2_smem, s>>>(g, sp, omega);
        else
            k2_select<false><<<nb, p.k2_threads, p.k2_smem, s>>>(g, sp, omega);
        g_launches += 2;
    }
    if (cudaError_t e = cudaGetLastError()) return cuda_fail(e, "kernel launch");
    return IMF_OK;
}

int imf_workspace_status(void* workspace, void* stream) {
    int h = 0;
    if (!workspace) return IMF_ERR_INVALID;
    if (cudaMemcpyAsync(&h, workspace, sizeof(int), cudaMemcpyDeviceToHost, (cudaStream_t)stream) !=
        cudaSuccess)
        return IMF_ERR_CUDA;
    if (cudaStreamSynchronize((cudaStream_t)stream) != cudaSuccess) return IMF_ERR_CUDA;
    return h ? IMF_ERR_DEFECT : IMF_OK;
}

static size_t extent_bytes(const imf_image* im) {
    const long long last = (long long)(im->batch - 1) * im->stride_b +
                           (long long)(im->height - 1) * im->stride_y +
                           (long long)(im->width - 1) * im->stride_x +
                           (long long)(im->channels - 1) * im->stride_c;
    return (size_t)(last + 1) * dtype_size(im->dtype);
}

int imf_filter_host(const imf_image* src, imf_image* dst, const imf_kernel* kernel, int32_t target,
                    const int32_t* target_map, int32_t tmin, int32_t tmax, const imf_options* opt,
                    void* stream) {
    if (!src || !dst || !kernel || !opt) return IMF_ERR_INVALID;
    cudaStream_t s = (cudaStream_t)stream;
    if (!target_map) tmin = tmax = target;
    Plan p;
    int st = make_plan(src, kernel, opt, tmin, tmax, &p);
    if (st) return st;
    const size_t sb = extent_bytes(src), db = extent_bytes(dst);
    const size_t tb = target_map ? (size_t)p.g.out_h * p.g.out_w * 4 : 0;
    void *dsrc = nullptr, *ddst = nullptr, *dws = nullptr, *dtm = nullptr;
    int rc = IMF_OK;
    if (cudaMallocAsync(&dsrc, sb, s) || cudaMallocAsync(&ddst, db, s) ||
        cudaMallocAsync(&dws, p.ws_total, s) || (tb && cudaMallocAsync(&dtm, tb, s))) {
        rc = IMF_ERR_CUDA;
    }
    if (!rc && cudaMemcpyAsync(dsrc, src->data, sb, cudaMemcpyHostToDevice, s)) rc = IMF_ERR_CUDA;
    if (!rc && tb && cudaMemcpyAsync(dtm, target_map, tb, cudaMemcpyHostToDevice, s)) rc = IMF_ERR_CUDA;
    if (!rc) {
        imf_image ds = *src, dd = *dst;
        ds.data = dsrc;
        dd.data = ddst;
        rc = imf_filter(&ds, &dd, kernel, target, (const int32_t*)dtm, tmin, tmax, opt, dws, p.ws_total,
                        stream);
    }
    if (!rc && cudaMemcpyAsync(dst->data, ddst, db, cudaMemcpyDeviceToHost, s)) rc = IMF_ERR_CUDA;
    if (!rc) rc = imf_workspace_status(dws, stream);
    if (dsrc) cudaFreeAsync(dsrc, s);
    if (ddst) cudaFreeAsync(ddst, s);
    if (dws) cudaFreeAsync(dws, s);
    if (dtm) cudaFreeAsync(dtm, s);
    cudaStreamSynchronize(s);
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
