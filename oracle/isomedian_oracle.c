/*
 * isomedian_oracle.c -- CPU restatement of the reference rank-order filter.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker and the CPU
 * baseline for bench.py; it is never linked into, loaded by, or called from
 * the product path (paper_2505_22938_b200/), which runs on the GPU or fails.
 *
 * It restates, in plain C, the algorithm of the reference Python/numba
 * package `isomedian` (arXiv 2505.22938, /root/reference/pkg/src/isomedian):
 *
 *   fast engine  (the reference's filter_image, the CPU path we time):
 *     orc_filter_fast    <- tiling.py:213-249  (filter_image), :94-131 decompose,
 *                           :134-145 pad_image, :165-177 targets, :180-210 _run_column
 *     ordinal_transform  <- ordinal.py:126-172, _rank_by_bucket :62-79,
 *                           _rank_by_radix16 :82-106, float_order_key :109-123
 *     process_tile       <- core.py:175-221 (_process_tile) with _seed_state :47-60,
 *                           _slide_right :63-72, _slide_down :75-84, _refine :87-146,
 *                           _select_pivot :39-44, _segment_mask ordinal.py:188-199,
 *                           _inside ordinal.py:175-185
 *     forwarding         <- core.py:149-172 (_forwarded_states), :369-409
 *   brute engine (the reference's oracle):
 *     orc_filter_brute   <- oracle.py:36-121 (gather every window, pick rank t;
 *                           floats ordered through the u32 key, oracle.py:26-33)
 *
 * Data model at this ABI: one single-channel image of u32 *order keys*
 * (u8/u16 values unchanged, f32 mapped by float_order_key), row-major, plus
 * the dtype code that selects the reference's ranking routine (256-bucket,
 * 65536-bucket, or 2x16-bit radix).  The caller (oracle/__init__.py) maps
 * dtypes and channels exactly like filter_image's per-channel recursion.
 * Compile with -ffp-contract=off: the polygon test must round a*dx and b*dy
 * separately, as numba/numpy do.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

#define ORC_DT_U8 0
#define ORC_DT_U16 1
#define ORC_DT_F32 2

typedef struct {
    int code;          /* 0 circle, 1 square, 2 polygon (kernels.py:135) */
    int rad;
    int64_t lim;       /* (2r+1)^2 */
    int nplanes;
    const double *planes;  /* nplanes x 3 */
    int area;
    const int32_t *off_dx, *off_dy;
    int nrows;
    const int32_t *row_dy, *row_xlo, *row_xhi;
    int ncols;
    const int32_t *col_dx, *col_ytop, *col_ybot;
} orc_kernel;

/* ordinal.py:175-185 */
static inline int inside(const orc_kernel *k, int64_t dx, int64_t dy) {
    if (k->code == 0) return 4 * (dx * dx + dy * dy) <= k->lim;
    if (k->code == 1) return -k->rad <= dx && dx <= k->rad && -k->rad <= dy && dy <= k->rad;
    for (int i = 0; i < k->nplanes; i++) {
        const double *p = k->planes + 3 * i;
        double a = p[0] * (double)dx;
        double b = p[1] * (double)dy;
        if (a + b > p[2]) return 0;
    }
    return 1;
}

/* ---------------------------------------------------------------- ordinal */

typedef struct {
    int h, w, n;
    int32_t *ranks;   /* h*w */
    int32_t *pos_x, *pos_y;
    uint32_t *values; /* keys in ascending order */
} orc_tile;

typedef struct {   /* per-worker scratch, sized for the largest tile */
    int32_t *hist;   /* 65536 */
    int64_t *hist64;
    int32_t *perm, *tmp, *rflat;
    uint32_t *keys;
    orc_tile ot;
    int32_t *m_out;
    int64_t *pivots, *counts;
    int64_t *seed_pivots, *seed_counts;
    int32_t *prev_m, *prev_offdx, *prev_offdy;
    int64_t *targets;
} orc_scratch;

/* ordinal.py:62-79: stable single-pass bucket ranks */
static void rank_by_bucket(const uint32_t *vals, int n, int nb, int32_t *hist, int32_t *out) {
    memset(hist, 0, sizeof(int32_t) * nb);
    for (int i = 0; i < n; i++) hist[vals[i]]++;
    int32_t total = 0;
    for (int k = 0; k < nb; k++) { int32_t c = hist[k]; hist[k] = total; total += c; }
    for (int i = 0; i < n; i++) out[i] = hist[vals[i]]++;
}

/* ordinal.py:82-106: stable ranks of u32 keys via two 16-bit counting passes */
static void rank_by_radix16(const uint32_t *keys, int n, int64_t *hist, int32_t *perm,
                            int32_t *tmp, int32_t *out) {
    for (int i = 0; i < n; i++) perm[i] = i;
    for (int shift = 0; shift <= 16; shift += 16) {
        memset(hist, 0, sizeof(int64_t) * 65536);
        for (int i = 0; i < n; i++) hist[(keys[perm[i]] >> shift) & 0xFFFF]++;
        int64_t total = 0;
        for (int k = 0; k < 65536; k++) { int64_t c = hist[k]; hist[k] = total; total += c; }
        for (int i = 0; i < n; i++) {
            uint32_t d = (keys[perm[i]] >> shift) & 0xFFFF;
            tmp[hist[d]++] = perm[i];
        }
        int32_t *t = perm; perm = tmp; tmp = t;
    }
    for (int v = 0; v < n; v++) out[perm[v]] = v;
}

/* ordinal.py:126-172 (no validity mask): tile is h x w keys, row stride `stride` */
static void ordinal_transform(const uint32_t *tile, int64_t stride, int h, int w, int dtype,
                              orc_scratch *s) {
    int n = h * w;
    orc_tile *ot = &s->ot;
    ot->h = h; ot->w = w; ot->n = n;
    for (int y = 0; y < h; y++) memcpy(s->keys + (int64_t)y * w, tile + y * stride, sizeof(uint32_t) * w);
    if (dtype == ORC_DT_U8) rank_by_bucket(s->keys, n, 256, s->hist, s->rflat);
    else if (dtype == ORC_DT_U16) rank_by_bucket(s->keys, n, 65536, s->hist, s->rflat);
    else rank_by_radix16(s->keys, n, s->hist64, s->perm, s->tmp, s->rflat);
    for (int i = 0; i < n; i++) {
        int32_t rk = s->rflat[i];
        ot->ranks[i] = rk;
        ot->pos_x[rk] = i % w;
        ot->pos_y[rk] = i / w;
        ot->values[rk] = s->keys[i];
    }
}

/* ------------------------------------------------------------------ core */

/* core.py:39-44 */
static inline int64_t select_pivot(int64_t m, int64_t n) {
    int64_t p = 64 * ((m + 32) >> 6);
    int64_t cap = 64 * ((n - 1) >> 6);
    return p <= cap ? p : cap;
}

/* ordinal.py:188-199 */
static inline uint64_t segment_mask(const orc_tile *ot, int64_t seg, int64_t cx, int64_t cy,
                                    const orc_kernel *k, int *pop) {
    int64_t base = seg * 64;
    int64_t end = base + 64 < ot->n ? base + 64 : ot->n;
    uint64_t mask = 0; int c = 0;
    for (int64_t v = base; v < end; v++) {
        if (inside(k, ot->pos_x[v] - cx, ot->pos_y[v] - cy)) { mask |= 1ull << (v - base); c++; }
    }
    *pop = c;
    return mask;
}

/* core.py:47-60 */
static void seed_state(const orc_tile *ot, int64_t cx, int64_t cy, const orc_kernel *k,
                       int64_t target, int64_t *hist, int64_t *piv, int64_t *cnt) {
    int64_t nbins = ((ot->n - 1) >> 6) + 1;
    memset(hist, 0, sizeof(int64_t) * nbins);
    for (int i = 0; i < k->area; i++) {
        int32_t v = ot->ranks[(cy + k->off_dy[i]) * ot->w + cx + k->off_dx[i]];
        hist[v >> 6]++;
    }
    int64_t c = 0, b = 0;
    while (c + hist[b] <= target) { c += hist[b]; b++; }
    *piv = 64 * b; *cnt = c;
}

/* core.py:63-72 */
static inline int64_t slide_right(const orc_tile *ot, int64_t cx, int64_t cy, int64_t pivot,
                                  int64_t count, const orc_kernel *k) {
    for (int i = 0; i < k->nrows; i++) {
        const int32_t *row = ot->ranks + (cy + k->row_dy[i]) * ot->w;
        if (row[cx + k->row_xhi[i]] < pivot) count++;
        if (row[cx + k->row_xlo[i]] < pivot) count--;
    }
    return count;
}

/* core.py:75-84 */
static inline int64_t slide_down(const orc_tile *ot, int64_t cx, int64_t cy, int64_t pivot,
                                 int64_t count, const orc_kernel *k) {
    for (int i = 0; i < k->ncols; i++) {
        int64_t x = cx + k->col_dx[i];
        if (ot->ranks[(cy + k->col_ybot[i] + 1) * ot->w + x] < pivot) count++;
        if (ot->ranks[(cy + k->col_ytop[i]) * ot->w + x] < pivot) count--;
    }
    return count;
}

static inline int64_t kth_bit(uint64_t mask, int64_t need) {
    int64_t seen = 0;
    for (int b = 0; b < 64; b++) {
        if ((mask >> b) & 1ull) { if (seen == need) return b; seen++; }
    }
    return -1;
}

/* Optional segment statistics (bench.py reports the measured S-bar of
 * 64-rank segments scanned per refined window).  Off by
 * default; one predictable branch per refine when off. */
static int g_seg_on = 0;
static long long g_seg_total = 0, g_refine_total = 0;

void orc_segment_stats(int enable, long long *segments, long long *refines) {
    if (segments) *segments = __atomic_load_n(&g_seg_total, __ATOMIC_RELAXED);
    if (refines) *refines = __atomic_load_n(&g_refine_total, __ATOMIC_RELAXED);
    if (enable >= 0) {
        g_seg_on = enable;
        __atomic_store_n(&g_seg_total, 0, __ATOMIC_RELAXED);
        __atomic_store_n(&g_refine_total, 0, __ATOMIC_RELAXED);
    }
}

static int64_t refine_(const orc_tile *ot, int64_t cx, int64_t cy, int64_t pivot, int64_t count,
                       int64_t target, const orc_kernel *k, int64_t *npiv_out, int64_t *ncnt_out,
                       long long *segs);

static int64_t refine(const orc_tile *ot, int64_t cx, int64_t cy, int64_t pivot, int64_t count,
                      int64_t target, const orc_kernel *k, int64_t *npiv_out, int64_t *ncnt_out) {
    long long segs = 0;
    int64_t m = refine_(ot, cx, cy, pivot, count, target, k, npiv_out, ncnt_out, &segs);
    if (g_seg_on) {
        __atomic_add_fetch(&g_seg_total, segs, __ATOMIC_RELAXED);
        __atomic_add_fetch(&g_refine_total, 1, __ATOMIC_RELAXED);
    }
    return m;
}

/* core.py:87-146; returns m (-1 on an inconsistent count) */
static int64_t refine_(const orc_tile *ot, int64_t cx, int64_t cy, int64_t pivot, int64_t count,
                       int64_t target, const orc_kernel *k, int64_t *npiv_out, int64_t *ncnt_out,
                       long long *segs) {
    int64_t n = ot->n;
    int64_t cap = 64 * ((n - 1) >> 6);
    int64_t s = pivot >> 6, c = count;
    int pop;
    if (count <= target) {
        for (;;) {
            if (s * 64 >= n) return -1;
            uint64_t mask = segment_mask(ot, s, cx, cy, k, &pop);
            (*segs)++;
            if (c + pop > target) {
                int64_t kb = kth_bit(mask, target - c);
                int64_t m = kb < 0 ? -1 : s * 64 + kb;
                int64_t npiv = 64 * ((m + 32) >> 6);
                if (npiv > cap) npiv = cap;
                *npiv_out = npiv;
                *ncnt_out = (npiv == 64 * s) ? c : c + pop;
                return m;
            }
            c += pop; s++;
        }
    } else {
        for (;;) {
            s--;
            if (s < 0) return -1;
            uint64_t mask = segment_mask(ot, s, cx, cy, k, &pop);
            (*segs)++;
            int64_t base_c = c - pop;
            if (base_c <= target) {
                int64_t kb = kth_bit(mask, target - base_c);
                int64_t m = kb < 0 ? -1 : s * 64 + kb;
                int64_t npiv = 64 * ((m + 32) >> 6);
                if (npiv > cap) npiv = cap;
                *npiv_out = npiv;
                *ncnt_out = (npiv == 64 * s) ? base_c : c;
                return m;
            }
            c = base_c;
        }
    }
}

/* core.py:149-172 */
static void forwarded_states(const orc_tile *ot, int64_t cx0, int64_t cy, const int32_t *seed_m,
                             const int64_t *seed_targets, int out_w, const orc_kernel *k,
                             int64_t *pivots, int64_t *counts) {
    for (int j = 0; j < out_w; j++) {
        int64_t cx = cx0 + j, m = seed_m[j];
        int64_t piv = select_pivot(m, ot->n);
        int64_t c = seed_targets[j];
        if (piv <= m) {
            for (int64_t v = piv; v < m; v++)
                if (inside(k, ot->pos_x[v] - cx, ot->pos_y[v] - cy)) c--;
        } else {
            for (int64_t v = m; v < piv; v++)
                if (inside(k, ot->pos_x[v] - cx, ot->pos_y[v] - cy)) c++;
        }
        pivots[j] = piv; counts[j] = c;
    }
}

/* core.py:175-221; targets out_h x out_w (row stride out_w); returns 0/1 */
static int process_tile(const orc_tile *ot, const orc_kernel *k, int64_t cx0, int64_t cy0,
                        const int64_t *targets, int out_h, int out_w, int seeded,
                        const int64_t *seed_pivots, const int64_t *seed_counts,
                        int32_t *m_out, int64_t *pivots, int64_t *counts, int64_t *hist) {
    int row_start;
    int64_t piv, c, m;
    if (seeded) {
        for (int j = 0; j < out_w; j++) { pivots[j] = seed_pivots[j]; counts[j] = seed_counts[j]; }
        row_start = 0;
    } else {
        seed_state(ot, cx0, cy0, k, targets[0], hist, &piv, &c);
        m = refine(ot, cx0, cy0, piv, c, targets[0], k, &piv, &c);
        if (m < 0) return 1;
        m_out[0] = (int32_t)m; pivots[0] = piv; counts[0] = c;
        for (int j = 1; j < out_w; j++) {
            c = slide_right(ot, cx0 + j - 1, cy0, piv, c, k);
            m = refine(ot, cx0 + j, cy0, piv, c, targets[j], k, &piv, &c);
            if (m < 0) return 1;
            m_out[j] = (int32_t)m; pivots[j] = piv; counts[j] = c;
        }
        row_start = 1;
    }
    for (int i = row_start; i < out_h; i++) {
        int64_t cy = cy0 + i;
        for (int j = 0; j < out_w; j++) {
            int64_t cx = cx0 + j;
            c = slide_down(ot, cx, cy - 1, pivots[j], counts[j], k);
            m = refine(ot, cx, cy, pivots[j], c, targets[(int64_t)i * out_w + j], k, &piv, &c);
            if (m < 0) return 1;
            m_out[(int64_t)i * out_w + j] = (int32_t)m; pivots[j] = piv; counts[j] = c;
        }
    }
    return 0;
}

/* ---------------------------------------------------------------- tiling */

typedef struct {
    const uint32_t *padded; int64_t pw;   /* padded image (H+2r or H) x pw */
    uint32_t *out; int out_h, out_w;
    const int64_t *target_map; int64_t target;   /* map nullable */
    const orc_kernel *k;
    int r, T, forwarding, dtype;
    int ncols_units;
    int next_unit; pthread_mutex_t mu;
    int status;
} orc_job;

static int alloc_scratch(orc_scratch *s, int max_side, int T) {
    int64_t nmax = (int64_t)max_side * max_side;
    memset(s, 0, sizeof(*s));
    s->hist = malloc(sizeof(int32_t) * 65536);
    s->hist64 = malloc(sizeof(int64_t) * 65536);
    s->perm = malloc(sizeof(int32_t) * nmax);
    s->tmp = malloc(sizeof(int32_t) * nmax);
    s->rflat = malloc(sizeof(int32_t) * nmax);
    s->keys = malloc(sizeof(uint32_t) * nmax);
    s->ot.ranks = malloc(sizeof(int32_t) * nmax);
    s->ot.pos_x = malloc(sizeof(int32_t) * nmax);
    s->ot.pos_y = malloc(sizeof(int32_t) * nmax);
    s->ot.values = malloc(sizeof(uint32_t) * nmax);
    s->m_out = malloc(sizeof(int32_t) * T * T);
    s->targets = malloc(sizeof(int64_t) * T * T);
    s->pivots = malloc(sizeof(int64_t) * T);
    s->counts = malloc(sizeof(int64_t) * T);
    s->seed_pivots = malloc(sizeof(int64_t) * T);
    s->seed_counts = malloc(sizeof(int64_t) * T);
    s->prev_m = malloc(sizeof(int32_t) * T);
    s->prev_offdx = malloc(sizeof(int32_t) * T);
    s->prev_offdy = malloc(sizeof(int32_t) * T);
    return s->hist && s->hist64 && s->perm && s->tmp && s->rflat && s->keys && s->ot.ranks &&
           s->ot.pos_x && s->ot.pos_y && s->ot.values && s->m_out && s->targets && s->pivots &&
           s->counts && s->seed_pivots && s->seed_counts && s->prev_m && s->prev_offdx && s->prev_offdy;
}

static void free_scratch(orc_scratch *s) {
    free(s->hist); free(s->hist64); free(s->perm); free(s->tmp); free(s->rflat); free(s->keys);
    free(s->ot.ranks); free(s->ot.pos_x); free(s->ot.pos_y); free(s->ot.values);
    free(s->m_out); free(s->targets); free(s->pivots); free(s->counts);
    free(s->seed_pivots); free(s->seed_counts); free(s->prev_m); free(s->prev_offdx); free(s->prev_offdy);
}

/* tiling.py:180-210 for one unit: a tile column (forwarding) or a single tile */
static int run_unit(orc_job *job, orc_scratch *s, int x0, int y_first, int y_last_excl) {
    const orc_kernel *k = job->k;
    int r = job->r, T = job->T;
    int tw = job->out_w - x0 < T ? job->out_w - x0 : T;
    int have_prev = 0;
    int64_t prev_in_y0 = 0, prev_cy_last = 0;
    for (int y0 = y_first; y0 < y_last_excl; y0 += T) {
        int th = job->out_h - y0 < T ? job->out_h - y0 : T;
        int seeded = job->forwarding && y0 > 0;
        int64_t in_y0 = y0 - (seeded ? 1 : 0);
        int in_h = th + 2 * r + (seeded ? 1 : 0), in_w = tw + 2 * r;
        ordinal_transform(job->padded + in_y0 * job->pw + x0, job->pw, in_h, in_w, job->dtype, s);
        const orc_tile *ot = &s->ot;
        int64_t cx0 = r, cy0 = r + (seeded ? 1 : 0);
        for (int i = 0; i < th; i++)
            for (int j = 0; j < tw; j++)
                s->targets[i * tw + j] = job->target_map
                    ? job->target_map[(int64_t)(y0 + i) * job->out_w + x0 + j] : job->target;
        if (seeded) {
            if (!have_prev) return 1;
            /* core.py:369-409: previous tile's last row re-anchored one row up */
            int64_t dy = prev_in_y0 - in_y0;
            int64_t cy = prev_cy_last + dy;
            for (int j = 0; j < tw; j++) {
                int64_t px = cx0 + j + s->prev_offdx[j];
                int64_t py = cy + s->prev_offdy[j];
                if (py < 0 || py >= ot->h || px < 0 || px >= ot->w) return 1;
                s->prev_m[j] = ot->ranks[py * ot->w + px];
            }
            int64_t seed_t[256];
            for (int j = 0; j < tw; j++)
                seed_t[j] = job->target_map ? job->target_map[(int64_t)(y0 - 1) * job->out_w + x0 + j]
                                            : job->target;
            forwarded_states(ot, cx0, cy, s->prev_m, seed_t, tw, k, s->seed_pivots, s->seed_counts);
        }
        if (process_tile(ot, k, cx0, cy0, s->targets, th, tw, seeded, s->seed_pivots,
                         s->seed_counts, s->m_out, s->pivots, s->counts, s->hist64))
            return 1;
        for (int i = 0; i < th; i++)
            for (int j = 0; j < tw; j++)
                job->out[(int64_t)(y0 + i) * job->out_w + x0 + j] = ot->values[s->m_out[i * tw + j]];
        if (job->forwarding) {
            int64_t cy_last = cy0 + th - 1;
            for (int j = 0; j < tw; j++) {
                int32_t m = s->m_out[(th - 1) * tw + j];
                s->prev_offdx[j] = ot->pos_x[m] - (int32_t)(cx0 + j);
                s->prev_offdy[j] = ot->pos_y[m] - (int32_t)cy_last;
            }
            have_prev = 1; prev_in_y0 = in_y0; prev_cy_last = cy_last;
        }
    }
    return 0;
}

static void *worker(void *arg) {
    orc_job *job = arg;
    orc_scratch s;
    int ok = alloc_scratch(&s, 257, job->T);
    int tiles_y = (job->out_h + job->T - 1) / job->T;
    for (;;) {
        pthread_mutex_lock(&job->mu);
        int u = job->next_unit++;
        int bad = job->status || !ok;
        if (!ok) job->status = 2;
        pthread_mutex_unlock(&job->mu);
        if (bad || u >= job->ncols_units) break;
        int st;
        if (job->forwarding) {
            st = run_unit(job, &s, u * job->T, 0, job->out_h);
        } else {
            int cx = u / tiles_y, ty = u % tiles_y;
            st = run_unit(job, &s, cx * job->T, ty * job->T, ty * job->T + 1);
        }
        if (st) { pthread_mutex_lock(&job->mu); job->status = st; pthread_mutex_unlock(&job->mu); }
    }
    free_scratch(&s);
    return NULL;
}

/*
 * Fast engine, one channel.  img: H x W keys (row-major).  boundary 0
 * replicate / 1 valid.  tile_size <= 0 selects the reference default
 * T = min(64, 256 - 2r - forwarding) (tiling.py:119).  target_map (nullable):
 * out_h x out_w int64 target ranks.  Returns 0 ok, 1 scan defect, 2 alloc,
 * 3 bad geometry.
 */
int orc_filter_fast(const uint32_t *img, int H, int W, int dtype, int boundary,
                    const orc_kernel *k, int64_t target, const int64_t *target_map,
                    int tile_size, int forwarding, int nthreads, uint32_t *out) {
    int r = k->rad;
    int out_h = boundary ? H - 2 * r : H, out_w = boundary ? W - 2 * r : W;
    if (out_h <= 0 || out_w <= 0) return 3;
    int T = tile_size > 0 ? tile_size : (64 < 256 - 2 * r - (forwarding ? 1 : 0) ? 64 : 256 - 2 * r - (forwarding ? 1 : 0));
    if (T < 1 || T + 2 * r + (forwarding ? 1 : 0) > 256) return 3;
    /* tiling.py:134-145: replicate pads with edge values (np.pad mode="edge") */
    int64_t ph = boundary ? H : H + 2 * r, pw = boundary ? W : W + 2 * r;
    uint32_t *padded = malloc(sizeof(uint32_t) * ph * pw);
    if (!padded) return 2;
    for (int64_t y = 0; y < ph; y++) {
        int64_t sy = boundary ? y : y - r;
        sy = sy < 0 ? 0 : (sy >= H ? H - 1 : sy);
        for (int64_t x = 0; x < pw; x++) {
            int64_t sx = boundary ? x : x - r;
            sx = sx < 0 ? 0 : (sx >= W ? W - 1 : sx);
            padded[y * pw + x] = img[sy * W + sx];
        }
    }
    orc_job job;
    memset(&job, 0, sizeof(job));
    job.padded = padded; job.pw = pw; job.out = out; job.out_h = out_h; job.out_w = out_w;
    job.target_map = target_map; job.target = target; job.k = k; job.r = r; job.T = T;
    job.forwarding = forwarding; job.dtype = dtype;
    int tiles_x = (out_w + T - 1) / T, tiles_y = (out_h + T - 1) / T;
    job.ncols_units = forwarding ? tiles_x : tiles_x * tiles_y;
    pthread_mutex_init(&job.mu, NULL);
    int nt = nthreads < 1 ? 1 : nthreads;
    if (nt > job.ncols_units) nt = job.ncols_units;
    if (nt <= 1) {
        worker(&job);
    } else {
        pthread_t *th = malloc(sizeof(pthread_t) * nt);
        for (int i = 0; i < nt; i++) pthread_create(&th[i], NULL, worker, &job);
        for (int i = 0; i < nt; i++) pthread_join(th[i], NULL);
        free(th);
    }
    pthread_mutex_destroy(&job.mu);
    free(padded);
    return job.status;
}

/* ----------------------------------------------------------------- brute */

static uint32_t quickselect(uint32_t *a, int n, int t) {
    int lo = 0, hi = n - 1;
    while (lo < hi) {
        uint32_t pv = a[lo + (hi - lo) / 2];
        int i = lo, j = hi;
        while (i <= j) {
            while (a[i] < pv) i++;
            while (a[j] > pv) j--;
            if (i <= j) { uint32_t x = a[i]; a[i] = a[j]; a[j] = x; i++; j--; }
        }
        if (t <= j) hi = j; else if (t >= i) lo = i; else return a[t];
    }
    return a[t];
}

typedef struct {
    const uint32_t *img; int H, W, boundary; const orc_kernel *k;
    int64_t target; const int64_t *target_map; uint32_t *out; int out_h, out_w;
    int next_row; pthread_mutex_t mu;
} brute_job;

static void *brute_worker(void *arg) {
    brute_job *b = arg;
    const orc_kernel *k = b->k;
    int r = k->rad;
    uint32_t *buf = malloc(sizeof(uint32_t) * k->area);
    for (;;) {
        pthread_mutex_lock(&b->mu);
        int y = b->next_row++;
        pthread_mutex_unlock(&b->mu);
        if (y >= b->out_h) break;
        for (int x = 0; x < b->out_w; x++) {
            /* center in image coordinates; replicate clamps (np.pad edge) */
            int64_t cy = b->boundary ? y + r : y, cx = b->boundary ? x + r : x;
            for (int i = 0; i < k->area; i++) {
                int64_t sy = cy + k->off_dy[i], sx = cx + k->off_dx[i];
                sy = sy < 0 ? 0 : (sy >= b->H ? b->H - 1 : sy);
                sx = sx < 0 ? 0 : (sx >= b->W ? b->W - 1 : sx);
                buf[i] = b->img[sy * b->W + sx];
            }
            int64_t t = b->target_map ? b->target_map[(int64_t)y * b->out_w + x] : b->target;
            b->out[(int64_t)y * b->out_w + x] = quickselect(buf, k->area, (int)t);
        }
    }
    free(buf);
    return NULL;
}

/* oracle.py:52-121 for one channel (keys in, keys out) */
int orc_filter_brute(const uint32_t *img, int H, int W, int boundary, const orc_kernel *k,
                     int64_t target, const int64_t *target_map, int nthreads, uint32_t *out) {
    int r = k->rad;
    brute_job b;
    memset(&b, 0, sizeof(b));
    b.img = img; b.H = H; b.W = W; b.boundary = boundary; b.k = k; b.target = target;
    b.target_map = target_map; b.out = out;
    b.out_h = boundary ? H - 2 * r : H; b.out_w = boundary ? W - 2 * r : W;
    if (b.out_h <= 0 || b.out_w <= 0) return 3;
    pthread_mutex_init(&b.mu, NULL);
    int nt = nthreads < 1 ? 1 : nthreads;
    pthread_t *th = malloc(sizeof(pthread_t) * nt);
    for (int i = 0; i < nt; i++) pthread_create(&th[i], NULL, brute_worker, &b);
    for (int i = 0; i < nt; i++) pthread_join(th[i], NULL);
    free(th);
    pthread_mutex_destroy(&b.mu);
    return 0;
}

/* Exposed for the oracle's own tests of the rank transform (test_ordinal.py:9-63). */
int orc_ordinal_transform(const uint32_t *tile, int h, int w, int dtype, int32_t *ranks,
                          int32_t *pos_x, int32_t *pos_y, uint32_t *values) {
    orc_scratch s;
    if (h < 1 || w < 1 || h > 256 || w > 256) return 3;
    if (!alloc_scratch(&s, 256, 1)) { free_scratch(&s); return 2; }
    ordinal_transform(tile, w, h, w, dtype, &s);
    int n = h * w;
    memcpy(ranks, s.ot.ranks, sizeof(int32_t) * n);
    memcpy(pos_x, s.ot.pos_x, sizeof(int32_t) * n);
    memcpy(pos_y, s.ot.pos_y, sizeof(int32_t) * n);
    memcpy(values, s.ot.values, sizeof(uint32_t) * n);
    free_scratch(&s);
    return 0;
}
