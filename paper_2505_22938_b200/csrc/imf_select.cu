// imf_select.cu -- K2: per-output-pixel rank selection on sm_100a.
//
// One CTA solves one T_w x T_h output tile from the tile's omega (K1 output).
// Shared memory holds the rank -> position map omega (u16 per rank, packed
// x | y << 8, the paper's omnigram) and the full-precision
// ordinal image I (u16 rank per pixel) of the (T+2r)^2 input tile.
//
// Window state (the reference's pivot/count cursor, core.py module docstring
// and :228-237): a pivot rank P and cnt = #{window pixels with rank < P}.
// Because I keeps exact ranks, the pivot can be ANY rank, so after a window is
// solved its state is simply (P, cnt) = (m, t): the solution rank and the
// target rank (exactly t window pixels rank below the t-th smallest).  The
// reference rounds the pivot to a multiple of 64 to fit its SIMD layout
// (core.py:39-44); the output does not depend on the pivot choice because the
// median is a selection, so both produce the same m.
//
//   A. one direct seed per tile (window at the centre of the tile's middle
//      seed row): every warp histograms part of the window into 32 rank bins
//      (warp ballots), giving a pivot with an exact count, then a
//      warp-collaborative omega scan to the target   (core.py:47-60, :87-146)
//   B. the other seed rows' centre windows: vertical slide deltas at the seed
//      pivot computed in parallel, prefix-summed, then warp-collaborative
//      refines                                          (core.py:75-84)
//   C. every seed-row window: horizontal slide deltas at its row's pivot in
//      parallel, prefix-summed, per-thread refine      (core.py:63-72)
//   D. vertical sweeps up and down from every seed row, one thread per
//      (column, group, direction): slide + refine + write C[m]
//                                                       (core.py:75-84, :87-146, :366)
// The refine walks omega from the pivot toward the target rank testing
// membership of each rank's pixel in the window (ordinal.py:175-199): eight
// ranks per step per thread (phase C/D) or sixty-four per warp step (A/B).
#include "imf_kernels.cuh"

namespace imf {

constexpr unsigned FULLM = 0xffffffffu;
constexpr uint16_t OMEGA_SENTINEL = 0xffffu;  // (255, 255): outside every window (S <= 255)
constexpr int OMEGA_PAD = 8;                  // sentinel entries on both sides of omega

struct Ctx {
    const Geom* g;
    const SelParams* p;
    const uint16_t* om;   // omega, om[-8..-1] and om[N..Npad+7] are sentinels
    const uint16_t* I;    // ordinal image, row stride Sw
    const int* span;      // 2r+1 packed spans (non-circle kernels)
    int N, Sw, r;
};

template <bool CIRCLE>
__device__ __forceinline__ bool inside(const Ctx& c, int x, int y, int cx, int cy) {
    if (CIRCLE) {
        const int dx = x - cx, dy = y - cy;
        return dx * dx + dy * dy <= c.p->R2;
    } else {
        const int dyi = y - cy + c.r;
        if ((unsigned)dyi > (unsigned)(2 * c.r)) return false;
        const int sp = c.span[dyi];
        const int xlo = (int)(short)(sp & 0xffff);
        return (unsigned)(x - cx - xlo) < (unsigned)(sp >> 16);
    }
}

template <bool CIRCLE>
__device__ __forceinline__ bool inside_e(const Ctx& c, uint32_t e, int cx, int cy) {
    return inside<CIRCLE>(c, (int)(e & 0xffu), (int)(e >> 8), cx, cy);
}

// Membership bits of ranks v..v+7 (bit i = rank v+i); v in [-8, N].
template <bool CIRCLE>
__device__ __forceinline__ uint32_t test8(const Ctx& c, int v, int cx, int cy) {
    uint32_t e[8];
#pragma unroll
    for (int i = 0; i < 8; i++) e[i] = c.om[v + i];
    uint32_t m = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) m |= (inside_e<CIRCLE>(c, e[i], cx, cy) ? 1u : 0u) << i;
    return m;
}

// Per-thread refine from an exact state (P, cnt): returns the t-th smallest
// rank of the window (core.py:87-146 restated for exact pivots), or -1 if the
// walk leaves [0, N) (inconsistent state: core.py:31-36 ScanDefectError).
template <bool CIRCLE>
__device__ int refine_thread(const Ctx& c, int cx, int cy, int P, int cnt, int t) {
    // One loop for both directions, so lanes of a warp walking up and lanes
    // walking down share iterations instead of serializing two loops.
    const bool up = cnt <= t;
    int need = up ? t - cnt : cnt - t - 1;  // members to skip (from P outward)
    const int step = up ? 8 : -8;
    for (int v = up ? P : P - 8;; v += step) {
        if (up ? v >= c.N : v <= -8) return -1;
        const uint32_t m = test8<CIRCLE>(c, v, cx, cy);
        const int pc = __popc(m);
        if (need < pc) return v + (int)__fns(m, 0, up ? need + 1 : pc - need);
        need -= pc;
    }
}

// Warp-collaborative refine: all lanes hold the same window;
// lane l tests ranks v0+2l and v0+2l+1 of each 64-rank block.
template <bool CIRCLE>
__device__ int refine_warp(const Ctx& c, int cx, int cy, int P, int cnt, int t) {
    const int lane = threadIdx.x & 31;
    const unsigned lt = lanemask_lt();
    const bool up = cnt <= t;
    int need = up ? t - cnt : cnt - t - 1;
    for (int v0 = up ? P : P - 64;; v0 += up ? 64 : -64) {
        if (up ? v0 >= c.N : v0 + 64 <= 0) return -1;
        const int v = v0 + 2 * lane;
        const bool i0 = v >= 0 && v < c.N && inside_e<CIRCLE>(c, c.om[v], cx, cy);
        const bool i1 = v + 1 >= 0 && v + 1 < c.N && inside_e<CIRCLE>(c, c.om[v + 1], cx, cy);
        const unsigned b0 = __ballot_sync(FULLM, i0), b1 = __ballot_sync(FULLM, i1);
        const int pc = __popc(b0) + __popc(b1);
        if (need < pc) {
            const int k = up ? need : pc - 1 - need;  // index from the bottom of the block
            const int pre = __popc(b0 & lt) + __popc(b1 & lt);
            const bool h0 = i0 && pre == k;
            const bool h1 = i1 && pre + (i0 ? 1 : 0) == k;
            const unsigned hb = __ballot_sync(FULLM, h0 || h1);
            const int L = __ffs(hb) - 1;
            const int off = __shfl_sync(FULLM, h0 ? 0 : 1, L);
            return v0 + 2 * L + off;
        }
        need -= pc;
    }
}

__device__ __forceinline__ int target_at(const Geom& g, const SelParams& p, const TileCoord& tc,
                                         int row, int col) {
    if (!p.tmap) return p.target;
    const int y = min(tc.oy0 + row, g.out_h - 1), x = min(tc.ox0 + col, g.out_w - 1);
    return __ldg(p.tmap + (long long)y * g.out_w + x);
}

// Output = C[m]: the input value at omega[m]'s position (core.py:366).
__device__ __forceinline__ void write_out(const Ctx& c, const TileCoord& tc, int m, int row, int col) {
    const Geom& g = *c.g;
    const int oy = tc.oy0 + row, ox = tc.ox0 + col;
    if (oy >= g.out_h || ox >= g.out_w) return;
    const uint32_t e = c.om[m];
    const long long so = src_offset(g, tc, (int)(e >> 8), (int)(e & 0xff));
    const long long d = tc.b * g.d_b + (long long)oy * g.d_y + (long long)ox * g.d_x + tc.c * g.d_c;
    if (g.dtype == DT_U8) {
        ((uint8_t*)g.dst)[d] = __ldg((const uint8_t*)tc.src + so);
    } else if (g.dtype == DT_U16) {
        ((uint16_t*)g.dst)[d] = __ldg((const uint16_t*)tc.src + so);
    } else {
        ((uint32_t*)g.dst)[d] = __ldg((const uint32_t*)tc.src + so);
    }
}

// acc += (a < P) for a, P in [0, 2^16): the sign bit of a - P (IADD + LEA.HI).
__device__ __forceinline__ void acc_lt(unsigned& acc, unsigned a, unsigned P) {
    asm("{\n\t.reg .u32 t;\n\tsub.u32 t, %1, %2;\n\tshr.u32 t, t, 31;\n\tadd.u32 %0, %0, t;\n\t}"
        : "+r"(acc) : "r"(a), "r"(P));
}

// Count change of a slide, from a BYTE-offset table in the constant bank
// (__grid_constant__ kernel parameter): + #[I[b+e] < P] - #[I[b+x] < P].
__device__ __forceinline__ int slide_delta(const unsigned char* __restrict__ Ib, const int2* tab,
                                           int n, int P, bool swap) {
    unsigned ein = 0, eout = 0;
#pragma unroll 4
    for (int k = 0; k < n; k++) {
        const int2 o = tab[k];
        acc_lt(ein, *reinterpret_cast<const uint16_t*>(Ib + o.x), (unsigned)P);
        acc_lt(eout, *reinterpret_cast<const uint16_t*>(Ib + o.y), (unsigned)P);
    }
    return swap ? (int)eout - (int)ein : (int)ein - (int)eout;
}

// Warp-collaborative slide delta: lanes split the n table entries.
__device__ __forceinline__ int slide_delta_warp(const unsigned char* __restrict__ Ib, const int2* tab,
                                                int n, int P, int lane) {
    unsigned ein = 0, eout = 0;
    for (int k = lane; k < n; k += 32) {
        const int2 o = tab[k];
        acc_lt(ein, *reinterpret_cast<const uint16_t*>(Ib + o.x), (unsigned)P);
        acc_lt(eout, *reinterpret_cast<const uint16_t*>(Ib + o.y), (unsigned)P);
    }
    return (int)__reduce_add_sync(FULLM, ein) - (int)__reduce_add_sync(FULLM, eout);
}

template <bool CIRCLE, bool OMG>
__global__ void __launch_bounds__(512) k2_select(Geom g, SelParams p, const __grid_constant__ KTab kt,
                                                 const uint16_t* __restrict__ omega_in) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nwarps = blockDim.x >> 5;
    const int N = g.N, Npad = g.Npad, Sw = g.Sw, r = g.r;
    const int Tw = g.Tw, Th = g.Th, G = p.G;
    const TileCoord tc = tile_coord(g, g.tile_begin + blockIdx.x);

    const uint16_t* om_g = omega_in + (long long)blockIdx.x * (Npad + 2 * OMEGA_SLOT_PAD) + OMEGA_SLOT_PAD;
    uint16_t* om_s = reinterpret_cast<uint16_t*>(smem) + OMEGA_PAD;
    const uint16_t* om = OMG ? om_g : om_s;
    uint16_t* I = OMG ? reinterpret_cast<uint16_t*>(smem) : om_s + Npad + OMEGA_PAD;
    int* st_P = reinterpret_cast<int*>(I + ((N + 7) & ~7));
    int* st_C = st_P + G * Tw;
    int* deltas = st_C + G * Tw;                   // max(G*Tw, Th) entries
    int* hist = deltas + max(G * Tw, Th);          // 32 bins
    int* seedP = hist + 32;                        // G
    int* seedC = seedP + G;                        // G
    // shared copies of the offset tables for lane-divergent indexing (the
    // constant bank serializes divergent addresses; uniform loops use kt.*)
    int2* vtab_s = reinterpret_cast<int2*>((reinterpret_cast<uintptr_t>(seedC + G) + 7) & ~uintptr_t(7));
    int2* htab_s = vtab_s + p.ncols;
    int* span_s = reinterpret_cast<int*>(htab_s + p.nrows);

    const int2* vtab = kt.v;
    const int2* htab = kt.h;
    const Ctx c{&g, &p, om, I, span_s, N, Sw, r};

    // ---- 0. stage omega and build the ordinal image -----------------------
    {
        const uint4* src = reinterpret_cast<const uint4*>(om_g);
        uint4* dst = reinterpret_cast<uint4*>(om_s);
        for (int i = tid; i < (Npad >> 3); i += blockDim.x) {
            const uint4 v = src[i];
            if (!OMG) dst[i] = v;
            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int q = 0; q < 8; q++) {
                const int rank = (i << 3) + q;
                if (rank < N) {
                    const uint32_t e = (q & 1) ? (w[q >> 1] >> 16) : (w[q >> 1] & 0xffffu);
                    I[(int)(e >> 8) * Sw + (int)(e & 0xffu)] = (uint16_t)rank;
                }
            }
        }
        if (!OMG && tid < OMEGA_PAD) {
            om_s[-OMEGA_PAD + tid] = OMEGA_SENTINEL;
            om_s[Npad + tid] = OMEGA_SENTINEL;
        }
        if (tid < 32) hist[tid] = 0;
        for (int i = tid; i < p.ncols; i += blockDim.x) vtab_s[i] = kt.v[i];
        for (int i = tid; i < p.nrows; i += blockDim.x) htab_s[i] = kt.h[i];
        for (int i = tid; i < 2 * r + 1; i += blockDim.x) span_s[i] = kt.span[i];
    }
    __syncthreads();

    const int R = Th / G;                 // rows per group; seed row at local R/2
    const int g0 = G >> 1;                // group of the direct seed
    const int cs = Tw >> 1;               // seed column
    auto seed_row = [&](int gi) { return gi * R + (R >> 1); };

    // ---- A. direct seed: 32-bin rank histogram split over all warps -------
    const int sh = max(0, 32 - __clz(max(N - 1, 1)) - 5);  // 32 bins of 2^sh ranks cover [0, N)
    {
        const int cx = cs + r, cy = seed_row(g0) + r;
        const uint16_t* Ic = I + cy * Sw + cx;
        unsigned lm[5];
#pragma unroll
        for (int b = 0; b < 5; b++) lm[b] = ((lane >> b) & 1) ? 0u : FULLM;
        int cntb = 0;
        for (int k = wid; k < p.nrows; k += nwarps) {
            const int2 hp = htab[k];  // byte offsets (2*(dy*Sw + xhi), 2*(dy*Sw + xlo))
            const int hx = hp.x >> 1;
            for (int o0 = hp.y >> 1; o0 < hx; o0 += 32) {
                const int o = o0 + lane;
                const bool ok = o < hx;
                const unsigned b = ok ? (unsigned)(Ic[o] >> sh) : 0u;
                unsigned m = __ballot_sync(FULLM, ok);
#pragma unroll
                for (int bit = 0; bit < 5; bit++) m &= ~(__ballot_sync(FULLM, (b >> bit) & 1u) ^ ~lm[bit]);
                cntb += __popc(m);
            }
        }
        if (cntb) atomicAdd(&hist[lane], cntb);
    }
    __syncthreads();
    if (wid == 0) {
        const int row = seed_row(g0);
        const int tgt = target_at(g, p, tc, row, cs);
        const int tot = hist[lane];
        int cum = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(FULLM, cum, o);
            if (lane >= o) cum += v;
        }
        const int B = __ffs(__ballot_sync(FULLM, cum > tgt)) - 1;
        const int cnt = __shfl_sync(FULLM, cum - tot, B);
        const int m = refine_warp<CIRCLE>(c, cs + r, row + r, B << sh, cnt, tgt);
        if (lane == 0) {
            if (m < 0) atomicOr(p.status, 1);
            seedP[g0] = max(m, 0);
            seedC[g0] = tgt;
        }
    }
    __syncthreads();

    // ---- B. other seed rows: vertical deltas at the direct seed's pivot ----
    const unsigned char* Ib0 = reinterpret_cast<const unsigned char*>(I);
    const int rowB = 2 * Sw;  // bytes per ordinal-image row
    const int ytop = seed_row(0), ybot = seed_row(G - 1);
    if (G > 1) {
        const int P0 = seedP[g0];
        for (int y = ytop + tid; y < ybot; y += blockDim.x) {  // step y -> y+1 at column cs
            deltas[y] = slide_delta(Ib0 + (y + r) * rowB + 2 * (cs + r), vtab, p.ncols, P0, false);
        }
        __syncthreads();
        for (int gi = wid; gi < G; gi += nwarps) {
            if (gi == g0) continue;
            const int y0 = seed_row(g0), y1 = seed_row(gi);
            int part = 0;
            if (y1 > y0) {
                for (int y = y0 + lane; y < y1; y += 32) part += deltas[y];
            } else {
                for (int y = y1 + lane; y < y0; y += 32) part -= deltas[y];
            }
            const int cnt = seedC[g0] + (int)__reduce_add_sync(FULLM, (unsigned)part);
            const int tgt = target_at(g, p, tc, y1, cs);
            const int m = refine_warp<CIRCLE>(c, cs + r, y1 + r, P0, cnt, tgt);
            if (lane == 0) {
                if (m < 0) atomicOr(p.status, 1);
                seedP[gi] = max(m, 0);
                seedC[gi] = tgt;
            }
        }
        __syncthreads();
    }

    // ---- C. seed rows: horizontal deltas at the row pivot, then refine ----
    for (int u = tid; u < G * Tw; u += blockDim.x) {  // step j -> j+1 of seed row gi
        const int gi = u / Tw, j = u - gi * Tw;
        if (j + 1 < Tw)
            deltas[u] = slide_delta(Ib0 + (seed_row(gi) + r) * rowB + 2 * (j + r), htab, p.nrows,
                                    seedP[gi], false);
    }
    __syncthreads();
    for (int u = tid; u < G * Tw; u += blockDim.x) {
        const int gi = u / Tw, j = u - gi * Tw, row = seed_row(gi);
        const int P = seedP[gi];
        int cnt = seedC[gi];
        if (j > cs) {
            for (int i = cs; i < j; i++) cnt += deltas[gi * Tw + i];
        } else {
            for (int i = j; i < cs; i++) cnt -= deltas[gi * Tw + i];
        }
        const int tgt = target_at(g, p, tc, row, j);
        int m = (j == cs) ? P : refine_thread<CIRCLE>(c, j + r, row + r, P, cnt, tgt);
        if (m < 0) {
            atomicOr(p.status, 1);
            m = 0;
        }
        st_P[u] = m;
        st_C[u] = tgt;
    }
    __syncthreads();

    // ---- D. vertical sweeps --------------------------------------------------
    for (int u = tid; u < G * Tw * 2; u += blockDim.x) {
        const int j = u % Tw, rest = u / Tw, gi = rest >> 1;
        const bool down = (rest & 1) == 0;
        const int row0 = seed_row(gi);
        const int rend = (gi == G - 1) ? Th : (gi + 1) * R;  // exclusive
        int P = st_P[gi * Tw + j], cnt = st_C[gi * Tw + j];
        if (down) write_out(c, tc, P, row0, j);
        const int cx = j + r;
        const unsigned char* Ic = Ib0 + 2 * cx;
        const int nsteps = down ? (rend - 1 - row0) : (row0 - gi * R);
        int row = row0;
        for (int step = 0; step < nsteps; step++) {
            if (down) {
                cnt += slide_delta(Ic + (row + r) * rowB, vtab, p.ncols, P, false);
                // test hook: an inconsistent count (core.py:31-36 defect path)
                if (p.debug_defect && blockIdx.x == 0 && g.tile_begin == 0 && u == 0 && step == 0) cnt += 1 << 20;
                row++;
            } else {
                cnt += slide_delta(Ic + (row + r - 1) * rowB, vtab, p.ncols, P, true);
                row--;
            }
            const int tgt = target_at(g, p, tc, row, j);
            const int m = refine_thread<CIRCLE>(c, cx, row + r, P, cnt, tgt);
            if (m < 0) {
                atomicOr(p.status, 1);
                break;
            }
            write_out(c, tc, m, row, j);
            P = m;
            cnt = tgt;
        }
    }
}

template __global__ void k2_select<true, false>(Geom, SelParams, const __grid_constant__ KTab, const uint16_t*);
template __global__ void k2_select<false, false>(Geom, SelParams, const __grid_constant__ KTab, const uint16_t*);
template __global__ void k2_select<true, true>(Geom, SelParams, const __grid_constant__ KTab, const uint16_t*);
template __global__ void k2_select<false, true>(Geom, SelParams, const __grid_constant__ KTab, const uint16_t*);

size_t k2_smem_bytes(int N, int Npad, int ncols, int nrows, int r, int G, int Tw, int Th, bool omg) {
    const int gt = G * Tw;
    const size_t tabs = 8 * (size_t)(ncols + nrows) + 4 * (size_t)(2 * r + 1) + 8;
    return (omg ? 0 : 2 * (size_t)(Npad + 2 * OMEGA_PAD)) + 2 * (size_t)((N + 7) & ~7) +
           4 * (size_t)(2 * gt + (gt > Th ? gt : Th) + 32 + 2 * G + 2) + tabs;
}

}  // namespace imf
