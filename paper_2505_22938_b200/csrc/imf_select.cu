// imf_select.cu -- K2: per-output-pixel rank selection on sm_100a.
//
// One CTA solves one T_w x T_h output tile from the tile's omega (K1 output):
//
//   0. stage omega (swizzled, 16-B chunks) and build the quantized ordinal
//      image Iq in shared memory
//   1. direct seeds: G seed rows x K seeds, one warp each: 32-bin histogram of
//      Iq over the window -> a pivot with an exact count -> warp-collaborative
//      64-rank segment refine (ballot/popc)          (core.py:47-60 _seed_state,
//                                                      PAPER.md:285-287)
//   2. seed rows: every column's count at its seed's pivot from a prefix of
//      horizontal slide deltas, then a per-thread refine
//                                                     (core.py:63-72 _slide_right)
//   3. vertical sweeps up and down from each seed row, one thread per
//      (column, group, direction): count update from the entering/exiting
//      kernel-column pixels, refine, write C[m]       (core.py:75-84 _slide_down,
//                                                      :87-146 _refine, :366)
//
// Pivot/count invariant (core.py module docstring): a window carries a pivot P
// (multiple of 2^qs) and count = #{window pixels with rank < P}; every slide
// keeps it exact, the refine walks 64-rank segments of omega from P to the
// target rank.  Because the median is a selection, any exact walk returns the
// same rank m, so the output equals the reference bit for bit.
#include "imf_common.cuh"

namespace imf {



constexpr unsigned FULLM = 0xffffffffu;

struct Ctx {
    const Geom* g;
    const SelParams* p;
    const uint16_t* om;   // swizzled omega
    const uint8_t* Iq;
    const int* span;      // 2r+1 packed spans
    int N, Sw, r;
};

template <bool CIRCLE>
__device__ __forceinline__ bool inside(const Ctx& c, int x, int y, int cx, int cy) {
    if (CIRCLE) {
        int dx = x - cx, dy = y - cy;
        return dx * dx + dy * dy <= c.p->R2;
    } else {
        int dyi = y - cy + c.r;
        if ((unsigned)dyi > (unsigned)(2 * c.r)) return false;
        int sp = c.span[dyi];
        int xlo = (int)(short)(sp & 0xffff);
        int w = sp >> 16;
        return (unsigned)(x - cx - xlo) < (unsigned)w;
    }
}

// Occupancy mask of ranks [64s, 64s+64) in the window centred at (cx, cy)
// (ordinal.py:188-199).  Sixteen-byte loads of the swizzled segment.
template <bool CIRCLE>
__device__ __forceinline__ uint64_t seg_mask(const Ctx& c, int s, int cx, int cy) {
    const uint4* seg = reinterpret_cast<const uint4*>(c.om + (s << 6));
    uint32_t lo = 0, hi = 0;
#pragma unroll
    for (int ch = 0; ch < 8; ch++) {
        uint4 v = seg[ch ^ (s & 7)];
        uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int q = 0; q < 4; q++) {
            int b = ch * 8 + q * 2;
            uint32_t e = w[q];
            bool i0 = inside<CIRCLE>(c, e & 0xff, (e >> 8) & 0xff, cx, cy);
            bool i1 = inside<CIRCLE>(c, (e >> 16) & 0xff, e >> 24, cx, cy);
            if (b < 32) {
                lo |= (i0 ? 1u : 0u) << b;
                lo |= (i1 ? 1u : 0u) << (b + 1);
            } else {
                hi |= (i0 ? 1u : 0u) << (b - 32);
                hi |= (i1 ? 1u : 0u) << (b - 31);
            }
        }
    }
    uint64_t m = ((uint64_t)hi << 32) | lo;
    int rem = c.N - (s << 6);
    if (rem < 64) m &= (rem <= 0) ? 0ull : ((1ull << rem) - 1ull);
    return m;
}

__device__ __forceinline__ int kth_bit(uint64_t m, int need) {
    uint32_t lo = (uint32_t)m, hi = (uint32_t)(m >> 32);
    int pl = __popc(lo);
    if (need < pl) return (int)__fns(lo, 0, need + 1);
    return 32 + (int)__fns(hi, 0, need - pl + 1);
}

__device__ __forceinline__ int quant_pivot(const SelParams& p, int m) {
    int P = ((m + (1 << (p.qs - 1))) >> p.qs) << p.qs;
    return P < p.P_lo ? p.P_lo : (P > p.P_hi ? p.P_hi : P);
}

// Per-thread refine (core.py:87-146).  On entry (piv, cnt) is an exact state of
// window (cx, cy); returns the solution rank m and re-anchors (piv, cnt) at the
// quantized pivot nearest m.  Returns -1 on an inconsistent count.
template <bool CIRCLE>
__device__ int refine_thread(const Ctx& c, int cx, int cy, int& piv, int& cnt, int tgt) {
    int s = piv >> 6, cc = cnt, pop;
    uint64_t mask;
    if (cc <= tgt) {
        for (;;) {
            if ((s << 6) >= c.N) return -1;
            mask = seg_mask<CIRCLE>(c, s, cx, cy);
            pop = __popcll(mask);
            if (cc + pop > tgt) break;
            cc += pop;
            s++;
        }
    } else {
        for (;;) {
            s--;
            if (s < 0) return -1;
            mask = seg_mask<CIRCLE>(c, s, cx, cy);
            pop = __popcll(mask);
            cc -= pop;
            if (cc <= tgt) break;
        }
    }
    const int m = (s << 6) + kth_bit(mask, tgt - cc);
    int np = quant_pivot(*c.p, m);
    int nc;
    if (np == (s << 6)) {
        nc = cc;
    } else if (np == ((s + 1) << 6)) {
        nc = cc + pop;
    } else if (np > (s << 6)) {
        nc = cc + pop;
        for (int t = s + 1; (t << 6) < np; t++) nc += __popcll(seg_mask<CIRCLE>(c, t, cx, cy));
    } else {
        nc = cc;
        for (int t = s - 1; (t << 6) >= np; t--) nc -= __popcll(seg_mask<CIRCLE>(c, t, cx, cy));
    }
    piv = np;
    cnt = nc;
    return m;
}

// Warp-collaborative segment occupancy: lane l tests ranks 64s+2l and 64s+2l+1.
template <bool CIRCLE>
__device__ __forceinline__ void seg_ballot(const Ctx& c, int s, int cx, int cy, int lane,
                                           unsigned& b0, unsigned& b1, bool& in0, bool& in1) {
    const uint32_t* om32 = reinterpret_cast<const uint32_t*>(c.om);
    int ch = lane >> 2;
    uint32_t e = om32[(s << 5) + (((ch ^ (s & 7)) << 2) | (lane & 3))];
    int v = (s << 6) + 2 * lane;
    in0 = v < c.N && inside<CIRCLE>(c, e & 0xff, (e >> 8) & 0xff, cx, cy);
    in1 = v + 1 < c.N && inside<CIRCLE>(c, (e >> 16) & 0xff, e >> 24, cx, cy);
    b0 = __ballot_sync(FULLM, in0);
    b1 = __ballot_sync(FULLM, in1);
}

// Warp-collaborative refine: all lanes hold the same window.
template <bool CIRCLE>
__device__ int refine_warp(const Ctx& c, int cx, int cy, int& piv, int& cnt, int tgt) {
    const int lane = threadIdx.x & 31;
    int s = piv >> 6, cc = cnt, pop;
    unsigned b0, b1;
    bool in0, in1;
    if (cc <= tgt) {
        for (;;) {
            if ((s << 6) >= c.N) return -1;
            seg_ballot<CIRCLE>(c, s, cx, cy, lane, b0, b1, in0, in1);
            pop = __popc(b0) + __popc(b1);
            if (cc + pop > tgt) break;
            cc += pop;
            s++;
        }
    } else {
        for (;;) {
            s--;
            if (s < 0) return -1;
            seg_ballot<CIRCLE>(c, s, cx, cy, lane, b0, b1, in0, in1);
            pop = __popc(b0) + __popc(b1);
            cc -= pop;
            if (cc <= tgt) break;
        }
    }
    const int need = tgt - cc;
    const unsigned lt = lanemask_lt();
    const int pre = __popc(b0 & lt) + __popc(b1 & lt);
    const bool h0 = in0 && pre == need;
    const bool h1 = in1 && pre + (in0 ? 1 : 0) == need;
    const unsigned hb = __ballot_sync(FULLM, h0 || h1);
    const int L = __ffs(hb) - 1;
    const int off = __shfl_sync(FULLM, h0 ? 0 : 1, L);
    const int m = (s << 6) + 2 * L + off;
    int np = quant_pivot(*c.p, m);
    int nc;
    if (np == (s << 6)) {
        nc = cc;
    } else if (np == ((s + 1) << 6)) {
        nc = cc + pop;
    } else if (np > (s << 6)) {
        nc = cc + pop;
        for (int t = s + 1; (t << 6) < np; t++) {
            seg_ballot<CIRCLE>(c, t, cx, cy, lane, b0, b1, in0, in1);
            nc += __popc(b0) + __popc(b1);
        }
    } else {
        nc = cc;
        for (int t = s - 1; (t << 6) >= np; t--) {
            seg_ballot<CIRCLE>(c, t, cx, cy, lane, b0, b1, in0, in1);
            nc -= __popc(b0) + __popc(b1);
        }
    }
    piv = np;
    cnt = nc;
    return m;
}

__device__ __forceinline__ int target_at(const Geom& g, const SelParams& p, const TileCoord& tc,
                                         int row, int col) {
    if (!p.tmap) return p.target;
    int y = min(tc.oy0 + row, g.out_h - 1), x = min(tc.ox0 + col, g.out_w - 1);
    return __ldg(p.tmap + (long long)y * g.out_w + x);
}

// Output = C[m]: the input value at omega[m]'s position (core.py:366).
__device__ __forceinline__ void write_out(const Ctx& c, const TileCoord& tc, int m, int row, int col) {
    const Geom& g = *c.g;
    const int oy = tc.oy0 + row, ox = tc.ox0 + col;
    if (oy >= g.out_h || ox >= g.out_w) return;
    const uint32_t e = c.om[omega_index(m)];
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

template <bool CIRCLE>
__global__ void __launch_bounds__(512) k2_select(Geom g, SelParams p,
                                                 const uint16_t* __restrict__ omega_in) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nwarps = blockDim.x >> 5;
    const int N = g.N, Npad = g.Npad, Sw = g.Sw, r = g.r;
    const int Tw = g.Tw, Th = g.Th, G = p.G, K = p.K;
    const TileCoord tc = tile_coord(g, g.tile_begin + blockIdx.x);

    uint16_t* om = reinterpret_cast<uint16_t*>(smem);
    uint8_t* Iq = reinterpret_cast<uint8_t*>(om + Npad);
    int* ktab = reinterpret_cast<int*>(Iq + ((N + 15) & ~15));
    const int ktab_n = 2 * p.ncols + 2 * p.nrows + 2 * r + 1;
    uint16_t* shist = reinterpret_cast<uint16_t*>(ktab + ((ktab_n + 3) & ~3));
    const int nhist = min(nwarps, G * K);
    int* st_m = reinterpret_cast<int*>(shist + nhist * 1024);
    int* st_p = st_m + G * Tw;
    int* st_c = st_p + G * Tw;
    int* deltas = st_c + G * Tw;

    const int2* vtab = reinterpret_cast<const int2*>(ktab);
    const int2* htab = reinterpret_cast<const int2*>(ktab + 2 * p.ncols);
    Ctx c{&g, &p, om, Iq, ktab + 2 * p.ncols + 2 * p.nrows, N, Sw, r};

    // ---- 0. stage omega (swizzled) and build Iq -------------------------
    {
        const uint4* src = reinterpret_cast<const uint4*>(omega_in + (long long)blockIdx.x * Npad);
        uint4* dst = reinterpret_cast<uint4*>(om);
        for (int i = tid; i < (Npad >> 3); i += blockDim.x) {
            uint4 v = src[i];
            const int s = i >> 3;
            dst[(s << 3) | ((i & 7) ^ (s & 7))] = v;
            uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int q = 0; q < 8; q++) {
                const int rank = (i << 3) + q;
                if (rank < N) {
                    const uint32_t e = (q & 1) ? (w[q >> 1] >> 16) : (w[q >> 1] & 0xffff);
                    int qv = (rank >> p.qs) - p.qb;
                    qv = qv < 0 ? 0 : (qv > 255 ? 255 : qv);
                    Iq[(int)(e >> 8) * Sw + (int)(e & 0xff)] = (uint8_t)qv;
                }
            }
        }
        for (int i = tid; i < ktab_n; i += blockDim.x) ktab[i] = __ldg(p.ktab + i);
    }
    __syncthreads();

    const int R = Th / G;  // rows per group; seed row at local R/2
    auto blk_lo = [&](int k) { return (k * Tw) / K; };
    auto seed_col = [&](int k) { return (blk_lo(k) + blk_lo(k + 1)) >> 1; };

    // ---- 1. direct seeds (one warp each) ----------------------------------
    for (int sd = wid; sd < G * K; sd += nwarps) {
        const int gi = sd / K, ki = sd % K;
        const int row = gi * R + (R >> 1), col = seed_col(ki);
        const int cx = col + r, cy = row + r;
        const int tgt = target_at(g, p, tc, row, col);
        uint16_t* h = shist + (wid % nhist) * 1024;
        for (int i = lane; i < 1024; i += 32) h[i] = 0;
        __syncwarp();
        const uint8_t* Ic = Iq + cy * Sw + cx;
        for (int k = 0; k < p.nrows; k++) {
            const int2 hp = htab[k];  // (dy*Sw + xhi, dy*Sw + xlo)
            for (int o = hp.y + lane; o < hp.x; o += 32) h[((Ic[o] >> 3) << 5) + lane]++;
        }
        __syncwarp();
        int tot = 0;
        for (int b = 0; b < 32; b++) {
            int v = __reduce_add_sync(FULLM, (unsigned)h[(b << 5) + lane]);
            if (lane == b) tot = v;
        }
        int cum = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int v = __shfl_up_sync(FULLM, cum, o);
            if (lane >= o) cum += v;
        }
        const int B = __ffs(__ballot_sync(FULLM, cum > tgt)) - 1;
        int pq, cnt;
        if (B == 0) {
            pq = 8;
            cnt = __shfl_sync(FULLM, cum, 0);
        } else {
            pq = 8 * B;
            cnt = __shfl_sync(FULLM, cum - tot, B);
        }
        int piv = (pq + p.qb) << p.qs;
        const int m = refine_warp<CIRCLE>(c, cx, cy, piv, cnt, tgt);
        if (m < 0 && lane == 0) atomicOr(p.status, 1);
        if (lane == 0) {
            st_m[gi * Tw + col] = m < 0 ? 0 : m;
            st_p[gi * Tw + col] = piv;
            st_c[gi * Tw + col] = cnt;
        }
    }
    __syncthreads();

    // ---- 2. seed rows: horizontal slide deltas at the seed pivot ----------
    for (int u = tid; u < G * Tw; u += blockDim.x) {
        const int gi = u / Tw, j = u % Tw;
        int ki = 0;
        while (ki + 1 < K && j >= blk_lo(ki + 1)) ki++;
        const int sc = seed_col(ki);
        if (j + 1 < blk_lo(ki + 1) && j + 1 < Tw) {
            const int row = gi * R + (R >> 1);
            const int pq = (st_p[gi * Tw + sc] >> p.qs) - p.qb;
            const uint8_t* Ic = Iq + (row + r) * Sw + (j + r);
            int d = 0;
            for (int k = 0; k < p.nrows; k++) {
                const int2 hp = htab[k];
                d += (Ic[hp.x] < pq) - (Ic[hp.y] < pq);
            }
            deltas[u] = d;
        }
    }
    __syncthreads();
    for (int u = tid; u < G * Tw; u += blockDim.x) {
        const int gi = u / Tw, j = u % Tw;
        int ki = 0;
        while (ki + 1 < K && j >= blk_lo(ki + 1)) ki++;
        const int sc = seed_col(ki);
        if (j == sc) continue;
        int piv = st_p[gi * Tw + sc], cnt = st_c[gi * Tw + sc];
        if (j > sc) {
            for (int i = sc; i < j; i++) cnt += deltas[gi * Tw + i];
        } else {
            for (int i = j; i < sc; i++) cnt -= deltas[gi * Tw + i];
        }
        const int row = gi * R + (R >> 1);
        const int m = refine_thread<CIRCLE>(c, j + r, row + r, piv, cnt, target_at(g, p, tc, row, j));
        if (m < 0) atomicOr(p.status, 1);
        st_m[u] = m < 0 ? 0 : m;
        st_p[u] = piv;
        st_c[u] = cnt;
    }
    __syncthreads();

    // ---- 3. vertical sweeps --------------------------------------------------
    for (int u = tid; u < G * Tw * 2; u += blockDim.x) {
        const int j = u % Tw, rest = u / Tw, gi = rest >> 1, down = (rest & 1) == 0;
        const int row0 = gi * R + (R >> 1);
        const int rend = (gi == G - 1) ? Th : (gi + 1) * R;  // exclusive
        int m = st_m[gi * Tw + j], piv = st_p[gi * Tw + j], cnt = st_c[gi * Tw + j];
        const int cx = j + r;
        if (down) write_out(c, tc, m, row0, j);
        int row = row0;
        const int nsteps = down ? (rend - 1 - row0) : (row0 - gi * R);
        for (int step = 0; step < nsteps; step++) {
            const int pq = (piv >> p.qs) - p.qb;
            int d = 0;
            if (down) {
                const uint8_t* Ib = Iq + (row + r) * Sw + cx;
                for (int k = 0; k < p.ncols; k++) {
                    const int2 o = vtab[k];
                    d += (Ib[o.x] < pq) - (Ib[o.y] < pq);
                }
                row++;
            } else {
                const uint8_t* Ib = Iq + (row + r - 1) * Sw + cx;
                for (int k = 0; k < p.ncols; k++) {
                    const int2 o = vtab[k];
                    d += (Ib[o.y] < pq) - (Ib[o.x] < pq);
                }
                row--;
            }
            cnt += d;
            m = refine_thread<CIRCLE>(c, cx, row + r, piv, cnt, target_at(g, p, tc, row, j));
            if (m < 0) {
                atomicOr(p.status, 1);
                break;
            }
            write_out(c, tc, m, row, j);
        }
    }
}

template __global__ void k2_select<true>(Geom, SelParams, const uint16_t*);
template __global__ void k2_select<false>(Geom, SelParams, const uint16_t*);

size_t k2_smem_bytes(int N, int Npad, int ncols, int nrows, int r, int G, int K, int Tw, int nwarps) {
    const int ktab_n = 2 * ncols + 2 * nrows + 2 * r + 1;
    const int nhist = nwarps < G * K ? nwarps : G * K;
    return 2 * (size_t)Npad + (size_t)((N + 15) & ~15) + 4 * (size_t)((ktab_n + 3) & ~3) +
           2048 * (size_t)nhist + 4 * (size_t)(4 * G * Tw);
}

}  // namespace imf
