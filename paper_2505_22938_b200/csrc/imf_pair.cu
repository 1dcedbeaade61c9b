// imf_pair.cu -- K2 fast path: per-output-pixel rank selection with two
// windows per thread and packed 15-bit rank compares (sm_100a).
//
// Same algorithm and phases as k2_select (imf_select.cu: direct seed, seed-row
// centres, seed rows, vertical sweeps -- core.py:47-60, :63-84, :87-146), with
// the two inner loops re-laid-out for the B200 SM:
//
// * Slides (core.py:63-84, 2 tests per kernel column/row per window).  A
//   thread owns the windows of two horizontally adjacent output pixels.  Their
//   entering / exiting pixels are horizontally adjacent too, so ONE 32-bit
//   shared load returns both windows' ranks (I[o], I[o+1]).  With tile ranks
//   below 2^15 (N <= 32768) the two "rank >= pivot" tests are one add:
//       d = (I[o+1] << 16 | I[o]) + ((0x8000 - P_B) << 16 | (0x8000 - P_A))
//   leaves [I >= P] in bits 15 and 31 (no carry crosses the halves), and
//   acc += (d & 0x80008000) >> 15 (LOP3 + LEA.HI) counts both.  Offsets come
//   from the constant bank and the load uses the [R + UR] form, so a kernel
//   column costs 2 LDS + 6 integer ops for 4 tests (reference: 4 tests = 8 ops).
//   Offsets whose pixel pair is not 4-byte aligned read the two enclosing words
//   and PRMT the middle halves.
// * Refine (core.py:87-146, ordinal.py:175-199).  Eight ranks per step from one
//   LDS.128 of omega.  Circle membership 4(dx^2+dy^2) <= (2r+1)^2 (kernels.py:
//   70-71) is evaluated on packed bytes: omega entry x | y << 8 plus a
//   per-window constant gives (dx+128, dy+128) bytes for two ranks at once,
//   XOR 0x80 makes them signed, and IDP.4A squares-and-adds them against
//   -(r(r+1)+1); the sign bit is the membership bit (funnel-shifted into the
//   step mask).  Wide tiles, squares and x/y-symmetric polygons take |dx|,
//   |dy| bytes from VABSDIFF4 of the raw entries against cx | cy << 8 and
//   test them against r(r+1), r or a per-|dy| table;
//   other polygons use a per-dy range table, any kernel the span table
//   (kernels.py:127-182).
//
// Layout (shared memory): omega (rank -> x | y << 8, 8 sentinel entries each
// side, 16-byte aligned so rank 8k starts a 16-byte chunk), then the ordinal
// image I (u16 rank per input-tile pixel, row stride Sw), then per-window state.
#include "imf_kernels.cuh"

namespace imf {

__device__ __forceinline__ uint32_t lds32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}

__device__ __forceinline__ uint32_t lds16(uint32_t a) {
    unsigned short v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
    return v;
}

__device__ __forceinline__ uint4 lds128(uint32_t a) {
    uint4 q;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(q.x), "=r"(q.y), "=r"(q.z), "=r"(q.w)
                 : "r"(a));
    return q;
}

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t s) {
    uint32_t r;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(s));
    return r;
}

// acc += (d & 0x80008000) >> 15: counts [I >= P] of both halves (LOP3 + LEA.HI).
__device__ __forceinline__ void acc_ge2(uint32_t& acc, uint32_t d) {
    asm("{\n\t.reg .u32 t;\n\tand.b32 t, %1, 0x80008000;\n\tshr.u32 t, t, 15;\n\tadd.u32 %0, %0, t;\n\t}"
        : "+r"(acc)
        : "r"(d));
}

// Packed pivot constant: halves (0x8000 - PA, 0x8000 - PB).
__device__ __forceinline__ uint32_t pivot_k(int PA, int PB) {
    return (uint32_t)(0x8000 - PA) | ((uint32_t)(0x8000 - PB) << 16);
}

// Two test words at once: bits 15 / 31 of d1 and d2 (the [I >= P] answers of
// windows A / B) are the top bits of bytes 1 / 3; PRMT gathers them into one
// word as bytes [A1, A2, B1, B2] and acc += (x & 0x80808080) >> 7 counts all
// four in byte lanes (LOP3 + LEA.HI): 5 instructions per 4 tests instead of 6.
__device__ __forceinline__ void acc_ge4(uint32_t& acc, uint32_t d1, uint32_t d2) {
    const uint32_t x = prmt(d1, d2, 0x7351);
    asm("{\n\t.reg .u32 t;\n\tand.b32 t, %1, 0x80808080;\n\tshr.u32 t, t, 7;\n\tadd.u32 %0, %0, t;\n\t}"
        : "+r"(acc)
        : "r"(x));
}

// Four tests into ONE dot product: PRMT in sign-replicate mode gathers the
// answer bytes of d1 and d2 as [A1, A2, B1, B2] = 0xff (I >= P) or 0x00, and
// IDP.4A against the unsigned weights [1, 1, 128, 128] accumulates -(A + 128 B)
// (2 instructions per 4 tests instead of PRMT + LOP3 + LEA.HI).  A run of
// acc_dp4 calls may count at most 127 A-tests before dp4_unpack.
__device__ __forceinline__ void acc_dp4(int& acc, uint32_t d1, uint32_t d2) {
    const uint32_t x = prmt(d1, d2, 0xFBD9);
    asm("dp4a.s32.u32 %0, %1, %2, %0;" : "+r"(acc) : "r"(x), "r"(0x80800101u));
}

// -(A + 128 B) with A <= 127 -> packed (A | B << 16).
__device__ __forceinline__ uint32_t dp4_unpack(int acc) {
    const uint32_t v = (uint32_t)(-acc);
    return (v & 127u) | ((v >> 7) << 16);
}

// Byte-lane counters [A1, A2, B1, B2] -> packed (A | B << 16).
__device__ __forceinline__ uint32_t unpack4(uint32_t acc) {
    return (acc & 0x00ff00ffu) + ((acc >> 8) & 0x00ff00ffu);
}

// Packed counts of [I >= P] over the vertical list at window-pair base `b`
// (entering and exiting lists; byte-lane accumulators, <= 2 * 124 + 1 columns).
template <int U>  // column-loop unroll: 4 (round-2 end, with the 2-instruction acc_dp4: circles 8 -> 4 c2 / c5 -0.5 to -1 %, 16 +9 %, 2 +2 %)
__device__ __forceinline__ void vcount(uint32_t b, const int2* __restrict__ v, int ne, int n, uint32_t K,
                                       uint32_t& ge_in, uint32_t& ge_out) {
    // one entry per kernel column, alternating parity: each of the even
    // (aligned) and odd lists holds <= 125 columns (build_pair_tab checks
    // <= 127), so each list is one acc_dp4 run
    int ai = 0, ao = 0;
    uint32_t ri = 0, ro = 0;
    int k = 0;
#pragma unroll U
    for (; k + 1 < ne; k += 2) {
        const int2 o0 = v[k], o1 = v[k + 1];
        acc_dp4(ai, lds32(b + o0.x) + K, lds32(b + o1.x) + K);
        acc_dp4(ao, lds32(b + o0.y) + K, lds32(b + o1.y) + K);
    }
    if (k < ne) {
        const int2 o = v[k];
        acc_ge2(ri, lds32(b + o.x) + K);
        acc_ge2(ro, lds32(b + o.y) + K);
    }
    ri += dp4_unpack(ai);
    ro += dp4_unpack(ao);
    ai = ao = 0;
#pragma unroll U
    for (k = ne; k + 1 < n; k += 2) {
        const int2 o0 = v[k], o1 = v[k + 1];
        acc_dp4(ai, prmt(lds32(b + o0.x), lds32(b + o0.x + 4), 0x5432) + K,
                prmt(lds32(b + o1.x), lds32(b + o1.x + 4), 0x5432) + K);
        acc_dp4(ao, prmt(lds32(b + o0.y), lds32(b + o0.y + 4), 0x5432) + K,
                prmt(lds32(b + o1.y), lds32(b + o1.y + 4), 0x5432) + K);
    }
    if (k < n) {
        const int2 o = v[k];
        acc_ge2(ri, prmt(lds32(b + o.x), lds32(b + o.x + 4), 0x5432) + K);
        acc_ge2(ro, prmt(lds32(b + o.y), lds32(b + o.y + 4), 0x5432) + K);
    }
    ge_in = dp4_unpack(ai) + ri;
    ge_out = dp4_unpack(ao) + ro;
}

// Packed count of [I >= P] over one horizontal list (acc_dp4 runs when both
// parity lists hold <= 127 rows -- a row's entering column parity follows the
// kernel's shape, so e.g. a large square puts every row in one list).
__device__ __forceinline__ uint32_t hcount(uint32_t b, const int* __restrict__ h, int ne, int n, uint32_t K) {
    uint32_t rr = 0;
    int k = 0;
    if (ne <= 127 && n - ne <= 127) {
        int a = 0;
#pragma unroll 2
        for (; k + 1 < ne; k += 2) acc_dp4(a, lds32(b + h[k]) + K, lds32(b + h[k + 1]) + K);
        if (k < ne) acc_ge2(rr, lds32(b + h[k]) + K);
        rr += dp4_unpack(a);
        a = 0;
#pragma unroll 2
        for (k = ne; k + 1 < n; k += 2)
            acc_dp4(a, prmt(lds32(b + h[k]), lds32(b + h[k] + 4), 0x5432) + K,
                    prmt(lds32(b + h[k + 1]), lds32(b + h[k + 1] + 4), 0x5432) + K);
        if (k < n) acc_ge2(rr, prmt(lds32(b + h[k]), lds32(b + h[k] + 4), 0x5432) + K);
        return dp4_unpack(a) + rr;
    }
    uint32_t a = 0;
#pragma unroll 2
    for (; k + 1 < ne; k += 2) acc_ge4(a, lds32(b + h[k]) + K, lds32(b + h[k + 1]) + K);
    if (k < ne) acc_ge2(rr, lds32(b + h[k]) + K);
#pragma unroll 2
    for (k = ne; k + 1 < n; k += 2)
        acc_ge4(a, prmt(lds32(b + h[k]), lds32(b + h[k] + 4), 0x5432) + K,
                prmt(lds32(b + h[k + 1]), lds32(b + h[k + 1] + 4), 0x5432) + K);
    if (k < n) acc_ge2(rr, prmt(lds32(b + h[k]), lds32(b + h[k] + 4), 0x5432) + K);
    return unpack4(a) + rr;
}

// Per-half difference lo(a) - lo(b), hi(a) - hi(b).
__device__ __forceinline__ void half_diff(uint32_t a, uint32_t b, int& lo, int& hi) {
    lo = (int)(a & 0xffffu) - (int)(b & 0xffffu);
    hi = (int)(a >> 16) - (int)(b >> 16);
}

// Index of the k-th (0-based) set bit of an 8-bit mask.
__device__ __forceinline__ int nth_bit8(uint32_t m, int k) {
    int pos = 0;
    int c = __popc(m & 0xfu);
    if (k >= c) { k -= c; m >>= 4; pos = 4; }
    c = __popc(m & 0x3u);
    if (k >= c) { k -= c; m >>= 2; pos += 2; }
    if (k >= (int)(m & 1u)) pos += 1;
    return pos;
}

struct PairCtx {
    uint32_t om_a;        // shared address of omega rank 0
    const uint16_t* om;   // generic pointer to omega rank 0
    const int* span;      // shared span table (2r+1)
    int N, r, R2p1;
    uint32_t rowk_a;      // SH_POLY: 256-entry per-(dy+128) range table; SH_POLYSYM: 128-byte table
    int nR2p1;            // -(r(r+1)+1)
    uint32_t x80;         // 0x80808080 in a register (SH_CIRCLE's LOP3 operand)
};

__device__ __forceinline__ uint32_t lds8(uint32_t a) {
    unsigned short v;
    asm volatile("ld.shared.u8 %0, [%1];" : "=h"(v) : "r"(a));
    return v;
}

__device__ __forceinline__ uint32_t lds32c(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}

// Membership bits of ranks v0..v0+7 (bit i = rank v0+i) of the window at (cx, cy).
template <int SHAPE, bool OMG>
__device__ __forceinline__ uint32_t test8(const PairCtx& c, int v0, uint32_t Kc, int cx, int cy) {
    uint4 q;
    if (OMG)  // omega in its L2-resident global slot (16-byte aligned)
        q = __ldg(reinterpret_cast<const uint4*>(c.om + v0));
    else
        q = lds128(c.om_a + 2 * v0);
    const uint32_t w[4] = {q.x, q.y, q.z, q.w};
    uint32_t m = 0;
    if (SHAPE == SH_CIRCLE) {
        // each rank's signed bytes isolated by ONE LOP3 ((a ^ 0x80808080) & mask,
        // the XOR constant held in a register) and squared against themselves:
        // 2 LOP3 + 2 IDP.4A per two ranks (b & mask against the full b needs 3
        // LOP3; VABSDIFF4 on the raw entries, as below, measured 1.7 % slower)
#pragma unroll
        for (int i = 3; i >= 0; i--) {
            const uint32_t a = w[i] + Kc;
            uint32_t blo, bhi;
            asm("lop3.b32 %0, %1, %2, 0x0000ffff, 0x28;" : "=r"(blo) : "r"(a), "r"(c.x80));
            asm("lop3.b32 %0, %1, %2, 0xffff0000, 0x28;" : "=r"(bhi) : "r"(a), "r"(c.x80));
            const int slo = __dp4a((int)blo, (int)blo, c.nR2p1);
            const int shi = __dp4a((int)bhi, (int)bhi, c.nR2p1);
            m = __funnelshift_l((uint32_t)shi, m, 1);
            m = __funnelshift_l((uint32_t)slo, m, 1);
        }
    } else if (SHAPE == SH_CIRCLEW) {
        // Wide tiles (|dx| up to 254): VABSDIFF4 of the raw entries x | y << 8
        // against cx | cy << 8 (Kc, both halves) gives |dx|, |dy| as unsigned
        // bytes; each rank's pair masked out by one LOP3 and squared by an
        // unsigned IDP.4A against -(r(r+1)+1): the sign bit is membership
        // (sums <= 2 * 255^2, no wrap).  3.5 instructions per rank.
#pragma unroll
        for (int i = 3; i >= 0; i--) {
            const uint32_t z = __vabsdiffu4(w[i], Kc);
            const uint32_t blo = z & 0xffffu, bhi = z & 0xffff0000u;
            const uint32_t slo = __dp4a(blo, blo, (unsigned)c.nR2p1);
            const uint32_t shi = __dp4a(bhi, bhi, (unsigned)c.nR2p1);
            m = __funnelshift_l(shi, m, 1);
            m = __funnelshift_l(slo, m, 1);
        }
    } else if (SHAPE == SH_SQUARE) {
        // VABSDIFF4 of the raw entries against cx | cy << 8 gives |dx|, |dy|
        // per byte (<= 127 for tile pixels), + (127 - r) per byte sets bit 7
        // exactly where |d| > r (no carry leaves a tile pixel's byte); a rank is
        // outside iff either of its bytes has bit 7: z | z << 8 holds the
        // outside bits in bits 15 (low rank) and 31 (high rank), complemented
        // once per 8 ranks
        const uint32_t K127 = (uint32_t)(127 - c.r) * 0x01010101u;
#pragma unroll
        for (int i = 3; i >= 0; i--) {
            const uint32_t z = __vabsdiffu4(w[i], Kc) + K127;
            const uint32_t o = z | (z << 8);  // bits 15 / 31: OUTSIDE
            m = __funnelshift_l(o, m, 1);
            m = __funnelshift_l(o << 16, m, 1);
        }
        m = ~m & 0xffu;  // outside bits -> membership, once per 8 ranks
    } else if (SHAPE == SH_POLYSYM) {
        // kernels symmetric in x and y (the regular polygons of kernels.py:45-64):
        // inside iff |dx| <= h(|dy|).  VABSDIFF4 gives |dx|, |dy| bytes of two
        // ranks; a 128-byte shared table gives 127 - h(|dy|) (128 for rows
        // outside the kernel), so |dx| + that has bit 7 exactly outside
        // (<= 255: no carry leaves a byte); bits 7 / 23 are the two ranks'
        // outside bits, complemented once per 8 ranks
#pragma unroll
        for (int i = 3; i >= 0; i--) {
            const uint32_t z = __vabsdiffu4(w[i], Kc);
            const uint32_t t0 = lds8(c.rowk_a + prmt(z, 0u, 0x4441u));
            const uint32_t t1 = lds8(c.rowk_a + prmt(z, 0u, 0x4443u));
            const uint32_t o = z + prmt(t0, t1, 0x5410u);  // bits 7 / 23: OUTSIDE
            m = __funnelshift_l(o << 8, m, 1);
            m = __funnelshift_l(o << 24, m, 1);
        }
        m = ~m & 0xffu;  // outside bits -> membership, once per 8 ranks
    } else if (SHAPE == SH_POLY) {
        // row table T[dy+128] = (0x8000 - (128+xlo)) | (0x8000 - (128+xhi)) << 16
        // (0 for rows outside the kernel): with the dx byte h in both halves,
        // bit 15 of h*0x10001 + T is [dx >= xlo] and bit 31 is [dx >= xhi]
#pragma unroll
        for (int i = 3; i >= 0; i--) {
            const uint32_t a = w[i] + Kc;
            const uint32_t T1 = lds32c(c.rowk_a + 4 * (a >> 24)), T0 = lds32c(c.rowk_a + 4 * ((a >> 8) & 0xffu));
            const uint32_t d1 = prmt(a, 0u, 0x4242u) + T1, d0 = prmt(a, 0u, 0x4040u) + T0;
            m = __funnelshift_l((d1 << 16) & ~d1, m, 1);
            m = __funnelshift_l((d0 << 16) & ~d0, m, 1);
        }
    } else {
#pragma unroll
        for (int i = 0; i < 8; i++) {
            const uint32_t e = (i & 1) ? (w[i >> 1] >> 16) : (w[i >> 1] & 0xffffu);
            const int dy = (int)(e >> 8) - cy + c.r;
            bool in = false;
            if ((unsigned)dy <= (unsigned)(2 * c.r)) {
                const int sp = c.span[dy];
                in = (unsigned)((int)(e & 0xffu) - cx - (int)(short)(sp & 0xffff)) < (unsigned)(sp >> 16);
            }
            m |= (in ? 1u : 0u) << i;
        }
    }
    return m;
}


// Both windows of a pair (columns cx and cx+1, same row) walk in the same
// loop, one 8-rank step of EACH per iteration (independent work, so the two
// LDS.128 + membership chains overlap): a warp iterates max over lanes of
// max(steps_A, steps_B) rather than of steps_A + steps_B.  The loop only
// locates the 8-rank block holding each answer; the bit search runs once after
// it.  Ranks >= N hold the 0xffff sentinel, which the packed circle test and
// the span test both place outside every window, so the last block needs no
// mask; a walk leaving [0, N) (inconsistent state, core.py:31-36) yields -1.
struct Walk {
    int v0, need, step;
    uint32_t Kc, msk;
    bool up, done;
};

// Returns the first block's mask (ranks on the walk's side of P).
__device__ __forceinline__ uint32_t walk_init(Walk& w, int P, int cnt, int t, int cx, int cy) {
    w.up = cnt <= t;
    w.need = w.up ? t - cnt : cnt - t - 1;
    uint32_t mask;
    if (w.up) {
        w.v0 = P & ~7;
        mask = (0xffu << (P - w.v0)) & 0xffu;
    } else {
        w.v0 = (P - 1) & ~7;  // P == 0: v0 = -8, reported as a defect
        mask = (P > 0) ? (1u << (P - w.v0)) - 1u : 0xffu;
    }
    w.step = w.up ? 8 : -8;
    w.Kc = (uint32_t)((128 - cx) + ((128 - cy) << 8)) * 0x10001u;
    w.done = false;
    w.msk = 0;
    return mask;
}

// Per-window constant of the membership test: (cx | cy << 8) in both halves
// for the VABSDIFF4 tests, walk_init's (128 - cx, 128 - cy) form for SH_CIRCLE
// and SH_POLY.
template <int SHAPE>
__device__ __forceinline__ uint32_t window_key(int cx, int cy) {
    if (SHAPE == SH_CIRCLEW || SHAPE == SH_SQUARE || SHAPE == SH_POLYSYM)
        return ((uint32_t)cx | ((uint32_t)cy << 8)) * 0x10001u;
    return (uint32_t)((128 - cx) + ((128 - cy) << 8)) * 0x10001u;
}

// One 8-rank step.  A finished walk keeps v0 at its answer's block (msk: that
// block's membership bits, need: in-window ranks to skip in it); a walk that
// leaves [0, N) stops with v0 outside it (a defect).
template <int SHAPE, bool OMG>
__device__ __forceinline__ void walk_step(const PairCtx& c, Walk& w, uint32_t mask, int cx, int cy) {
    if (w.done) return;
    if ((unsigned)w.v0 >= (unsigned)c.N) {
        w.done = true;
        return;
    }
    const uint32_t m = test8<SHAPE, OMG>(c, w.v0, w.Kc, cx, cy) & mask;
    const int pc = __popc(m);
    if (w.need < pc) {
        w.done = true;
        w.msk = m;
    } else {
        w.need -= pc;
        w.v0 += w.step;
    }
}

// Two 8-rank blocks per step (v0 and v0 + step): half the trip count of the
// warp's longest walk for ~1.7x the work of a step (fewer loop / branch
// overheads per block).  The second block may lie past either end of [0, N):
// it then reads the sentinel entries (outside every window) next to omega.
template <int SHAPE, bool OMG>
__device__ __forceinline__ void walk_step2(const PairCtx& c, Walk& w, uint32_t mask, int cx, int cy) {
    if (w.done) return;
    if ((unsigned)w.v0 >= (unsigned)c.N) {
        w.done = true;
        return;
    }
    const uint32_t m1 = test8<SHAPE, OMG>(c, w.v0, w.Kc, cx, cy) & mask;
    const uint32_t m2 = test8<SHAPE, OMG>(c, w.v0 + w.step, w.Kc, cx, cy);
    const int p1 = __popc(m1), p2 = __popc(m2);
    if (w.need < p1) {
        w.done = true;
        w.msk = m1;
    } else if (w.need < p1 + p2) {
        w.done = true;
        w.msk = m2;
        w.need -= p1;
        w.v0 += w.step;
    } else {
        w.need -= p1 + p2;
        w.v0 += 2 * w.step;
    }
}

__device__ __forceinline__ int walk_result(const PairCtx& c, const Walk& w) {
    if ((unsigned)w.v0 >= (unsigned)c.N) return -1;
    return w.v0 + nth_bit8(w.msk, w.up ? w.need : __popc(w.msk) - 1 - w.need);
}

// t-th smallest rank of the window at (cx, cy) from the exact state (P, cnt):
// walk omega from P toward the target 8 ranks per step (core.py:87-146 with an
// exact pivot).  -1 if the walk leaves [0, N) (core.py:31-36).
template <int SHAPE, bool OMG>
__device__ int refine8(const PairCtx& c, int cx, int cy, int P, int cnt, int t) {
    Walk w;
    const uint32_t mask = walk_init(w, P, cnt, t, cx, cy);
    w.Kc = window_key<SHAPE>(cx, cy);
    walk_step2<SHAPE, OMG>(c, w, mask, cx, cy);
    while (!w.done) walk_step2<SHAPE, OMG>(c, w, 0xffu, cx, cy);
    return walk_result(c, w);
}

#ifdef IMF_STATS
__device__ unsigned long long g_stats[256];  // [0..63] lane steps/window-pair, [64..127] warp trip counts
#endif

template <int SHAPE, bool OMG>
__device__ __forceinline__ void refine8x2(const PairCtx& c, int cx, int cy, int PA, int cntA, int tA, int PB,
                                          int cntB, int tB, int& mA, int& mB) {
    Walk a, b;
    const uint32_t ma = walk_init(a, PA, cntA, tA, cx, cy);
    const uint32_t mb = walk_init(b, PB, cntB, tB, cx + 1, cy);
    a.Kc = window_key<SHAPE>(cx, cy);
    b.Kc = window_key<SHAPE>(cx + 1, cy);
    // first blocks (partial masks) peeled; then full blocks
    walk_step<SHAPE, OMG>(c, a, ma, cx, cy);
    walk_step<SHAPE, OMG>(c, b, mb, cx + 1, cy);
#ifdef IMF_STATS
    int nit = 1;
#endif
    while (!(a.done && b.done)) {
#ifdef IMF_STATS
        nit++;
#endif
        walk_step2<SHAPE, OMG>(c, a, 0xffu, cx, cy);
        walk_step2<SHAPE, OMG>(c, b, 0xffu, cx + 1, cy);
    }
    mA = walk_result(c, a);
    mB = walk_result(c, b);
#ifdef IMF_STATS
    atomicAdd(&g_stats[min(nit, 63)], 1ull);
    const int mx = __reduce_max_sync(__activemask(), nit);
    if ((threadIdx.x & 31) == __ffs(__activemask()) - 1) atomicAdd(&g_stats[64 + min(mx, 63)], 1ull);
#endif
}

// The pair's two walks one after the other in ONE loop (a lane switches to
// window B when A is done): a warp iterates max over lanes of (steps_A +
// steps_B) single-walk iterations instead of max over lanes of max(steps_A,
// steps_B) double iterations -- never more work, less when the pair's walk
// lengths differ (IMF_REFINE=1).
template <int SHAPE, bool OMG>
__device__ __forceinline__ void refine8x2_seq(const PairCtx& c, int cx, int cy, int PA, int cntA, int tA, int PB,
                                              int cntB, int tB, int& mA, int& mB) {
    Walk w;
    uint32_t mk = walk_init(w, PA, cntA, tA, cx, cy);
    w.Kc = window_key<SHAPE>(cx, cy);
    int cxc = cx;
    bool second = false;
    for (;;) {
        walk_step2<SHAPE, OMG>(c, w, mk, cxc, cy);
        mk = 0xffu;
        if (w.done) {
            if (second) break;
            mA = walk_result(c, w);
            mk = walk_init(w, PB, cntB, tB, cx + 1, cy);
            w.Kc = window_key<SHAPE>(cx + 1, cy);
            cxc = cx + 1;
            second = true;
        }
    }
    mB = walk_result(c, w);
#ifdef IMF_STATS
    // [128..]: pairs, same direction, sum |PA-PB|, sum |mA-PA|, sum |mB-PB|, sum union length (same dir)
    {
        const bool upA = cntA <= tA, upB = cntB <= tB;
        atomicAdd(&g_stats[128], 1ull);
        if (upA == upB) {
            atomicAdd(&g_stats[129], 1ull);
            const int lo = min(min(PA, PB), min(mA, mB)), hi = max(max(PA, PB), max(mA, mB));
            atomicAdd(&g_stats[133], (unsigned long long)(hi - lo));
        }
        atomicAdd(&g_stats[130], (unsigned long long)abs(PA - PB));
        atomicAdd(&g_stats[131], (unsigned long long)abs(mA - PA));
        atomicAdd(&g_stats[132], (unsigned long long)abs(mB - PB));
    }
#endif
}

// Gather C[m] (the input value at omega[m]'s position, core.py:366) and the
// flat destination index; the store is issued later so the L2 latency of the
// gather overlaps the next slide.
struct Pend {
    uint32_t v;
    long long d;
    bool ok;
};

__device__ __forceinline__ void store_out(const Geom& g, const Pend& o) {
    if (!o.ok) return;
    if (g.dtype == DT_U8)
        ((uint8_t*)g.dst)[o.d] = (uint8_t)o.v;
    else if (g.dtype == DT_U16)
        ((uint16_t*)g.dst)[o.d] = (uint16_t)o.v;
    else
        ((uint32_t*)g.dst)[o.d] = o.v;
}

// Phase-D output path of one thread: the pair's destination index advances by
// one output row per step, and the source of C[m] -- input-tile pixel (x, y)
// of omega[m] -- is base + y*s_y + x*s_x with 32-bit strides when the tile's
// input box lies inside the image (no clamp; src_offset otherwise).
struct PairOut {
    long long d;        // destination element index of window A at the current row
    long long dx;       // destination stride between A and B (one output column)
    long long drow;     // destination stride of one output row
    long long sbase;    // interior tiles: element offset of input-tile pixel (0, 0)
    int sy, sx;         // interior tiles: 32-bit source strides
    bool interior;
    bool okA, okB;      // the pair's columns lie inside the output
};

// (omega in shared memory: read through its shared address, an LDS, not a
// generic load of the generic pointer)
template <bool OMG>
__device__ __forceinline__ Pend gather_pair(const Geom& g, const TileCoord& tc, const PairOut& po,
                                            const uint16_t* om, uint32_t om_a, int m, bool okrow, bool okcol,
                                            long long d) {
    Pend o;
    o.ok = okrow && okcol;
    o.d = d;
    o.v = 0;
    if (o.ok) {
        const uint32_t e = OMG ? (uint32_t)om[m] : lds16(om_a + 2 * m);
        const int ly = (int)(e >> 8), lx = (int)(e & 0xff);
        const long long so = po.interior ? po.sbase + (ly * po.sy + lx * po.sx) : src_offset(g, tc, ly, lx);
        if (g.dtype == DT_U8)
            o.v = __ldg((const uint8_t*)tc.src + so);
        else if (g.dtype == DT_U16)
            o.v = __ldg((const uint16_t*)tc.src + so);
        else
            o.v = __ldg((const uint32_t*)tc.src + so);
    }
    return o;
}

__device__ __forceinline__ int target_at2(const Geom& g, const PairParams& p, const TileCoord& tc, int row,
                                          int col) {
    if (!p.tmap) return p.target;
    const int y = min(tc.oy0 + row, g.out_h - 1), x = min(tc.ox0 + col, g.out_w - 1);
    return __ldg(p.tmap + (long long)y * g.out_w + x);
}

// Warp-collaborative refine for the few seed windows (lane l tests ranks
// v0+2l, v0+2l+1 of each 64-rank block), generic membership.
template <int SHAPE>
__device__ int refine_warp2(const PairCtx& c, int cx, int cy, int P, int cnt, int t) {
    const int lane = threadIdx.x & 31;
    const unsigned lt = lanemask_lt();
    const bool up = cnt <= t;
    int need = up ? t - cnt : cnt - t - 1;
    const int R2 = c.R2p1 - 1;
    auto inside = [&](int v) -> bool {
        if (v < 0 || v >= c.N) return false;
        const uint32_t e = c.om[v];
        const int dx = (int)(e & 0xffu) - cx, dyr = (int)(e >> 8) - cy;
        if (SHAPE == SH_CIRCLE || SHAPE == SH_CIRCLEW) return dx * dx + dyr * dyr <= R2;
        if (SHAPE == SH_SQUARE) return max(abs(dx), abs(dyr)) <= c.r;
        const int dy = dyr + c.r;
        if ((unsigned)dy > (unsigned)(2 * c.r)) return false;
        const int sp = c.span[dy];
        return (unsigned)(dx - (int)(short)(sp & 0xffff)) < (unsigned)(sp >> 16);
    };
    for (int v0 = up ? P : P - 64;; v0 += up ? 64 : -64) {
        if (up ? v0 >= c.N : v0 + 64 <= 0) return -1;
        const int v = v0 + 2 * lane;
        const bool i0 = inside(v), i1 = inside(v + 1);
        const unsigned b0 = __ballot_sync(0xffffffffu, i0), b1 = __ballot_sync(0xffffffffu, i1);
        const int pc = __popc(b0) + __popc(b1);
        if (need < pc) {
            const int k = up ? need : pc - 1 - need;
            const int pre = __popc(b0 & lt) + __popc(b1 & lt);
            const bool h0 = i0 && pre == k;
            const bool h1 = i1 && pre + (i0 ? 1 : 0) == k;
            const unsigned hb = __ballot_sync(0xffffffffu, h0 || h1);
            const int L = __ffs(hb) - 1;
            const int off = __shfl_sync(0xffffffffu, h0 ? 0 : 1, L);
            return v0 + 2 * L + off;
        }
        need -= pc;
    }
}

// Is rank v's pixel in the window at (cx, cy)?  (ordinal.py:175-185)
template <int SHAPE>
__device__ __forceinline__ bool inside1(const PairCtx& c, int v, int cx, int cy) {
    const uint32_t e = c.om[v];
    const int dx = (int)(e & 0xffu) - cx, dyr = (int)(e >> 8) - cy;
    if (SHAPE == SH_CIRCLE || SHAPE == SH_CIRCLEW) return dx * dx + dyr * dyr <= c.R2p1 - 1;
    if (SHAPE == SH_SQUARE) return max(abs(dx), abs(dyr)) <= c.r;
    const int dy = dyr + c.r;
    if ((unsigned)dy > (unsigned)(2 * c.r)) return false;
    const int sp = c.span[dy];
    return (unsigned)(dx - (int)(short)(sp & 0xffff)) < (unsigned)(sp >> 16);
}

// Solved window (answer m, target t) -> slide state (pivot P, count below P).
// With halved ranks (hs) the ordinal image holds rank >> 1, which compares
// exactly only against EVEN pivots: P = m & ~1, and when m is odd the count
// below P is t minus [rank m-1 is in the window].
template <int SHAPE>
__device__ __forceinline__ void to_state(const PairCtx& c, int hs, int m, int t, int cx, int cy, int& P,
                                         int& cnt) {
    P = m;
    cnt = t;
    if (hs && (m & 1)) {
        P = m - 1;
        cnt = t - (inside1<SHAPE>(c, m - 1, cx, cy) ? 1 : 0);
    }
}

template <int SHAPE, bool OMG>
__global__ void __launch_bounds__(512, 2) k2_pair(Geom g, PairParams p, const __grid_constant__ PairTab kt,
                                               const uint16_t* __restrict__ omega_in) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nwarps = blockDim.x >> 5;
    const int N = g.N, Npad = g.Npad, Sw = g.Sw, r = g.r;
    const int T = g.Tw, TY = g.Th, G = p.G, TH = T >> 1;  // T: tile columns, TY: tile rows
    const int hs = p.hs;
    // chunk-relative tile: the chunk's bottom image-border tile rows first (slow:
    // their windows reach into the clamped margin, long all-tie walks), so
    // they do not form the launch's tail
    const int bt = chunk_tile_ranges(g);
    const TileCoord tc = tile_coord(g, g.tile_begin + bt);

    const uint16_t* om_g = omega_in + (long long)bt * (Npad + 2 * OMEGA_SLOT_PAD) + OMEGA_SLOT_PAD;
    // omega: shared copy (8 sentinels before rank 0), or the global slot (OMG)
    uint16_t* om_sh = reinterpret_cast<uint16_t*>(smem) + 8;
    const uint16_t* om = OMG ? om_g : om_sh;
    uint16_t* I = OMG ? reinterpret_cast<uint16_t*>(smem) : om_sh + Npad + 8;  // 16-byte aligned
    const int Ipad = (Sw * g.Sh + 15) & ~7;  // I covers the whole Sw x Sh input tile
    int* st_P = reinterpret_cast<int*>(I + Ipad);
    int* st_C = st_P + G * T;
    int* deltas = st_C + G * T;                // max(G*T, TY) entries
    int* hist = deltas + max(G * T, TY);       // 32 bins
    int* seedP = hist + 32;                    // G
    int* seedC = seedP + G;                    // G
    int* span_s = seedC + G;                   // 2r+1
    uint32_t* rowk = reinterpret_cast<uint32_t*>(span_s + 2 * r + 1);  // 256 (SH_POLY)
    uint32_t* gsc = rowk + 256;                                         // 2 * G * 32 (grouped phase C)
    int* rowd = reinterpret_cast<int*>(gsc + 64 * G);                   // TY + 1 (grouped seed counts)

    // ---- 0. stage omega, build the ordinal image --------------------------
    {
        const uint4* src = reinterpret_cast<const uint4*>(om_g);
        uint4* dst = reinterpret_cast<uint4*>(om_sh);
        for (int i = tid; i < (Npad >> 3); i += blockDim.x) {
            const uint4 v = src[i];
            if (!OMG) dst[i] = v;
            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int q = 0; q < 8; q++) {
                const int rank = (i << 3) + q;
                if (rank < N) {
                    const uint32_t e = (q & 1) ? (w[q >> 1] >> 16) : (w[q >> 1] & 0xffffu);
                    I[(int)(e >> 8) * Sw + (int)(e & 0xffu)] = (uint16_t)(rank >> hs);
                }
            }
        }
        if (!OMG && tid < 8) {
            om_sh[-8 + tid] = 0xffffu;  // sentinels: outside every window
            om_sh[Npad + tid] = 0xffffu;
        }
        for (int i = Sw * g.Sh + tid; i < Ipad; i += blockDim.x) I[i] = 0;
        if (tid < 32) hist[tid] = 0;
        for (int i = tid; i <= TY; i += blockDim.x) rowd[i] = 0;
        for (int i = tid; i < 2 * r + 1; i += blockDim.x) span_s[i] = kt.span[i];
        if (SHAPE == SH_POLYSYM) {  // 127 - h(|dy|), h = the row's half-width (xlo = -h); 256 entries
            for (int i = tid; i < 256; i += blockDim.x) {  // (|dy| of the sentinel entries exceeds 127)
                int v = 128;
                if (i <= r) {
                    const int sp = kt.span[i + r];
                    if (sp >> 16) v = 127 + (int)(short)(sp & 0xffff);
                }
                reinterpret_cast<uint8_t*>(rowk)[i] = (uint8_t)v;
            }
        }
        if (SHAPE == SH_POLY) {
            for (int i = tid; i < 256; i += blockDim.x) {
                const int dy = i - 128;
                uint32_t v = 0;  // rows outside the kernel: never inside
                if (dy >= -r && dy <= r) {
                    const int sp = kt.span[dy + r];
                    const int xlo = (int)(short)(sp & 0xffff), xhi = xlo + (sp >> 16);
                    if (sp >> 16) v = (uint32_t)(0x8000 - (128 + xlo)) | ((uint32_t)(0x8000 - (128 + xhi)) << 16);
                }
                rowk[i] = v;
            }
        }
    }
    __syncthreads();

    const uint32_t I_a = (uint32_t)__cvta_generic_to_shared(I);
    // omega's shared address and -(r(r+1)+1) held in registers (opaque to the
    // compiler, which would otherwise rebuild them inside every refine step)
    uint32_t om_a = OMG ? 0u : (uint32_t)__cvta_generic_to_shared(om_sh);
    const int nR2p1 = p.nR2p1;
    uint32_t x80 = 0x80808080u;
    asm volatile("" : "+r"(om_a), "+r"(x80));
    const PairCtx c{om_a, om, span_s, N, r, p.R2p1, (uint32_t)__cvta_generic_to_shared(rowk), nR2p1, x80};
    const int R = TY / G;
    const int g0 = G >> 1;
    const int cs = (T >> 1) & ~1;  // seed column (even: a pair base)
    auto seed_row = [&](int gi) { return gi * R + (R >> 1); };

    // ---- A. direct seed: 32-bin rank histogram over the window ------------
    const int sh = max(0, 32 - __clz(max(((N - 1) >> hs), 1)) - 5);  // 32 bins over I's range
    const int ytop = seed_row(0), ybot = seed_row(G - 1);
    if (!p.grouped) {
    {
        const int cx = cs + r, cy = seed_row(g0) + r;
        unsigned lm[5];
#pragma unroll
        for (int b = 0; b < 5; b++) lm[b] = ((lane >> b) & 1) ? 0u : 0xffffffffu;
        int cntb = 0;
        for (int dy = wid; dy <= 2 * r; dy += nwarps) {
            const int sp = span_s[dy];
            const int w = sp >> 16;
            if (w <= 0) continue;
            const uint16_t* row = I + (cy - r + dy) * Sw + cx + (int)(short)(sp & 0xffff);
            for (int o0 = 0; o0 < w; o0 += 32) {
                const int o = o0 + lane;
                const bool ok = o < w;
                const unsigned b = ok ? (unsigned)(row[o] >> sh) : 0u;
                unsigned m = __ballot_sync(0xffffffffu, ok);
#pragma unroll
                for (int bit = 0; bit < 5; bit++)
                    m &= ~(__ballot_sync(0xffffffffu, (b >> bit) & 1u) ^ ~lm[bit]);
                cntb += __popc(m);
            }
        }
        if (cntb) atomicAdd(&hist[lane], cntb);
    }
    __syncthreads();
    if (wid == 0) {
        const int row = seed_row(g0);
        const int tgt = target_at2(g, p, tc, row, cs);
        const int tot = hist[lane];
        int cum = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, cum, o);
            if (lane >= o) cum += v;
        }
        const int B = __ffs(__ballot_sync(0xffffffffu, cum > tgt)) - 1;
        const int cnt = __shfl_sync(0xffffffffu, cum - tot, B);
        const int m = refine_warp2<SHAPE>(c, cs + r, row + r, B << (sh + hs), cnt, tgt);
        if (lane == 0) {
            if (m < 0) atomicOr(p.status, 1);
            seedP[g0] = max(m, 0);
            seedC[g0] = tgt;
        }
    }
    __syncthreads();

    // ---- B. other seed rows' centre windows: vertical deltas at column cs --
    if (G > 1) {
        int P0, C0;
        to_state<SHAPE>(c, hs, seedP[g0], seedC[g0], cs + r, seed_row(g0) + r, P0, C0);
        const uint32_t K0 = pivot_k(P0 >> hs, P0 >> hs);
        for (int y = ytop + tid; y < ybot; y += blockDim.x) {  // step y -> y+1 at column cs
            uint32_t gi_, go_;
            vcount<4>(I_a + 2 * (y * Sw + cs), kt.v, p.nv_even, p.nv, K0, gi_, go_);
            deltas[y] = (int)(go_ & 0xffffu) - (int)(gi_ & 0xffffu);
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
            const int cnt = C0 + (int)__reduce_add_sync(0xffffffffu, (unsigned)part);
            const int tgt = target_at2(g, p, tc, y1, cs);
            const int m = refine_warp2<SHAPE>(c, cs + r, y1 + r, P0, cnt, tgt);
            if (lane == 0) {
                if (m < 0) atomicOr(p.status, 1);
                seedP[gi] = max(m, 0);
                seedC[gi] = tgt;
            }
        }
        __syncthreads();
    }

    }  // !grouped (phases A, B)

    // ---- C+D grouped: with one warp pair per seed-row group (T <= 64), each
    // group does its own seed row and then its sweeps, synchronized by a named
    // barrier of its 64 threads only -- no CTA-wide wait for the slowest
    // group's seed-row refines.
    if (p.grouped) {
        const int q = lane, rest = wid, gi = rest % G, half = rest / G;  // half 0: down warp
        const int row = seed_row(gi);
        auto gbar = [&]() { asm volatile("bar.sync %0, 64;" ::"r"(1 + gi) : "memory"); };
        // this group's seed: the centre window of its seed row.  The counts
        // below the even pivot N/2 of ALL groups' seed windows come from one
        // CTA-wide pass -- the top group's window in full plus the down-slide
        // deltas of column cs between the seed rows (rowd[TY], rowd[y]) --
        // then each group walks warp-collaboratively to its target
        // (core.py:47-60, :87-146).
        const int Pg = (N >> 1) & ~1;
        {
            const int Pq = Pg >> hs;
            {
                const int cx = cs + r, cy = ytop + r;
                int cnt = 0;
                for (int dy = wid; dy <= 2 * r; dy += nwarps) {
                    const int sp = span_s[dy];
                    const int w = sp >> 16;
                    const uint16_t* rowp = I + (cy - r + dy) * Sw + cx + (int)(short)(sp & 0xffff);
                    for (int o0 = 0; o0 < w; o0 += 32) {
                        const int o = o0 + lane;
                        cnt += __popc(__ballot_sync(0xffffffffu, o < w && (int)rowp[o] < Pq));
                    }
                }
                if (lane == 0 && cnt) atomicAdd(&rowd[TY], cnt);
            }
            // down-slide deltas (entering < Pq) - (exiting < Pq) of the column-cs
            // window from row y to y+1: warps = rows, lanes = kernel columns
            // (their offsets loaded once into registers), one warp reduction
            // per row.  (Lanes = rows would put the lanes 2*Sw bytes apart:
            // 16-way shared bank conflicts.)
            if (ybot > ytop) {
                int2 ov[8];  // entering / exiting byte offsets of columns lane + 32i (nv <= 249)
#pragma unroll
                for (int i = 0; i < 8; i++) {
                    const int k = lane + 32 * i;
                    ov[i] = make_int2(0, 0);
                    if (k < p.nv) {
                        const int2 o = kt.v[k];
                        const int adj = k >= p.nv_even ? 2 : 0;  // odd entries: the high half of the word
                        ov[i] = make_int2(o.x + adj, o.y + adj);
                    }
                }
                const int nvk = (p.nv + 31) >> 5;
                for (int y = ytop + wid; y < ybot; y += nwarps) {
                    const uint32_t b = I_a + 2 * (y * Sw + cs);
                    int d = 0;
#pragma unroll
                    for (int i = 0; i < 8; i++)
                        if (i < nvk && lane + 32 * i < p.nv)
                            d += ((int)lds16(b + ov[i].x) < Pq) - ((int)lds16(b + ov[i].y) < Pq);
                    d = (int)__reduce_add_sync(0xffffffffu, (unsigned)d);
                    if (lane == 0) rowd[y] = d;
                }
            }
        }
        __syncthreads();
        if (half == 0) {
            int part = 0;
            for (int y = ytop + lane; y < row; y += 32) part += rowd[y];
            const int cnt = rowd[TY] + (int)__reduce_add_sync(0xffffffffu, (unsigned)part);
            const int tgt = target_at2(g, p, tc, row, cs);
            const int m = refine_warp2<SHAPE>(c, cs + r, row + r, Pg, cnt, tgt);
            if (lane == 0) {
                if (m < 0) atomicOr(p.status, 1);
                seedP[gi] = max(m, 0);
                seedC[gi] = tgt;
            }
        }
        gbar();
        int P, C0;
        to_state<SHAPE>(c, hs, seedP[gi], seedC[gi], cs + r, row + r, P, C0);
        uint32_t* gin = gsc + gi * 64;  // [0..32): entering counts, [32..64): exiting counts
        if (q < TH) {  // pair-step (2q, 2q+1): the down warp counts entering, the up warp exiting
            const uint32_t K = pivot_k(P >> hs, P >> hs);
            const uint32_t b = I_a + 2 * (row * Sw + 2 * q);
            gin[half * 32 + q] = half ? hcount(b, kt.hx, p.nhx_even, p.nh, K)
                                      : hcount(b, kt.he, p.nhe_even, p.nh, K);
        }
        gbar();
        // the down warp turns the step deltas into prefix sums by one warp
        // scan: pref[k] = sum of deltas of steps 0..k-1, kept for k = 1..T in
        // deltas[gi*T + k - 1] (pref[0] = 0), so window j's count below P is
        // C0 + pref[j] - pref[cs] with no per-thread loop over the steps
        if (half == 0) {
            int d0 = 0, d1 = 0;
            if (q < TH) half_diff(gin[32 + q], gin[q], d0, d1);
            const int pr = d0 + d1;
            int incl = pr;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, incl, o);
                if (q >= o) incl += t;
            }
            if (q < TH) {
                deltas[gi * T + 2 * q] = incl - pr + d0;  // pref[2q + 1]
                deltas[gi * T + 2 * q + 1] = incl;        // pref[2q + 2]
            }
        }
        gbar();
        // (giving one warp the columns far from cs and the other the near ones
        // measured slower on the smooth field, no faster on noise)
        const int j = half * 32 + q;
        if (j < T) {
            auto pref = [&](int k) { return k ? deltas[gi * T + k - 1] : 0; };
            const int cnt = C0 + pref(j) - pref(cs);
            const int tgt = target_at2(g, p, tc, row, j);
            int m = (j == cs) ? seedP[gi] : refine8<SHAPE, OMG>(c, j + r, row + r, P, cnt, tgt);
            if (m < 0) {
                atomicOr(p.status, 1);
                m = 0;
            }
            st_P[gi * T + j] = m;
            st_C[gi * T + j] = tgt;
        }
        gbar();
    } else {
    // ---- C. seed rows: horizontal deltas (pairs of steps) at the row pivot --
    for (int u = tid; u < G * TH; u += blockDim.x) {  // steps 2q -> 2q+1, 2q+1 -> 2q+2 of row gi
        const int gi = u / TH, q = u - gi * TH;
        int P, C0;
        to_state<SHAPE>(c, hs, seedP[gi], seedC[gi], cs + r, seed_row(gi) + r, P, C0);
        const uint32_t K = pivot_k(P >> hs, P >> hs);
        const uint32_t b = I_a + 2 * (seed_row(gi) * Sw + 2 * q);
        const uint32_t ge_in = hcount(b, kt.he, p.nhe_even, p.nh, K);
        const uint32_t ge_out = hcount(b, kt.hx, p.nhx_even, p.nh, K);
        int d0, d1;
        half_diff(ge_out, ge_in, d0, d1);
        deltas[gi * T + 2 * q] = d0;
        deltas[gi * T + 2 * q + 1] = d1;
    }
    __syncthreads();
    for (int u = tid; u < G * T; u += blockDim.x) {
        const int gi = u / T, j = u - gi * T, row = seed_row(gi);
        int P, cnt;
        to_state<SHAPE>(c, hs, seedP[gi], seedC[gi], cs + r, row + r, P, cnt);
        if (j > cs) {
            for (int i = cs; i < j; i++) cnt += deltas[gi * T + i];
        } else {
            for (int i = j; i < cs; i++) cnt -= deltas[gi * T + i];
        }
        const int tgt = target_at2(g, p, tc, row, j);
        int m = (j == cs) ? seedP[gi] : refine8<SHAPE, OMG>(c, j + r, row + r, P, cnt, tgt);
        if (m < 0) {
            atomicOr(p.status, 1);
            m = 0;
        }
        st_P[u] = m;
        st_C[u] = tgt;
    }
    __syncthreads();
    }  // !grouped

    // ---- D. vertical sweeps: thread = (direction, group, column pair) ------
    // lanes of a (direction, group) padded to whole warps: every warp sweeps
    // one row band in one direction (uniform trip counts, one I row per load)
    const int THP = (TH + 31) & ~31;
    for (int u = tid; u < 2 * G * THP; u += blockDim.x) {
        const int q = u % THP, rest = u / THP, gi = rest % G;
        if (q >= TH) continue;
        const bool down = rest < G;
        const int row0 = seed_row(gi);
        const int rend = (gi == G - 1) ? TY : (gi + 1) * R;  // exclusive
        const int j0 = 2 * q, j1 = j0 + 1;
        const int mA0 = st_P[gi * T + j0], mB0 = st_P[gi * T + j1];
        int PA, cA, PB, cB;
        to_state<SHAPE>(c, hs, mA0, st_C[gi * T + j0], j0 + r, row0 + r, PA, cA);
        to_state<SHAPE>(c, hs, mB0, st_C[gi * T + j1], j1 + r, row0 + r, PB, cB);
        PairOut po;
        {
            const int X0 = tc.ox0 - r + g.vshift, Y0 = tc.oy0 - r + g.vshift;
            po.interior = X0 >= 0 && Y0 >= 0 && X0 + Sw <= g.W && Y0 + g.Sh <= g.H &&
                          (long long)(g.H - 1) * g.s_y + (long long)(g.W - 1) * g.s_x < (1ll << 31);
            po.sbase = (long long)Y0 * g.s_y + (long long)X0 * g.s_x;
            po.sy = (int)g.s_y;
            po.sx = (int)g.s_x;
            po.dx = g.d_x;
            po.drow = g.d_y;
            po.d = tc.b * g.d_b + tc.c * g.d_c + (long long)(tc.oy0 + row0) * g.d_y + (long long)(tc.ox0 + j0) * g.d_x;
            po.okA = tc.ox0 + j0 < g.out_w;
            po.okB = tc.ox0 + j1 < g.out_w;
        }
        Pend wa{0, 0, false}, wb{0, 0, false};
        if (down) {
            const bool okr = tc.oy0 + row0 < g.out_h;
            wa = gather_pair<OMG>(g, tc, po, om, c.om_a, mA0, okr, po.okA, po.d);
            wb = gather_pair<OMG>(g, tc, po, om, c.om_a, mB0, okr, po.okB, po.d + po.dx);
        }
        const int nsteps = down ? (rend - 1 - row0) : (row0 - gi * R);
        // test hook: an inconsistent count (core.py:31-36 defect path)
        const bool dbg = p.debug_defect && bt == 0 && g.tile_begin == 0 && u == 0;
        int row = row0;
        for (int s = 0; s < nsteps; s++) {
            const uint32_t K = pivot_k(PA >> hs, PB >> hs);
            uint32_t ge_in, ge_out;
            int dA, dB;
            if (down) {
                vcount<4>(I_a + 2 * (row * Sw + j0), kt.v, p.nv_even, p.nv, K, ge_in, ge_out);
                half_diff(ge_out, ge_in, dA, dB);
                row++;
            } else {
                vcount<4>(I_a + 2 * ((row - 1) * Sw + j0), kt.v, p.nv_even, p.nv, K, ge_in, ge_out);
                half_diff(ge_in, ge_out, dA, dB);
                row--;
            }
            store_out(g, wa);
            store_out(g, wb);
            cA += dA;
            cB += dB;
            if (dbg && s == 0) cA += 1 << 20;
            const int tA = target_at2(g, p, tc, row, j0);
            const int tB = target_at2(g, p, tc, row, j1);
            int mA, mB;
            if (p.refine_mode & 1)
                refine8x2_seq<SHAPE, OMG>(c, j0 + r, row + r, PA, cA, tA, PB, cB, tB, mA, mB);
            else
                refine8x2<SHAPE, OMG>(c, j0 + r, row + r, PA, cA, tA, PB, cB, tB, mA, mB);
            if ((mA | mB) < 0) {
                atomicOr(p.status, 1);
                mA = max(mA, 0);
                mB = max(mB, 0);
            }
            po.d += down ? po.drow : -po.drow;
            const bool okr = tc.oy0 + row < g.out_h;
            wa = gather_pair<OMG>(g, tc, po, om, c.om_a, mA, okr, po.okA, po.d);
            wb = gather_pair<OMG>(g, tc, po, om, c.om_a, mB, okr, po.okB, po.d + po.dx);
            to_state<SHAPE>(c, hs, mA, tA, j0 + r, row + r, PA, cA);
            to_state<SHAPE>(c, hs, mB, tB, j1 + r, row + r, PB, cB);
        }
        store_out(g, wa);
        store_out(g, wb);
    }
}

#define IMF_K2P(S, O) \
    template __global__ void k2_pair<S, O>(Geom, PairParams, const __grid_constant__ PairTab, const uint16_t*);
IMF_K2P(SH_SPAN, false)
IMF_K2P(SH_CIRCLE, false)
IMF_K2P(SH_SQUARE, false)
IMF_K2P(SH_SPAN, true)
IMF_K2P(SH_CIRCLE, true)
IMF_K2P(SH_SQUARE, true)
IMF_K2P(SH_POLY, false)
IMF_K2P(SH_POLY, true)
IMF_K2P(SH_POLYSYM, false)
IMF_K2P(SH_POLYSYM, true)
IMF_K2P(SH_CIRCLEW, false)
IMF_K2P(SH_CIRCLEW, true)
#undef IMF_K2P

size_t k2_pair_smem_bytes(int N, int Npad, int NI, int r, int G, int T, int TY, bool omg) {
    const int Ipad = (NI + 15) & ~7;
    const int gt = G * T;
    return (omg ? 0 : 2 * (size_t)(Npad + 16)) + 2 * (size_t)Ipad +
           4 * (size_t)(2 * gt + (gt > TY ? gt : TY) + 32 + 2 * G + 2 * r + 1 + 256 + 64 * G + TY + 1) + 16;
}

// Host: build the pair tables for input-tile row stride Sw.  Returns false if
// an offset list would overflow PT_MAX.
bool build_pair_tab(const int* row_dy, const int* row_xlo, const int* row_xhi, int nrows, const int* col_dx,
                    const int* col_ytop, const int* col_ybot, int ncols, int r, int Sw, PairTab& t,
                    PairParams& p) {
    if (ncols > PT_MAX || nrows > PT_MAX || 2 * r + 1 > PT_MAX) return false;
    memset(&t, 0, sizeof(t));
    // element offset of a pixel relative to the pair base (row*Sw + 2q): (r + dy)*Sw + r + dx
    auto put_v = [&](int k, int e, int x, bool odd) {
        t.v[k] = odd ? make_int2(2 * (e - 1), 2 * (x - 1)) : make_int2(2 * e, 2 * x);
    };
    int k = 0;
    for (int pass = 0; pass < 2; pass++) {
        for (int i = 0; i < ncols; i++) {
            const int e = (r + col_ybot[i] + 1) * Sw + r + col_dx[i];
            const int x = (r + col_ytop[i]) * Sw + r + col_dx[i];
            const bool odd = (e & 1) != 0;  // e and x share the parity of r + dx (Sw even)
            if (odd == (pass == 1)) put_v(k++, e, x, odd);
        }
        if (pass == 0) p.nv_even = k;
    }
    p.nv = ncols;
    if (p.nv_even > 127 || ncols - p.nv_even > 127) return false;  // vcount's acc_dp4 runs
    auto fill_h = [&](int* dst, bool hi, int& ne) {
        int kk = 0;
        for (int pass = 0; pass < 2; pass++) {
            for (int i = 0; i < nrows; i++) {
                const int o = (r + row_dy[i]) * Sw + r + (hi ? row_xhi[i] : row_xlo[i]);
                const bool odd = (o & 1) != 0;
                if (odd == (pass == 1)) dst[kk++] = odd ? 2 * (o - 1) : 2 * o;
            }
            if (pass == 0) ne = kk;
        }
    };
    fill_h(t.he, true, p.nhe_even);
    fill_h(t.hx, false, p.nhx_even);
    p.nh = nrows;
    for (int i = 0; i < nrows; i++)
        t.span[row_dy[i] + r] = (row_xlo[i] & 0xffff) | ((row_xhi[i] - row_xlo[i]) << 16);
    return true;
}

}  // namespace imf

#ifdef IMF_STATS
extern "C" int imf_stats(unsigned long long* out, int reset) {
    if (cudaMemcpyFromSymbol(out, imf::g_stats, sizeof(imf::g_stats))) return 2;
    if (reset) {
        static const unsigned long long z[256] = {};
        cudaMemcpyToSymbol(imf::g_stats, z, sizeof(z));
    }
    return 0;
}
#endif
