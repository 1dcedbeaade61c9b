// imf_k1.cuh -- device helpers shared by the K1 (ordinal transform) kernels:
// omega scratch slots, the packed 16-bit histogram scan.
#pragma once
#include "imf_kernels.cuh"

namespace imf {

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

// store_omega through the TMA engine: one thread issues a bulk shared->global
// copy of the Npad entries (cp.async.bulk), the pads are stored by 16 threads,
// and the issuing thread waits for the copy to finish reading shared memory
// before the CTA exits (the other threads are free at once).
__device__ __forceinline__ void store_omega_bulk(const Geom& g, const uint16_t* om_s, uint16_t* om_g) {
    if (threadIdx.x == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the scatter's stores -> async proxy
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(om_g),
                     "r"((uint32_t)__cvta_generic_to_shared(om_s)), "r"(2 * g.Npad)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
    if (threadIdx.x < OMEGA_SLOT_PAD) {
        om_g[-OMEGA_SLOT_PAD + (int)threadIdx.x] = 0xffffu;
        om_g[g.Npad + threadIdx.x] = 0xffffu;
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
        unsigned long long sqacc = 0;  // this lane's sum of squared counters (sumsq)
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
            if (starts || sumsq) {
                const uint32_t cw[4] = {q.x, q.y, q.z, q.w}, bw[4] = {b0, b1, b2, b3};
#pragma unroll
                for (int k = 0; k < 4; k++) {
                    const uint32_t lo = cw[k] & 0xffffu, hi = cw[k] >> 16, e0 = bw[k], e1 = bw[k] + lo;
                    if (starts) {  // bit at every non-empty counter's first position (bucket starts)
                        if (lo) atomicOr(&starts[e0 >> 5], 1u << (e0 & 31));
                        if (hi) atomicOr(&starts[e1 >> 5], 1u << (e1 & 31));
                    }
                    sqacc += (unsigned long long)(lo * lo) + (unsigned long long)(hi * hi);
                }
            }
            q.x = b0 | ((b0 + (q.x & 0xffffu)) << 16);
            q.y = b1 | ((b1 + (q.y & 0xffffu)) << 16);
            q.z = b2 | ((b2 + (q.z & 0xffffu)) << 16);
            q.w = b3 | ((b3 + (q.w & 0xffffu)) << 16);
            wb[i0 + lane] = q;
            const uint32_t last = __shfl_sync(0xffffffffu, incl, 31);
            carry += (last & 0xffffu) + (last >> 16);
        }
        if (sumsq) {
            // clamp per lane at 2^26 (> kMaxSumSq: the tile falls back anyway) so
            // the 32-bit warp sum cannot wrap
            const unsigned wsq = __reduce_add_sync(0xffffffffu, (unsigned)min(sqacc, 1ull << 26));
            if (lane == 0 && wsq) atomicAdd(sumsq, (unsigned long long)wsq);
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

// hist16_exclusive_scan without bucket-start / sum-of-squares outputs, for
// 1024-thread CTAs and NW = 32768 words: lane l of warp w owns the 32
// CONSECUTIVE words [w*1024 + 32l, +32) (8 uint4 chunks), so the lane scans
// them sequentially in registers and the warp needs ONE shuffle scan (not one
// per chunk row).  Chunk loads are rotated by lane ((i + l) & 7) so a warp's
// 32 LDS.128 hit all 8 bank quads (4 wavefronts, conflict-free); the in-order
// prefix of chunk k is rebuilt from P = (sum of the lane's chunks before its
// first rotated chunk) and a running sum reset where the rotation wraps.
__device__ __forceinline__ void hist16_scan_lanes(uint32_t* hw) {
    constexpr int NW = 32768, PER = 1024, CH = 8;  // words per warp, chunks per lane
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    __shared__ uint32_t wt[32];
    uint4* wb = reinterpret_cast<uint4*>(hw + wid * PER + lane * 32);
    const int a = lane & (CH - 1);  // the lane's first chunk in rotated order
    uint32_t tot = 0, pre = 0;      // packed: all chunks / chunks before chunk a
#pragma unroll
    for (int i = 0; i < CH; i++) {
        const uint4 q = wb[(a + i) & (CH - 1)];
        const uint32_t cs = q.x + q.y + q.z + q.w;
        tot += cs;
        if (i >= CH - a) pre += cs;  // rotated position i holds chunk (a + i) - CH < a
    }
    const uint32_t T = (tot & 0xffffu) + (tot >> 16);
    uint32_t incl = T;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) wt[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        const uint32_t v = wt[lane];
        uint32_t x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += t;
        }
        wt[lane] = x - v;
    }
    __syncthreads();
    const uint32_t base = wt[wid] + incl - T;  // counters before the lane's first word
    // running exclusive prefix, unpacked: per word (counters lo, hi) the
    // output is s | (s + lo) << 16 and s advances by lo + hi -- LOP3, IADD,
    // LEA.HI and one PRMT per word
    uint32_t s = base + (pre & 0xffffu) + (pre >> 16);
    auto step = [&](uint32_t w) {
        const uint32_t e0 = s, e1 = s + (w & 0xffffu);
        s = e1 + (w >> 16);
        uint32_t r;
        asm("prmt.b32 %0, %1, %2, 0x5410;" : "=r"(r) : "r"(e0), "r"(e1));
        return r;
    };
#pragma unroll
    for (int i = 0; i < CH; i++) {
        const int k = (a + i) & (CH - 1);
        if (k == 0) s = base;  // wrapped to the lane's first chunk
        uint4 q = wb[k];
        q.x = step(q.x);
        q.y = step(q.y);
        q.z = step(q.z);
        q.w = step(q.w);
        wb[k] = q;
    }
    (void)NW;
}

}  // namespace imf
