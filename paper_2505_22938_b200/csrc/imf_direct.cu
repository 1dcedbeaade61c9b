// imf_direct.cu -- direct selection for tiny windows (area <= 32, e.g. circle
// or square r <= 2) on sm_100a.
//
// For a window of at most 32 pixels the rank machinery (tile sort + pivot
// walks through a rank space far sparser than the window) costs more than
// selecting directly: each thread loads its window's u32 order keys
// (ordinal.py:109-123; u8/u16 values unchanged) from a shared-memory input tile
// into registers, sorts them with a 32-element bitonic network (240
// compare-exchanges, padded with 0xffffffff keys that sort last), and outputs
// the key of rank t decoded back to the value (core.py:366: the t-th smallest
// of the window multiset -- the definition, oracle.py:88-121).
#include "imf_kernels.cuh"

namespace imf {


__device__ __forceinline__ void cx_swap(uint32_t& a, uint32_t& b, bool up) {
    const uint32_t lo = min(a, b), hi = max(a, b);
    a = up ? lo : hi;
    b = up ? hi : lo;
}

template <int DT>
__global__ void __launch_bounds__(1024) k_direct(Geom g, const __grid_constant__ DirectTab dt, int target,
                                                 const int* __restrict__ tmap) {
    extern __shared__ __align__(16) uint32_t keys[];  // Sw x Sh input tile
    const TileCoord tc = tile_coord(g, g.tile_begin + blockIdx.x);
    const int Sw = g.Sw, Sh = g.Sh, n = Sw * Sh;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int y = i / Sw, x = i - y * Sw;
        keys[i] = load_key(g, tc, y, x);
    }
    __syncthreads();
    const int tx = threadIdx.x % g.Tw, ty = threadIdx.x / g.Tw;
    if (ty >= g.Th) return;
    const int oy = tc.oy0 + ty, ox = tc.ox0 + tx;
    if (oy >= g.out_h || ox >= g.out_w) return;
    const uint32_t* c = keys + (ty + g.r) * Sw + tx + g.r;
    uint32_t k[32];
#pragma unroll
    for (int i = 0; i < 32; i++) k[i] = i < dt.area ? c[dt.off[i]] : 0xffffffffu;
    // bitonic sort, ascending
#pragma unroll
    for (int size = 2; size <= 32; size <<= 1)
#pragma unroll
        for (int stride = size >> 1; stride > 0; stride >>= 1)
#pragma unroll
            for (int i = 0; i < 32; i++) {
                const int j = i ^ stride;
                if (j > i) cx_swap(k[i], k[j], (i & size) == 0);
            }
    const int t = tmap ? __ldg(tmap + (long long)oy * g.out_w + ox) : target;
    uint32_t key = k[0];
#pragma unroll
    for (int i = 1; i < 32; i++)
        if (i == t) key = k[i];
    const long long d = tc.b * g.d_b + (long long)oy * g.d_y + (long long)ox * g.d_x + tc.c * g.d_c;
    if (DT == DT_U8) {
        ((uint8_t*)g.dst)[d] = (uint8_t)key;
    } else if (DT == DT_U16) {
        ((uint16_t*)g.dst)[d] = (uint16_t)key;
    } else {
        // inverse of float_key: keys with the top bit set came from non-negative floats
        ((uint32_t*)g.dst)[d] = (key & 0x80000000u) ? (key & 0x7fffffffu) : ~key;
    }
}

template __global__ void k_direct<DT_U8>(Geom, const __grid_constant__ DirectTab, int, const int*);
template __global__ void k_direct<DT_U16>(Geom, const __grid_constant__ DirectTab, int, const int*);
template __global__ void k_direct<DT_F32>(Geom, const __grid_constant__ DirectTab, int, const int*);

}  // namespace imf
