// imf_kernels.cuh -- declarations shared between the kernel translation units
// (imf_sort.cu: K1, imf_select.cu / imf_pair.cu: K2, imf_direct.cu: K0) and
// the launch planner (imf_api.cu).  Each kernel source is compiled on its own
// (separate .o, no -rdc: only host launch stubs cross translation units) and
// explicitly instantiates the template kernels the planner launches.
#pragma once
#include <cuda.h>  // CUtensorMap (TMA descriptors; encoded through the runtime's driver entry point)

#include "imf_common.cuh"

namespace imf {

// ---- K1 (imf_sort.cu) -------------------------------------------------------
constexpr int kCoarse = 4096;          // f32 adaptive buckets: coarse bins on key >> 20
constexpr int kAdaptiveMinN = 16384;   // below this many tile pixels: plain top-16-bit buckets
constexpr int kRunMin = 1024;          // replicate-edge copy groups this large rank as one run
constexpr int kRunMinFloor = 2;

template <int DT, bool GMEM>
__global__ void __launch_bounds__(1024) k1_sort(Geom g, uint16_t* __restrict__ omega_out,
                                               unsigned char* __restrict__ gscratch,
                                               long long gscratch_stride, const int* __restrict__ only);
template <int DT>
__global__ void __launch_bounds__(1024) k1_count(Geom g, uint16_t* __restrict__ omega_out);
template <int DT, int NK, bool TMA>
__global__ void __launch_bounds__(1024) k1_count_reg(Geom g, uint16_t* __restrict__ omega_out,
                                                     const __grid_constant__ CUtensorMap tmap);
__global__ void __launch_bounds__(1024) k1_count_g(Geom g, uint16_t* __restrict__ omega_out);
template <int NK, bool GENT, bool FP>
__global__ void __launch_bounds__(1024) k1_f32_bucket(Geom g, uint16_t* __restrict__ omega_out,
                                                     int* __restrict__ fallback, uint32_t* __restrict__ gent,
                                                     long long gent_stride, unsigned long long max_sumsq);
__global__ void __launch_bounds__(1024) k1_f32_bucket_g(Geom g, uint16_t* __restrict__ omega_out,
                                                       int* __restrict__ fallback,
                                                       uint32_t* __restrict__ gent, long long gent_stride,
                                                       unsigned long long max_sumsq);
__global__ void __launch_bounds__(1024) k_coarse_hist(Geom g, int y0, int y1, uint32_t* __restrict__ counts);
__global__ void __launch_bounds__(1024) k_coarse_alloc(uint32_t* __restrict__ tab);

size_t k1_f32_bucket_g_smem_bytes(int N);
size_t k1_f32_bucket_smem_bytes(int N);
size_t k1_count_g_smem_bytes();
size_t k1_count_smem_bytes(int dtype, int Npad);
size_t k1_smem_bytes(int dtype, int Npad, int nwarps, bool gmem);
size_t k1_gscratch_bytes(int dtype, int Npad);

// ---- K2 general path (imf_select.cu) ---------------------------------------
template <bool CIRCLE, bool OMG>
__global__ void __launch_bounds__(512) k2_select(Geom g, SelParams p, const __grid_constant__ KTab kt,
                                                 const uint16_t* __restrict__ omega_in);
size_t k2_smem_bytes(int N, int Npad, int ncols, int nrows, int r, int G, int Tw, int Th, bool omg);

// ---- K2 fast path (imf_pair.cu) --------------------------------------------
// Membership test families of the pair kernel (template parameter SHAPE).
constexpr int SH_SPAN = 0;    // any convex kernel: per-row span table (kernels.py:127-182)
constexpr int SH_CIRCLE = 1;  // 4(dx^2+dy^2) <= (2r+1)^2 (kernels.py:70-71), packed bytes + IDP.4A
constexpr int SH_SQUARE = 2;  // |dx|, |dy| <= r (kernels.py:72-73), VABSDIFF4 on packed bytes
constexpr int SH_POLY = 3;    // any convex kernel, per-row range constants looked up by dy byte
constexpr int SH_CIRCLEW = 4; // circle, any tile (T + r > 128): unsigned-byte IDP.4A on x, y (see test8)
constexpr int SH_POLYSYM = 5; // convex kernel symmetric in x and y: |dx| <= h(|dy|), VABSDIFF4 + byte table

constexpr int PT_MAX = 250;  // >= kernel rows / columns (2r+1, r <= 124)

// Byte offsets into I relative to a window pair's base 2*(row*Sw + 2q), in
// the constant bank.  Every list holds its 4-byte-aligned entries first; the
// rest ("odd") store the offset of the aligned word BEFORE the pixel pair.
struct PairTab {
    int2 v[PT_MAX];  // per kernel column: (enter, exit) of a down slide
    int he[PT_MAX];  // per kernel row: pixel entering on a right slide
    int hx[PT_MAX];  // per kernel row: pixel exiting on a right slide
    int span[PT_MAX];  // per dy + r: (xlo & 0xffff) | width << 16 (kernels.py:127-182 rows)
};

struct PairParams {
    int shape;       // SH_*: membership test family (packed ones require T + r <= 128)
    int R2p1;        // r(r+1) + 1
    int nR2p1;       // -(r(r+1) + 1), the membership tests' IDP.4A addend (read from the constant bank)
    int nv, nv_even;
    int nh, nhe_even, nhx_even;
    int target;
    const int* tmap;
    int G;
    int grouped;     // phase C+D per seed-row group (named barriers), needs 64 threads per group
    int hs;          // 1: I holds rank >> 1 (tiles with 32768 < N <= 65536), pivots even
    int* status;
    int debug_defect;  // test hook (IMF_FLAG_DEBUG_DEFECT): corrupt one slide count in tile 0
    int refine_mode;   // phase-D refine: 0 both walks per iteration, 1 walks in sequence (IMF_REFINE)
};

template <int SHAPE, bool OMG>
__global__ void __launch_bounds__(512, 2) k2_pair(Geom g, PairParams p, const __grid_constant__ PairTab kt,
                                                  const uint16_t* __restrict__ omega_in);
size_t k2_pair_smem_bytes(int N, int Npad, int NI, int r, int G, int T, int TY, bool omg);
bool build_pair_tab(const int* row_dy, const int* row_xlo, const int* row_xhi, int nrows, const int* col_dx,
                    const int* col_ytop, const int* col_ybot, int ncols, int r, int Sw, PairTab& t,
                    PairParams& p);

// ---- K0 direct selection (imf_direct.cu) -----------------------------------
struct DirectTab {
    int area;
    int off[32];  // window offsets dy * Sw + dx relative to the window centre
};

template <int DT>
__global__ void __launch_bounds__(1024) k_direct(Geom g, const __grid_constant__ DirectTab dt, int target,
                                                 const int* __restrict__ tmap);

}  // namespace imf
