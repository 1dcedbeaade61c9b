/*
 * isomedian_b200.h -- C ABI of the B200 rank-order (circular median) filter.
 *
 * Drop-in native boundary for the hot path of the reference package
 * `isomedian` (arXiv 2505.22938).  One call replaces the body of
 *   filter_image(image, FilterParams)          /root/reference/pkg/src/isomedian/tiling.py:213-249
 * i.e. padding (tiling.py:134-145), tiling (tiling.py:94-131), the per-tile
 * ordinal transform (ordinal.py:126-172: _rank_by_bucket :62-79,
 * _rank_by_radix16 :82-106, float_order_key :109-123) and the per-tile
 * selection (core.py:175-221 _process_tile, the numba native boundary
 * declared at core.py:176-181), plus the per-channel recursion
 * (tiling.py:219-221) for HWC images and image batches.
 *
 * The host prologue stays with the caller, exactly as in the reference:
 * validation and error messages (tiling.py:216-226, kernels.py:36-42),
 * kernel rasterization (kernels.py:127-182 make_kernel) and target ranks
 * (kernels.py:185-192, tiling.py:165-177) are computed on the host and
 * passed in (the Python mirror lives in paper_2505_22938_b200/).
 *
 * Conventions: plain C types only; every pointer in imf_image.data and
 * target_map is DEVICE memory for imf_filter and HOST memory for
 * imf_filter_host; kernel tables are host memory.  No call allocates
 * except imf_filter_host; no call throws; all return an IMF_* status.
 * Calls are re-entrant (no mutable global state besides a launch counter).
 */
#ifndef ISOMEDIAN_B200_H
#define ISOMEDIAN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define IMF_OK 0
#define IMF_ERR_INVALID 1     /* bad argument (host-side validation should catch first) */
#define IMF_ERR_CUDA 2        /* CUDA runtime error */
#define IMF_ERR_DEFECT 3      /* pivot/count scan exhausted: core.py:31-36 ScanDefectError */
#define IMF_ERR_WORKSPACE 4   /* workspace too small */
#define IMF_ERR_UNSUPPORTED 5 /* geometry the kernels cannot tile (e.g. radius > 124) */

#define IMF_DTYPE_U8 0
#define IMF_DTYPE_U16 1
#define IMF_DTYPE_F32 2

#define IMF_BOUNDARY_REPLICATE 0 /* np.pad(mode="edge") by r: tiling.py:134-140 */
#define IMF_BOUNDARY_VALID 1     /* output (H-2r, W-2r): tiling.py:102-105,141-144 */

#define IMF_SHAPE_CIRCLE 0  /* kernels.py:70-71 */
#define IMF_SHAPE_SQUARE 1  /* kernels.py:72-73 */
#define IMF_SHAPE_POLYGON 2 /* kernels.py:45-64,74-78 (rasterized by the caller) */

/* Rasterized kernel = reference KernelShape (kernels.py:81-124).  Row spans
 * are half-open [row_xlo, row_xhi); column extents inclusive. */
typedef struct imf_kernel {
    int32_t shape_code;
    int32_t radius; /* 0..124 (kernels.py:24) */
    int32_t area;
    int32_t nrows;
    const int32_t* row_dy;
    const int32_t* row_xlo;
    const int32_t* row_xhi;
    int32_t ncols;
    const int32_t* col_dx;
    const int32_t* col_ytop;
    const int32_t* col_ybot;
} imf_kernel;

/* A batch of (H, W, C) images; strides in ELEMENTS (any layout, e.g. HWC
 * interleaved or planar).  One (H, W) plane per (batch, channel) is filtered
 * independently, as the reference's per-channel recursion does. */
typedef struct imf_image {
    void* data;
    int32_t dtype;
    int32_t batch, height, width, channels;
    int64_t stride_b, stride_y, stride_x, stride_c;
} imf_image;

typedef struct imf_options {
    int32_t boundary;      /* IMF_BOUNDARY_* */
    int32_t tile_size;     /* output tile side; 0 = auto.  Output-neutral (tiling.py:110-119) */
    int32_t seed_rows;     /* seed rows per tile; 0 = auto (tuning knob, output-neutral) */
    int32_t seeds_per_row; /* direct seeds per seed row; 0 = auto */
    int32_t flags;         /* IMF_FLAG_* */
    int32_t row_begin;     /* output stripe [row_begin, row_end) of every plane; */
    int32_t row_end;       /*   row_end == 0 = all output rows (SURVEY 8(b) sketch) */
    int32_t reserved;
} imf_options;

#define IMF_FLAG_PROFILE 1      /* per-kernel CUDA-event timing, see imf_profile_last */
#define IMF_FLAG_KEEP_STATUS 2  /* do not clear the workspace status word (stripe 2..n of one job) */
#define IMF_FLAG_DEBUG_DEFECT 4 /* test hook: corrupt one window's slide count in the first tile so its
                                   segment scan leaves the rank array and the call reports IMF_ERR_DEFECT
                                   (reference test_core.py:124-130).  Rank paths only (window area > 32) */

/* Bytes of device workspace imf_filter needs for this problem. */
size_t imf_workspace_size(const imf_image* src, const imf_kernel* kernel, const imf_options* opt);

/*
 * Filter `src` into `dst` (device memory, distinct buffers) on `stream`
 * (a cudaStream_t, NULL = legacy default stream).  Selection rank per output
 * pixel: `target` when target_map is NULL, else target_map[y*out_w + x]
 * (device int32, shared by every plane).  [tmin, tmax] must bound the targets
 * in use (both == target for a scalar percentile).  The call is asynchronous;
 * scan defects are reported by imf_workspace_status() after the stream
 * completes.
 */
int imf_filter(const imf_image* src, imf_image* dst, const imf_kernel* kernel, int32_t target,
               const int32_t* target_map, int32_t tmin, int32_t tmax, const imf_options* opt,
               void* workspace, size_t workspace_bytes, void* stream);

/*
 * Multi-percentile "bracket" (core.py:412-426 bracket_filter):
 * n outputs dsts[0..n) at scalar selection ranks targets[0..n), one ordinal
 * transform (K1) per tile shared by all n selections.  Same conventions and
 * workspace size as imf_filter.
 */
int imf_filter_bracket(const imf_image* src, imf_image* dsts, int32_t n, const int32_t* targets,
                       const imf_kernel* kernel, const imf_options* opt, void* workspace,
                       size_t workspace_bytes, void* stream);

/* Synchronizes `stream` and returns IMF_OK or IMF_ERR_DEFECT for the last
 * imf_filter that used `workspace`. */
int imf_workspace_status(void* workspace, void* stream);

/*
 * Synchronous host-memory variant for FFI callers (cgo / JNI / ctypes): copies
 * src to the current device, filters, copies the result back to dst.  Images
 * whose rows are outermost within each plane group (HW, HWC, NHWC) are
 * pipelined in output-row stripes: the upload of stripe i+1, the filter of
 * stripe i and the download of stripe i-1 run concurrently (three streams,
 * event-ordered); batches of more than two such images reuse two device
 * image slots (image b in slot b % 2).  Device buffers come from the
 * stream-ordered pool (cudaMallocAsync); the streams, events and pinned
 * status words it uses are kept per (calling thread, device) and released
 * when the thread exits.  Host buffers should be pinned for
 * full copy bandwidth.  dst must be dense (every byte of its extent belongs
 * to an element, e.g. C-contiguous: row ranges are copied back as whole byte
 * ranges), else IMF_ERR_INVALID.  opt->row_begin/row_end select an output
 * row range: only the input rows it reads are uploaded and only its output
 * rows of dst are written (one device's stripe of a multi-device job; needs
 * row-outermost src and dst).
 */
int imf_filter_host(const imf_image* src, imf_image* dst, const imf_kernel* kernel, int32_t target,
                    const int32_t* target_map, int32_t tmin, int32_t tmax, const imf_options* opt,
                    void* stream);

const char* imf_strerror(int status);
int imf_version(void);                  /* 100 * major + minor */
const char* imf_last_error(void);       /* detail of the last IMF_ERR_CUDA on this thread */
uint64_t imf_launch_count(void);        /* kernels launched by this process (diagnostic) */

/* Per-kernel device time of the last imf_filter on this thread that ran with
 * opt->flags & IMF_FLAG_PROFILE (events on its stream; that call synchronizes). */
int imf_profile_last(float* sort_ms, float* select_ms, int32_t* launches, int64_t* tiles,
                     int32_t* tile_side, int32_t* qshift);

/*
 * Ordinal transform of ONE tile (device-side counterpart of the reference's
 * per-tile ordinal_transform, ordinal.py:126-172; for invariant checks as in
 * the reference's test_ordinal.py): runs the call's K1 on tile `tile` (index
 * as the filter enumerates them: channel fastest, then tile column, tile row,
 * image) and copies
 * its omega -- the rank -> position map, x | y << 8 in input-tile coordinates
 * -- to host memory omega[0..N).  Only the tile's footprint is ranked (when
 * the planner uses one); ties are in arbitrary order (output-neutral for the
 * filter).  info[8] receives N, the input tile's image origin x0, y0 (before
 * clamping: replicate tiles read clamp(x0 + x), clamp(y0 + y)), its extent
 * Sw, Sh, channel, image, and whether a footprint was applied.  Synchronous.
 */
int imf_tile_omega(const imf_image* src, const imf_kernel* kernel, const imf_options* opt, int64_t tile,
                   uint16_t* omega, int32_t capacity, int32_t* info, void* workspace, size_t workspace_bytes,
                   void* stream);

/*
 * The launch plan the library would use for this call (host only, no CUDA
 * work; diagnostics and tests): info[16] = output tile Tw, Th; input tile Sw,
 * Sh; ranked pixels per tile N (the footprint when one is used) and Npad;
 * tiles in the call; tiles per chunk; chunk streams; selection kernel (0
 * direct, 1 general, 2 pair); footprint used; K1 tile loads by TMA (when the
 * data pointer is 16-byte aligned); halved ranks; seed rows; workspace bytes;
 * ordinal-transform family (0 radix, 1 f32 buckets, 2 f32 buckets with global
 * entries, 3 counting sort, 4 counting sort with omega in global memory).
 */
int imf_plan_info(const imf_image* src, const imf_kernel* kernel, const imf_options* opt, int64_t* info);

/* Kernel paths the last imf_filter / imf_filter_bracket on this thread took
 * (diagnostic): IMF_FEATURE_K1_TMA = the ordinal transform loaded its tile
 * boxes with TMA (cp.async.bulk.tensor). */
#define IMF_FEATURE_K1_TMA 1u
uint32_t imf_last_features(void);

/* Measured int32 add throughput of the current device (ops/s): the
 * denominator of the selection kernel's integer roofline. */
int imf_int_peak(double* ops_per_s, double* ms);

#ifdef __cplusplus
}
#endif
#endif /* ISOMEDIAN_B200_H */
