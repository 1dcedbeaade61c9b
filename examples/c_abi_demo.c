/*
 * A plain-C caller of the drop-in boundary (include/isomedian_b200.h): what a
 * cgo / JNI / N-API binding compiles down to.  Builds a circle kernel's span
 * tables the way kernels.py:127-182 rasterizes them (4(dx^2+dy^2) <= (2r+1)^2,
 * kernels.py:70-71), filters a u16 RGB image through imf_filter_host (host
 * buffers in and out) and checks every output against a brute-force median
 * (sort each clamped window, take rank t = floor(p(area-1) + 0.5)).
 *
 *   gcc -O2 -Iinclude examples/c_abi_demo.c -Lpaper_2505_22938_b200 -lisomedian_b200 \
 *       -Wl,-rpath,$PWD/paper_2505_22938_b200 -o /tmp/c_abi_demo
 *   /tmp/c_abi_demo            # filter on cuda:0 and check
 *   /tmp/c_abi_demo --plan     # host-only: plan and workspace size (no GPU needed)
 *   /tmp/c_abi_demo --device   # device pointers: imf_filter on a stream with a caller-owned
 *                              # workspace (build with -DWITH_CUDART -I/usr/local/cuda/include
 *                              # -L/usr/local/cuda/lib64 -lcudart)
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "isomedian_b200.h"
#ifdef WITH_CUDART
#include <cuda_runtime.h>
#endif

enum { R = 6, H = 57, W = 83, C = 3 };

static int cmp_u16(const void* a, const void* b) {
    return (int)*(const uint16_t*)a - (int)*(const uint16_t*)b;
}

int main(int argc, char** argv) {
    const int side = 2 * R + 1;
    int32_t row_dy[2 * R + 1], row_xlo[2 * R + 1], row_xhi[2 * R + 1];
    int32_t col_dx[2 * R + 1], col_ytop[2 * R + 1], col_ybot[2 * R + 1];
    int area = 0;
    for (int i = 0; i < side; i++) {
        const int d = i - R;
        int ext = 0;  /* largest e with d^2 + e^2 <= r(r+1) */
        while ((ext + 1) * (ext + 1) + d * d <= R * (R + 1)) ext++;
        row_dy[i] = d, row_xlo[i] = -ext, row_xhi[i] = ext + 1;  /* half-open */
        col_dx[i] = d, col_ytop[i] = -ext, col_ybot[i] = ext;     /* inclusive */
        area += 2 * ext + 1;
    }
    const imf_kernel k = {IMF_SHAPE_CIRCLE, R, area, side, row_dy, row_xlo, row_xhi,
                          side, col_dx, col_ytop, col_ybot};
    const int32_t t = (int32_t)floor(0.5 * (area - 1) + 0.5);  /* kernels.py:185-192, p = 0.5 */

    uint16_t* src = malloc(sizeof(uint16_t) * H * W * C);
    uint16_t* dst = malloc(sizeof(uint16_t) * H * W * C);
    uint32_t s = 12345u;
    for (int i = 0; i < H * W * C; i++) {
        s = s * 1664525u + 1013904223u;
        src[i] = (uint16_t)(s >> 16);
    }
    imf_image is = {src, IMF_DTYPE_U16, 1, H, W, C, (int64_t)H * W * C, W * C, C, 1};
    imf_image os = {dst, IMF_DTYPE_U16, 1, H, W, C, (int64_t)H * W * C, W * C, C, 1};
    imf_options opt;
    memset(&opt, 0, sizeof(opt));
    opt.boundary = IMF_BOUNDARY_REPLICATE;

    printf("library version %d, workspace %zu bytes\n", imf_version(), imf_workspace_size(&is, &k, &opt));
    if (argc > 1 && strcmp(argv[1], "--plan") == 0) {
        int64_t info[16];
        const int st = imf_plan_info(&is, &k, &opt, info);
        printf("plan: status %d, tile %lldx%lld, ranked pixels per tile %lld\n", st, (long long)info[0],
               (long long)info[1], (long long)info[4]);
        return st;
    }
    int st;
    if (argc > 1 && strcmp(argv[1], "--device") == 0) {
#ifdef WITH_CUDART
        /* the asynchronous entry: device buffers, caller-owned workspace, a stream */
        const size_t bytes = sizeof(uint16_t) * H * W * C, ws_bytes = imf_workspace_size(&is, &k, &opt);
        void *dsrc, *ddst, *ws;
        cudaStream_t stream;
        if (cudaMalloc(&dsrc, bytes) || cudaMalloc(&ddst, bytes) || cudaMalloc(&ws, ws_bytes) ||
            cudaStreamCreate(&stream))
            return 2;
        cudaMemcpyAsync(dsrc, src, bytes, cudaMemcpyHostToDevice, stream);
        imf_image ds = is, dd = os;
        ds.data = dsrc;
        dd.data = ddst;
        st = imf_filter(&ds, &dd, &k, t, NULL, t, t, &opt, ws, ws_bytes, stream);
        cudaMemcpyAsync(dst, ddst, bytes, cudaMemcpyDeviceToHost, stream);
        if (st == IMF_OK) st = imf_workspace_status(ws, stream);  /* synchronizes the stream */
        cudaFree(dsrc), cudaFree(ddst), cudaFree(ws), cudaStreamDestroy(stream);
#else
        fprintf(stderr, "--device needs a -DWITH_CUDART build\n");
        return 2;
#endif
    } else {
        st = imf_filter_host(&is, &os, &k, t, NULL, t, t, &opt, NULL);
    }
    if (st != IMF_OK) {
        fprintf(stderr, "imf_filter: %s (%s)\n", imf_strerror(st), imf_last_error());
        return 1;
    }
    uint16_t win[(2 * R + 1) * (2 * R + 1)];
    long bad = 0;
    for (int c = 0; c < C; c++)
        for (int y = 0; y < H; y++)
            for (int x = 0; x < W; x++) {
                int n = 0;
                for (int i = 0; i < side; i++)
                    for (int dx = row_xlo[i]; dx < row_xhi[i]; dx++) {
                        int yy = y + row_dy[i], xx = x + dx;  /* replicate = clamped (tiling.py:134-140) */
                        yy = yy < 0 ? 0 : (yy >= H ? H - 1 : yy);
                        xx = xx < 0 ? 0 : (xx >= W ? W - 1 : xx);
                        win[n++] = src[(yy * W + xx) * C + c];
                    }
                qsort(win, (size_t)n, sizeof(uint16_t), cmp_u16);
                bad += win[t] != dst[(y * W + x) * C + c];
            }
    printf("%dx%dx%d u16, circle r=%d (area %d, t=%d): %ld mismatches vs brute force\n", H, W, C, R, area, t, bad);
    free(src);
    free(dst);
    return bad ? 1 : 0;
}
