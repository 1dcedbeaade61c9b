// dev aid: minimal TMA load probe; ./tma_probe V  (V selects a variant)
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>

__global__ void k(uint16_t* out, const __grid_constant__ CUtensorMap tm, const CUtensorMap* gtm, int bw, int bh,
                  int variant, int c0) {
    extern __shared__ __align__(128) unsigned char smem[];
    uint32_t bar = (uint32_t)__cvta_generic_to_shared(smem);
    uint32_t dst = (uint32_t)__cvta_generic_to_shared(smem + 128);
    const uint64_t desc = (variant & 4) ? reinterpret_cast<uint64_t>(gtm) : reinterpret_cast<uint64_t>(&tm);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(1) : "memory");
        if (variant & 1) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        else asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bw * bh * 2) : "memory");
        if (variant & 2)
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                         ::"r"(dst), "l"(desc), "r"(c0), "r"(c0), "r"(bar) : "memory");
        else
            asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                         ::"r"(dst), "l"(desc), "r"(c0), "r"(c0), "r"(0), "r"(0), "r"(bar) : "memory");
    }
    __syncthreads();
    asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(bar), "r"(0) : "memory");
    const uint16_t* s = reinterpret_cast<const uint16_t*>(smem + 128);
    for (int i = threadIdx.x; i < bw * bh; i += blockDim.x) out[i] = s[i];
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main(int argc, char** argv) {
    const int variant = argc > 1 ? atoi(argv[1]) : 0, c0 = argc > 2 ? atoi(argv[2]) : 0;
    const int W = 256, H = 256, bw = 48, bh = 40;
    uint16_t *d, *o;
    cudaMalloc(&d, W * H * 2);
    cudaMalloc(&o, bw * bh * 2);
    uint16_t* h = new uint16_t[W * H];
    for (int i = 0; i < W * H; i++) h[i] = (uint16_t)i;
    cudaMemcpy(d, h, W * H * 2, cudaMemcpyHostToDevice);
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &f, 12000, cudaEnableDefault, &q);
    EncodeTiledFn enc = (EncodeTiledFn)f;
    CUtensorMap tm;
    const int rank = (variant & 2) ? 2 : 4;
    cuuint64_t dims[4] = {W, H, 1, 1}, str[3] = {W * 2, (cuuint64_t)W * H * 2, (cuuint64_t)W * H * 2};
    cuuint32_t box[4] = {bw, bh, 1, 1}, es[4] = {1, 1, 1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT16, rank, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    CUtensorMap* gtm;
    cudaMalloc(&gtm, sizeof(CUtensorMap));
    cudaMemcpy(gtm, &tm, sizeof(CUtensorMap), cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
    k<<<1, 128, 100000>>>(o, tm, gtm, bw, bh, variant, c0);
    cudaError_t e = cudaDeviceSynchronize();
    uint16_t* ho = new uint16_t[bw * bh];
    cudaMemcpy(ho, o, bw * bh * 2, cudaMemcpyDeviceToHost);
    printf("variant %d c0 %d: encode %d launch %s; box[5][7] = %d (expect %d)\n", variant, c0, (int)r,
           cudaGetErrorString(e), ho[5 * bw + 7], (c0 + 5) * W + c0 + 7);
    return 0;
}
