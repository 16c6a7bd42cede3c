// TMA tiled load of an 8-bit 4-D tensor (the int8 gather's grid-digit box) on sm_100a.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/tma_test tools/tma_test.cu -lcuda
#include <cstdio>
#include <vector>
#include <cstdlib>

#include <cuda.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k_load(const __grid_constant__ CUtensorMap map, int c0, int c1, int c2, int c3, uint8_t *out,
                       int bytes, int variant) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(sa(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(sa(&bar)), "r"(bytes) : "memory");
        if (variant == 0)
            asm volatile(
                "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
                "%5}], [%6];\n" ::"r"(sa(sm)),
                "l"(&map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(sa(&bar))
                : "memory");
        else
            asm volatile(
                "cp.async.bulk.tensor.4d.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
                "%5}], [%6];\n" ::"r"(sa(sm)),
                "l"(&map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(sa(&bar))
                : "memory");
    }
    uint32_t ok = 0;
    while (!ok)
        asm volatile(
            "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(ok)
            : "r"(sa(&bar))
            : "memory");
    for (int i = threadIdx.x; i < bytes; i += blockDim.x) out[i] = sm[i];
}

int main(int argc, char **argv) {
    const int C0 = argc > 1 ? atoi(argv[1]) : 5, BOXR = argc > 2 ? atoi(argv[2]) : 80, BOXC = argc > 3 ? atoi(argv[3]) : 16, NDB = argc > 4 ? atoi(argv[4]) : 6;
    const int P2 = 96, R = 160, ND = 6, N0 = 8;
    std::vector<uint8_t> h((size_t)P2 * R * ND * N0);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (uint8_t)(i * 131 + 7);
    uint8_t *d, *o;
    cudaMalloc(&d, h.size());
    cudaMemcpy(d, h.data(), h.size(), cudaMemcpyHostToDevice);
    const int bytes = BOXC * BOXR * NDB;
    cudaMalloc(&o, bytes);
    CUtensorMap map;
    cuuint64_t dims[4] = {(cuuint64_t)P2, (cuuint64_t)R, (cuuint64_t)ND, (cuuint64_t)N0};
    cuuint64_t strides[3] = {(cuuint64_t)P2, (cuuint64_t)P2 * R, (cuuint64_t)P2 * R * ND};
    cuuint32_t box[4] = {(cuuint32_t)BOXC, (cuuint32_t)BOXR, (cuuint32_t)NDB, 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    for (auto l2 : {CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE})
        for (int variant = 0; variant < 2; ++variant) {
            CUresult r = cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, d, dims, strides, box, estr,
                                                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, l2,
                                                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            cudaFuncSetAttribute(k_load, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
            const int c0 = C0, c1 = 33, c2 = 0, c3 = 3;
            k_load<<<1, 128, 65536>>>(map, c0, c1, c2, c3, o, bytes, variant);
            cudaError_t e = cudaDeviceSynchronize();
            std::vector<uint8_t> got(bytes);
            cudaMemcpy(got.data(), o, bytes, cudaMemcpyDeviceToHost);
            int bad = 0;
            for (int dg = 0; dg < NDB; ++dg)
                for (int rr = 0; rr < BOXR; ++rr)
                    for (int c = 0; c < BOXC; ++c) {
                        size_t gi = (((size_t)c3 * ND + dg) * R + (c1 + rr)) * P2 + c0 + c;
                        bad += got[(dg * BOXR + rr) * BOXC + c] != h[gi];
                    }
            printf("c0 %d boxr %d boxc %d nd %d encode %d l2 %d variant %d: %s, %d mismatches\n", C0, BOXR, BOXC, NDB, (int)r, (int)l2, variant, cudaGetErrorString(e),
                   bad);
            if (e != cudaSuccess) return 1;
        }
    return 0;
}
