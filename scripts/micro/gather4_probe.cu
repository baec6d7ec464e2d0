// Probe of the TMA tile::gather4 load (sm_100a) with a 128-B-swizzled 2-D
// tensor map: which box height the map needs, how many bytes the copy
// delivers, and where each 16-B chunk of the 4 gathered rows lands in shared
// memory.  Every wait is bounded (no hang if the byte count is wrong).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -o gather4_probe gather4_probe.cu
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__global__ void probe(const __grid_constant__ CUtensorMap tmap, int r0, int r1, int r2, int r3,
                      int col, uint32_t expect, uint8_t* out, int* status) {
    __shared__ __align__(1024) uint8_t buf[4096];
    __shared__ __align__(8) uint64_t bar;
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) buf[i] = 0xAA;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)),
                     "r"(expect)
                     : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(buf)),
            "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3),
            "r"(smem_u32(&bar))
            : "memory");
        int done = 0;
        for (long it = 0; it < 20000000 && !done; ++it) {
            uint32_t ok;
            asm volatile(
                "{\n\t.reg .pred p;\n\t"
                "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\t"
                "selp.u32 %0, 1, 0, p;\n\t}"
                : "=r"(ok)
                : "r"(smem_u32(&bar))
                : "memory");
            done = ok;
        }
        *status = done ? 0 : 1;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) out[i] = buf[i];
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                              CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                              CUtensorMapFloatOOBfill);

int main() {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
        printf("no cuTensorMapEncodeTiled\n");
        return 1;
    }
    auto encode = reinterpret_cast<EncodeFn>(f);
    const int R = 256, C = 192;  // rows x halfs (384 B per row)
    std::vector<uint16_t> img((size_t)R * C);
    for (int r = 0; r < R; ++r)
        for (int c = 0; c < C; ++c) img[(size_t)r * C + c] = (uint16_t)((r << 8) | c);
    uint16_t* dimg;
    cudaMalloc(&dimg, img.size() * 2);
    cudaMemcpy(dimg, img.data(), img.size() * 2, cudaMemcpyHostToDevice);
    uint8_t* dout;
    int* dst;
    cudaMalloc(&dout, 4096);
    cudaMalloc(&dst, 4);
    const int rows[4] = {5, 200, 3, 77};
    for (int boxh : {1, 4}) {
        for (int col : {0, 64, 128}) {
            CUtensorMap m;
            cuuint64_t gdim[2] = {(cuuint64_t)C, (cuuint64_t)R};
            cuuint64_t gstr[1] = {(cuuint64_t)C * 2};
            cuuint32_t box[2] = {64, (cuuint32_t)boxh};
            cuuint32_t es[2] = {1, 1};
            CUresult cr = encode(&m, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, dimg, gdim, gstr, box, es,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (cr != CUDA_SUCCESS) {
                printf("boxh=%d: encode failed %d\n", boxh, (int)cr);
                continue;
            }
            cudaMemset(dst, 0xFF, 4);
            probe<<<1, 128>>>(m, rows[0], rows[1], rows[2], rows[3], col, 4 * 128, dout, dst);
            cudaError_t e = cudaDeviceSynchronize();
            int st = -1;
            std::vector<uint8_t> out(4096);
            cudaMemcpy(&st, dst, 4, cudaMemcpyDeviceToHost);
            cudaMemcpy(out.data(), dout, 4096, cudaMemcpyDeviceToHost);
            printf("boxh=%d col=%d: %s status=%d\n", boxh, col, cudaGetErrorString(e), st);
            if (e != cudaSuccess) return 2;
            // each 16-B chunk of the first 8 x 128 B: which (row, col) it holds
            for (int j = 0; j < 8; ++j) {
                printf("  smem row %d:", j);
                for (int p = 0; p < 8; ++p) {
                    uint16_t v;
                    memcpy(&v, &out[j * 128 + p * 16], 2);
                    if (v == 0xAAAA) printf("   --   ");
                    else printf(" %3d:%3d", v >> 8, v & 0xFF);
                }
                printf("\n");
            }
        }
    }
    return 0;
}
