// Does TMA tile::gather4 work on this GPU, and with which box shape / swizzle?
// nvcc -gencode arch=compute_100a,code=sm_100a -o gather4_test gather4_test.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <vector>

__global__ void k(const __grid_constant__ CUtensorMap tm, int r0, int r1, int r2, int r3, uint16_t* out) {
    __shared__ __align__(1024) unsigned char buf[8 * 128];
    __shared__ __align__(8) uint64_t bar;
    uint32_t dst = (uint32_t)__cvta_generic_to_shared(buf) + 512;
    uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(512) : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
            "%4, %5, %6}], [%7];" ::"r"(dst),
            "l"(&tm), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(b)
            : "memory");
        asm volatile(
            "{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(b)
            : "memory");
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 256; i += blockDim.x) out[i] = ((uint16_t*)(buf + 512))[i];
}

int main() {
    const int rows = 64, cols = 64;
    std::vector<uint16_t> h(rows * cols);
    for (int r = 0; r < rows; r++)
        for (int c = 0; c < cols; c++) h[r * cols + c] = (uint16_t)(r * 100 + c);
    uint16_t *d, *o;
    cudaMalloc(&d, h.size() * 2);
    cudaMalloc(&o, 512);
    cudaMemcpy(d, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
    for (int boxh : {1}) {
        for (int sw : {0, 1}) {
            CUtensorMap m;
            cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
            cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
            cuuint32_t box[2] = {64u, (cuuint32_t)boxh};
            cuuint32_t es[2] = {1u, 1u};
            CUresult r = cuTensorMapEncodeTiled(&m, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, d, dims, strides, box, es,
                                                CU_TENSOR_MAP_INTERLEAVE_NONE,
                                                sw ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                                                CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r != CUDA_SUCCESS) { printf("box h %d sw %d: encode failed %d\n", boxh, sw, r); continue; }
            cudaMemset(o, 0xff, 512);
            k<<<1, 32>>>(m, 3, 10, -1, 70, o);
            cudaError_t e = cudaDeviceSynchronize();
            std::vector<uint16_t> ho(256);
            cudaMemcpy(ho.data(), o, 512, cudaMemcpyDeviceToHost);
            printf("box h %d sw %d: %s\n", boxh, sw, cudaGetErrorString(e));
            int rr[4] = {3, 10, -1, 70};
            int bad = 0;
            for (int i = 0; i < 4; i++)
                for (int j = 0; j < 8; j++) {
                    const int r = 4 + i;  // tile row of this gathered row
                    const int pos = sw ? ((j ^ (r & 7)) * 8) : j * 8;
                    const uint16_t exp = (rr[i] >= 0 && rr[i] < 64) ? (uint16_t)(rr[i] * 100 + j * 8) : 0;
                    if (ho[i * 64 + pos] != exp) bad++;
                }
            printf("  layout check (rows at +512, sw128 by absolute row): bad=%d\n", bad);
            if (e != cudaSuccess) return 1;
        }
    }
    return 0;
}
