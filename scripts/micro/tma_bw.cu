// Per-SM streaming bandwidth of 2-D TMA tile loads (box 64 x 128 bf16 = 16 KB, SW128) into a
// ring of STAGES slots, consumer just releases slots.  Grid = 1 / 20 / 148 CTAs; data either
// L2-resident (8 MB matrix) or streamed from HBM (1 GB matrix).
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(const __grid_constant__ CUtensorMap tm, int rows_total, int iters, int stages, long long* out) {
    extern __shared__ __align__(1024) unsigned char sm[];
    unsigned char* ring = (unsigned char*)(((uintptr_t)sm + 1023) & ~1023);
    __shared__ __align__(8) uint64_t full[8], empty[8];
    const int tid = threadIdx.x;
    if (tid == 0) {
        for (int s = 0; s < stages; s++) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(full + s)));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(empty + s)));
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    long long t0 = clock64();
    if (tid == 0) {
        for (int i = 0; i < iters; i++) {
            const int s = i % stages;
            if (i >= stages) {
                asm volatile("{.reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W;}" ::"r"(sa(empty + s)), "r"(((i / stages) & 1) ^ 1));
            }
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(full + s)), "r"(16384));
            const int row = ((blockIdx.x * 131 + i * 7) * 128) % rows_total;
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                         ::"r"(sa(ring + s * 16384)), "l"(&tm), "r"(0), "r"(row), "r"(sa(full + s)) : "memory");
        }
    } else if (tid == 32) {
        for (int i = 0; i < iters; i++) {
            const int s = i % stages;
            asm volatile("{.reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W;}" ::"r"(sa(full + s)), "r"((i / stages) & 1));
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(empty + s)));
        }
        out[blockIdx.x] = clock64() - t0;
    }
}
int main() {
    PFN_cuTensorMapEncodeTiled_v12000 enc;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    long long* out; cudaMalloc(&out, 8 * 148);
    for (int big = 0; big < 2; big++) {
        const long long rows = big ? (1LL << 19) : (1LL << 15);  // x 64 cols x 2 B: 64 MB / 4 MB
        void* d; cudaMalloc(&d, rows * 64 * 2); cudaMemset(d, 1, rows * 64 * 2);
        CUtensorMap tm;
        cuuint64_t dims[2] = {64, (cuuint64_t)rows}; cuuint64_t st[1] = {128}; cuuint32_t box[2] = {64, 128}, es[2] = {1, 1};
        enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 16384 + 1024);
        for (int stages : {2, 4, 8}) for (int grid : {1, 20, 148}) {
            const int iters = 400;
            for (int r = 0; r < 2; r++) k<<<grid, 64, 8 * 16384 + 1024>>>(tm, (int)rows, iters, stages, out);
            long long h[148]; cudaMemcpy(h, out, 8 * grid, cudaMemcpyDeviceToHost);
            double mx = 0; for (int i = 0; i < grid; i++) mx = h[i] > mx ? h[i] : mx;
            const double us = mx / 1.965e3;
            printf("%s stages %d grid %3d: %.1f GB/s per CTA, %.0f GB/s total\n", big ? "HBM" : "L2 ", stages, grid,
                   iters * 16384.0 / us / 1e3, grid * iters * 16384.0 / us / 1e3);
        }
        cudaFree(d);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
