// TMA streaming with the exact operand pattern of the VM's split-K GEMM item for M=256, N=1280,
// K=11520 (BN=128, S=7): CTA (z, tm, tn) streams A[tm*128.., k-range] and B[tn*128.., k-range]
// through a 4-slot ring; consumer = plain release (no MMA).  Per-CTA GB/s.
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) | ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
__global__ void k(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb, int S, int kb, long long* out, int mma) {
    extern __shared__ __align__(1024) unsigned char sm[];
    unsigned char* ring = (unsigned char*)(((uintptr_t)sm + 1023) & ~1023);
    __shared__ __align__(8) uint64_t full[8], empty[8];
    __shared__ uint32_t tslot;
    const int stages = 4;
    if (threadIdx.x >= 32 && threadIdx.x < 64) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(sa(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    const int tid = threadIdx.x;
    const int item = blockIdx.x, z = item % S, tile = item / S, tn = tile % 10, tm = tile / 10;
    const int per = (kb + S - 1) / S, kb0 = z * per, nk = min(kb, kb0 + per) - kb0;
    if (tid == 0) {
        for (int s = 0; s < stages; s++) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(full + s)));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(empty + s)));
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tslot;
    long long t0 = clock64();
    if (tid == 0) {
        for (int i = 0; i < nk; i++) {
            const int s = i % stages;
            if (i >= stages)
                asm volatile("{.reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W;}" ::"r"(sa(empty + s)), "r"(((i / stages) & 1) ^ 1));
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(full + s)), "r"(32768));
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                         ::"r"(sa(ring + s * 32768)), "l"(&ta), "r"((kb0 + i) * 64), "r"(tm * 128), "r"(sa(full + s)) : "memory");
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                         ::"r"(sa(ring + s * 32768 + 16384)), "l"(&tb), "r"((kb0 + i) * 64), "r"(tn * 128), "r"(sa(full + s)) : "memory");
        }
    } else if (tid == 32) {
        const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(128 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
        for (int i = 0; i < nk; i++) {
            const int s = i % stages;
            asm volatile("{.reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W;}" ::"r"(sa(full + s)), "r"((i / stages) & 1));
            asm volatile("tcgen05.fence::after_thread_sync;");
            if (mma) {
                const uint32_t a0 = sa(ring + s * 32768), b0 = a0 + 16384;
                for (int kk = 0; kk < 4; kk++) {
                    const uint32_t acc = (i > 0 || kk > 0) ? 1u : 0u;
                    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                                 ::"r"(tmem), "l"(desc(a0 + kk * 32)), "l"(desc(b0 + kk * 32)), "r"(idesc), "r"(acc));
                }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(empty + s)) : "memory");
            } else {
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(empty + s)));
            }
        }
        out[2 * blockIdx.x] = clock64() - t0;
        out[2 * blockIdx.x + 1] = nk;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x >= 32 && threadIdx.x < 64) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
}
int main() {
    PFN_cuTensorMapEncodeTiled_v12000 enc;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    const int M = 256, N = 1280, K = 11520;
    void *a, *b; cudaMalloc(&a, (size_t)M * K * 2); cudaMalloc(&b, (size_t)N * K * 2);
    cudaMemset(a, 1, (size_t)M * K * 2); cudaMemset(b, 1, (size_t)N * K * 2);
    CUtensorMap ta, tb;
    cuuint64_t da[2] = {(cuuint64_t)K, (cuuint64_t)M}, db[2] = {(cuuint64_t)K, (cuuint64_t)N}, st[1] = {(cuuint64_t)K * 2};
    cuuint32_t box[2] = {64, 128}, es[2] = {1, 1};
    enc(&ta, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, a, da, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    enc(&tb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, b, db, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    long long* out; cudaMalloc(&out, 16 * 148);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 32768 + 1024);
    for (int mma : {0, 1}) for (int S : {7, 1}) {
        const int grid = 20 * S;
        for (int r = 0; r < 3; r++) k<<<grid, 64, 4 * 32768 + 1024>>>(ta, tb, S, K / 64, out, mma);
        long long h[296]; cudaMemcpy(h, out, 16 * grid, cudaMemcpyDeviceToHost);
        double mx = 0; for (int i = 0; i < grid; i++) mx = h[2 * i] > mx ? h[2 * i] : mx;
        const double us = mx / 1.965e3;
        printf("mma %d S=%d grid %d: %.1f us, %.1f GB/s per CTA, %.0f GB/s total\n", mma, S, grid, us, h[1] * 32768.0 / us / 1e3, grid * h[1] * 32768.0 / us / 1e3);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
