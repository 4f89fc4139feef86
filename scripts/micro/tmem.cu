// tcgen05.ld latency: x16 / x32 / x64 loads each followed by wait::ld, one warp per TMEM lane quarter.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(128, 1) k(long long* out) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"((uint32_t)__cvta_generic_to_shared(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t t = slot + ((uint32_t)(warp * 32) << 16);
    uint32_t acc = 0;
    long long c0 = clock64();
    for (int i = 0; i < 64; i++) {
        uint32_t u[16];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]), "=r"(u[7]), "=r"(u[8]), "=r"(u[9]), "=r"(u[10]), "=r"(u[11]), "=r"(u[12]), "=r"(u[13]), "=r"(u[14]), "=r"(u[15]) : "r"(t + (i % 8) * 16));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        acc += u[0] + u[15];
    }
    long long c1 = clock64();
    for (int i = 0; i < 16; i++) {
        uint32_t u[64];
#define R(j) "=r"(u[j])
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
            : R(0),R(1),R(2),R(3),R(4),R(5),R(6),R(7),R(8),R(9),R(10),R(11),R(12),R(13),R(14),R(15),R(16),R(17),R(18),R(19),R(20),R(21),R(22),R(23),R(24),R(25),R(26),R(27),R(28),R(29),R(30),R(31),
              R(32),R(33),R(34),R(35),R(36),R(37),R(38),R(39),R(40),R(41),R(42),R(43),R(44),R(45),R(46),R(47),R(48),R(49),R(50),R(51),R(52),R(53),R(54),R(55),R(56),R(57),R(58),R(59),R(60),R(61),R(62),R(63) : "r"(t + (i % 4) * 64));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        for (int j = 0; j < 64; j++) acc += u[j];
    }
    long long c2 = clock64();
    if (threadIdx.x == 0) { out[0] = (c1 - c0) / 64; out[1] = (c2 - c1) / 16; out[2] = acc; }
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}
int main() {
    long long* o; cudaMalloc(&o, 32);
    for (int r = 0; r < 3; r++) k<<<1, 128>>>(o);
    long long h[3]; cudaMemcpy(h, o, 24, cudaMemcpyDeviceToHost);
    printf("tcgen05.ld x16+wait: %lld cy; x64+wait: %lld cy (%s)\n", h[0], h[1], cudaGetErrorString(cudaGetLastError()));
}
