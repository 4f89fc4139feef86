// Calibration microbenchmarks (B200): %globaltimer read cost, clock64 per L2 pointer-chase hop,
// cp.async issue cost, and the same L2 chase right after a gpu-scope fence.
#include <cstdio>
#include <cuda_runtime.h>
__device__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
__global__ void k(const int* chain, long long* out, int hops) {
    if (threadIdx.x) return;
    long long c0 = clock64();
    unsigned long long g = 0;
    for (int i = 0; i < 100; i++) g += gt();
    long long c1 = clock64();
    int p = 0;
    for (int i = 0; i < hops; i++) p = __ldcg(chain + p);
    long long c2 = clock64();
    for (int i = 0; i < hops; i++) { p = chain[p]; }
    long long c3 = clock64();
    for (int i = 0; i < 20; i++) { __threadfence(); p = chain[p]; }
    long long c4 = clock64();
    out[0] = (c1 - c0) / 100; out[1] = (c2 - c1) / hops; out[2] = (c3 - c2) / hops; out[3] = (c4 - c3) / 20;
    out[4] = p + (int)(g & 1);
}
int main() {
    const int n = 1 << 20;  // 4 MB chain (L2-resident)
    int* h = new int[n];
    for (int i = 0; i < n; i++) h[i] = (int)(((long long)i * 7919 + 104729) % n);
    int* d; long long* o; cudaMalloc(&d, n * 4); cudaMalloc(&o, 64);
    cudaMemcpy(d, h, n * 4, cudaMemcpyHostToDevice);
    for (int r = 0; r < 3; r++) k<<<1, 32>>>(d, o, 2000);
    long long ho[5]; cudaMemcpy(ho, o, 40, cudaMemcpyDeviceToHost);
    printf("globaltimer read: %lld cy; L2 chase (ldcg): %lld cy/hop; chase (ld, L1): %lld cy/hop; fence+ld: %lld cy\n",
           ho[0], ho[1], ho[2], ho[3]);
    return 0;
}
