// L2 latency seen by one CTA while the other CTAs poll a global flag (the VM's dependency wait).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(const int* chain, long long* out, int hops, int* flag, int mode, int ns) {
    if (blockIdx.x == 0) {
        if (threadIdx.x) return;
        long long c1 = clock64();
        int p = 0;
        for (int i = 0; i < hops; i++) p = __ldcg(chain + p);
        long long c2 = clock64();
        out[0] = (c2 - c1) / hops;
        out[1] = p;
        __threadfence();
        atomicExch(flag, 1);
        return;
    }
    if (threadIdx.x) return;
    if (mode == 0) return;
    int v;
    do {
        asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
        if (mode == 2) __nanosleep(ns);
    } while (v == 0);
}
int main() {
    const int n = 1 << 20;
    int* h = new int[n];
    for (int i = 0; i < n; i++) h[i] = (int)(((long long)i * 7919 + 104729) % n);
    int *d, *f; long long* o; cudaMalloc(&d, n * 4); cudaMalloc(&o, 64); cudaMalloc(&f, 4);
    cudaMemcpy(d, h, n * 4, cudaMemcpyHostToDevice);
    int modes[4][2] = {{0, 0}, {1, 0}, {2, 32}, {2, 1000}};
    for (auto& m : modes) {
        long long ho[2];
        for (int r = 0; r < 3; r++) {
            cudaMemset(f, 0, 4);
            k<<<148, 32>>>(d, o, 4000, f, m[0], m[1]);
        }
        cudaMemcpy(ho, o, 16, cudaMemcpyDeviceToHost);
        printf("pollers mode %d sleep %4d ns: L2 chase %lld cy/hop\n", m[0], m[1], ho[0]);
    }
    return 0;
}
