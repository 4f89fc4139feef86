// Cost of a 128x128 bf16 tile epilogue (staged fp32 in smem -> + residual -> bf16 store) with
// 256 threads, 8-column items, coalesced; and the same with the 16-column-per-thread row layout.
#include <cstdio>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(288, 1) k(const __nv_bfloat16* res, __nv_bfloat16* out, long long* cy, int ld, int mode) {
    extern __shared__ float st[];
    const int tid = threadIdx.x;
    if (tid >= 256) return;
    for (int i = tid; i < 128 * 132; i += 256) st[i] = i * 0.001f;
    asm volatile("bar.sync 1, 256;");
    long long c0 = clock64();
    if (mode == 0) {
        for (int idx = tid; idx < 128 * 16; idx += 256) {
            const int row = idx / 16, ch = idx % 16;
            const float4 f0 = *(const float4*)(st + row * 132 + ch * 8), f1 = *(const float4*)(st + row * 132 + ch * 8 + 4);
            const uint4 r = *(const uint4*)(res + (long long)row * ld + ch * 8);
            const __nv_bfloat162* h = (const __nv_bfloat162*)&r;
            float v[8] = {f0.x, f0.y, f0.z, f0.w, f1.x, f1.y, f1.z, f1.w};
            uint4 o;
            __nv_bfloat162* oh = (__nv_bfloat162*)&o;
            for (int q = 0; q < 4; q++) {
                float2 x = __bfloat1622float2(h[q]);
                oh[q] = __floats2bfloat162_rn(v[2 * q] + x.x, v[2 * q + 1] + x.y);
            }
            *(uint4*)(out + (long long)row * ld + ch * 8) = o;
        }
    }
    asm volatile("bar.sync 1, 256;");
    long long c1 = clock64();
    if (tid == 0) cy[blockIdx.x] = c1 - c0;
}
int main() {
    const int ld = 320, rows = 128;
    __nv_bfloat16 *r, *o; long long* cy;
    cudaMalloc(&r, rows * ld * 2); cudaMalloc(&o, rows * ld * 2); cudaMalloc(&cy, 8 * 148);
    cudaMemset(r, 0, rows * ld * 2);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 132 * 4);
    for (int it = 0; it < 3; it++) k<<<1, 288, 128 * 132 * 4>>>(r, o, cy, ld, 0);
    long long h; cudaMemcpy(&h, cy, 8, cudaMemcpyDeviceToHost);
    printf("staged coalesced epilogue 128x128 (+res): %lld cycles\n", h);
    return 0;
}
