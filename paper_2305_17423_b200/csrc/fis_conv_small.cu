// 3x3 conv with few input channels (the latent stem conv: C_in = 4, K = 36; unet.py:447
// conv_in over the noisy latent, sparse.py:184-223 over the active pixels) on the FMA pipes.
//
// K = 9 * C_in is too narrow for a 64-wide tensor-core K block per tap, and the generic SIMT
// GEMM (fis_gemm_simt.cu) spends its time in per-element gathers and per-element stores. Here
// one CTA = 64 output rows x all N output channels:
//   * the weights [N][K] are staged transposed ([K][N], fp32) in shared memory before the
//     programmatic-launch wait (they are static);
//   * each row's 9 taps resolve once (select-on-read: fresh compact row / cached slab pixel /
//     zero padding, build_sel) and its K input values are staged as fp32;
//   * thread item = (row, 16 consecutive output channels), a warp = 32 rows of one channel group:
//     K x 16 FMAs from shared memory (weights broadcast), then
//     the shared fused row epilogue (bias, time bias, cached-stat GN + SiLU, step update,
//     records; fis_tc.cuh::row_epilogue) with 16-byte stores.
#include "fis_tc.cuh"

namespace fis {
namespace small {

using namespace fis::tc;

// ROWS output rows per tile: 32 (320 threads) for large M; 8 (160 threads) when 32-row tiles would
// leave most SMs idle (the batch-1 stem conv: 400 rows = 13 tiles of 32 -> 50 tiles of 8: 19 -> 14.7 us)
constexpr int MAX_N = 640;

__host__ __device__ inline int smem_bytes(int k, int n, int rows) {
    return (k * n + rows * (k + 1) + 6 * n) * 4 + rows * 9 * 4 + 64;
}

template <int ROWS>
__global__ void __launch_bounds__(ROWS == 32 ? 320 : 160, 2) conv_small_kernel(const fis_gemm_args a) {
    constexpr int THREADS = ROWS == 32 ? 320 : 160;
    extern __shared__ __align__(16) float sm[];
    const int K = a.k, N = a.n, cin = a.src[0].c;
    float* ws = sm;                  // [K][N]
    float* as = ws + K * N;          // [ROWS][K + 1]
    EpiTab tb;
    tb.bias = as + ROWS * (K + 1);
    tb.b2 = tb.bias + N;
    tb.mean = tb.b2 + N;
    tb.rstd = tb.mean + N;
    tb.gamma = tb.rstd + N;
    tb.beta = tb.gamma + N;
    int* sel = (int*)(tb.beta + N);  // [ROWS][9]
    const int tid = threadIdx.x;
    const int ls = ltr_begin(13);
    const int t = cur_step(a.step);  // host-written before the step
    {
        // weights: bf16 rows packed back to back (ld == K, even): 4-byte pairs, 8 loads in flight
        // per thread, transposed into [K][N] fp32
        const char* bbase = ref_base(a.b, t);
        if (a.b.dtype == FIS_BF16 && a.b.ld == K && !(K & 1) && !(((uintptr_t)bbase) & 3)) {
            const int pairs = N * K / 2;
            const __nv_bfloat162* w2 = (const __nv_bfloat162*)bbase;
            for (int i0 = tid; i0 < pairs; i0 += 8 * THREADS) {
                __nv_bfloat162 u[8];
#pragma unroll
                for (int j = 0; j < 8; j++) {
                    const int i = i0 + j * THREADS;
                    if (i < pairs) u[j] = w2[i];
                }
#pragma unroll
                for (int j = 0; j < 8; j++) {
                    const int i = i0 + j * THREADS;
                    if (i >= pairs) break;
                    const int e = 2 * i, n = e / K, k = e - n * K;  // K even: a pair never crosses rows
                    const float2 f = __bfloat1622float2(u[j]);
                    ws[k * N + n] = f.x;
                    ws[(k + 1) * N + n] = f.y;
                }
            }
        } else {
            for (int i = tid; i < N * K; i += THREADS) {
                const int n = i / K, k = i - n * K;
                ws[k * N + n] = load_elem(bbase, a.b.dtype, (long long)n * a.b.ld + k);
            }
        }
    }
    // the first tile's select-on-read table before the dependency wait: row lists and pixel maps are
    // plan data (no kernel of the step writes them)
    const int ntiles = (a.m + ROWS - 1) / ROWS;
    if ((int)blockIdx.x < ntiles && tid < ROWS) {
        const int r = (int)blockIdx.x * ROWS + tid;
        const int p = r < a.m ? (a.rows ? __ldg(a.rows + r) : r) : -1;
        build_sel(a, p, 0, sel + tid * 9);
    }
    pdl_trigger();
    pdl_wait();
    ltr(ls, 2);
    const EpiCtx e = make_epi(a, t);
    for (int c = tid; c < N; c += THREADS) {
        tb.bias[c] = a.bias ? __ldg(a.bias + c) : 0.f;
        tb.b2[c] = e.bias2 ? load_elem(e.bias2, a.bias2.dtype, c) : 0.f;
        tb.gamma[c] = 0.f;
        tb.beta[c] = 0.f;
        if (a.epi == FIS_EPI_GN_SILU) {
            const int g = c / e.cpg;
            const float rstd = (float)(1.0 / sqrt((double)e.var[g] + (double)a.eps));
            const float scale = rstd * __ldg(a.gamma + c);
            tb.mean[c] = scale;
            tb.rstd[c] = fmaf(-e.mean[g], scale, __ldg(a.beta + c));
        } else {
            tb.mean[c] = 0.f;
            tb.rstd[c] = 0.f;
        }
    }
#pragma unroll 1
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {  // persistent: weights staged once
    const int m0 = tile * ROWS;
    if (tile != (int)blockIdx.x && tid < ROWS) {
        const int r = m0 + tid;
        const int p = r < a.m ? (a.rows ? __ldg(a.rows + r) : r) : -1;
        build_sel(a, p, 0, sel + tid * 9);
    }
    __syncthreads();
    if (tile == (int)blockIdx.x) ltr(ls, 3);
    {
        const fis_src& s = a.src[0];
        const char* fb = s.fresh.ptr ? ref_base(s.fresh, t) : nullptr;
        const char* cb = s.cache.ptr ? ref_base(s.cache, t) : nullptr;
        // one (row, tap) per thread per pass: its cin values (fp32 x 4 = one 16-byte load)
        const bool vec = cin == 4 && s.fresh.dtype == FIS_F32 && (s.fresh.ld & 3) == 0 &&
                         (!cb || (s.cache.dtype == FIS_F32 && (s.cache.ld & 3) == 0));
#pragma unroll 1
        for (int i = tid; i < ROWS * 9; i += THREADS) {
            const int row = i / 9, tap = i - row * 9;
            const int q = sel[row * 9 + tap];
            float* dst = as + row * (K + 1) + tap * cin;
            if (q == SEL_ZERO) {
                for (int c = 0; c < cin; c++) dst[c] = 0.f;
            } else if (vec) {
                const float4 f = q >= 0 ? __ldcg((const float4*)((const float*)fb + (long long)q * s.fresh.ld))
                                        : __ldcg((const float4*)((const float*)cb + (long long)(-2 - q) * s.cache.ld));
                dst[0] = f.x; dst[1] = f.y; dst[2] = f.z; dst[3] = f.w;
            } else {
                for (int c = 0; c < cin; c++)
                    dst[c] = q >= 0 ? load_elem(fb, s.fresh.dtype, (long long)q * s.fresh.ld + c)
                                    : load_elem(cb, s.cache.dtype, (long long)(-2 - q) * s.cache.ld + c);
            }
        }
    }
    __syncthreads();
    if (tile == (int)blockIdx.x) ltr(ls, 4);
    const int groups = N / 16;
#pragma unroll 1
    for (int item = tid; item < ROWS * groups; item += THREADS) {
        // a warp = the rows of 32 / ROWS 16-channel groups: weight reads are (near-)broadcasts, the
        // row reads (pitch K + 1, odd) hit distinct banks
        const int g = item / ROWS, row = item - g * ROWS;
        const int r = m0 + row;
        if (r >= a.m) continue;
        float v[16];
#pragma unroll
        for (int j = 0; j < 16; j++) v[j] = 0.f;
        const float* ar = as + row * (K + 1);
        const float* wc = ws + g * 16;
#pragma unroll 4
        for (int k = 0; k < K; k++) {
            const float x = ar[k];
            const float4* w4 = (const float4*)(wc + k * N);
#pragma unroll
            for (int q = 0; q < 4; q++) {
                const float4 w = w4[q];
                v[4 * q] = fmaf(x, w.x, v[4 * q]);
                v[4 * q + 1] = fmaf(x, w.y, v[4 * q + 1]);
                v[4 * q + 2] = fmaf(x, w.z, v[4 * q + 2]);
                v[4 * q + 3] = fmaf(x, w.w, v[4 * q + 3]);
            }
        }
        if (tile == (int)blockIdx.x && item == tid) ltr(ls, 5);
        row_epilogue_any(a, e, tb, r, g * 16, 0, v);
    }
    if (tile == (int)blockIdx.x) ltr(ls, 6);
    __syncthreads();  // the next tile's row tables / inputs overwrite this one's
    }
    ltr(ls, 7);
}

}  // namespace small
}  // namespace fis

// Shapes this kernel takes: one 3x3 conv source with C_in <= 8 (no upsample), N a multiple of 16
// (<= 640), row-major outputs. Host-only.
int fis_conv_small_ok(const fis_gemm_args* a) {
    if (a->a_mode != FIS_A_CONV3X3 || a->nsrc != 1 || a->src[0].up || a->src[0].c > 8 || a->k != 9 * a->src[0].c)
        return 0;
    if (a->n % 16 || a->n > fis::small::MAX_N || a->d_trans || a->n_split > 0) return 0;
    return fis::small::smem_bytes(a->k, a->n, 32) <= 200 * 1024;
}

int fis_conv_small_launch(const fis_gemm_args* a, cudaStream_t stream) {
    using namespace fis::small;
    const bool small_m = (a->m + 31) / 32 < 64;  // (the dense 4096-row stem keeps 32-row tiles: measured)
    const int rows = small_m ? 8 : 32;
    const int smem = smem_bytes(a->k, a->n, rows);
    static bool configured = false;
    if (!configured) {
        if (cudaFuncSetAttribute(conv_small_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024) !=
                cudaSuccess ||
            cudaFuncSetAttribute(conv_small_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024) !=
                cudaSuccess)
            return FIS_ERR_UNSUPPORTED;
        configured = true;
    }
    // persistent CTAs (the weights are staged once per CTA), 2 per SM when registers allow
    const int tiles = (a->m + rows - 1) / rows;
    const dim3 grid(tiles < 2 * 148 ? tiles : 2 * 148);
    const cudaError_t e = small_m ? fis_launch(conv_small_kernel<8>, grid, dim3(160), smem, stream, *a)
                                  : fis_launch(conv_small_kernel<32>, grid, dim3(320), smem, stream, *a);
    return e == cudaSuccess ? FIS_OK : FIS_ERR_LAUNCH;
}

FIS_LTR_SETTER(fis_ltr_set_small)
