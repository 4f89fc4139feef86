// SIMT fp32-accumulate gather-GEMM (the fp32-parity path and the path for
// shapes the tcgen05 kernel does not take: C_in % 8 != 0, N % 16 != 0).
//
// D[r,n] = epi( sum_k A[r,k] * B[n,k] ), A gathered on the fly:
//   FIS_A_ROWS    : A[r,k] = a[row(r)*lda + k]
//   FIS_A_CONV3X3 : k = tap*Cin + c, pixel p = rows[r], neighbour q = p + (ky-1, kx-1),
//                   zero outside the image (same padding, tensors.py:97-113), channel c
//                   taken from concat(src0, src1) with select-on-read + nearest upsample.
// Split-K partials are reduced in fixed split order by the last-arriving CTA, so
// results are bitwise deterministic run to run (test_unet.py:303-312 semantics).
#include "fis_common.cuh"

namespace fis {

constexpr int SBM = 64, SBN = 64, SBK = 16, STHREADS = 256;

struct ConvGeom {
    int cin, c0;
};

__device__ __forceinline__ float gather_a(const fis_gemm_args& a, int t, const char* f0, const char* c0p,
                                          const char* f1, const char* c1p, const char* abase, int r, int k,
                                          int p, int oy, int ox) {
    if (a.a_mode == FIS_A_ROWS) {
        return load_elem(abase, a.a.dtype, (long long)p * a.a.ld + k);
    }
    const int cin = a.src[0].c + (a.nsrc > 1 ? a.src[1].c : 0);
    const int tap = k / cin;
    int c = k - tap * cin;
    const int y = oy + tap / 3 - 1, x = ox + tap % 3 - 1;
    if (y < 0 || x < 0 || y >= a.out_h || x >= a.out_w) return 0.f;
    const bool second = c >= a.src[0].c;
    const fis_src& s = second ? a.src[1] : a.src[0];
    if (second) c -= a.src[0].c;
    const int sy = s.up ? (y >> 1) : y, sx = s.up ? (x >> 1) : x;
    const int img = p / (a.out_h * a.out_w);  // stacked images (batched requests)
    return src_value(s, second ? f1 : f0, second ? c1p : c0p, img * s.h * s.w + sy * s.w + sx, c);
}

__global__ void __launch_bounds__(STHREADS) gemm_simt_kernel(const fis_gemm_args a) {
    const int ls = ltr_begin(3);
    __shared__ float As[SBK][SBM + 4];
    __shared__ float Bs[SBK][SBN + 4];
    __shared__ int rowp[SBM], rowy[SBM], rowx[SBM];
    __shared__ int s_last;
    pdl_trigger();
    pdl_wait();
    ltr(ls, 2);
    const int t = cur_step(a.step);
    const int tid = threadIdx.x;
    const int n0 = blockIdx.x * SBN, m0 = blockIdx.y * SBM;
    const int ktiles = (a.k + SBK - 1) / SBK;
    const int kper = (ktiles + a.splits - 1) / a.splits;
    const int kt0 = blockIdx.z * kper, kt1 = min(ktiles, kt0 + kper);

    const char* abase = a.a.ptr ? ref_base(a.a, t) : nullptr;
    const char* f0 = a.nsrc > 0 && a.src[0].fresh.ptr ? ref_base(a.src[0].fresh, t) : nullptr;
    const char* c0p = a.nsrc > 0 && a.src[0].cache.ptr ? ref_base(a.src[0].cache, t) : nullptr;
    const char* f1 = a.nsrc > 1 && a.src[1].fresh.ptr ? ref_base(a.src[1].fresh, t) : nullptr;
    const char* c1p = a.nsrc > 1 && a.src[1].cache.ptr ? ref_base(a.src[1].cache, t) : nullptr;
    const char* bbase = ref_base(a.b, t);

    if (tid < SBM) {
        int r = m0 + tid;
        int p = r < a.m ? (a.rows ? __ldg(a.rows + r) : r) : 0;
        rowp[tid] = p;
        if (a.a_mode == FIS_A_CONV3X3) {
            const int lp = p % (a.out_h * a.out_w);  // pixel within its stacked image
            rowy[tid] = lp / a.out_w;
            rowx[tid] = lp - (lp / a.out_w) * a.out_w;
        }
    }
    __syncthreads();

    const int tx = tid % 16, ty = tid / 16;  // 16x16 threads, 4x4 outputs each
    float acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; i++)
#pragma unroll
        for (int j = 0; j < 4; j++) acc[i][j] = 0.f;

    const int lk = tid % SBK, lr = tid / SBK;  // loader: 16 k x 16 rows per pass
    for (int kt = kt0; kt < kt1; kt++) {
        const int k = kt * SBK + lk;
#pragma unroll
        for (int i = 0; i < 4; i++) {
            const int row = lr + 16 * i;
            const int r = m0 + row;
            float v = 0.f;
            if (r < a.m && k < a.k && rowp[row] >= 0)  // rowp < 0: framing row at an image border
                v = gather_a(a, t, f0, c0p, f1, c1p, abase, r, k, rowp[row], rowy[row], rowx[row]);
            As[lk][row] = v;
            const int n = n0 + row;
            float bv = 0.f;
            if (n < a.n && k < a.k) bv = load_elem(bbase, a.b.dtype, (long long)n * a.b.ld + k);
            Bs[lk][row] = bv;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < SBK; kk++) {
            float av[4], bv[4];
#pragma unroll
            for (int i = 0; i < 4; i++) av[i] = As[kk][ty * 4 + i];
#pragma unroll
            for (int j = 0; j < 4; j++) bv[j] = Bs[kk][tx * 4 + j];
#pragma unroll
            for (int i = 0; i < 4; i++)
#pragma unroll
                for (int j = 0; j < 4; j++) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
        }
        __syncthreads();
    }

    const EpiCtx e = make_epi(a, t);
    if (a.splits <= 1) {
#pragma unroll 1
        for (int i = 0; i < 4; i++) {
            const int r = m0 + ty * 4 + i;
            if (r >= a.m) continue;
#pragma unroll
            for (int j = 0; j < 4; j++) {
                const int n = n0 + tx * 4 + j;
                if (n < a.n) epilogue_store(a, e, r, n, acc[i][j]);
            }
        }
        return;
    }
    // split-K: publish partial, last CTA reduces in split order
    float* wsz = a.ws + (long long)blockIdx.z * a.m * a.n;
#pragma unroll
    for (int i = 0; i < 4; i++) {
        const int r = m0 + ty * 4 + i;
        if (r >= a.m) continue;
#pragma unroll
        for (int j = 0; j < 4; j++) {
            const int n = n0 + tx * 4 + j;
            if (n < a.n) __stcg(wsz + (long long)r * a.n + n, acc[i][j]);
        }
    }
    __threadfence();
    __syncthreads();
    const int tile = blockIdx.y * gridDim.x + blockIdx.x;
    if (tid == 0) {
        int old = atomicAdd(a.counters + tile, 1);
        s_last = (old == a.splits - 1);
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
#pragma unroll 1
    for (int i = 0; i < 4; i++) {
        const int r = m0 + ty * 4 + i;
        if (r >= a.m) continue;
#pragma unroll 1
        for (int j = 0; j < 4; j++) {
            const int n = n0 + tx * 4 + j;
            if (n >= a.n) continue;
            float s = 0.f;
            for (int z = 0; z < a.splits; z++) s += __ldcg(a.ws + ((long long)z * a.m + r) * a.n + n);
            epilogue_store(a, e, r, n, s);
        }
    }
    if (tid == 0) a.counters[tile] = 0;
}

}  // namespace fis

int fis_gemm_simt_launch(const fis_gemm_args* a, cudaStream_t stream) {
    dim3 grid((a->n + fis::SBN - 1) / fis::SBN, (a->m + fis::SBM - 1) / fis::SBM, a->splits > 1 ? a->splits : 1);
    return fis_launch(fis::gemm_simt_kernel, grid, dim3(fis::STHREADS), 0, stream, *a) == cudaSuccess ? FIS_OK
                                                                                               : FIS_ERR_LAUNCH;
}

FIS_LTR_SETTER(fis_ltr_set_simt)
