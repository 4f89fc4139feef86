// Mask generation (K1): fused single-CTA kernels.
//
// fis_mask_detect : accumulate_diff -> min-max -> Otsu -> threshold -> dilate
//                   (masks.py:117-192), bit-exact against numpy: the per-pixel
//                   channel mean and step sum follow numpy's outer-axis order, and
//                   Otsu's class sums reproduce numpy's pairwise summation tree
//                   (8-way unrolled leaves of <=128, halving splits) over the full
//                   masked vector, so the objective matches to the last bit.
// fis_mask_plan   : OR-pool pyramid, row-major active-pixel lists + pixel->row
//                   maps, active 2x2-tile lists (gather-plan origins) per level,
//                   via warp ballots and a block-wide prefix sum.
#include "fis_common.cuh"

namespace fis {

constexpr int MT = 1024;

// numpy pairwise_sum (float64, contiguous) over v[off, off+n) with masking:
// keep = (x >= eps) == want_ge ; masked-out entries contribute +0.0
__device__ double pw_sum(const float* v, int off, int n, double eps, bool want_ge) {
    auto val = [&](int j) -> double {
        const double x = (double)v[off + j];
        return ((x >= eps) == want_ge) ? x : 0.0;
    };
    if (n < 8) {
        double res = 0.0;
        for (int i = 0; i < n; i++) res = __dadd_rn(res, val(i));
        return res;
    }
    if (n <= 128) {
        double r[8];
#pragma unroll
        for (int j = 0; j < 8; j++) r[j] = val(j);
        int i = 8;
        for (; i < n - (n % 8); i += 8) {
#pragma unroll
            for (int j = 0; j < 8; j++) r[j] = __dadd_rn(r[j], val(i + j));
        }
        double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                               __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
        for (; i < n; i++) res = __dadd_rn(res, val(i));
        return res;
    }
    int n2 = n / 2;
    n2 -= n2 % 8;
    return __dadd_rn(pw_sum(v, off, n2, eps, want_ge), pw_sum(v, off + n2, n - n2, eps, want_ge));
}

__device__ __forceinline__ double block_reduce_minmax(double v, bool is_max, double* sh) {
    // 1024 threads, fixed tree
    for (int o = 16; o; o >>= 1) {
        double w = __shfl_xor_sync(0xffffffffu, v, o);
        v = is_max ? fmax(v, w) : fmin(v, w);
    }
    const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
    if (lane == 0) sh[warp] = v;
    __syncthreads();
    if (warp == 0) {
        v = sh[lane];
        for (int o = 16; o; o >>= 1) {
            double w = __shfl_xor_sync(0xffffffffu, v, o);
            v = is_max ? fmax(v, w) : fmin(v, w);
        }
        if (lane == 0) sh[32] = v;
    }
    __syncthreads();
    double r = sh[32];
    __syncthreads();
    return r;
}

__global__ void __launch_bounds__(MT, 1) mask_detect_kernel(const fis_mask_detect_args a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int hw = a.h * a.w;
    double* acc = (double*)smem;                  // [hw]
    float* v = (float*)(smem + (size_t)hw * 8);   // [hw]
    __shared__ double sh[33];
    __shared__ double part[256][4][2];
    __shared__ int pcnt[256][4];
    __shared__ double obj_s[256];
    __shared__ int valid_s[256];
    __shared__ int best_s;
    const int tid = threadIdx.x;
    pdl_trigger();
    pdl_wait();

    // Σ_t mean_c |x - y|  (masks.py:136-137): channel order sequential, then /C
    if (a.values_in) {
        // otsu_threshold on a given (non-degenerate) DiffMap
        for (int q = tid; q < hw; q += MT) { v[q] = a.values_in[q]; a.values[q] = v[q]; }
        __syncthreads();
    } else {
        for (int q = tid; q < hw; q += MT) {
            double s = 0.0;
            for (int t = a.t1; t <= a.t2; t++) {
                const float* x = (const float*)((const char*)a.x.ptr + (long long)(t - 1) * a.x.step_stride) + (long long)q * a.x.ld;
                const float* y = (const float*)((const char*)a.y.ptr + (long long)(t - 1) * a.y.step_stride) + (long long)q * a.y.ld;
                double d = 0.0;
                for (int c = 0; c < a.c; c++) d = __dadd_rn(d, fabs(__dsub_rn((double)x[c], (double)y[c])));
                d = __ddiv_rn(d, (double)a.c);
                s = (t == a.t1) ? d : __dadd_rn(s, d);
            }
            acc[q] = s;
        }
        __syncthreads();
        double lo = 1e300, hi = -1e300;
        for (int q = tid; q < hw; q += MT) {
            lo = fmin(lo, acc[q]);
            hi = fmax(hi, acc[q]);
        }
        lo = block_reduce_minmax(lo, false, sh);
        hi = block_reduce_minmax(hi, true, sh);
        const bool degenerate = (hi == lo);
        for (int q = tid; q < hw; q += MT) {
            float f = 0.f;
            if (!degenerate) {
                f = (float)__ddiv_rn(__dsub_rn(acc[q], lo), __dsub_rn(hi, lo));
                f = fminf(fmaxf(f, 0.f), 1.f);
            }
            v[q] = f;
            a.values[q] = f;
        }
        __syncthreads();
        if (degenerate) {
            for (int q = tid; q < hw; q += MT) { a.raw_mask[q] = 0; a.mask[q] = 0; }
            if (tid == 0) { a.result[0] = 1.0; a.result[1] = 0.0; a.flags[0] = 1; a.flags[1] = 1; }
            return;
        }
    }
    // Otsu over 256 midpoints; thread = (candidate, one of the <=4 subtrees formed by the top
    // two levels of numpy's pairwise recursion), so the f64 sums keep numpy's exact grouping.
    {
        const int i = tid >> 2, qq = tid & 3;
        const double eps = ((double)i + 0.5) / 256.0;
        int off = 0, len = 0;
        if (hw <= 128) {
            if (qq == 0) len = hw;
        } else {
            int h0 = hw / 2;
            h0 -= h0 % 8;
            const int half = qq >> 1, hoff = half ? h0 : 0, hlen = half ? hw - h0 : h0;
            if (hlen <= 128) {
                if ((qq & 1) == 0) { off = hoff; len = hlen; }
            } else {
                int q0 = hlen / 2;
                q0 -= q0 % 8;
                off = hoff + ((qq & 1) ? q0 : 0);
                len = (qq & 1) ? hlen - q0 : q0;
            }
        }
        part[i][qq][0] = len ? pw_sum(v, off, len, eps, false) : 0.0;
        part[i][qq][1] = len ? pw_sum(v, off, len, eps, true) : 0.0;
        int c = 0;
        for (int j = off; j < off + len; j++) c += ((double)v[j] >= eps);
        pcnt[i][qq] = c;
    }
    __syncthreads();
    if (tid < 256) {
        const int i = tid;
        double s1, s2;
        if (hw <= 128) {
            s1 = part[i][0][0];
            s2 = part[i][0][1];
        } else {
            int h0 = hw / 2;
            h0 -= h0 % 8;
            const bool splitA = h0 > 128, splitB = (hw - h0) > 128;
            const double a1 = splitA ? __dadd_rn(part[i][0][0], part[i][1][0]) : part[i][0][0];
            const double a2 = splitA ? __dadd_rn(part[i][0][1], part[i][1][1]) : part[i][0][1];
            const double b1 = splitB ? __dadd_rn(part[i][2][0], part[i][3][0]) : part[i][2][0];
            const double b2 = splitB ? __dadd_rn(part[i][2][1], part[i][3][1]) : part[i][2][1];
            s1 = __dadd_rn(a1, b1);
            s2 = __dadd_rn(a2, b2);
        }
        const long long n2 = (long long)pcnt[i][0] + pcnt[i][1] + pcnt[i][2] + pcnt[i][3];
        const long long n1 = hw - n2;
        const bool ok = n1 > 0 && n2 > 0;
        valid_s[i] = ok;
        double o = -INFINITY;
        if (ok) {
            const double m1 = __ddiv_rn(s1, (double)n1), m2 = __ddiv_rn(s2, (double)n2);
            const double dm = __dsub_rn(m1, m2);
            o = __dmul_rn(__ddiv_rn((double)(n1 * n2), __dmul_rn((double)hw, (double)hw)), __dmul_rn(dm, dm));
        }
        obj_s[i] = o;
    }
    __syncthreads();
    if (tid == 0) {
        int best = -1;
        double bo = -INFINITY;
        for (int i = 0; i < 256; i++)
            if (valid_s[i] && (best < 0 || obj_s[i] > bo)) { best = i; bo = obj_s[i]; }
        best_s = best;
        if (best < 0) {
            a.result[0] = 1.0; a.result[1] = 0.0; a.flags[0] = 1; a.flags[1] = 0;
        } else {
            a.result[0] = ((double)best + 0.5) / 256.0; a.result[1] = bo; a.flags[0] = 0; a.flags[1] = 0;
        }
    }
    __syncthreads();
    const int best = best_s;
    const float eps32 = best < 0 ? 2.f : (float)(((double)best + 0.5) / 256.0);
    unsigned char* raw = (unsigned char*)acc;  // reuse
    for (int q = tid; q < hw; q += MT) {
        const unsigned char b = (best >= 0) && (v[q] >= eps32);
        raw[q] = b;
        a.raw_mask[q] = b;
    }
    __syncthreads();
    const int r = a.radius;
    for (int q = tid; q < hw; q += MT) {
        const int y = q / a.w, x = q % a.w;
        unsigned char o = 0;
        for (int yy = max(0, y - r); yy <= min(a.h - 1, y + r) && !o; yy++)
            for (int xx = max(0, x - r); xx <= min(a.w - 1, x + r); xx++)
                if (raw[yy * a.w + xx]) { o = 1; break; }
        a.mask[q] = o;
    }
}

// block exclusive scan of one int per thread (MT threads); returns total via *tot
__device__ int block_excl_scan(int x, int* sh, int* tot) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int inc = x;
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) sh[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        int w = sh[lane];
        int wi = w;
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += y;
        }
        sh[32 + lane] = wi - w;
        if (lane == 31) sh[64] = wi;
    }
    __syncthreads();
    const int res = sh[32 + warp] + inc - x;
    *tot = sh[64];
    __syncthreads();
    return res;
}

// compacts active entries of bits[0..n) in order; writes list[] and optional index[]
__device__ int compact_list(const unsigned char* bits, int n, int* list, int* index, int* sh) {
    const int per = (n + MT - 1) / MT;
    const int b = threadIdx.x * per, e = min(n, b + per);
    int cnt = 0;
    for (int q = b; q < e; q++) cnt += bits[q] != 0;
    int tot;
    int pos = block_excl_scan(cnt, sh, &tot);
    for (int q = b; q < e; q++) {
        if (bits[q]) {
            if (list) list[pos] = q;
            if (index) index[q] = pos;
            pos++;
        } else if (index) {
            index[q] = -1;
        }
    }
    return tot;
}

__global__ void __launch_bounds__(MT, 1) mask_plan_kernel(const fis_mask_plan_args a) {
    extern __shared__ __align__(16) unsigned char sm[];
    __shared__ int sh[72];
    pdl_trigger();
    pdl_wait();
    unsigned char* cur = sm;  // level bits
    unsigned char* tb = sm + a.h * a.w;  // tile bits scratch
    int h = a.h, w = a.w;
    const int r = a.radius;
    for (int q = threadIdx.x; q < h * w; q += MT) {
        const int y = q / w, x = q % w;
        unsigned char o = 0;
        for (int yy = max(0, y - r); yy <= min(h - 1, y + r) && !o; yy++)
            for (int xx = max(0, x - r); xx <= min(w - 1, x + r); xx++)
                if (a.mask[yy * w + xx]) { o = 1; break; }
        cur[q] = o;
    }
    __syncthreads();
    for (int l = 0; l < a.levels; l++) {
        if (l > 0) {
            const int nh = h / 2, nw = w / 2;
            // in-place safe: read children before overwrite using a second buffer
            for (int q = threadIdx.x; q < nh * nw; q += MT) {
                const int y = q / nw, x = q % nw;
                const unsigned char* p = cur + (2 * y) * w + 2 * x;
                tb[q] = p[0] | p[1] | p[w] | p[w + 1];
            }
            __syncthreads();
            for (int q = threadIdx.x; q < nh * nw; q += MT) cur[q] = tb[q];
            __syncthreads();
            h = nh; w = nw;
        }
        if (a.bits[l])
            for (int q = threadIdx.x; q < h * w; q += MT) a.bits[l][q] = cur[q];
        const int n = compact_list(cur, h * w, a.rows[l], a.index[l], sh);
        if (threadIdx.x == 0) a.counts[l] = n;
        // active 2x2 tiles on a regular grid (sparse.py:81-88), clipped at the border
        const int th = (h + 1) / 2, tw = (w + 1) / 2;
        for (int q = threadIdx.x; q < th * tw; q += MT) {
            const int y = q / tw, x = q % tw;
            unsigned char o = 0;
            for (int dy = 0; dy < 2; dy++)
                for (int dx = 0; dx < 2; dx++)
                    if (2 * y + dy < h && 2 * x + dx < w) o |= cur[(2 * y + dy) * w + 2 * x + dx];
            tb[q] = o;
        }
        __syncthreads();
        const int nt = compact_list(tb, th * tw, a.tiles[l], nullptr, sh);
        if (threadIdx.x == 0) a.counts[a.levels + l] = nt;
        __syncthreads();
    }
}

}  // namespace fis

extern "C" long long fis_mask_detect_smem(int h, int w) { return (long long)h * w * 12; }

extern "C" int fis_mask_detect(const fis_mask_detect_args* a, void* stream) {
    const int hw = a->h * a->w;
    if (hw < 1 || a->t1 < 1 || a->t2 < a->t1 || a->c < 1) return FIS_ERR_SHAPE;
    const size_t smem = (size_t)fis_mask_detect_smem(a->h, a->w);
    if (cudaFuncSetAttribute(fis::mask_detect_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return FIS_ERR_UNSUPPORTED;
    return fis_launch(fis::mask_detect_kernel, dim3(1), dim3(fis::MT), smem, (cudaStream_t)stream, *a) == cudaSuccess
               ? FIS_OK : FIS_ERR_LAUNCH;
}

extern "C" int fis_mask_plan(const fis_mask_plan_args* a, void* stream) {
    if (a->levels < 1 || a->levels > FIS_MAX_LEVELS) return FIS_ERR_SHAPE;
    const size_t smem = (size_t)a->h * a->w * 2;
    if (cudaFuncSetAttribute(fis::mask_plan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return FIS_ERR_UNSUPPORTED;
    return fis_launch(fis::mask_plan_kernel, dim3(1), dim3(fis::MT), smem, (cudaStream_t)stream, *a) == cudaSuccess
               ? FIS_OK : FIS_ERR_LAUNCH;
}
