// Row-wise / element-wise kernels of the sparse edit step: group-norm statistics
// and application (+SiLU), scaled row softmax with controlled-mode column pinning,
// select-on-read 2x2 average pooling and full-map materialisation.
// All reductions use a fixed order, so outputs are bitwise deterministic.
#include <cstdlib>
#include "fis_common.cuh"
#include <type_traits>

namespace fis {

// ---- group norm statistics (tensors.py:129-146): two-pass f64, rounded to f32
__global__ void __launch_bounds__(256) gn_stats_kernel(const fis_gn_stats_args a) {
    const int ls = ltr_begin(11);
    const int t = cur_step(a.step);  // host-written before the step: read before the wait
    pdl_trigger();
    pdl_wait();
    ltr(ls, 2);
    const int g = blockIdx.x, img = blockIdx.y;  // one CTA per (group, stacked image)
    const int cpg = a.c / a.groups;
    const long long cnt = (long long)a.hw * cpg;
    const char* x = ref_base(a.x, t) + (long long)img * a.hw * a.x.ld * (a.x.dtype == FIS_BF16 ? 2 : 4);
    __shared__ double red[256];
    if (a.x.dtype == FIS_BF16 && (cpg % 8) == 0 && (a.x.ld % 8) == 0 && (((uintptr_t)x) & 15) == 0) {
        // bf16 activations (perf mode): 16-byte loads, fp32 per-thread partials, f64 block sums;
        // still two-pass and in a fixed order (deterministic)
        const int vpg = cpg / 8, items = a.hw * vpg;
        const __nv_bfloat16* xb = (const __nv_bfloat16*)x + g * cpg;
        float ps = 0.f;
        for (int i = threadIdx.x; i < items; i += blockDim.x) {
            const int q = i / vpg, v = i - q * vpg;
            const uint4 u = *(const uint4*)(xb + (long long)q * a.x.ld + v * 8);
            const __nv_bfloat162* h = (const __nv_bfloat162*)&u;
#pragma unroll
            for (int k = 0; k < 4; k++) {
                const float2 f = __bfloat1622float2(h[k]);
                ps += f.x + f.y;
            }
        }
        red[threadIdx.x] = (double)ps;
        __syncthreads();
        for (int o = 128; o; o >>= 1) {
            if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
            __syncthreads();
        }
        const double mean = red[0] / (double)cnt;
        const float mf = (float)mean;
        __syncthreads();
        float pv = 0.f;
        for (int i = threadIdx.x; i < items; i += blockDim.x) {
            const int q = i / vpg, v = i - q * vpg;
            const uint4 u = *(const uint4*)(xb + (long long)q * a.x.ld + v * 8);
            const __nv_bfloat162* h = (const __nv_bfloat162*)&u;
#pragma unroll
            for (int k = 0; k < 4; k++) {
                const float2 f = __bfloat1622float2(h[k]);
                const float d0 = f.x - mf, d1 = f.y - mf;
                pv = fmaf(d0, d0, fmaf(d1, d1, pv));
            }
        }
        red[threadIdx.x] = (double)pv;
        __syncthreads();
        for (int o = 128; o; o >>= 1) {
            if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            ((float*)ref_base(a.mean, t))[img * a.groups + g] = mf;
            ((float*)ref_base(a.var, t))[img * a.groups + g] = (float)(red[0] / (double)cnt);
        }
        return;
    }
    double s = 0.0;
    // thread = pixel (strided), inner loop over the group's contiguous channels (32-bit index math)
    for (int q = threadIdx.x; q < a.hw; q += blockDim.x) {
        const long long base = (long long)q * a.x.ld + g * cpg;
        for (int c = 0; c < cpg; c++) s += (double)load_elem(x, a.x.dtype, base + c);
    }
    red[threadIdx.x] = s;
    __syncthreads();
    for (int o = 128; o; o >>= 1) {
        if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    const double mean = red[0] / (double)cnt;
    __syncthreads();
    double v = 0.0;
    for (int q = threadIdx.x; q < a.hw; q += blockDim.x) {
        const long long base = (long long)q * a.x.ld + g * cpg;
        for (int c = 0; c < cpg; c++) {
            const double d = (double)load_elem(x, a.x.dtype, base + c) - mean;
            v += d * d;
        }
    }
    red[threadIdx.x] = v;
    __syncthreads();
    for (int o = 128; o; o >>= 1) {
        if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        ((float*)ref_base(a.mean, t))[img * a.groups + g] = (float)mean;
        ((float*)ref_base(a.var, t))[img * a.groups + g] = (float)(red[0] / (double)cnt);
    }
}

// ---- normalise with given stats (+SiLU) (tensors.py:149-180, unet.py:291-293)
__global__ void gn_apply_kernel(const fis_gn_apply_args a) {
    const int ls = ltr_begin(7);
    const int t = cur_step(a.step);  // host-written before the step: read before the wait
    pdl_trigger();
    pdl_wait();
    ltr(ls, 2);
    const char* x = ref_base(a.x, t);
    const float* mean = (const float*)ref_base(a.mean, t);
    const float* var = (const float*)ref_base(a.var, t);
    char* yn = a.y_norm.ptr ? ref_base(a.y_norm, t) : nullptr;
    char* ys = a.y_silu.ptr ? ref_base(a.y_silu, t) : nullptr;
    const int cpg = a.c / a.groups;
    const int total = a.rows * a.c;
    const bool bf16_out = (!yn || a.y_norm.dtype == FIS_BF16) && (!ys || a.y_silu.dtype == FIS_BF16);
    if (bf16_out && a.x.dtype == FIS_BF16 && cpg >= 8 && (a.c % 8) == 0 && (a.x.ld % 8) == 0 &&
        (!yn || (a.y_norm.ld % 8) == 0) &&
        (!ys || (a.y_silu.ld % 8) == 0) && ((((uintptr_t)x) | ((uintptr_t)yn) | ((uintptr_t)ys)) & 15) == 0) {
        // bf16 perf mode, 8 channels (one group) per thread: 16-byte loads / stores
        const int cv = a.c / 8, totalv = a.rows * cv;
        for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < totalv; e += gridDim.x * blockDim.x) {
            const int r = e / cv, c = (e - r * cv) * 8;
            const int xr = a.x_rows ? __ldg(a.x_rows + r) : r;
            const int yr = a.y_rows ? __ldg(a.y_rows + r) : r;
            // 8 channels span at most two groups (cpg >= 8): g0 below `split`, g0 + 1 from it
            const int gi = (a.row_img ? __ldg(a.row_img + r) : (a.img_rows > 0 ? r / a.img_rows : 0)) * a.groups;
            const int g0 = c / cpg, split = (g0 + 1) * cpg - c;
            // fp32 1/sqrt (IEEE sqrt and divide): the per-item f64 sqrt + divide made this kernel
            // issue-bound (r02, stacked step: 380 instructions per 8 channels, 23 us for 22 MB)
            const float rstd0 = __frcp_rn(__fsqrt_rn(var[gi + g0] + a.eps));
            const float mu0 = mean[gi + g0];
            float rstd1 = rstd0, mu1 = mu0;
            if (split < 8) {
                rstd1 = __frcp_rn(__fsqrt_rn(var[gi + g0 + 1] + a.eps));
                mu1 = mean[gi + g0 + 1];
            }
            const uint4 u = *(const uint4*)((const __nv_bfloat16*)x + (long long)xr * a.x.ld + c);
            const __nv_bfloat162* h = (const __nv_bfloat162*)&u;
            uint4 on, os;
            __nv_bfloat162* hn = (__nv_bfloat162*)&on;
            __nv_bfloat162* hs = (__nv_bfloat162*)&os;
            // gamma / beta as two 16-byte loads each (scalar loads made this kernel L1-bound)
            float ga[8], be[8];
            *(float4*)ga = __ldg((const float4*)(a.gamma + c));
            *(float4*)(ga + 4) = __ldg((const float4*)(a.gamma + c + 4));
            *(float4*)be = __ldg((const float4*)(a.beta + c));
            *(float4*)(be + 4) = __ldg((const float4*)(a.beta + c + 4));
#pragma unroll
            for (int k = 0; k < 4; k++) {
                const float2 f = __bfloat1622float2(h[k]);
                const bool s0 = 2 * k >= split, s1 = 2 * k + 1 >= split;
                const float y0 = fmaf((f.x - (s0 ? mu1 : mu0)) * (s0 ? rstd1 : rstd0), ga[2 * k], be[2 * k]);
                const float y1 = fmaf((f.y - (s1 ? mu1 : mu0)) * (s1 ? rstd1 : rstd0), ga[2 * k + 1], be[2 * k + 1]);
                hn[k] = __floats2bfloat162_rn(y0, y1);
                hs[k] = __floats2bfloat162_rn(__fdividef(y0, 1.0f + __expf(-y0)), __fdividef(y1, 1.0f + __expf(-y1)));
            }
            if (yn) *(uint4*)((__nv_bfloat16*)yn + (long long)yr * a.y_norm.ld + c) = on;
            if (ys) *(uint4*)((__nv_bfloat16*)ys + (long long)yr * a.y_silu.ld + c) = os;
        }
        return;
    }
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
        const int r = e / a.c, c = e - (e / a.c) * a.c;
        const int xr = a.x_rows ? __ldg(a.x_rows + r) : r;
        const int yr = a.y_rows ? __ldg(a.y_rows + r) : r;
        const int g = (a.row_img ? __ldg(a.row_img + r) : (a.img_rows > 0 ? r / a.img_rows : 0)) * a.groups + c / cpg;
        float y;
        if (bf16_out) {
            // bf16 mode: fp32 normalisation (the fp32-parity mode keeps the reference's f64)
            const float rstd = (float)(1.0 / sqrt((double)var[g] + (double)a.eps));
            y = fmaf((load_elem(x, a.x.dtype, (long long)xr * a.x.ld + c) - mean[g]) * rstd, a.gamma[c], a.beta[c]);
            if (yn) store_elem(yn, a.y_norm.dtype, (long long)yr * a.y_norm.ld + c, y);
            if (ys) store_elem(ys, a.y_silu.dtype, (long long)yr * a.y_silu.ld + c, __fdividef(y, 1.0f + __expf(-y)));
            continue;
        }
        const double xv = (double)load_elem(x, a.x.dtype, (long long)xr * a.x.ld + c);
        const double y64 = (xv - (double)mean[g]) / sqrt((double)var[g] + (double)a.eps) * (double)a.gamma[c] +
                           (double)a.beta[c];
        y = (float)y64;
        if (yn) store_elem(yn, a.y_norm.dtype, (long long)yr * a.y_norm.ld + c, y);
        if (ys) {
            const double yd = (double)y;
            store_elem(ys, a.y_silu.dtype, (long long)yr * a.y_silu.ld + c, (float)(yd / (1.0 + exp(-yd))));
        }
    }
}

// ---- scaled row softmax; one warp per row (tensors.py:183-192, unet.py:555-566)
__global__ void softmax_kernel(const fis_softmax_args a) {
    const int ls = ltr_begin(8);
    const int t = cur_step(a.step);  // host-written before the step: read before the wait
    pdl_trigger();
    pdl_wait();
    ltr(ls, 2);
    const int warps = blockDim.x / 32;
    const int row = blockIdx.x * warps + threadIdx.x / 32;
    const int lane = threadIdx.x & 31;
    if (row >= a.rows) return;
    char* pb = ref_base(a.p, t);
    char* mb = a.map.ptr ? ref_base(a.map, t) : nullptr;
    const float* cached = a.cached.ptr ? (const float*)ref_base(a.cached, t) + (long long)row * a.cached.ld : nullptr;
    const long long prow = (long long)row * a.p.ld;
    if (a.verbatim) {
        for (int j = lane; j < a.cols; j += 32) {
            const float v = cached[j];
            store_elem(pb, a.p.dtype, prow + j, v);
            if (mb) ((float*)mb)[(long long)row * a.map.ld + j] = v;
        }
    } else if (a.npairs == 0 && a.cols <= 32 * 16) {
        // one pass: the row lives in registers (<= 16 values per lane), all loads in flight
        // (same max / sum / normalise arithmetic as the multi-pass loop below)
        const float* s = (const float*)ref_base(a.s, t) + (long long)row * a.s.ld;
        float x[16];
        float m = -INFINITY;
#pragma unroll
        for (int k = 0; k < 16; k++) {
            const int j = lane + 32 * k;
            x[k] = j < a.cols ? s[j] * a.scale : -INFINITY;
        }
#pragma unroll
        for (int k = 0; k < 16; k++) m = fmaxf(m, x[k]);
        m = warp_max(m);
        float sum = 0.f;
#pragma unroll
        for (int k = 0; k < 16; k++) {
            x[k] = lane + 32 * k < a.cols ? expf(x[k] - m) : 0.f;
            sum += x[k];
        }
        sum = warp_sum(sum);
        const float inv_sum = 1.0f / sum;
#pragma unroll
        for (int k = 0; k < 16; k++) {
            const int j = lane + 32 * k;
            if (j < a.cols) {
                const float v = x[k] * inv_sum;
                store_elem(pb, a.p.dtype, prow + j, v);
                if (mb) ((float*)mb)[(long long)row * a.map.ld + j] = v;
            }
        }
    } else {
        const float* s = (const float*)ref_base(a.s, t) + (long long)row * a.s.ld;
        float m = -INFINITY;
        for (int j = lane; j < a.cols; j += 32) m = fmaxf(m, s[j] * a.scale);
        m = warp_max(m);
        float sum = 0.f;
        for (int j = lane; j < a.cols; j += 32) sum += expf(s[j] * a.scale - m);
        sum = warp_sum(sum);
        const float inv_sum = 1.0f / sum;
        if (a.npairs == 0) {
            for (int j = lane; j < a.cols; j += 32) {
                const float v = expf(s[j] * a.scale - m) * inv_sum;
                store_elem(pb, a.p.dtype, prow + j, v);
                if (mb) ((float*)mb)[(long long)row * a.map.ld + j] = v;
            }
        } else {
            // pin shared-token columns to the cached map, renormalise rows (f32 sum, f64 divide)
            float rs = 0.f;
            for (int j = lane; j < a.cols; j += 32) {
                float v = expf(s[j] * a.scale - m) * inv_sum;
                for (int i = 0; i < a.npairs; i++)
                    if (__ldg(a.pair_new + i) == j) v = cached[__ldg(a.pair_old + i)];
                rs += v;
            }
            rs = warp_sum(rs);
            for (int j = lane; j < a.cols; j += 32) {
                float v = expf(s[j] * a.scale - m) * inv_sum;
                for (int i = 0; i < a.npairs; i++)
                    if (__ldg(a.pair_new + i) == j) v = cached[__ldg(a.pair_old + i)];
                const float o = (float)((double)v / (double)rs);
                store_elem(pb, a.p.dtype, prow + j, o);
                if (mb) ((float*)mb)[(long long)row * a.map.ld + j] = o;
            }
        }
    }
    for (int j = a.cols + lane; j < a.pad_cols; j += 32) store_elem(pb, a.p.dtype, prow + j, 0.f);
}

// ---- 2x2 average pool with select-on-read (unet.py:296-298; numpy order (a+b)+(c+d))
__global__ void pool2_kernel(const fis_pool_args a) {
    const int ls = ltr_begin(6);
    const int t = cur_step(a.step);  // host-written before the step: read before the wait
    pdl_trigger();
    pdl_wait();
    ltr(ls, 2);
    const char* fr = a.src.fresh.ptr ? ref_base(a.src.fresh, t) : nullptr;
    const char* ca = a.src.cache.ptr ? ref_base(a.src.cache, t) : nullptr;
    char* out = ref_base(a.out, t);
    const int cw = a.src.w / 2, chw = (a.src.h / 2) * cw;
    const int total = a.n * a.c;
    const bool vec = a.src.fresh.dtype == FIS_BF16 && (!a.src.index || a.src.cache.dtype == FIS_BF16) &&
                     a.out.dtype == FIS_BF16 && (a.c % 8) == 0 && (a.src.fresh.ld % 8) == 0 &&
                     (!a.src.index || (a.src.cache.ld % 8) == 0) && (a.out.ld % 8) == 0 &&
                     ((((uintptr_t)fr) | ((uintptr_t)ca) | ((uintptr_t)out)) & 15) == 0;
    if (vec) {  // 8 channels per thread: each of the 4 source rows selected once, read as one vector
        for (int e = (blockIdx.x * blockDim.x + threadIdx.x) * 8; e < total; e += gridDim.x * blockDim.x * 8) {
            const int i = e / a.c, c = e - (e / a.c) * a.c;
            const int P = a.rows ? __ldg(a.rows + i) : i;
            const int img = P / chw, lP = P - img * chw;  // stacked images (batched requests)
            const int py = lP / cw, px = lP - (lP / cw) * cw;
            const int q = img * a.src.h * a.src.w + (2 * py) * a.src.w + 2 * px;
            const int qs[4] = {q, q + 1, q + a.src.w, q + a.src.w + 1};
            uint4 u[4];
#pragma unroll
            for (int k = 0; k < 4; k++) u[k] = *(const uint4*)((const __nv_bfloat16*)src_row(a.src, fr, ca, qs[k]).p + c);
            uint4 o;
            __nv_bfloat162* oh = (__nv_bfloat162*)&o;
#pragma unroll
            for (int h = 0; h < 4; h++) {
                const float2 a0 = __bfloat1622float2(((const __nv_bfloat162*)&u[0])[h]);
                const float2 a1 = __bfloat1622float2(((const __nv_bfloat162*)&u[1])[h]);
                const float2 a2 = __bfloat1622float2(((const __nv_bfloat162*)&u[2])[h]);
                const float2 a3 = __bfloat1622float2(((const __nv_bfloat162*)&u[3])[h]);
                oh[h] = __floats2bfloat162_rn(__fmul_rn(__fadd_rn(__fadd_rn(a0.x, a1.x), __fadd_rn(a2.x, a3.x)), 0.25f),
                                              __fmul_rn(__fadd_rn(__fadd_rn(a0.y, a1.y), __fadd_rn(a2.y, a3.y)), 0.25f));
            }
            *(uint4*)((__nv_bfloat16*)out + (long long)i * a.out.ld + c) = o;
        }
        return;
    }
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
        const int i = e / a.c, c = e - (e / a.c) * a.c;
        const int P = a.rows ? __ldg(a.rows + i) : i;
        const int img = P / chw, lP = P - img * chw;
        const int py = lP / cw, px = lP - (lP / cw) * cw;
        const int q = img * a.src.h * a.src.w + (2 * py) * a.src.w + 2 * px;
        const float v00 = src_value(a.src, fr, ca, q, c), v01 = src_value(a.src, fr, ca, q + 1, c);
        const float v10 = src_value(a.src, fr, ca, q + a.src.w, c), v11 = src_value(a.src, fr, ca, q + a.src.w + 1, c);
        const float s = __fadd_rn(__fadd_rn(v00, v01), __fadd_rn(v10, v11));
        store_elem(out, a.out.dtype, (long long)i * a.out.ld + c, __fmul_rn(s, 0.25f));
    }
}

// ---- full-map materialisation: out[q] = select(q)
__global__ void materialize_kernel(const fis_materialize_args a) {
    const int ls = ltr_begin(9);
    const int t = cur_step(a.step);  // host-written before the step: read before the wait
    pdl_trigger();
    pdl_wait();
    ltr(ls, 2);
    const char* fr = a.src.fresh.ptr ? ref_base(a.src.fresh, t) : nullptr;
    const char* ca = a.src.cache.ptr ? ref_base(a.src.cache, t) : nullptr;
    char* out = ref_base(a.out, t);
    const int total = a.src.h * a.src.w * a.c;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
        const int q = e / a.c, c = e - (e / a.c) * a.c;
        store_elem(out, a.out.dtype, (long long)q * a.out.ld + c, src_value(a.src, fr, ca, q, c));
    }
}

// ---- nearest 2x upsample of a dense map (unet.py:301-302), 8 channels per thread
__global__ void up2_kernel(const fis_pool_args a) {
    const int ls = ltr_begin(10);
    const int t = cur_step(a.step);  // host-written before the step: read before the wait
    pdl_trigger();
    pdl_wait();
    ltr(ls, 2);
    const char* fr = ref_base(a.src.fresh, t);
    char* out = ref_base(a.out, t);
    const int ow = 2 * a.src.w, ohw = 4 * a.src.h * a.src.w, cv = a.c / 8;
    const long long total = (long long)a.n * cv;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
        const int p = (int)(e / cv), c = (int)(e - (long long)p * cv) * 8;
        const int img = p / ohw, lp = p - img * ohw;
        const int y = lp / ow, x = lp - y * ow;
        const long long q = (long long)img * a.src.h * a.src.w + (y >> 1) * a.src.w + (x >> 1);
        *(uint4*)((__nv_bfloat16*)out + (long long)p * a.out.ld + c) =
            *(const uint4*)((const __nv_bfloat16*)fr + q * a.src.fresh.ld + c);
    }
}

// ---- dense group norm in one launch (statistics + normalise + SiLU), bf16 maps, one CTA per
// (group, stacked image): the group's hw x cpg block is read three times from L2 instead of
// a statistics launch followed by a separate apply launch (same arithmetic as the pair)
// One-launch dense GroupNorm (+SiLU) of bf16 maps: a cluster of up to 8 CTAs per (group, image), each
// over a contiguous slice of the image's pixels; the two-pass statistics (sum -> f32 mean, then the
// centred sum of squares) are block-reduced in f64 and combined across the cluster through
// distributed shared memory in rank order (deterministic), then every CTA normalises its slice.
// VW bf16 channels per vector access: 8 (16-byte loads, channels-per-group % 8 == 0) or 2.

FIS_DEV double gn_block_sum(double v, double* red) {
    const int tid = threadIdx.x;
    red[tid] = v;
    __syncthreads();
    for (int o = 128; o; o >>= 1) {
        if (tid < o) red[tid] += red[tid + o];
        __syncthreads();
    }
    const double r = red[0];
    __syncthreads();
    return r;
}

// cluster-wide sum of one double per CTA (slot[0] of every CTA's shared memory, rank order)
FIS_DEV double gn_cluster_sum(double mine, double* slot) {
    if (threadIdx.x == 0) *slot = mine;
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    double s = 0.0;
    const uint32_t a = (uint32_t)__cvta_generic_to_shared(slot);
    uint32_t ncl;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(ncl));
    for (int r = 0; r < (int)ncl; r++) {
        uint32_t ra;
        double v;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(r));
        asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(ra) : "memory");
        s += v;
    }
    return s;
}

template <int VW>
__global__ void __launch_bounds__(256) gn_fused_kernel(const fis_gn_apply_args a) {
    using VT = typename std::conditional<VW == 8, uint4, uint32_t>::type;
    const int ls = ltr_begin(5);
    const int t = cur_step(a.step);  // host-written before the step: read before the wait
    pdl_trigger();
    pdl_wait();
    ltr(ls, 2);
    const int hw = a.img_rows;  // pixels per image (set by fis_gn)
    uint32_t ncl, crank;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(ncl));
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
    const int cl = (int)ncl, rank = (int)crank;
    const int g = blockIdx.x / cl, img = blockIdx.y, tid = threadIdx.x;
    const int cpg = a.c / a.groups, vpg = cpg / VW;
    const int per = (hw + cl - 1) / cl, q0 = min(hw, rank * per), q1 = min(hw, q0 + per);
    const int items = (q1 - q0) * vpg;
    const long long cnt = (long long)hw * cpg;
    const __nv_bfloat16* x = (const __nv_bfloat16*)ref_base(a.x, t) + (long long)(img * hw + q0) * a.x.ld + g * cpg;
    __shared__ double red[256];
    __shared__ double slot[2];
    float ps = 0.f;
    for (int i = tid; i < items; i += blockDim.x) {
        const int q = i / vpg, v = i - q * vpg;
        const VT u = *(const VT*)(x + (long long)q * a.x.ld + v * VW);
        const __nv_bfloat162* h = (const __nv_bfloat162*)&u;
#pragma unroll
        for (int k = 0; k < VW / 2; k++) {
            const float2 f = __bfloat1622float2(h[k]);
            ps += f.x + f.y;
        }
    }
    const float mf = (float)(gn_cluster_sum(gn_block_sum((double)ps, red), slot) / (double)cnt);
    float pv = 0.f;
    for (int i = tid; i < items; i += blockDim.x) {
        const int q = i / vpg, v = i - q * vpg;
        const VT u = *(const VT*)(x + (long long)q * a.x.ld + v * VW);
        const __nv_bfloat162* h = (const __nv_bfloat162*)&u;
#pragma unroll
        for (int k = 0; k < VW / 2; k++) {
            const float2 f = __bfloat1622float2(h[k]);
            const float d0 = f.x - mf, d1 = f.y - mf;
            pv = fmaf(d0, d0, fmaf(d1, d1, pv));
        }
    }
    const float vf = (float)(gn_cluster_sum(gn_block_sum((double)pv, red), slot + 1) / (double)cnt);
    if (tid == 0 && rank == 0) {
        ((float*)ref_base(a.mean, t))[img * a.groups + g] = mf;
        ((float*)ref_base(a.var, t))[img * a.groups + g] = vf;
    }
    const float rstd = (float)(1.0 / sqrt((double)vf + (double)a.eps));
    char* yn = a.y_norm.ptr ? ref_base(a.y_norm, t) : nullptr;
    char* ys = a.y_silu.ptr ? ref_base(a.y_silu, t) : nullptr;
    for (int i = tid; i < items; i += blockDim.x) {
        const int q = i / vpg, v = i - q * vpg;
        const int c = g * cpg + v * VW;
        const long long row = (long long)img * hw + q0 + q;
        const VT u = *(const VT*)(x + (long long)q * a.x.ld + v * VW);
        const __nv_bfloat162* h = (const __nv_bfloat162*)&u;
        VT on, os;
        __nv_bfloat162* hn = (__nv_bfloat162*)&on;
        __nv_bfloat162* hs = (__nv_bfloat162*)&os;
        float ga[VW], be[VW];
#pragma unroll
        for (int k = 0; k < VW; k += 2) {
            *(float2*)(ga + k) = __ldg((const float2*)(a.gamma + c + k));
            *(float2*)(be + k) = __ldg((const float2*)(a.beta + c + k));
        }
#pragma unroll
        for (int k = 0; k < VW / 2; k++) {
            const float2 f = __bfloat1622float2(h[k]);
            const float y0 = fmaf((f.x - mf) * rstd, ga[2 * k], be[2 * k]);
            const float y1 = fmaf((f.y - mf) * rstd, ga[2 * k + 1], be[2 * k + 1]);
            hn[k] = __floats2bfloat162_rn(y0, y1);
            hs[k] = __floats2bfloat162_rn(__fdividef(y0, 1.0f + __expf(-y0)), __fdividef(y1, 1.0f + __expf(-y1)));
        }
        if (yn) *(VT*)((__nv_bfloat16*)yn + row * a.y_norm.ld + c) = on;
        if (ys) *(VT*)((__nv_bfloat16*)ys + row * a.y_silu.ld + c) = os;
    }
    // peers read this CTA's slots: keep its shared memory until the whole cluster is done
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// Dense group norm of stacked images (thousands of (group, image) pairs: no cluster needed): one
// CTA per (image, GW_G groups) instead of per (group, image), so each pixel row contributes one
// contiguous GW_G * cpg-channel run (320 B at c = 1280) rather than an 80-byte fragment, the CTA
// count drops 4x and every thread keeps one 8-channel vector (its gamma / beta in registers).
// Per-thread fp32 partials, reduced in f64 in a fixed order (deterministic); mean first, then
// the centred sum of squares (same two-pass statistics as gn_fused_kernel).
constexpr int GW_G = 4;
__global__ void __launch_bounds__(256) gn_wide_kernel(const fis_gn_apply_args a) {
    const int ls = ltr_begin(5);
    const int t = cur_step(a.step);  // host-written before the step: read before the wait
    pdl_trigger();
    pdl_wait();
    ltr(ls, 2);
    const int hw = a.img_rows, img = blockIdx.y, gb = blockIdx.x * GW_G, tid = threadIdx.x;
    const int cpg = a.c / a.groups, vpg = cpg / 8, vpr = GW_G * vpg, rp = blockDim.x / vpr;
    const int v = tid % vpr, q0 = tid / vpr, gl = v / vpg;
    const int c = gb * cpg + v * 8;
    const long long cnt = (long long)hw * cpg;
    const __nv_bfloat16* x = (const __nv_bfloat16*)ref_base(a.x, t) + (long long)img * hw * a.x.ld + c;
    __shared__ double red[256];
    __shared__ float st[3][GW_G];  // mean, variance, 1 / sqrt(var + eps)
    auto group_sums = [&](float mine, int which) {
        red[tid] = (double)mine;
        __syncthreads();
        if (tid < GW_G) {
            double sum = 0.0;
            for (int q = 0; q < rp; q++)
                for (int w = 0; w < vpg; w++) sum += red[q * vpr + tid * vpg + w];
            st[which][tid] = (float)(sum / (double)cnt);
        }
        __syncthreads();
    };
    // pass 1 stages the CTA's slice (hw x vpr 16-byte vectors) in shared memory when it fits (the
    // host sizes the dynamic allocation), 8 loads in flight per thread; passes 2-3 read it back
    extern __shared__ uint4 xs[];
    const bool staged = a.x_rows == nullptr && (long long)hw * vpr * 16 <= 96 * 1024;
    float ps = 0.f;
    for (int q = q0; q < hw; q += 8 * rp) {
        uint4 u[8];
#pragma unroll
        for (int k = 0; k < 8; k++)
            if (q + k * rp < hw) u[k] = *(const uint4*)(x + (long long)(q + k * rp) * a.x.ld);
#pragma unroll
        for (int k = 0; k < 8; k++) {
            if (q + k * rp >= hw) break;
            if (staged) xs[(q + k * rp) * vpr + v] = u[k];
            const __nv_bfloat162* h = (const __nv_bfloat162*)&u[k];
#pragma unroll
            for (int e2 = 0; e2 < 4; e2++) {
                const float2 f = __bfloat1622float2(h[e2]);
                ps += f.x + f.y;
            }
        }
    }
    group_sums(ps, 0);
    const float mf = st[0][gl];
    float pv = 0.f;
    for (int q = q0; q < hw; q += rp) {
        const uint4 u = staged ? xs[q * vpr + v] : *(const uint4*)(x + (long long)q * a.x.ld);
        const __nv_bfloat162* h = (const __nv_bfloat162*)&u;
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const float2 f = __bfloat1622float2(h[k]);
            const float d0 = f.x - mf, d1 = f.y - mf;
            pv = fmaf(d0, d0, fmaf(d1, d1, pv));
        }
    }
    group_sums(pv, 1);
    if (tid < GW_G) {
        const float vf = st[1][tid];
        ((float*)ref_base(a.mean, t))[img * a.groups + gb + tid] = st[0][tid];
        ((float*)ref_base(a.var, t))[img * a.groups + gb + tid] = vf;
        st[2][tid] = (float)(1.0 / sqrt((double)vf + (double)a.eps));
    }
    __syncthreads();
    const float rstd = st[2][gl];
    float ga[8], be[8];
    *(float4*)ga = __ldg((const float4*)(a.gamma + c));
    *(float4*)(ga + 4) = __ldg((const float4*)(a.gamma + c + 4));
    *(float4*)be = __ldg((const float4*)(a.beta + c));
    *(float4*)(be + 4) = __ldg((const float4*)(a.beta + c + 4));
    char* yn = a.y_norm.ptr ? ref_base(a.y_norm, t) : nullptr;
    char* ys = a.y_silu.ptr ? ref_base(a.y_silu, t) : nullptr;
    for (int q = q0; q < hw; q += rp) {
        const long long row = (long long)img * hw + q;
        const uint4 u = staged ? xs[q * vpr + v] : *(const uint4*)(x + (long long)q * a.x.ld);
        const __nv_bfloat162* h = (const __nv_bfloat162*)&u;
        uint4 on, os;
        __nv_bfloat162* hn = (__nv_bfloat162*)&on;
        __nv_bfloat162* hs = (__nv_bfloat162*)&os;
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const float2 f = __bfloat1622float2(h[k]);
            const float y0 = fmaf((f.x - mf) * rstd, ga[2 * k], be[2 * k]);
            const float y1 = fmaf((f.y - mf) * rstd, ga[2 * k + 1], be[2 * k + 1]);
            hn[k] = __floats2bfloat162_rn(y0, y1);
            hs[k] = __floats2bfloat162_rn(__fdividef(y0, 1.0f + __expf(-y0)), __fdividef(y1, 1.0f + __expf(-y1)));
        }
        if (yn) *(uint4*)((__nv_bfloat16*)yn + row * a.y_norm.ld + c) = on;
        if (ys) *(uint4*)((__nv_bfloat16*)ys + row * a.y_silu.ld + c) = os;
    }
}

static int grid_for(long long total, int threads) {
    long long b = (total + threads - 1) / threads;
    if (b < 1) b = 1;
    if (b > 148 * 16) b = 148 * 16;
    return (int)b;
}

}  // namespace fis


extern "C" int fis_gn_stats(const fis_gn_stats_args* a, void* stream) {
    if (a->groups <= 0 || a->c % a->groups) return FIS_ERR_SHAPE;
    return fis_launch(fis::gn_stats_kernel, dim3(a->groups, a->n_img > 1 ? a->n_img : 1), dim3(256), 0, (cudaStream_t)stream, *a) == cudaSuccess ? FIS_OK : FIS_ERR_LAUNCH;
}

extern "C" int fis_gn_apply(const fis_gn_apply_args* a, void* stream);

// Dense group norm with its own statistics (written to mean/var per image): rows = n_img * img_rows
// (img_rows = 0: one image). bf16 maps with 8 | channels-per-group take the one-launch kernel;
// otherwise statistics + apply are two launches.
// one-launch GN (statistics + normalise per group) for bf16 maps: vector width 8 (16-byte
// accesses) when the channels per group allow, else 2 (bf16 pairs); 0 = two launches
static int gn_vec(const fis_gn_apply_args* a) {
    const int cpg = a->c / a->groups;
    for (int vw = 8; vw >= 2; vw -= 6) {
        if (a->x.dtype == FIS_BF16 && cpg % vw == 0 && (a->x.ld % vw) == 0 &&
            (!a->y_norm.ptr || (a->y_norm.dtype == FIS_BF16 && (a->y_norm.ld % vw) == 0)) &&
            (!a->y_silu.ptr || (a->y_silu.dtype == FIS_BF16 && (a->y_silu.ld % vw) == 0)) &&
            ((((uintptr_t)a->x.ptr) | ((uintptr_t)a->y_norm.ptr) | ((uintptr_t)a->y_silu.ptr)) & (2 * vw - 1)) == 0)
            return vw;
    }
    return 0;
}

// kernel launches one fis_gn call makes (1 fused, or 2: statistics + apply)
extern "C" int fis_gn_launches(const fis_gn_apply_args* a) {
    if (a->groups <= 0 || a->c % a->groups || a->rows == 0) return 0;
    return gn_vec(a) ? 1 : 2;
}

extern "C" int fis_gn(const fis_gn_apply_args* a, void* stream) {
    if (a->groups <= 0 || a->c % a->groups) return FIS_ERR_SHAPE;
    if (a->rows == 0) return FIS_OK;
    const int hw = a->img_rows > 0 ? a->img_rows : a->rows;
    if (a->rows % hw || a->x_rows || a->y_rows || a->row_img) return FIS_ERR_SHAPE;
    const int n_img = a->rows / hw;
    if (const int vw = gn_vec(a)) {
        fis_gn_apply_args ap = *a;
        ap.img_rows = hw;
        // a cluster of 8 CTAs per (group, image) when the (group, image) CTAs alone would leave most SMs
        // idle and the maps are large (r02 C2 dense step: L0 GN 78 -> 22 us, L1 49 -> 16 us); stacked
        // requests already give thousands of CTAs: one per (group, image), no cluster
        const int cl = hw >= 256 && (long long)a->groups * n_img < 148 ? 8 : 1;
        const dim3 grid(a->groups * cl, n_img);
        cudaError_t e;
        const int vpr = fis::GW_G * (a->c / a->groups) / 8;
        static int wide_off = getenv("FIS_GN_WIDE") && getenv("FIS_GN_WIDE")[0] == '0';
        if (!wide_off && cl == 1 && vw == 8 && a->groups % fis::GW_G == 0 && vpr <= 256) {
            // stacked images: one CTA per (image, GW_G groups), rows-per-pass x vectors-per-row threads
            const dim3 g2(a->groups / fis::GW_G, n_img);
            const long long st = (long long)hw * vpr * 16;
            const int smem = st <= 96 * 1024 ? (int)st : 0;
            static bool configured = false;
            if (!configured) {
                cudaFuncSetAttribute(fis::gn_wide_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
                configured = true;
            }
            return fis_launch(fis::gn_wide_kernel, g2, dim3((256 / vpr) * vpr), smem, (cudaStream_t)stream, ap) ==
                           cudaSuccess ? FIS_OK : FIS_ERR_LAUNCH;
        }
        if (cl > 1)
            e = vw == 8 ? fis_launch_cluster(fis::gn_fused_kernel<8>, grid, dim3(256), cl, (cudaStream_t)stream, ap)
                        : fis_launch_cluster(fis::gn_fused_kernel<2>, grid, dim3(256), cl, (cudaStream_t)stream, ap);
        else
            e = vw == 8 ? fis_launch(fis::gn_fused_kernel<8>, grid, dim3(256), 0, (cudaStream_t)stream, ap)
                        : fis_launch(fis::gn_fused_kernel<2>, grid, dim3(256), 0, (cudaStream_t)stream, ap);
        return e == cudaSuccess ? FIS_OK : FIS_ERR_LAUNCH;
    }
    fis_gn_stats_args st = {};
    st.hw = hw; st.c = a->c; st.groups = a->groups; st.x = a->x; st.mean = a->mean; st.var = a->var;
    st.step = a->step; st.n_img = n_img;
    const int rc = fis_gn_stats(&st, stream);
    if (rc != FIS_OK) return rc;
    fis_gn_apply_args ap = *a;
    ap.img_rows = n_img > 1 ? hw : 0;
    return fis_gn_apply(&ap, stream);
}

extern "C" int fis_gn_apply(const fis_gn_apply_args* a, void* stream) {
    if (a->groups <= 0 || a->c % a->groups) return FIS_ERR_SHAPE;
    if (a->rows == 0) return FIS_OK;
    long long total = (long long)a->rows * a->c;
    return fis_launch(fis::gn_apply_kernel, dim3(fis::grid_for(total, 256)), dim3(256), 0, (cudaStream_t)stream, *a) ==
                   cudaSuccess ? FIS_OK : FIS_ERR_LAUNCH;
}

extern "C" int fis_up2(const fis_pool_args* a, void* stream) {
    if (a->n == 0) return FIS_OK;
    if (a->src.index || a->src.fresh.dtype != FIS_BF16 || a->out.dtype != FIS_BF16 || a->c % 8 ||
        (a->src.fresh.ld % 8) || (a->out.ld % 8))
        return FIS_ERR_UNSUPPORTED;
    const long long total = (long long)a->n * (a->c / 8);
    return fis_launch(fis::up2_kernel, dim3(fis::grid_for(total, 256)), dim3(256), 0, (cudaStream_t)stream, *a) ==
                   cudaSuccess ? FIS_OK : FIS_ERR_LAUNCH;
}

extern "C" int fis_softmax(const fis_softmax_args* a, void* stream) {
    if (a->rows == 0) return FIS_OK;
    if (a->pad_cols < a->cols) return FIS_ERR_SHAPE;
    if ((a->verbatim || a->npairs) && !a->cached.ptr) return FIS_ERR_CACHE_MISS;
    const int warps = 8;
    return fis_launch(fis::softmax_kernel, dim3((a->rows + warps - 1) / warps), dim3(warps * 32), 0, (cudaStream_t)stream, *a) == cudaSuccess ? FIS_OK : FIS_ERR_LAUNCH;
}

extern "C" int fis_pool2(const fis_pool_args* a, void* stream) {
    if (a->n == 0) return FIS_OK;
    if (a->src.index && !a->src.cache.ptr) return FIS_ERR_CACHE_MISS;
    long long total = (long long)a->n * a->c;
    return fis_launch(fis::pool2_kernel, dim3(fis::grid_for(total, 256)), dim3(256), 0, (cudaStream_t)stream, *a) ==
                   cudaSuccess ? FIS_OK : FIS_ERR_LAUNCH;
}

extern "C" int fis_materialize(const fis_materialize_args* a, void* stream) {
    if (a->src.index && !a->src.cache.ptr) return FIS_ERR_CACHE_MISS;
    long long total = (long long)a->src.h * a->src.w * a->c;
    return fis_launch(fis::materialize_kernel, dim3(fis::grid_for(total, 256)), dim3(256), 0, (cudaStream_t)stream, *a) ==
                   cudaSuccess ? FIS_OK : FIS_ERR_LAUNCH;
}

FIS_LTR_SETTER(fis_ltr_set_ops)
