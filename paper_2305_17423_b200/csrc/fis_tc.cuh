// tcgen05 / cp.async / UMMA-descriptor helpers and the fused GEMM row epilogue shared by
// tcgen05 GEMM / conv kernels (fis_gemm_tc.cu, fis_gemm_big.cu, fis_gemm_pair.cu, fis_gemm_halo.cu).
#pragma once
#include "fis_common.cuh"
#include <climits>

namespace fis {
namespace tc {

constexpr int BM = 128, BK = 64;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(valid ? 16 : 0) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t* b) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(b)) : "memory");
}
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// L2 prefetch of one TMA box (no shared-memory destination, no completion): issued for operands
// that no kernel of the step writes (weights, per-edit text K/V) BEFORE griddepcontrol.wait, so
// their HBM latency overlaps the previous kernel and the main loop streams them from L2
__device__ __forceinline__ void tma_prefetch2d(const void* tmap, int c0, int c1) {
    asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(tmap), "r"(c0), "r"(c1)
                 : "memory");
}

// K-major, 128B-swizzled UMMA shared-memory descriptor (LBO=16B, SBO=1024B, version 1)
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

// byte offset of 16B chunk j of row r inside a SW128 K-major tile (rows of 128 B)
__device__ __forceinline__ uint32_t sw128_off(int r, int j) {
    return (uint32_t)((r >> 3) * 1024 + (r & 7) * 128 + ((j ^ (r & 7)) << 4));
}


// Per-column epilogue parameters of this CTA's BN columns, staged once in shared memory.
struct EpiTab {
    float* bias; float* b2; float* gamma; float* beta; float* mean; float* rstd;
};

__device__ __forceinline__ void load_row16(const char* base, int dtype, long long off, int nvalid, float* v) {
    if (dtype == FIS_BF16) {
        const __nv_bfloat16* p = (const __nv_bfloat16*)base + off;
        if (nvalid == 16 && ((uintptr_t)p & 15) == 0) {
#pragma unroll
            for (int q = 0; q < 2; q++) {
                uint4 u = FIS_LD_U4(p + 8 * q);
                const __nv_bfloat162* h = (const __nv_bfloat162*)&u;
#pragma unroll
                for (int k = 0; k < 4; k++) {
                    float2 f = __bfloat1622float2(h[k]);
                    v[8 * q + 2 * k] = f.x;
                    v[8 * q + 2 * k + 1] = f.y;
                }
            }
        } else {
#pragma unroll
            for (int j = 0; j < 16; j++) if (j < nvalid) v[j] = load_elem((const char*)p, FIS_BF16, j);
        }
    } else {
        const float* p = (const float*)base + off;
        if (nvalid == 16 && ((uintptr_t)p & 15) == 0) {
#pragma unroll
            for (int q = 0; q < 4; q++) {
                float4 f = FIS_LD_F4(p + 4 * q);
                v[4 * q] = f.x; v[4 * q + 1] = f.y; v[4 * q + 2] = f.z; v[4 * q + 3] = f.w;
            }
        } else {
#pragma unroll
            for (int j = 0; j < 16; j++) if (j < nvalid) v[j] = load_elem((const char*)p, FIS_F32, j);
        }
    }
}

__device__ __forceinline__ void store_row16(char* base, int dtype, long long off, int nvalid, const float* v) {
    if (dtype == FIS_BF16) {
        __nv_bfloat16* p = (__nv_bfloat16*)base + off;
        if (nvalid == 16 && ((uintptr_t)p & 15) == 0) {
#pragma unroll
            for (int q = 0; q < 2; q++) {
                uint4 u;
                __nv_bfloat162* h = (__nv_bfloat162*)&u;
#pragma unroll
                for (int k = 0; k < 4; k++) h[k] = __floats2bfloat162_rn(v[8 * q + 2 * k], v[8 * q + 2 * k + 1]);
                *(uint4*)(p + 8 * q) = u;
            }
        } else {
#pragma unroll
            for (int j = 0; j < 16; j++) if (j < nvalid) p[j] = __float2bfloat16_rn(v[j]);
        }
    } else {
        float* p = (float*)base + off;
        if (nvalid == 16 && ((uintptr_t)p & 15) == 0) {
#pragma unroll
            for (int q = 0; q < 4; q++) *(float4*)(p + 4 * q) = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        } else {
#pragma unroll
            for (int j = 0; j < 16; j++) if (j < nvalid) p[j] = v[j];
        }
    }
}

// Fused epilogue of one 16-column chunk of one output row (v holds the fp32 accumulators).
// Same arithmetic, in the same order, as fis::epilogue_store (fis_common.cuh).
template <int MODE>
__device__ __forceinline__ void row_epilogue(const fis_gemm_args& a, const EpiCtx& e, const EpiTab& tb, int r,
                                             int c0, int n0, float* v) {
    const int n = n0 + c0;
    const int nvalid = min(16, a.n - n);
    if (nvalid <= 0) return;
    const int orow = a.d_rows ? __ldg(a.d_rows + r) : r;
    if (orow < 0) return;  // a framing row of a halo-mode conv: computed, not stored
#pragma unroll
    for (int j = 0; j < 16; j++) v[j] = __fadd_rn(v[j] * a.alpha, tb.bias[c0 + j]);
    if (e.pre) store_row16(e.pre, a.pre.dtype, (long long)orow * a.pre.ld + n, nvalid, v);
    if (e.bias2) {
#pragma unroll
        for (int j = 0; j < 16; j++) v[j] = __fadd_rn(v[j], tb.b2[c0 + j]);
    }
    if (MODE == FIS_EPI_GN_SILU) {
        float y[16];
#pragma unroll
        // bf16 tensor-core path: cached-stat GN + SiLU in fp32 (the fp32-parity SIMT path,
        // epilogue_store, keeps the reference's f64 arithmetic)
        for (int j = 0; j < 16; j++)
            y[j] = fmaf(v[j], tb.mean[c0 + j], tb.rstd[c0 + j]);  // tables hold GN scale / shift
        if (e.pre2) store_row16(e.pre2, a.pre2.dtype, (long long)orow * a.pre2.ld + n, nvalid, y);
#pragma unroll
        for (int j = 0; j < 16; j++) v[j] = __fdividef(y[j], 1.0f + __expf(-y[j]));
    } else if (MODE == FIS_EPI_STEP) {
        float l[16];
        load_row16(e.lat, a.lat.dtype, (long long)orow * a.lat.ld + n, nvalid, l);
#pragma unroll
        for (int j = 0; j < 16; j++) v[j] = __fsub_rn(l[j], __fmul_rn(a.step_scale, v[j]));
    }
    if (e.res) {
        float q[16];
        load_row16(e.res, a.res.dtype, (long long)orow * a.res.ld + n, nvalid, q);
#pragma unroll
        for (int j = 0; j < 16; j++) v[j] = __fadd_rn(v[j], q[j]);
    }
    char* dbase = e.d;
    int dt = a.d.dtype, dld = a.d.ld, dn = n, trans = a.d_trans;
    if (a.n_split > 0 && n >= a.n_split) {  // fused QKV: V part goes transposed to d2
        dbase = e.d2; dt = a.d2.dtype; dld = a.d2.ld; dn = n - a.n_split; trans = a.d2_trans;
    }
    if (trans) {
#pragma unroll
        for (int j = 0; j < 16; j++)
            if (j < nvalid) store_elem(dbase, dt, (long long)(dn + j) * dld + orow, v[j]);
    } else {
        store_row16(dbase, dt, (long long)orow * dld + dn, nvalid, v);
    }
}

__device__ __forceinline__ void row_epilogue_any(const fis_gemm_args& a, const EpiCtx& e, const EpiTab& tb, int r,
                                                 int c0, int n0, float* v) {
    if (a.epi == FIS_EPI_GN_SILU) row_epilogue<FIS_EPI_GN_SILU>(a, e, tb, r, c0, n0, v);
    else if (a.epi == FIS_EPI_STEP) row_epilogue<FIS_EPI_STEP>(a, e, tb, r, c0, n0, v);
    else row_epilogue<FIS_EPI_NONE>(a, e, tb, r, c0, n0, v);
}

// Per-row gather geometry, computed once per CTA: the row's pixel p (ROWS: A row) and,
// for CONV, its (y, x); valid=false rows (beyond M) load zeros.
struct RowGeo {
    int p, oy, ox;
    bool valid;
};

constexpr int SEL_ZERO = INT_MIN;

// Select-on-read decisions of one output row for every 3x3 tap of source segment `seg`:
// >= 0 fresh row (or full-map pixel), <= -2 cache pixel (-2 - q), SEL_ZERO = zero padding.
__device__ __forceinline__ void build_sel(const fis_gemm_args& a, int p, int seg, int* out9) {
    const fis_src& s = a.src[seg];
    if (p < 0) {  // framing row at the image border (halo-mode rows): zeros
#pragma unroll
        for (int tap = 0; tap < 9; tap++) out9[tap] = SEL_ZERO;
        return;
    }
    // pixels of several stacked images (batched requests): image = p / (out_h * out_w); taps never
    // cross an image border; the source pixel is offset by the image's h * w source pixels
    const int ipx = a.out_h * a.out_w;
    const int img = p / ipx, lp = p - img * ipx;
    const int oy = lp / a.out_w, ox = lp - (lp / a.out_w) * a.out_w;
    const int qimg = img * s.h * s.w;
#pragma unroll
    for (int tap = 0; tap < 9; tap++) {
        const int y = oy + tap / 3 - 1, x = ox + tap % 3 - 1;
        int v = SEL_ZERO;
        if (y >= 0 && x >= 0 && y < a.out_h && x < a.out_w) {
            const int q = qimg + (s.up ? (y >> 1) : y) * s.w + (s.up ? (x >> 1) : x);
            if (s.index) {
                const int i = __ldg(s.index + q);
                v = i >= 0 ? i : -2 - q;
            } else {
                v = q;
            }
        }
        out9[tap] = v;
    }
}

}  // namespace tc
}  // namespace fis
