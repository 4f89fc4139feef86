// Shared device helpers for libfisedit (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include "../../include/fisedit.h"

#define FIS_DEV __device__ __forceinline__

namespace fis {

// Programmatic dependent launch: every kernel is launched with programmatic stream
// serialization; it lets its own dependents launch immediately (they are only scheduled
// once all of this grid's CTAs are resident) and waits for its predecessor's memory
// before touching global data. Inside a captured CUDA graph this overlaps each kernel's
// launch + prologue with the previous kernel's tail.
FIS_DEV void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
FIS_DEV void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

FIS_DEV int cur_step(const int* step) { return step ? __ldg(step) : 0; }

// Launch trace (profiling builds only: `python -m paper_2305_17423_b200.build --trace` compiles with
// FIS_TRACE into libfisedit_trace.so, loaded with FIS_LIB=libfisedit_trace.so). CTA (0,0,0) of every
// kernel takes the next slot of the installed buffer (atomic counter at buf[0]) and records
// %globaltimer phase stamps at buf[16 + 16 * slot + phase]; phase 15 = kernel kind. Production builds
// compile every probe to nothing: each probe is a dependent global load on the issuing thread's path.
static __device__ unsigned long long* g_ltr = nullptr;
FIS_DEV unsigned long long ltr_now() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#ifdef FIS_TRACE
FIS_DEV int ltr_begin(int kind) {
    unsigned long long* b = g_ltr;
    if (!b || (blockIdx.x | blockIdx.y | blockIdx.z) || threadIdx.x) return -1;
    const unsigned long long t = ltr_now();
    const int s = (int)atomicAdd(b, 1ull);
    if (s >= 4096) return -1;
    b[16 + 16 * s] = t;
    b[16 + 16 * s + 15] = (unsigned long long)kind;
    return s;
}
FIS_DEV void ltr(int slot, int phase) {
    if (slot >= 0) g_ltr[16 + 16 * slot + phase] = ltr_now();
}
#else
FIS_DEV int ltr_begin(int) { return -1; }
FIS_DEV void ltr(int, int) {}
#endif
#ifdef FIS_TRACE
#define FIS_LTR_SETTER(fn) \
    extern "C" int fn(unsigned long long* p) { return cudaMemcpyToSymbol(fis::g_ltr, &p, sizeof(p)) == cudaSuccess ? 0 : 1; }
#else
#define FIS_LTR_SETTER(fn) \
    extern "C" int fn(unsigned long long*) { return FIS_ERR_UNSUPPORTED; }
#endif

FIS_DEV char* ref_base(const fis_ref& r, int t) {
    return (char*)r.ptr + (long long)t * r.step_stride;
}

#define FIS_LD_U16(p) (*(const unsigned short*)(p))
#define FIS_LD_F32(p) (*(const float*)(p))
#define FIS_LD_U4(p) (*(const uint4*)(p))
#define FIS_LD_F4(p) (*(const float4*)(p))

FIS_DEV float load_elem(const char* base, int dtype, long long idx) {
    if (dtype == FIS_BF16) return __uint_as_float((uint32_t)FIS_LD_U16((const __nv_bfloat16*)base + idx) << 16);
    return FIS_LD_F32((const float*)base + idx);
}

FIS_DEV void store_elem(char* base, int dtype, long long idx, float v) {
    if (dtype == FIS_BF16) ((__nv_bfloat16*)base)[idx] = __float2bfloat16_rn(v);
    else ((float*)base)[idx] = v;
}

// Value of a selectable source at source pixel q, channel c (select-on-read).
FIS_DEV float src_value(const fis_src& s, const char* fresh, const char* cache, int q, int c) {
    if (s.index) {
        int i = __ldg(s.index + q);
        if (i >= 0) return load_elem(fresh, s.fresh.dtype, (long long)i * s.fresh.ld + c);
        return load_elem(cache, s.cache.dtype, (long long)q * s.cache.ld + c);
    }
    return load_elem(fresh, s.fresh.dtype, (long long)q * s.fresh.ld + c);
}

// Source row pointer (and dtype/ld) for pixel q, used by vectorised gathers.
struct RowPtr { const char* p; int dtype; };
FIS_DEV RowPtr src_row(const fis_src& s, const char* fresh, const char* cache, int q) {
    if (s.index) {
        int i = __ldg(s.index + q);
        if (i >= 0) return {fresh + (long long)i * s.fresh.ld * (s.fresh.dtype == FIS_BF16 ? 2 : 4), s.fresh.dtype};
        return {cache + (long long)q * s.cache.ld * (s.cache.dtype == FIS_BF16 ? 2 : 4), s.cache.dtype};
    }
    return {fresh + (long long)q * s.fresh.ld * (s.fresh.dtype == FIS_BF16 ? 2 : 4), s.fresh.dtype};
}

FIS_DEV float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
FIS_DEV float warp_max(float v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Epilogue shared by the SIMT and tcgen05 GEMMs. Applies bias / time-bias /
// GN(cached stats)+SiLU / step update / residual and stores. r = GEMM row.
struct EpiCtx {
    char* d2;
    char* d; char* pre; char* pre2; char* res; char* lat; char* bias2;
    const float* mean; const float* var;
    int cpg;  // channels per group
};

FIS_DEV EpiCtx make_epi(const fis_gemm_args& a, int t) {
    EpiCtx e;
    e.d = ref_base(a.d, t);
    e.d2 = a.d2.ptr ? ref_base(a.d2, t) : nullptr;
    e.pre = a.pre.ptr ? ref_base(a.pre, t) : nullptr;
    e.pre2 = a.pre2.ptr ? ref_base(a.pre2, t) : nullptr;
    e.res = a.res.ptr ? ref_base(a.res, t) : nullptr;
    e.lat = a.lat.ptr ? ref_base(a.lat, t) : nullptr;
    e.bias2 = a.bias2.ptr ? ref_base(a.bias2, t) : nullptr;
    e.mean = a.gn_mean.ptr ? (const float*)ref_base(a.gn_mean, t) : nullptr;
    e.var = a.gn_var.ptr ? (const float*)ref_base(a.gn_var, t) : nullptr;
    e.cpg = a.groups > 0 ? a.n / a.groups : 1;
    return e;
}

FIS_DEV void epilogue_store(const fis_gemm_args& a, const EpiCtx& e, int r, int n, float acc) {
    float v = acc * a.alpha;
    if (a.bias) v = __fadd_rn(v, __ldg(a.bias + n));
    const int orow = a.d_rows ? __ldg(a.d_rows + r) : r;
    if (orow < 0) return;  // framing row of a halo-mode conv
    if (e.pre) store_elem(e.pre, a.pre.dtype, (long long)orow * a.pre.ld + n, v);
    if (e.bias2) v = __fadd_rn(v, load_elem(e.bias2, a.bias2.dtype, n));
    if (a.epi == FIS_EPI_GN_SILU) {
        // normalize_with_group_stats (tensors.py:149-180) in f64, then SiLU in f64 (unet.py:291-293)
        const int g = n / e.cpg;
        const double y64 = ((double)v - (double)e.mean[g]) / sqrt((double)e.var[g] + (double)a.eps) *
                               (double)__ldg(a.gamma + n) + (double)__ldg(a.beta + n);
        const float y = (float)y64;
        if (e.pre2) store_elem(e.pre2, a.pre2.dtype, (long long)orow * a.pre2.ld + n, y);
        const double yd = (double)y;
        v = (float)(yd / (1.0 + exp(-yd)));
    } else if (a.epi == FIS_EPI_STEP) {
        const float l = load_elem(e.lat, a.lat.dtype, (long long)orow * a.lat.ld + n);
        v = __fsub_rn(l, __fmul_rn(a.step_scale, v));
    }
    if (e.res) v = __fadd_rn(v, load_elem(e.res, a.res.dtype, (long long)orow * a.res.ld + n));
    if (a.n_split > 0 && n >= a.n_split) {
        const int n2 = n - a.n_split;
        if (a.d2_trans) store_elem(e.d2, a.d2.dtype, (long long)n2 * a.d2.ld + orow, v);
        else store_elem(e.d2, a.d2.dtype, (long long)orow * a.d2.ld + n2, v);
        return;
    }
    if (a.d_trans) store_elem(e.d, a.d.dtype, (long long)n * a.d.ld + orow, v);
    else store_elem(e.d, a.d.dtype, (long long)orow * a.d.ld + n, v);
}

}  // namespace fis

#include <stdlib.h>
// Launch with the PDL attribute (FIS_PDL=0 in the environment disables it).
inline bool fis_pdl_enabled() {
    static int on = -1;
    if (on < 0) {
        const char* e = getenv("FIS_PDL");
        on = (e && e[0] == '0') ? 0 : 1;
    }
    return on == 1;
}

template <typename Arg>
inline cudaError_t fis_launch(void (*kernel)(Arg), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                              const Arg& arg) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = fis_pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, arg);
}

// the same with a thread-block cluster of cl CTAs along x
template <typename Arg>
inline cudaError_t fis_launch_cluster(void (*kernel)(Arg), dim3 grid, dim3 block, int cl, cudaStream_t stream,
                                      const Arg& arg) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cl;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = fis_pdl_enabled() ? 2 : 1;
    return cudaLaunchKernelEx(&cfg, kernel, arg);
}
