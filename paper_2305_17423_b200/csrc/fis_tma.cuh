// Host-side TMA tensor-map encoding shared by the step VM and the persistent GEMM.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstring>
#include <stdint.h>

// cuTensorMapEncodeTiled resolved through the runtime (no link-time libcuda dependency: the
// library must load on hosts without a driver; there the plan simply uses no TMA)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static inline EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (EncodeTiledFn)p;
        cudaGetLastError();
    }
    return fn;
}

// 2D bf16 tensor map [rows][cols] (row stride ld elements), box {64, box_rows}, 128-byte swizzle,
// zero fill outside the matrix.  false when TMA cannot address it.
static inline bool encode_2d(void* out128, const void* base, long long rows, long long cols, long long ld, int box_rows) {
    if (!base || rows <= 0 || cols <= 0 || (((uintptr_t)base) & 15) || ((ld * 2) % 16) || ld < cols) return false;
    CUtensorMap m;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)(ld * 2)};
    cuuint32_t box[2] = {64u, (cuuint32_t)box_rows};
    cuuint32_t es[2] = {1u, 1u};
    EncodeTiledFn enc = encode_fn();
    if (!enc) return false;
    const CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                                              strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return false;
    std::memcpy(out128, &m, 128);
    return true;
}


// 2D bf16 tensor map with 32-column boxes {32, box_rows} and 64-byte swizzle (epilogue tiles whose
// width is a multiple of 32 columns; row r's 16-byte chunk j sits at chunk j ^ ((r >> 1) & 3)).
static inline bool encode_2d_sw64(void* out128, const void* base, long long rows, long long cols, long long ld,
                                  int box_rows) {
    if (!base || rows <= 0 || cols <= 0 || (((uintptr_t)base) & 15) || ((ld * 2) % 16) || ld < cols) return false;
    CUtensorMap m;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)(ld * 2)};
    cuuint32_t box[2] = {32u, (cuuint32_t)box_rows};
    cuuint32_t es[2] = {1u, 1u};
    EncodeTiledFn enc = encode_fn();
    if (!enc) return false;
    const CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return false;
    std::memcpy(out128, &m, 128);
    return true;
}
