// C-ABI entry points of libfisedit.so that are not defined next to their kernels.
#include "fis_common.cuh"

int fis_gemm_simt_launch(const fis_gemm_args* a, cudaStream_t stream);
int fis_gemm_tc_launch(const fis_gemm_args* a, cudaStream_t stream);
int fis_gemm_tc_supported(const fis_gemm_args* a);

extern "C" {

int fis_abi_version(void) { return FIS_ABI_VERSION; }

const char* fis_last_error(void) { return cudaGetErrorString(cudaPeekAtLastError()); }

int fis_device_sm_count(void) {
    int dev = 0, n = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return -1;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
    return n;
}

long long fis_gemm_ws_floats(int m, int n, int splits) { return splits > 1 ? (long long)splits * m * n : 0; }

int fis_gemm_counters(int m, int n) {
    // enough for the smallest tile shape of either implementation (64x16)
    return ((m + 63) / 64) * ((n + 15) / 16);
}

int fis_gemm(const fis_gemm_args* a, void* stream) {
    if (a->m < 0 || a->n <= 0 || a->k <= 0) return FIS_ERR_SHAPE;
    if (a->m == 0) return FIS_OK;
    if (a->a_mode == FIS_A_CONV3X3) {
        if (a->nsrc < 1 || a->nsrc > 2) return FIS_ERR_SHAPE;
        const int cin = a->src[0].c + (a->nsrc > 1 ? a->src[1].c : 0);
        if (a->k != 9 * cin) return FIS_ERR_SHAPE;
        for (int i = 0; i < a->nsrc; i++)
            if (a->src[i].index && !a->src[i].cache.ptr) return FIS_ERR_CACHE_MISS;
    } else if (a->a_mode != FIS_A_ROWS) {
        return FIS_ERR_UNSUPPORTED;
    }
    if (a->epi == FIS_EPI_GN_SILU && (a->groups <= 0 || a->n % a->groups || !a->gn_mean.ptr || !a->gn_var.ptr))
        return a->gn_mean.ptr ? FIS_ERR_SHAPE : FIS_ERR_CACHE_MISS;
    if (a->splits > 1 && (!a->ws || !a->counters)) return FIS_ERR_SHAPE;
    if (a->impl == 2 || (a->impl == 0 && fis_gemm_tc_supported(a)))
        return fis_gemm_tc_launch(a, (cudaStream_t)stream);
    return fis_gemm_simt_launch(a, (cudaStream_t)stream);
}

}  // extern "C"
