// C-ABI entry points of libfisedit.so that are not defined next to their kernels.
#include "fis_common.cuh"

int fis_gemm_simt_launch(const fis_gemm_args* a, cudaStream_t stream);
int fis_gemm_tc_launch(const fis_gemm_args* a, cudaStream_t stream);
int fis_gemm_tc_supported(const fis_gemm_args* a);
int fis_gemm_tc_choose_splits(int m, int n, int k);
int fis_gemm_tf32_supported(const fis_gemm_args* a);
int fis_gemm_tf32_choose_splits(int m, int n, int k);
int fis_gemm_tf32_launch(const fis_gemm_args* a, cudaStream_t stream);
int fis_gemm_halo_ok(const fis_gemm_args* a);
int fis_gemm_halo_launch(const fis_gemm_args* a, cudaStream_t stream);
int fis_gemm_big_eligible(const fis_gemm_args* a);
int fis_gemm_big_launch(const fis_gemm_args* a, cudaStream_t stream);
int fis_conv_small_ok(const fis_gemm_args* a);
int fis_gemm_pair_ok(const fis_gemm_args* a, int single_bn);
int fis_gemm_pair_launch(const fis_gemm_args* a, cudaStream_t stream);
int fis_gemm_big_bn(int n);
int fis_conv_small_launch(const fis_gemm_args* a, cudaStream_t stream);

extern "C" {
int fis_ltr_set_tc(unsigned long long* p);
int fis_ltr_set_attn(unsigned long long* p);
int fis_ltr_set_simt(unsigned long long* p);
int fis_ltr_set_ops(unsigned long long* p);
int fis_ltr_set_big(unsigned long long* p);
int fis_ltr_set_small(unsigned long long* p);
int fis_ltr_set_pair(unsigned long long* p);
int fis_ltr_set_short(unsigned long long* p);

int fis_trace_launches(unsigned long long* buf) {
    return fis_ltr_set_tc(buf) | fis_ltr_set_attn(buf) | fis_ltr_set_simt(buf) | fis_ltr_set_ops(buf) |
           fis_ltr_set_big(buf) | fis_ltr_set_small(buf) | fis_ltr_set_pair(buf) |
           fis_ltr_set_short(buf);
}

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

static int sm_count_cached(void) {
    static int n = 0;
    if (n <= 0) n = fis_device_sm_count();
    return n > 0 ? n : 148;
}

// Split-K so that the grid covers the SMs once (tcgen05: 1 CTA/SM, 128xBN tiles, 64-wide K
// blocks; SIMT: 64x64 tiles, 16-wide K tiles), keeping >= 4 K blocks per split and
// bounded by the workspace capacity.
static int fis_choose_splits(const fis_gemm_args* a, bool tc) {
    const int sms = sm_count_cached();
    long long tiles, kb;
    int minper, target;
    if (tc) {
        // split-K CTAs form one thread-block cluster per tile (DSMEM reduction, no workspace);
        // S is the largest cluster size whose clusters all fit in one wave
        return fis_gemm_tc_choose_splits(a->m, a->n, a->k);
    } else {
        tiles = (long long)((a->m + 63) / 64) * ((a->n + 63) / 64);
        kb = (a->k + 15) / 16;
        minper = 16;
        target = 2 * sms;
    }
    long long s = target / (tiles > 0 ? tiles : 1);
    if (s > kb / minper) s = kb / minper;
    if (s > 32) s = 32;
    if (s < 2) return 1;
    while (s > 1 && (long long)s * a->m * a->n > a->ws_floats) s--;
    // no empty splits: round so every split gets ceil(kb/s) blocks
    const long long per = (kb + s - 1) / s;
    s = (kb + per - 1) / per;
    return (int)(s < 1 ? 1 : s);
}

// Which kernel fis_gemm would run for these arguments: 0 SIMT, 1 per-op tcgen05, 2 persistent
// large-M tcgen05 (csrc/fis_gemm_big.cu), 3 per-op tcgen05 3xTF32 (fp32 operands), 4 halo-staged
// persistent gather conv (csrc/fis_gemm_halo.cu), 5 few-input-channel 3x3 conv on the FMA pipes
// (csrc/fis_conv_small.cu), 6 persistent 2-SM (CTA pair, cta_group::2) GEMM with TMA-staged A
// (csrc/fis_gemm_pair.cu). Host-only query (no launch).
int fis_gemm_kernel_kind(const fis_gemm_args* a) {
    if (a->impl == 3) return fis_gemm_tf32_supported(a) ? 3 : 0;
    if (a->impl == 0 && fis_conv_small_ok(a)) return 5;
    if (a->impl == 0 && fis_gemm_halo_ok(a)) return 4;
    const bool tc = a->impl == 2 || (a->impl == 0 && fis_gemm_tc_supported(a));
    if (!tc) return 0;
    if (a->impl == 0 && fis_gemm_big_eligible(a)) return fis_gemm_pair_ok(a, fis_gemm_big_bn(a->n)) ? 6 : 2;
    return 1;
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
    const bool tc = a->impl == 2 || (a->impl == 0 && fis_gemm_tc_supported(a));
    // the latent stem conv (C_in = 4): FMA pipes, weights and taps staged once per 64 rows
    if (a->impl == 0 && fis_conv_small_ok(a)) {
        const int rc = fis_conv_small_launch(a, (cudaStream_t)stream);
        if (rc != FIS_ERR_UNSUPPORTED) return rc;
    }
    // halo-mode gathered convs of the stacked step: staged once per kernel row (fis_gemm_halo.cu)
    if (a->impl == 0 && fis_gemm_halo_ok(a)) {
        const int rc = fis_gemm_halo_launch(a, (cudaStream_t)stream);
        if (rc != FIS_ERR_UNSUPPORTED) return rc;
    }
    // large M (stacked requests): persistent tcgen05 kernel with TMA weights (fis_gemm_big.cu)
    if (tc && a->impl == 0 && fis_gemm_big_eligible(a)) {
        if (fis_gemm_pair_ok(a, fis_gemm_big_bn(a->n))) {  // 2-SM tiles: half the B traffic per SM
            const int rc = fis_gemm_pair_launch(a, (cudaStream_t)stream);
            if (rc != FIS_ERR_UNSUPPORTED) return rc;
        }
        const int rc = fis_gemm_big_launch(a, (cudaStream_t)stream);
        if (rc != FIS_ERR_UNSUPPORTED) return rc;
    }
    fis_gemm_args g = *a;
    if (a->impl == 3 && fis_gemm_tf32_supported(a)) {  // fp32 operands on the tensor cores (3xTF32)
        if (g.splits <= 0) g.splits = fis_gemm_tf32_choose_splits(a->m, a->n, a->k);
        return fis_gemm_tf32_launch(&g, (cudaStream_t)stream);
    }
    if (g.splits <= 0) g.splits = fis_choose_splits(&g, tc);
    if (!tc && g.splits > 1 && (!g.ws || !g.counters)) return FIS_ERR_SHAPE;
    return tc ? fis_gemm_tc_launch(&g, (cudaStream_t)stream) : fis_gemm_simt_launch(&g, (cudaStream_t)stream);
}

}  // extern "C"
