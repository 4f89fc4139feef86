// tcgen05 (5th-gen tensor core) bf16 gather-GEMM — placeholder until the
// sm_100a kernel lands; reports "unsupported" so dispatch uses the SIMT path.
#include "fis_common.cuh"

int fis_gemm_tc_supported(const fis_gemm_args*) { return 0; }

int fis_gemm_tc_launch(const fis_gemm_args*, cudaStream_t) { return FIS_ERR_UNSUPPORTED; }
