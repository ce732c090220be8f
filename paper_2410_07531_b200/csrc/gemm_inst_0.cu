// gemm_inst_0.cu -- explicit instantiations of the CTA-pair GEMM (gemm_sm100.cuh).
#include "gemm_sm100.cuh"

namespace rgo_gk {
RGO_GEMM_VARIANT(true, EPI_NONE, OUT_BF16)
RGO_GEMM_VARIANT(true, EPI_NONE, OUT_E4M3)
}  // namespace rgo_gk
