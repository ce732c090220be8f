// gemm_inst_1.cu -- explicit instantiations of the CTA-pair GEMM (gemm_sm100.cuh).
#include "gemm_sm100.cuh"

namespace rgo_gk {
RGO_GEMM_VARIANT(true, EPI_SWIGLU, OUT_E4M3)
RGO_GEMM_VARIANT(true, EPI_SWIGLU, OUT_BF16)
}  // namespace rgo_gk
