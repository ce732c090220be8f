// tma_host.cu -- host-side TMA tensor-map construction (driver entry point
// fetched through the runtime, so the library does not link libcuda).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <mutex>

#include "tma_host.h"

namespace rgo {

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

bool make_tmap(CUtensorMap* map, const void* base, CUtensorMapDataType dtype, uint32_t rank,
               const uint64_t* dims, const uint64_t* strides_bytes, const uint32_t* box,
               CUtensorMapSwizzle swizzle) {
    auto fn = encode_fn();
    if (!fn) return false;
    // The driver encoder needs a current context; a host thread that has not
    // touched the runtime yet (torch's autograd workers, user threads) has
    // none until the runtime binds the device's primary context.
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaSetDevice(dev) != cudaSuccess) return false;
    cuuint32_t elem_strides[5] = {1, 1, 1, 1, 1};
    cuuint64_t d[5], s[4];
    cuuint32_t b[5];
    for (uint32_t i = 0; i < rank; ++i) {
        d[i] = dims[i];
        b[i] = box[i];
        if (i + 1 < rank) s[i] = strides_bytes[i];
    }
    CUresult r = fn(map, dtype, rank, const_cast<void*>(base), d, s, b, elem_strides,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

}  // namespace rgo
