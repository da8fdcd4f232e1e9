// tma_host.h — host-side TMA tensor-map encoding shared by the tensor-core kernels.
// The encoder comes from the driver via cudaGetDriverEntryPoint, so the library needs
// no -lcuda and still loads on a GPU-less host.
#pragma once

#include <cuda.h>  // CUtensorMap / enums only
#include <cuda_runtime.h>

#include <string>

#include "hc_internal.h"
#include "hc_launch.cuh"

namespace hcb {

using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline EncodeTiled tma_encoder() {
    static EncodeTiled fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        cuda_check(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q),
                   "cudaGetDriverEntryPoint(cuTensorMapEncodeTiled)");
        if (!p || q != cudaDriverEntryPointSuccess) throw cuda_error("cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<EncodeTiled>(p);
    }
    return fn;
}

}  // namespace hcb
