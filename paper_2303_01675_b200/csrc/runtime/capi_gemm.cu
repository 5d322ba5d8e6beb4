// C-ABI entry points for the GEMM kernel and the error channel.
#include <cuda_runtime.h>

#include <string>

#include "../../../include/ptk.h"
#include "../kernels/gemm_sm100.h"
#include "errors.h"

extern "C" int ptk_gemm(const ptk_gemm_desc* desc, void* stream) {
    if (desc == nullptr) return ptk::set_error(PTK_ERR_ARG, "ptk_gemm: null descriptor");
    ptk::GemmPlan plan;
    int rc = ptk::gemm_prepare(*desc, &plan);
    if (rc != PTK_OK) return ptk::set_error(rc, "ptk_gemm: prepare failed (shape/alignment)");
    rc = ptk::gemm_run(plan, static_cast<cudaStream_t>(stream));
    if (rc != PTK_OK) return ptk::set_error(rc, std::string("ptk_gemm: launch failed: ") +
                                                     cudaGetErrorString(cudaGetLastError()));
    return PTK_OK;
}
