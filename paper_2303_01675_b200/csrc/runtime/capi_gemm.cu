// C-ABI entry points for the GEMM kernel and the error channel.
#include <cuda_runtime.h>

#include <string>

#include "../../../include/ptk.h"
#include "../kernels/attention_sm100.h"
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

extern "C" int ptk_gemm_plan_info(const ptk_gemm_desc* desc, int* info) {
    if (desc == nullptr || info == nullptr) return ptk::set_error(PTK_ERR_ARG, "ptk_gemm_plan_info: null argument");
    ptk::GemmPlan plan;
    const int rc = ptk::gemm_prepare(*desc, &plan);
    if (rc != PTK_OK) return ptk::set_error(rc, "ptk_gemm_plan_info: prepare failed (shape/alignment)");
    info[0] = plan.args.bn;
    info[1] = plan.grid;
    info[2] = plan.args.num_tiles;
    info[3] = plan.multicast ? 1 : 0;
    return PTK_OK;
}

extern "C" int ptk_flash_forward(const void* qkv, void* o, float* lse, int b, int s, int H, int d, int causal,
                                 void* stream) {
    ptk::FlashPlan p;
    cudaError_t e = ptk::flash_prepare(qkv, o, lse, b, s, H, d, &p, causal);
    if (e != cudaSuccess) return ptk::set_error(PTK_ERR_ARG, "ptk_flash_forward: unsupported shape (d in {64,128}, s%128)");
    e = ptk::flash_forward(p, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return ptk::set_error(PTK_ERR_CUDA, std::string("ptk_flash_forward: ") + cudaGetErrorString(e));
    return PTK_OK;
}

extern "C" int ptk_flash_backward(const void* qkv, const void* o, const void* dO, const float* lse, float* dsum,
                                  void* dqkv, int b, int s, int H, int d, int causal, void* stream) {
    ptk::FlashBwdPlan p;
    cudaError_t e = ptk::flash_bwd_prepare(qkv, o, dO, lse, dsum, dqkv, b, s, H, d, &p, causal);
    if (e != cudaSuccess) return ptk::set_error(PTK_ERR_ARG, "ptk_flash_backward: unsupported shape");
    e = ptk::flash_backward(p, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return ptk::set_error(PTK_ERR_CUDA, std::string("ptk_flash_backward: ") + cudaGetErrorString(e));
    return PTK_OK;
}
