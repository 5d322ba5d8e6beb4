// See preload.h.
#include <cuda.h>
#include <cuda_runtime.h>

#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "preload.h"

namespace ptk {

namespace {

template <typename Fn>
Fn entry(const char* name) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
        return nullptr;
    return reinterpret_cast<Fn>(p);
}

}  // namespace

void preload_module_of(const void* kernel) {
    using GetModule = CUresult (*)(CUmodule*, CUfunction);
    using Count = CUresult (*)(unsigned int*, CUmodule);
    using Enumerate = CUresult (*)(CUfunction*, unsigned int, CUmodule);
    using Load = CUresult (*)(CUfunction);
    static const GetModule get_module = entry<GetModule>("cuFuncGetModule");
    static const Count count = entry<Count>("cuModuleGetFunctionCount");
    static const Enumerate enumerate = entry<Enumerate>("cuModuleEnumerateFunctions");
    static const Load load = entry<Load>("cuFuncLoad");
    if (!get_module || !count || !enumerate || !load) return;  // older driver: loading stays lazy
    cudaFunction_t f = nullptr;
    if (cudaGetFuncBySymbol(&f, kernel) != cudaSuccess) throw std::runtime_error("preload: cudaGetFuncBySymbol failed");
    CUmodule mod = nullptr;
    unsigned int n = 0;
    if (get_module(&mod, reinterpret_cast<CUfunction>(f)) != CUDA_SUCCESS || count(&n, mod) != CUDA_SUCCESS)
        throw std::runtime_error("preload: module query failed");
    std::vector<CUfunction> fs(n);
    if (n > 0 && enumerate(fs.data(), n, mod) != CUDA_SUCCESS) throw std::runtime_error("preload: enumerate failed");
    for (CUfunction fn : fs)
        if (load(fn) != CUDA_SUCCESS) throw std::runtime_error("preload: cuFuncLoad failed");
}

void preload_all_kernels() {
    static std::once_flag once;
    std::call_once(once, [] {
        preload_gemm_kernels();
        preload_attention_kernels();
        preload_gpt_kernels();
        preload_emulator_kernels();
    });
}

}  // namespace ptk
