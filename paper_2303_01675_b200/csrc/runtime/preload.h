// Eager loading of this library's kernels.
//
// CUDA 12 loads modules and functions lazily, on first launch.  Loading a
// function while other streams of the context hold work that waits on the
// stream being launched into (two pipeline stages of one process on one GPU,
// each waiting on the other's arrival flags) serialises against that work and
// deadlocks.  preload_all_kernels() loads every function of each translation
// unit's module up front (cuModuleEnumerateFunctions + cuFuncLoad), once per
// process; GptStage and Executor call it from their constructors.
#pragma once

namespace ptk {

void preload_module_of(const void* kernel);  // all functions of the module holding `kernel`
void preload_all_kernels();

// one per translation unit with kernels
void preload_gemm_kernels();
void preload_attention_kernels();
void preload_gpt_kernels();
void preload_emulator_kernels();

}  // namespace ptk
