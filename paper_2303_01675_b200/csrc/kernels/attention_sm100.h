// Fused causal attention (flash-style) on tcgen05 — host interface.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace ptk {

struct FlashPlan {
    alignas(64) CUtensorMap tmQK;  // qkv viewed as {d, s, 3H, b}, box {64, 128}
    alignas(64) CUtensorMap tmV;   // same view, box {64, 64} (V as the MN-major B operand)
    alignas(64) CUtensorMap tmO;   // o viewed as {d, s, H, b}, box {64, 128}: the epilogue's TMA stores
    __nv_bfloat16* o = nullptr;    // [b*s][H*d]
    float* lse = nullptr;          // [b][H][s] (log2 units of scaled scores)
    int b = 0, s = 0, H = 0, d = 0;
    float scale_log2 = 0.f;
    int causal = 1;
};

// qkv: bf16 [b][s][3][H][d] (the QKV projection output, row stride 3*H*d).
cudaError_t flash_prepare(const void* qkv, void* o, float* lse, int b, int s, int H, int d, FlashPlan* p,
                          int causal = 1);
cudaError_t flash_forward(const FlashPlan& p, cudaStream_t st);

struct FlashBwdPlan {
    alignas(64) CUtensorMap tmQKV;  // qkv as {d, s, 3H, b}, box {64, 128}
    alignas(64) CUtensorMap tmDO;   // dO [b*s][H*d] as {d, s, H, b}, box {64, 128}
    alignas(64) CUtensorMap tmDQKV;  // dqkv as {d, s, 3H, b}, box {64, 128}: the epilogue's TMA stores
    const __nv_bfloat16* o = nullptr;
    const __nv_bfloat16* dO = nullptr;
    const float* lse = nullptr;
    float* dsum = nullptr;         // scratch [b][H][s]
    __nv_bfloat16* dqkv = nullptr;  // [b*s][3*H*d]
    int b = 0, s = 0, H = 0, d = 0;
    float scale_log2 = 0.f;
    int causal = 1;
    // optional fp32 [b*s/32][3*H*d]: += per-32-row column sums of dqkv as stored (the QKV bias
    // gradient, fused into the dQ / dK / dV epilogues; one owner per entry, fixed order)
    float* col_part = nullptr;
};

// dqkv (all three sections) from qkv, the forward output o, its gradient dO and lse.
cudaError_t flash_bwd_prepare(const void* qkv, const void* o, const void* dO, const float* lse, float* dsum,
                              void* dqkv, int b, int s, int H, int d, FlashBwdPlan* p, int causal = 1);
cudaError_t flash_backward(const FlashBwdPlan& p, cudaStream_t st);

}  // namespace ptk
