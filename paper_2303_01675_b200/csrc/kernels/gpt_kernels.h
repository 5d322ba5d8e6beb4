// Host launchers for the memory-bound GPT stage kernels (gpt_kernels.cu).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace ptk {

cudaError_t layernorm_fwd(const __nv_bfloat16* x, const __nv_bfloat16* g, const __nv_bfloat16* b, __nv_bfloat16* y,
                          float* mean, float* rstd, int rows, int h, float eps, cudaStream_t st);
// 1-D parameter gradients (LayerNorm affine, biases) accumulate into
// per-parameter partials float[kVecParts][cols] over the micro-batches of an
// iteration; vec_grad_finalize adds them into the gradient (fixed order) and
// clears them.  rows % kVecParts == 0.
#ifndef PTK_VEC_PARTS
#define PTK_VEC_PARTS 256
#endif
constexpr int kVecParts = PTK_VEC_PARTS;
struct VecGradSeg {
    float* grad;
    float* part;
    int cols;
};
// dx = LN'(dy) (+ resid); part_g/part_b += the gamma/beta column partials;
// part_out (optional) += the column partials of dx as stored (the bias grad
// of the GEMM whose output gradient dx is).  h in {256, 512, 768, 1024, 2048, 4096}.
cudaError_t layernorm_bwd(const __nv_bfloat16* dy, const __nv_bfloat16* x, const float* mean, const float* rstd,
                          const __nv_bfloat16* g, const __nv_bfloat16* resid, __nv_bfloat16* dx, float* part_g,
                          float* part_b, float* part_out, int rows, int h, cudaStream_t st);
// part[p][c] += sum over row block p of m[r][c]  (cols % 8 == 0).
cudaError_t colsum_partial(const __nv_bfloat16* m, float* part, int rows, int cols, cudaStream_t st);
// segs_dev: device array of nseg segments; max_cols: the widest segment.
cudaError_t vec_grad_finalize(const VecGradSeg* segs_dev, int nseg, int max_cols, cudaStream_t st);
// logits overwritten by dlogits * grad_scale; loss_out[0] += sum(row losses) * loss_scale.
cudaError_t cross_entropy(__nv_bfloat16* logits, const int32_t* labels, float* loss_rows, float* loss_out, int rows,
                          int vocab, float grad_scale, float loss_scale, cudaStream_t st);
cudaError_t embedding_fwd(const int32_t* tok, const __nv_bfloat16* wte, const __nv_bfloat16* wpe, __nv_bfloat16* x,
                          int rows, int seq, int h, cudaStream_t st);
// order: int32 scratch [rows] (token-sorted positions).
cudaError_t embedding_bwd(const int32_t* tok, const __nv_bfloat16* dx, float* dwte, float* dwpe, int32_t* order,
                          int rows, int seq, int h, int vocab, cudaStream_t st);
// out = dy * gelu'(pre) (tanh form), n % 8 == 0
cudaError_t dgelu_mul(const __nv_bfloat16* dy, const __nv_bfloat16* pre, __nv_bfloat16* out, int64_t n,
                      cudaStream_t st);
cudaError_t adamw_step(float* w, float* g, float* m, float* v, __nv_bfloat16* wb, int64_t n, float lr, float b1,
                       float b2, float eps, float wd, int step, cudaStream_t st);
cudaError_t init_normal(float* w, int64_t n, uint64_t seed, float std, float mean, cudaStream_t st);
cudaError_t cast_to_bf16(const float* src, __nv_bfloat16* dst, int64_t n, cudaStream_t st);

}  // namespace ptk
