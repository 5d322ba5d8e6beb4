// One GPT pipeline stage on one B200: parameters (fp32 master + bf16 compute
// copy + fp32 grads + AdamW moments, each one flat buffer), the activation
// stash (one slot per in-flight micro-batch), scratch, and the fwd/bwd
// sequences of sm_100a kernels.  This is the real compute behind the
// reference's compute_duration() (proj/src/model.cpp:43-47).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <memory>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../../include/ptk.h"
#include "../kernels/attention_sm100.h"
#include "../kernels/gemm_sm100.h"
#include "../kernels/gpt_kernels.h"

namespace ptk {

struct ParamInfo {
    std::string name;
    int64_t offset = 0;  // elements into the flat buffers
    int64_t numel = 0;
    int64_t rows = 0, cols = 0;
};

// Prepared-GEMM cache keyed by the descriptor bytes (tensor maps are bound
// to buffer addresses; every address the stage uses is stable).
class GemmCache {
  public:
    const GemmPlan& get(const ptk_gemm_desc& d);

  private:
    std::unordered_map<std::string, std::unique_ptr<GemmPlan>> plans_;
};

struct GemmTiming {
    bool armed = false;    // user switch
    bool enabled = false;  // active for the current micro-batch (sampled)
    int stride = 8;        // time the GEMMs of one micro-batch in `stride`
    std::vector<cudaEvent_t> pool;
    size_t used = 0;
    std::vector<double> flops;  // per recorded launch pair
    double total_flops = 0.0;
    double total_ms = 0.0;
    long launches = 0;
};

class GptStage {
  public:
    explicit GptStage(const ptk_gpt_config& cfg);
    ~GptStage();

    const ptk_gpt_config& cfg() const { return cfg_; }
    int tokens() const { return cfg_.micro_batch_size * cfg_.seq; }

    // x_in: device bf16 [T, h] activations (ignored on the embedding stage,
    // which reads `tok`); x_out: where the stage output goes (ignored on the
    // head stage, which computes the loss from `labels`).
    void forward(int slot, const int32_t* tok, const __nv_bfloat16* x_in, const int32_t* labels,
                 __nv_bfloat16* x_out, cudaStream_t st);
    // dy: device bf16 [T, h] gradient of this stage's output (ignored on the
    // head stage); dx: gradient of the input (ignored on the embedding stage).
    void backward(int slot, const int32_t* tok, const __nv_bfloat16* dy, __nv_bfloat16* dx, cudaStream_t st);
    // Folds the 1-D parameter partials of the micro-batches run so far into
    // grads() (one launch; idempotent).  optimizer_step() calls it first.
    void finalize_grads(cudaStream_t st);
    // Paired weight gradients: runs the deferred micro-batch's weight-gradient GEMMs alone.
    void flush_wgrads(cudaStream_t st);
    // Runtime switch (buffers exist only if the stage was created with cfg.wgrad_pairs).
    void set_wgrad_pairs(bool on);
    bool wgrad_pairs_on() const { return pairs_on_; }
    void optimizer_step(float lr, float wd, cudaStream_t st);
    void zero_grads(cudaStream_t st);

    float* loss_accumulator() { return loss_acc_; }
    const std::vector<ParamInfo>& params() const { return params_; }
    float* master() { return master_; }
    __nv_bfloat16* weights() { return wbf_; }
    float* grads() { return grad_; }
    int64_t param_count() const { return total_; }
    size_t stash_bytes_per_slot() const { return stash_per_slot_; }

    // Run subsequent micro-batches with b <= the allocated maximum (plan switch).
    // When b divides the allocated maximum, every stash slot is split into
    // b_max / b virtual slots (sample-granular stash): virtual_slots() grows.
    void set_micro_batch(int b, int micro_batches);
    int virtual_slots() const { return vslots_; }
    int slot_split() const { return vsplit_; }  // virtual slots per physical slot
    long launches() const { return launches_; }
    void reset_launches() { launches_ = 0; }

    GemmTiming& gemm_timing() { return timing_; }
    // Synchronises the recorded GEMM event pairs into totals and recycles them.
    void collect_timing();

  private:
    struct LayerW {  // element offsets (-1: block on another stage)
        int64_t ln1_g = -1, ln1_b = -1, w_qkv = -1, b_qkv = -1, w_o = -1, b_o = -1;
        int64_t ln2_g = -1, ln2_b = -1, w_fc1 = -1, b_fc1 = -1, w_fc2 = -1, b_fc2 = -1;
    };
    struct LayerStash {
        __nv_bfloat16 *x_in = nullptr, *ln1 = nullptr, *qkv = nullptr, *attn_o = nullptr, *x_mid = nullptr,
                      *ln2 = nullptr, *fc1_pre = nullptr, *fc1_act = nullptr;
        float *mean1 = nullptr, *rstd1 = nullptr, *mean2 = nullptr, *rstd2 = nullptr, *lse = nullptr;
    };
    // GPT: ln1/ln2 hold the pre-LN outputs, x_mid the post-attention residual.
    // BERT (post-LN): ln1 holds y = attn + x (pre-LN1), x_mid = LN1(y),
    //                 ln2 holds z = ffn + x_mid (pre-LN2); the layer output is LN2(z).
    struct HeadStash {
        __nv_bfloat16 *x_fin, *xf, *dlogits;
        float *meanf, *rstdf;
        __nv_bfloat16 *t_pre, *t_act;  // BERT MLM transform
    };
    struct EmbStash {  // BERT: embedding sum before its LayerNorm
        __nv_bfloat16* sum;
        float *mean, *rstd;
    };
    bool bert() const { return cfg_.arch == 1; }
    // half-layer stage boundaries: the first layer may lack its attention block, the last its MLP block
    bool has_attn(int li) const { return !(li == 0 && cfg_.skip_first_attn); }
    bool has_mlp(int li) const { return !(li == L_ - 1 && cfg_.skip_last_mlp); }
    void bert_layer_forward(int li, LayerStash& s, const __nv_bfloat16* x_in, __nv_bfloat16* x_out, cudaStream_t st);
    void bert_layer_backward(int li, LayerStash& s, const __nv_bfloat16* dy, __nv_bfloat16* dx, cudaStream_t st);
    void attention_forward(LayerStash& s, cudaStream_t st);
    void attention_backward(LayerStash& s, float* bqkv_part, cudaStream_t st);

    struct InitSpec {
        int64_t offset, numel;
        uint64_t seed;
        float std, mean;
    };
    std::vector<InitSpec> init_;

    int64_t add_param(const std::string& name, int64_t rows, int64_t cols, float std, float mean, uint64_t seed);
    void gemm(ptk_gemm_desc d, cudaStream_t st);
    void layer_forward(int li, LayerStash& s, const __nv_bfloat16* x_in, __nv_bfloat16* x_out, cudaStream_t st);
    void layer_backward(int li, LayerStash& s, const __nv_bfloat16* dy, __nv_bfloat16* dx, cudaStream_t st);
    void* alloc(size_t bytes);
    void kl(int n, cudaError_t e, const char* what);

    ptk_gpt_config cfg_;
    int L_ = 0;  // layers on this stage
    int b_max_ = 1;
    long launches_ = 0;
    std::vector<ParamInfo> params_;
    std::vector<LayerW> lw_;
    int64_t wte_ = -1, wpe_ = -1, lnf_g_ = -1, lnf_b_ = -1, w_head_ = -1;
    int64_t lne_g_ = -1, lne_b_ = -1, w_t_ = -1, b_t_ = -1;  // BERT embedding LN, MLM transform
    std::vector<EmbStash> emb_;
    int64_t total_ = 0;
    float *master_ = nullptr, *grad_ = nullptr, *adam_m_ = nullptr, *adam_v_ = nullptr;
    __nv_bfloat16* wbf_ = nullptr;
    int step_ = 0;

    std::vector<std::vector<LayerStash>> stash_;  // [slot][layer]
    std::vector<HeadStash> head_;                 // [slot]
    // views of the physical slots at the current micro-batch size
    std::vector<std::vector<LayerStash>> vstash_;  // [virtual slot][layer]
    std::vector<HeadStash> vhead_;
    std::vector<EmbStash> vemb_;
    int vslots_ = 0, vsplit_ = 1;
    void build_virtual_slots();
    size_t stash_per_slot_ = 0;

    // scratch (one micro-batch in flight on the compute stream at a time)
    int32_t* order_ = nullptr;
    float *dsum_ = nullptr, *loss_rows_ = nullptr, *loss_acc_ = nullptr;
    __nv_bfloat16 *g_a_ = nullptr, *g_b_ = nullptr, *d_pre_ = nullptr, *d_ln_ = nullptr,
                  *d_attn_ = nullptr, *dqkv_ = nullptr, *dx_mid_ = nullptr, *dy_ = nullptr;
    // paired weight gradients (cfg.wgrad_pairs): the deferred micro-batch's gradient-side
    // operands live in per-layer buffers (the scratch pointers are switched to them while it runs)
    struct DeferBufs {
        __nv_bfloat16 *out = nullptr, *d_pre = nullptr, *dx_mid = nullptr, *dqkv = nullptr, *d_ln = nullptr,
                      *dy = nullptr;
    };
    std::vector<DeferBufs> dbuf_;
    __nv_bfloat16 *dhead_g_ = nullptr, *dhead_dy_ = nullptr;
    bool pairs_on_ = false;
    int wg_mode_ = 0;                        // 0 direct, 1 deferring (first of a pair), 2 pairing (second)
    int wg_count_ = 0;                       // backwards since the last flush (pairing phase)
    std::vector<ptk_gemm_desc> wg_pending_;  // the deferred micro-batch's weight-gradient GEMMs
    void wgrad(const ptk_gemm_desc& d, cudaStream_t st);
    void use_scratch(int layer);             // layer >= 0: deferral buffers of that layer; -1: shared scratch
    __nv_bfloat16 *s_d_pre_ = nullptr, *s_d_ln_ = nullptr, *s_dqkv_ = nullptr, *s_dx_mid_ = nullptr,
                  *s_dy_ = nullptr;  // the shared scratch set

    // 1-D parameter gradient partials: grad offset -> float[kVecParts][cols]
    std::unordered_map<int64_t, float*> vparts_;
    VecGradSeg* vsegs_ = nullptr;  // device table for vec_grad_finalize
    int nvseg_ = 0, vseg_max_cols_ = 0;
    size_t vparts_bytes_ = 0;
    float* vp(int64_t offset);

    std::vector<void*> allocs_;
    GemmCache cache_;
    std::unordered_map<std::string, std::unique_ptr<FlashPlan>> flash_fwd_;
    std::unordered_map<std::string, std::unique_ptr<FlashBwdPlan>> flash_bwd_;
    GemmTiming timing_;
};

}  // namespace ptk
