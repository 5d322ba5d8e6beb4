// GPT stage forward/backward on sm_100a.  See gpt_stage.h and DESIGN.md §4.
//
// Per layer forward (T = b*s tokens, h hidden, H heads, d = h/H):
//   ln1 = LN(x)                          qkv = ln1·Wqkvᵀ + b           (tcgen05 GEMM)
//   o, lse = causal flash attention(qkv) (tcgen05, S/P never leave TMEM/smem)
//   x_mid = o·Woᵀ + b + x                (residual in the GEMM epilogue)
//   ln2 = LN(x_mid)                      pre = ln2·W1ᵀ + b, a = gelu(pre) (one epilogue)
//   x_out = a·W2ᵀ + b + x_mid
// Backward mirrors it; every weight gradient is a K = T GEMM accumulated in
// place (fp32, β = 1) in the order micro-batches are run — ascending on every
// device for every k, so gradients are bit-identical across k at fixed b.
#include "gpt_stage.h"
#include "preload.h"

#include <cmath>
#include <cstring>
#include <stdexcept>

#include "../kernels/gpt_kernels.h"
#include "errors.h"

namespace ptk {

namespace {

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

ptk_matrix mat(const void* p, int64_t ld, int mn = 0, int64_t bs0 = 0, int64_t bs1 = 0) {
    ptk_matrix m;
    std::memset(&m, 0, sizeof m);
    m.ptr = const_cast<void*>(p);
    m.ld = ld;
    m.mn_major = mn;
    m.batch_stride[0] = bs0;
    m.batch_stride[1] = bs1;
    return m;
}

ptk_gemm_desc desc(int m, int n, int k, ptk_matrix a, ptk_matrix b, ptk_matrix c, int epi) {
    ptk_gemm_desc d;
    std::memset(&d, 0, sizeof d);
    d.m = m;
    d.n = n;
    d.k = k;
    d.batch[0] = d.batch[1] = 1;
    d.a = a;
    d.b = b;
    d.c = c;
    d.epilogue = epi;
    d.multicast = 2;  // CTA-pair tcgen05 kernel for every dense BN=256 GEMM
    return d;
}

}  // namespace

const GemmPlan& GemmCache::get(const ptk_gemm_desc& d) {
    std::string key(reinterpret_cast<const char*>(&d), sizeof d);
    auto it = plans_.find(key);
    if (it != plans_.end()) return *it->second;
    auto p = std::make_unique<GemmPlan>();
    const int rc = gemm_prepare(d, p.get());
    if (rc != PTK_OK)
        throw std::runtime_error("gemm_prepare failed (" + std::to_string(rc) + ") m=" + std::to_string(d.m) +
                                 " n=" + std::to_string(d.n) + " k=" + std::to_string(d.k));
    return *plans_.emplace(std::move(key), std::move(p)).first->second;
}

void* GptStage::alloc(size_t bytes) {
    void* p = nullptr;
    ck(cudaMalloc(&p, bytes < 256 ? 256 : bytes), "cudaMalloc");
    allocs_.push_back(p);
    return p;
}

int64_t GptStage::add_param(const std::string& name, int64_t rows, int64_t cols, float std, float mean, uint64_t seed) {
    ParamInfo p;
    p.name = name;
    p.offset = total_;
    p.rows = rows;
    p.cols = cols;
    p.numel = rows * cols;
    total_ += (p.numel + 63) / 64 * 64;  // keep every tensor 128-byte aligned in bf16
    params_.push_back(p);
    init_.push_back({p.offset, p.numel, seed, std, mean});
    return p.offset;
}

GptStage::GptStage(const ptk_gpt_config& c) : cfg_(c) {
    preload_all_kernels();
    const int h = c.hidden, f = c.ffn, V = c.vocab;
    if (h % 256 || c.heads <= 0 || h % c.heads || (h / c.heads) % 64 || c.seq % 128 || f % 64 || V % 64)
        throw std::invalid_argument("GptStage: unsupported shape (h%256, d%64, seq%128, ffn%64, vocab%64)");
    if (c.arch != 0 && c.arch != 1) throw std::invalid_argument("GptStage: arch must be 0 (GPT) or 1 (BERT)");
    if (c.layer_begin < 0 || c.layer_end < c.layer_begin || c.layer_end > c.n_layer || c.slots < 1 ||
        c.micro_batch_size < 1 || c.micro_batches < 1)
        throw std::invalid_argument("GptStage: bad layer range / slots / batch");
    L_ = c.layer_end - c.layer_begin;
    b_max_ = c.micro_batch_size;
    if ((c.skip_first_attn && (c.has_embedding || L_ < 1)) || (c.skip_last_mlp && (c.has_head || L_ < 1)) ||
        (L_ == 1 && c.skip_first_attn && c.skip_last_mlp))
        throw std::invalid_argument("GptStage: half-layer boundaries need a layer block on this stage, no "
                                    "attention-less embedding stage and no MLP-less head stage");
    if (static_cast<int64_t>(c.micro_batch_size) * c.seq > 32LL * kVecParts)
        throw std::invalid_argument("GptStage: micro_batch_size * seq exceeds 32 * kVecParts tokens");
    const float proj_std = 0.02f / std::sqrt(2.f * c.n_layer);
    const uint64_t base = c.seed * 1000003ull;

    // ---- parameters (seeded per global tensor identity: any partition of the
    //      model into stages initialises identical weights)
    if (c.has_embedding) {
        wte_ = add_param("wte", V, h, 0.02f, 0.f, base + 1);
        wpe_ = add_param("wpe", c.seq, h, 0.02f, 0.f, base + 2);
        if (c.arch == 1) {
            lne_g_ = add_param("lne_g", 1, h, 0.f, 1.f, base + 6);
            lne_b_ = add_param("lne_b", 1, h, 0.f, 0.f, base + 7);
        }
    }
    for (int i = 0; i < L_; ++i) {
        const int l = c.layer_begin + i;
        const uint64_t s = base + 100 + 16ull * l;
        const std::string p = "h" + std::to_string(l) + ".";
        LayerW w;
        if (!(i == 0 && c.skip_first_attn)) {  // attention block
            w.ln1_g = add_param(p + "ln1_g", 1, h, 0.f, 1.f, s + 0);
            w.ln1_b = add_param(p + "ln1_b", 1, h, 0.f, 0.f, s + 1);
            w.w_qkv = add_param(p + "w_qkv", 3 * h, h, 0.02f, 0.f, s + 2);
            w.b_qkv = add_param(p + "b_qkv", 1, 3 * h, 0.f, 0.f, s + 3);
            w.w_o = add_param(p + "w_o", h, h, proj_std, 0.f, s + 4);
            w.b_o = add_param(p + "b_o", 1, h, 0.f, 0.f, s + 5);
        }
        if (!(i == L_ - 1 && c.skip_last_mlp)) {  // MLP block
            w.ln2_g = add_param(p + "ln2_g", 1, h, 0.f, 1.f, s + 6);
            w.ln2_b = add_param(p + "ln2_b", 1, h, 0.f, 0.f, s + 7);
            w.w_fc1 = add_param(p + "w_fc1", f, h, 0.02f, 0.f, s + 8);
            w.b_fc1 = add_param(p + "b_fc1", 1, f, 0.f, 0.f, s + 9);
            w.w_fc2 = add_param(p + "w_fc2", h, f, proj_std, 0.f, s + 10);
            w.b_fc2 = add_param(p + "b_fc2", 1, h, 0.f, 0.f, s + 11);
        }
        lw_.push_back(w);
    }
    if (c.has_head) {
        if (c.arch == 1) {
            w_t_ = add_param("w_t", h, h, 0.02f, 0.f, base + 8);
            b_t_ = add_param("b_t", 1, h, 0.f, 0.f, base + 9);
        }
        lnf_g_ = add_param("lnf_g", 1, h, 0.f, 1.f, base + 3);
        lnf_b_ = add_param("lnf_b", 1, h, 0.f, 0.f, base + 4);
        w_head_ = add_param("w_head", V, h, 0.02f, 0.f, base + 5);
    }
    master_ = static_cast<float*>(alloc(total_ * 4));
    grad_ = static_cast<float*>(alloc(total_ * 4));
    adam_m_ = static_cast<float*>(alloc(total_ * 4));
    adam_v_ = static_cast<float*>(alloc(total_ * 4));
    wbf_ = static_cast<__nv_bfloat16*>(alloc(total_ * 2));
    ck(cudaMemset(master_, 0, total_ * 4), "memset");
    ck(cudaMemset(grad_, 0, total_ * 4), "memset");
    ck(cudaMemset(adam_m_, 0, total_ * 4), "memset");
    ck(cudaMemset(adam_v_, 0, total_ * 4), "memset");
    for (const InitSpec& in : init_) ck(init_normal(master_ + in.offset, in.numel, in.seed, in.std, in.mean, 0), "init");
    ck(cast_to_bf16(master_, wbf_, total_, 0), "cast");

    // ---- activation stash
    const int64_t T = tokens();
    stash_.assign(c.slots, std::vector<LayerStash>(L_));
    head_.resize(c.slots);
    for (int sl = 0; sl < c.slots; ++sl) {
        size_t bytes = 0;
        for (int i = 0; i < L_; ++i) {
            LayerStash& s = stash_[sl][i];
            auto bf = [&](int64_t n) {
                bytes += n * 2;
                return static_cast<__nv_bfloat16*>(alloc(n * 2));
            };
            auto fl = [&](int64_t n) {
                bytes += n * 4;
                return static_cast<float*>(alloc(n * 4));
            };
            const bool A = has_attn(i), M = has_mlp(i);
            if (A) {
                s.x_in = (i == 0 && !c.has_embedding) ? nullptr : bf(T * h);  // layer 0 reads the stage input
                s.ln1 = bf(T * h);
                s.qkv = bf(T * 3 * h);
                s.attn_o = bf(T * h);
                s.mean1 = fl(T);
                s.rstd1 = fl(T);
                s.lse = fl(static_cast<int64_t>(c.micro_batch_size) * c.heads * c.seq);
            }
            // x_mid: the attention block's output; an MLP-only first layer reads the stage input
            // there, an attention-only last layer writes it straight to the stage output
            if (A && M) s.x_mid = bf(T * h);
            if (M) {
                s.ln2 = bf(T * h);
                s.fc1_pre = bf(T * f);
                s.fc1_act = bf(T * f);
                s.mean2 = fl(T);
                s.rstd2 = fl(T);
            }
        }
        if (c.has_head) {
            HeadStash& hs = head_[sl];
            hs.x_fin = static_cast<__nv_bfloat16*>(alloc(T * h * 2));
            hs.xf = static_cast<__nv_bfloat16*>(alloc(T * h * 2));
            hs.dlogits = static_cast<__nv_bfloat16*>(alloc(T * V * 2));
            hs.meanf = static_cast<float*>(alloc(T * 4));
            hs.rstdf = static_cast<float*>(alloc(T * 4));
            bytes += T * h * 4 + T * V * 2 + T * 8;
            hs.t_pre = hs.t_act = nullptr;
            if (c.arch == 1) {
                hs.t_pre = static_cast<__nv_bfloat16*>(alloc(T * h * 2));
                hs.t_act = static_cast<__nv_bfloat16*>(alloc(T * h * 2));
                bytes += T * h * 4;
            }
        }
        if (c.has_embedding && c.arch == 1) {
            EmbStash e;
            e.sum = static_cast<__nv_bfloat16*>(alloc(T * h * 2));
            e.mean = static_cast<float*>(alloc(T * 4));
            e.rstd = static_cast<float*>(alloc(T * 4));
            bytes += T * h * 2 + T * 8;
            emb_.push_back(e);
        }
        stash_per_slot_ = bytes;
    }
    // x_in of layer i>0 is layer i-1's output: point the stash there.
    // (layer_forward writes x_out of layer i into stash[i+1].x_in)

    // ---- scratch
    dsum_ = static_cast<float*>(alloc(static_cast<int64_t>(c.micro_batch_size) * c.heads * c.seq * 4));
    g_a_ = static_cast<__nv_bfloat16*>(alloc(T * h * 2));
    g_b_ = static_cast<__nv_bfloat16*>(alloc(T * h * 2));
    d_pre_ = static_cast<__nv_bfloat16*>(alloc(T * f * 2));
    d_ln_ = static_cast<__nv_bfloat16*>(alloc(T * h * 2));
    d_attn_ = static_cast<__nv_bfloat16*>(alloc(T * h * 2));
    dqkv_ = static_cast<__nv_bfloat16*>(alloc(T * 3 * h * 2));
    dx_mid_ = static_cast<__nv_bfloat16*>(alloc(T * h * 2));
    dy_ = static_cast<__nv_bfloat16*>(alloc(T * h * 2));
    s_d_pre_ = d_pre_;
    s_d_ln_ = d_ln_;
    s_dqkv_ = dqkv_;
    s_dx_mid_ = dx_mid_;
    s_dy_ = dy_;
    pairs_on_ = c.wgrad_pairs != 0;
    if (c.wgrad_pairs) {
        dbuf_.resize(L_);
        for (int i = 0; i < L_; ++i) {
            DeferBufs& d = dbuf_[i];
            auto bf = [&](int64_t n) { return static_cast<__nv_bfloat16*>(alloc(n * 2)); };
            d.out = bf(T * h);
            d.d_pre = bf(T * f);
            d.dx_mid = bf(T * h);
            d.dqkv = bf(T * 3 * h);
            d.d_ln = bf(T * h);
            d.dy = bf(T * h);
        }
        if (c.has_head) {
            dhead_g_ = static_cast<__nv_bfloat16*>(alloc(T * h * 2));
            dhead_dy_ = static_cast<__nv_bfloat16*>(alloc(T * h * 2));
        }
    }
    // 1-D parameter gradient partials (see vec_grad_finalize)
    {
        std::vector<VecGradSeg> segs;
        for (const ParamInfo& p : params_) {
            if (p.rows != 1) continue;
            float* part = static_cast<float*>(alloc(static_cast<size_t>(kVecParts) * p.cols * 4));
            ck(cudaMemset(part, 0, static_cast<size_t>(kVecParts) * p.cols * 4), "memset");
            vparts_[p.offset] = part;
            segs.push_back({grad_ + p.offset, part, static_cast<int>(p.cols)});
            vparts_bytes_ += static_cast<size_t>(kVecParts) * p.cols * 4;
            vseg_max_cols_ = std::max<int>(vseg_max_cols_, static_cast<int>(p.cols));
        }
        nvseg_ = static_cast<int>(segs.size());
        if (nvseg_ > 0) {
            vsegs_ = static_cast<VecGradSeg*>(alloc(segs.size() * sizeof(VecGradSeg)));
            ck(cudaMemcpy(vsegs_, segs.data(), segs.size() * sizeof(VecGradSeg), cudaMemcpyHostToDevice), "copy");
        }
    }
    loss_rows_ = static_cast<float*>(alloc(T * 4));
    order_ = static_cast<int32_t*>(alloc(T * 4));
    loss_acc_ = static_cast<float*>(alloc(64));
    ck(cudaMemset(loss_acc_, 0, 64), "memset");
    build_virtual_slots();
    ck(cudaDeviceSynchronize(), "stage init");
}

GptStage::~GptStage() {
    for (cudaEvent_t e : timing_.pool) cudaEventDestroy(e);
    for (void* p : allocs_) cudaFree(p);
}

void GptStage::kl(int n, cudaError_t e, const char* what) {
    ck(e, what);
    launches_ += n;
}

void GptStage::set_micro_batch(int b, int micro_batches) {
    if (b < 1 || b > b_max_) throw std::invalid_argument("set_micro_batch: b exceeds the allocated maximum");
    cfg_.micro_batch_size = b;
    cfg_.micro_batches = micro_batches;
    build_virtual_slots();
}

// Virtual slot v = (physical slot v / r, sample offset (v % r)·b) with r = b_max / b:
// every stash buffer is [b_max samples][per-sample extent], so a micro-batch of
// b samples occupies a contiguous sub-range of a physical slot.
void GptStage::build_virtual_slots() {
    const ptk_gpt_config& c = cfg_;
    const int b = c.micro_batch_size;
    const int r = (b_max_ % b == 0) ? b_max_ / b : 1;
    const int64_t s = c.seq, h = c.hidden, f = c.ffn;
    const int phys = static_cast<int>(stash_.size());
    vsplit_ = r;
    vslots_ = phys * r;
    vstash_.assign(vslots_, std::vector<LayerStash>(L_));
    vhead_.assign(c.has_head ? vslots_ : 0, HeadStash{});
    vemb_.assign(emb_.empty() ? 0 : vslots_, EmbStash{});
    auto off = [](auto* p, int64_t n) { return p == nullptr ? p : p + n; };
    for (int v = 0; v < vslots_; ++v) {
        const int ps = v / r;
        const int64_t j = static_cast<int64_t>(v % r) * b;  // first sample of this view
        for (int i = 0; i < L_; ++i) {
            const LayerStash& P = stash_[ps][i];
            LayerStash& V = vstash_[v][i];
            V.x_in = off(P.x_in, j * s * h);
            V.ln1 = off(P.ln1, j * s * h);
            V.qkv = off(P.qkv, j * s * 3 * h);
            V.attn_o = off(P.attn_o, j * s * h);
            V.x_mid = off(P.x_mid, j * s * h);
            V.ln2 = off(P.ln2, j * s * h);
            V.fc1_pre = off(P.fc1_pre, j * s * f);
            V.fc1_act = off(P.fc1_act, j * s * f);
            V.mean1 = off(P.mean1, j * s);
            V.rstd1 = off(P.rstd1, j * s);
            V.mean2 = off(P.mean2, j * s);
            V.rstd2 = off(P.rstd2, j * s);
            V.lse = off(P.lse, j * c.heads * s);
        }
        if (c.has_head) {
            const HeadStash& P = head_[ps];
            HeadStash& V = vhead_[v];
            V.x_fin = off(P.x_fin, j * s * h);
            V.xf = off(P.xf, j * s * h);
            V.dlogits = off(P.dlogits, j * s * c.vocab);
            V.meanf = off(P.meanf, j * s);
            V.rstdf = off(P.rstdf, j * s);
            V.t_pre = off(P.t_pre, j * s * h);
            V.t_act = off(P.t_act, j * s * h);
        }
        if (!emb_.empty()) {
            const EmbStash& P = emb_[ps];
            EmbStash& V = vemb_[v];
            V.sum = off(P.sum, j * s * h);
            V.mean = off(P.mean, j * s);
            V.rstd = off(P.rstd, j * s);
        }
    }
}

void GptStage::gemm(ptk_gemm_desc d, cudaStream_t st) {
    const GemmPlan& p = cache_.get(d);
    ++launches_;
    if (timing_.enabled) {
        if (timing_.used + 2 > timing_.pool.size()) {
            for (int i = 0; i < 256; ++i) {
                cudaEvent_t e;
                ck(cudaEventCreate(&e), "event");
                timing_.pool.push_back(e);
            }
        }
        ck(cudaEventRecord(timing_.pool[timing_.used], st), "event");
        const int rc = gemm_run(p, st);
        ck(cudaEventRecord(timing_.pool[timing_.used + 1], st), "event");
        timing_.used += 2;
        timing_.flops.push_back(p.flops);
        if (rc != PTK_OK) throw std::runtime_error("gemm launch failed");
        return;
    }
    if (gemm_run(p, st) != PTK_OK) throw std::runtime_error("gemm launch failed");
}

// Weight-gradient GEMM (fp32 accumulate into the gradient buffer).  With paired weight
// gradients, the first micro-batch of a pair only records the descriptor (its operands stay
// live: stash slot + per-layer deferral buffers); the second launches ONE GEMM with two K
// segments, deferred micro-batch first, so the fp32 gradient is read and written once per
// pair.  Pairs are (0,1), (2,3), ... in backward order, which is ascending for every plan, so
// gradients stay bit-identical across k and stage splits.
void GptStage::wgrad(const ptk_gemm_desc& d, cudaStream_t st) {
    // only GEMMs that run on the CTA-pair kernel anyway are paired (a two-segment GEMM needs it);
    // a narrow-tile weight gradient (BERT-large's 1024 x 1024 out-proj) stays per micro-batch
    if (wg_mode_ != 0) {
        const GemmPlan& p = cache_.get(d);
        if (!(p.multicast && p.args.bn == 256 && d.multicast == 2)) {
            gemm(d, st);
            return;
        }
    }
    if (wg_mode_ == 1) {
        wg_pending_.push_back(d);
        return;
    }
    if (wg_mode_ == 2) {
        for (size_t i = 0; i < wg_pending_.size(); ++i) {
            const ptk_gemm_desc& p = wg_pending_[i];
            if (p.c.ptr != d.c.ptr) continue;
            ptk_gemm_desc two = p;
            two.a2 = d.a;
            two.b2 = d.b;
            two.k2 = d.k;
            wg_pending_.erase(wg_pending_.begin() + static_cast<std::ptrdiff_t>(i));
            gemm(two, st);
            return;
        }
    }
    gemm(d, st);
}

void GptStage::set_wgrad_pairs(bool on) {
    if (on && !cfg_.wgrad_pairs) throw std::invalid_argument("set_wgrad_pairs: stage created without wgrad_pairs");
    if (!wg_pending_.empty()) throw std::logic_error("set_wgrad_pairs: a deferred micro-batch is pending");
    pairs_on_ = on;
    wg_count_ = 0;
}

void GptStage::flush_wgrads(cudaStream_t st) {
    for (const ptk_gemm_desc& d : wg_pending_) gemm(d, st);
    wg_pending_.clear();
    wg_count_ = 0;
}

void GptStage::use_scratch(int layer) {
    if (layer < 0) {
        d_pre_ = s_d_pre_;
        d_ln_ = s_d_ln_;
        dqkv_ = s_dqkv_;
        dx_mid_ = s_dx_mid_;
        dy_ = s_dy_;
        return;
    }
    const DeferBufs& b = dbuf_[static_cast<size_t>(layer)];
    d_pre_ = b.d_pre;
    d_ln_ = b.d_ln;
    dqkv_ = b.dqkv;
    dx_mid_ = b.dx_mid;
    dy_ = b.dy;
}

void GptStage::attention_forward(LayerStash& s, cudaStream_t st) {
    // fused attention (tcgen05): o = softmax(QKᵀ/√d [causal for GPT]) V, lse for the backward
    const ptk_gpt_config& c = cfg_;
    const int b = c.micro_batch_size, d = c.hidden / c.heads;
    const std::string key = std::to_string(reinterpret_cast<uintptr_t>(s.qkv)) + "." + std::to_string(b);
    auto it = flash_fwd_.find(key);
    if (it == flash_fwd_.end()) {
        auto p = std::make_unique<FlashPlan>();
        ck(flash_prepare(s.qkv, s.attn_o, s.lse, b, c.seq, c.heads, d, p.get(), bert() ? 0 : 1), "flash prepare");
        it = flash_fwd_.emplace(key, std::move(p)).first;
    }
    kl(1, flash_forward(*it->second, st), "flash fwd");
}

void GptStage::attention_backward(LayerStash& s, float* bqkv_part, cudaStream_t st) {
    // dqkv = flash backward (dK/dV per key block, dQ per query block; deterministic)
    const ptk_gpt_config& c = cfg_;
    const int b = c.micro_batch_size, d = c.hidden / c.heads;
    const std::string key = std::to_string(reinterpret_cast<uintptr_t>(s.qkv)) + "." + std::to_string(b) + "." +
                            std::to_string(reinterpret_cast<uintptr_t>(dqkv_));
    auto it = flash_bwd_.find(key);
    if (it == flash_bwd_.end()) {
        auto p = std::make_unique<FlashBwdPlan>();
        ck(flash_bwd_prepare(s.qkv, s.attn_o, d_attn_, s.lse, dsum_, dqkv_, b, c.seq, c.heads, d, p.get(),
                             bert() ? 0 : 1),
           "flash bwd prep");
        p->col_part = bqkv_part;  // dbqkv = column sums of dqkv, fused into the dQ/dK/dV epilogues
        it = flash_bwd_.emplace(key, std::move(p)).first;
    }
    kl(3, flash_backward(*it->second, st), "flash bwd");
}

void GptStage::bert_layer_forward(int li, LayerStash& s, const __nv_bfloat16* x_in, __nv_bfloat16* x_out,
                                  cudaStream_t st) {
    // post-LN: y = x + attn(x); x_mid = LN1(y); z = x_mid + ffn(x_mid); x_out = LN2(z)
    const ptk_gpt_config& c = cfg_;
    const LayerW& w = lw_[li];
    const int T = tokens(), h = c.hidden, f = c.ffn;
    const __nv_bfloat16* W = wbf_;
    const bool A = has_attn(li), M = has_mlp(li);
    // attention block (input x_in) -> x_mid; MLP block (input x_mid) -> x_out
    const __nv_bfloat16* xm = A ? (M ? s.x_mid : x_out) : x_in;
    if (A) {
        {
            ptk_gemm_desc g = desc(T, 3 * h, h, mat(x_in, h), mat(W + w.w_qkv, h), mat(s.qkv, 3 * h), PTK_EPI_BF16);
            g.bias = W + w.b_qkv;
            gemm(g, st);
        }
        attention_forward(s, st);
        {
            ptk_gemm_desc g = desc(T, h, h, mat(s.attn_o, h), mat(W + w.w_o, h), mat(s.ln1, h), PTK_EPI_BF16);
            g.bias = W + w.b_o;
            g.aux = mat(x_in, h);
            gemm(g, st);
        }
        kl(1, layernorm_fwd(s.ln1, W + w.ln1_g, W + w.ln1_b, const_cast<__nv_bfloat16*>(xm), s.mean1, s.rstd1, T, h,
                            1e-12f, st),
           "ln1");
    }
    if (M) {
        {
            ptk_gemm_desc g = desc(T, f, h, mat(xm, h), mat(W + w.w_fc1, h), mat(s.fc1_act, f), PTK_EPI_BIAS_GELU);
            g.bias = W + w.b_fc1;
            g.c2 = s.fc1_pre;
            gemm(g, st);
        }
        {
            ptk_gemm_desc g = desc(T, h, f, mat(s.fc1_act, f), mat(W + w.w_fc2, f), mat(s.ln2, h), PTK_EPI_BF16);
            g.bias = W + w.b_fc2;
            g.aux = mat(xm, h);
            gemm(g, st);
        }
        kl(1, layernorm_fwd(s.ln2, W + w.ln2_g, W + w.ln2_b, x_out, s.mean2, s.rstd2, T, h, 1e-12f, st), "ln2");
    }
}

void GptStage::bert_layer_backward(int li, LayerStash& s, const __nv_bfloat16* dy, __nv_bfloat16* dx,
                                   cudaStream_t st) {
    const ptk_gpt_config& c = cfg_;
    const LayerW& w = lw_[li];
    const int T = tokens(), h = c.hidden, f = c.ffn;
    const __nv_bfloat16* W = wbf_;
    float* G = grad_;
    const bool A = has_attn(li), M = has_mlp(li);
    // gradient w.r.t. x_mid: from the MLP block, or the incoming gradient of an attention-only layer
    const __nv_bfloat16* gxm = dy;
    if (M) {
        const __nv_bfloat16* xm = s.x_mid;  // an MLP-only first layer: the stage input (set by forward)
        // dz = LN2'(dy)
        kl(1, layernorm_bwd(dy, s.ln2, s.mean2, s.rstd2, W + w.ln2_g, nullptr, d_ln_, vp(w.ln2_g), vp(w.ln2_b),
                            vp(w.b_fc2) /* db2 = Σ dz, fused */, T, h, st),
           "ln2 bwd");
        {  // d_pre = dz W2 * gelu'(pre); db1 = Σ d_pre fused in the epilogue
            ptk_gemm_desc g = desc(T, f, h, mat(d_ln_, h), mat(W + w.w_fc2, f, 1), mat(d_pre_, f), PTK_EPI_DGELU);
            g.aux = mat(s.fc1_pre, f);
            g.col_part = vp(w.b_fc1);
            gemm(g, st);
        }
        wgrad(desc(h, f, T, mat(d_ln_, h, 1), mat(s.fc1_act, f, 1), mat(G + w.w_fc2, f), PTK_EPI_ACC_F32), st);
        __nv_bfloat16* out = A ? dx_mid_ : dx;  // an MLP-only first layer hands d(x_mid) to the previous stage
        {  // d_xmid = d_pre W1 + dz   (residual around the FFN)
            ptk_gemm_desc g = desc(T, h, f, mat(d_pre_, f), mat(W + w.w_fc1, h, 1), mat(out, h), PTK_EPI_BF16);
            g.aux = mat(d_ln_, h);
            gemm(g, st);
        }
        wgrad(desc(f, h, T, mat(d_pre_, f, 1), mat(xm, h, 1), mat(G + w.w_fc1, h), PTK_EPI_ACC_F32), st);
        gxm = out;
    }
    if (A) {
        // dy_ = LN1'(d_xmid)
        kl(1, layernorm_bwd(gxm, s.ln1, s.mean1, s.rstd1, W + w.ln1_g, nullptr, dy_, vp(w.ln1_g), vp(w.ln1_b),
                            vp(w.b_o) /* dbo = Σ dy_, fused */, T, h, st),
           "ln1 bwd");
        gemm(desc(T, h, h, mat(dy_, h), mat(W + w.w_o, h, 1), mat(d_attn_, h), PTK_EPI_BF16), st);
        wgrad(desc(h, h, T, mat(dy_, h, 1), mat(s.attn_o, h, 1), mat(G + w.w_o, h), PTK_EPI_ACC_F32), st);
        attention_backward(s, vp(w.b_qkv), st);
        wgrad(desc(3 * h, h, T, mat(dqkv_, 3 * h, 1), mat(s.x_in, h, 1), mat(G + w.w_qkv, h), PTK_EPI_ACC_F32), st);
        {  // dx = dqkv Wqkv + dy_   (residual around attention)
            ptk_gemm_desc g = desc(T, h, 3 * h, mat(dqkv_, 3 * h), mat(W + w.w_qkv, h, 1), mat(dx, h), PTK_EPI_BF16);
            g.aux = mat(dy_, h);
            gemm(g, st);
        }
    }
}

void GptStage::layer_forward(int li, LayerStash& s, const __nv_bfloat16* x_in, __nv_bfloat16* x_out,
                             cudaStream_t st) {
    const ptk_gpt_config& c = cfg_;
    const LayerW& w = lw_[li];
    const int T = tokens(), h = c.hidden, f = c.ffn;
    const __nv_bfloat16* W = wbf_;
    const bool A = has_attn(li), M = has_mlp(li);
    // attention block: x_mid = x + attn(LN1(x)); MLP block: x_out = x_mid + mlp(LN2(x_mid)).
    // An MLP-only first layer reads x_mid = the stage input; an attention-only last layer
    // writes x_mid straight to the stage output.
    const __nv_bfloat16* xm = A ? (M ? s.x_mid : x_out) : x_in;
    if (A) {
        kl(1, layernorm_fwd(x_in, W + w.ln1_g, W + w.ln1_b, s.ln1, s.mean1, s.rstd1, T, h, 1e-5f, st), "ln1");
        {
            ptk_gemm_desc g = desc(T, 3 * h, h, mat(s.ln1, h), mat(W + w.w_qkv, h), mat(s.qkv, 3 * h), PTK_EPI_BF16);
            g.bias = W + w.b_qkv;
            gemm(g, st);
        }
        attention_forward(s, st);
        {  // x_mid = o Woᵀ + b + x
            ptk_gemm_desc g = desc(T, h, h, mat(s.attn_o, h), mat(W + w.w_o, h), mat(xm, h), PTK_EPI_BF16);
            g.bias = W + w.b_o;
            g.aux = mat(x_in, h);
            gemm(g, st);
        }
    }
    if (M) {
        kl(1, layernorm_fwd(xm, W + w.ln2_g, W + w.ln2_b, s.ln2, s.mean2, s.rstd2, T, h, 1e-5f, st), "ln2");
        {
            ptk_gemm_desc g = desc(T, f, h, mat(s.ln2, h), mat(W + w.w_fc1, h), mat(s.fc1_act, f), PTK_EPI_BIAS_GELU);
            g.bias = W + w.b_fc1;
            g.c2 = s.fc1_pre;
            gemm(g, st);
        }
        {
            ptk_gemm_desc g = desc(T, h, f, mat(s.fc1_act, f), mat(W + w.w_fc2, f), mat(x_out, h), PTK_EPI_BF16);
            g.bias = W + w.b_fc2;
            g.aux = mat(xm, h);
            gemm(g, st);
        }
    }
}

void GptStage::layer_backward(int li, LayerStash& s, const __nv_bfloat16* dy, __nv_bfloat16* dx, cudaStream_t st) {
    const ptk_gpt_config& c = cfg_;
    const LayerW& w = lw_[li];
    const int T = tokens(), h = c.hidden, f = c.ffn;
    const __nv_bfloat16* W = wbf_;
    float* G = grad_;
    const bool A = has_attn(li), M = has_mlp(li);
    // gradient w.r.t. x_mid: from the MLP block, or the incoming gradient of an attention-only layer
    const __nv_bfloat16* gxm = dy;
    if (M) {
        // FC2: d_pre = (dy W2) * gelu'(pre); dW2 += dyᵀ a; db1 = Σ d_pre fused in the epilogue
        {
            ptk_gemm_desc g = desc(T, f, h, mat(dy, h), mat(W + w.w_fc2, f, 1), mat(d_pre_, f), PTK_EPI_DGELU);
            g.aux = mat(s.fc1_pre, f);
            g.col_part = vp(w.b_fc1);
            gemm(g, st);
        }
        wgrad(desc(h, f, T, mat(dy, h, 1), mat(s.fc1_act, f, 1), mat(G + w.w_fc2, f), PTK_EPI_ACC_F32), st);
        // db2 = Σ dy: fused into the LayerNorm backward that produced dy (the next layer's LN1 or the
        // head's final LN), except for the last layer of a stage whose dy arrives from the next stage
        if (li == L_ - 1 && !c.has_head) kl(1, colsum_partial(dy, vp(w.b_fc2), T, h, st), "db2");
        // FC1: d_ln2 = d_pre W1; dW1 += d_preᵀ ln2
        gemm(desc(T, h, f, mat(d_pre_, f), mat(W + w.w_fc1, h, 1), mat(d_ln_, h), PTK_EPI_BF16), st);
        wgrad(desc(f, h, T, mat(d_pre_, f, 1), mat(s.ln2, h, 1), mat(G + w.w_fc1, h), PTK_EPI_ACC_F32), st);
        // LN2 backward + residual: d(x_mid) = LN2'(d_ln2) + dy; an MLP-only first layer hands it to the
        // previous stage, whose attention block then owns db_o
        __nv_bfloat16* out = A ? dx_mid_ : dx;
        kl(1, layernorm_bwd(d_ln_, s.x_mid, s.mean2, s.rstd2, W + w.ln2_g, dy, out, vp(w.ln2_g), vp(w.ln2_b),
                            A ? vp(w.b_o) : nullptr /* dbo = Σ d(x_mid), fused */, T, h, st),
           "ln2 bwd");
        gxm = out;
    } else {
        // attention-only last layer: dy is d(x_mid) from the next stage; db_o = Σ dy here
        kl(1, colsum_partial(dy, vp(w.b_o), T, h, st), "dbo");
    }
    if (A) {
        // out-proj: d_attn = d(x_mid) Wo; dWo += d(x_mid)ᵀ o
        gemm(desc(T, h, h, mat(gxm, h), mat(W + w.w_o, h, 1), mat(d_attn_, h), PTK_EPI_BF16), st);
        wgrad(desc(h, h, T, mat(gxm, h, 1), mat(s.attn_o, h, 1), mat(G + w.w_o, h), PTK_EPI_ACC_F32), st);
        attention_backward(s, vp(w.b_qkv), st);
        // QKV: d_ln1 = dqkv Wqkv; dWqkv += dqkvᵀ ln1; dbqkv = Σ dqkv (fused in the flash backward)
        gemm(desc(T, h, 3 * h, mat(dqkv_, 3 * h), mat(W + w.w_qkv, h, 1), mat(d_ln_, h), PTK_EPI_BF16), st);
        wgrad(desc(3 * h, h, T, mat(dqkv_, 3 * h, 1), mat(s.ln1, h, 1), mat(G + w.w_qkv, h), PTK_EPI_ACC_F32), st);
        // LN1 backward + residual: dx = LN1'(d_ln1) + d(x_mid)
        kl(1, layernorm_bwd(d_ln_, s.x_in, s.mean1, s.rstd1, W + w.ln1_g, gxm, dx, vp(w.ln1_g), vp(w.ln1_b),
                            li > 0 ? vp(lw_[li - 1].b_fc2) : nullptr /* previous layer's db2 */, T, h, st),
           "ln1 bwd");
    }
}

void GptStage::forward(int slot, const int32_t* tok, const __nv_bfloat16* x_in, const int32_t* labels,
                       __nv_bfloat16* x_out, cudaStream_t st) {
    const ptk_gpt_config& c = cfg_;
    const int T = tokens(), h = c.hidden;
    auto& S = vstash_.at(static_cast<size_t>(slot));
    const __nv_bfloat16* W = wbf_;
    const __nv_bfloat16* cur = x_in;
    if (c.has_embedding && bert()) {  // BERT: LN(wte[tok] + wpe[pos])
        EmbStash& e = vemb_.at(static_cast<size_t>(slot));
        kl(1, embedding_fwd(tok, W + wte_, W + wpe_, e.sum, T, c.seq, h, st), "embedding");
        __nv_bfloat16* dst = L_ > 0 ? S[0].x_in : vhead_.at(static_cast<size_t>(slot)).x_fin;
        kl(1, layernorm_fwd(e.sum, W + lne_g_, W + lne_b_, dst, e.mean, e.rstd, T, h, 1e-12f, st), "emb ln");
        cur = dst;
    } else if (c.has_embedding) {
        kl(1, embedding_fwd(tok, W + wte_, W + wpe_, S[0].x_in, T, c.seq, h, st), "embedding");
        cur = S[0].x_in;
    } else if (L_ > 0) {
        // the stage input stays live until this slot's backward
        if (has_attn(0))
            S[0].x_in = const_cast<__nv_bfloat16*>(x_in);
        else
            S[0].x_mid = const_cast<__nv_bfloat16*>(x_in);
    }
    for (int i = 0; i < L_; ++i) {
        __nv_bfloat16* out = (i + 1 < L_) ? S[i + 1].x_in : (c.has_head ? vhead_.at(static_cast<size_t>(slot)).x_fin : x_out);
        if (bert())
            bert_layer_forward(i, S[i], cur, out, st);
        else
            layer_forward(i, S[i], cur, out, st);
        cur = out;
    }
    if (c.has_head) {
        HeadStash& hs = vhead_.at(static_cast<size_t>(slot));
        if (L_ == 0 && cur != hs.x_fin)
            ck(cudaMemcpyAsync(hs.x_fin, cur, static_cast<size_t>(T) * h * 2, cudaMemcpyDeviceToDevice, st), "copy");
        if (bert()) {  // MLM transform: t = gelu(x Wtᵀ + b), xf = LN(t)
            ptk_gemm_desc g = desc(T, h, h, mat(hs.x_fin, h), mat(W + w_t_, h), mat(hs.t_act, h), PTK_EPI_BIAS_GELU);
            g.bias = W + b_t_;
            g.c2 = hs.t_pre;
            gemm(g, st);
            kl(1, layernorm_fwd(hs.t_act, W + lnf_g_, W + lnf_b_, hs.xf, hs.meanf, hs.rstdf, T, h, 1e-12f, st), "lnh");
        } else {
            kl(1, layernorm_fwd(hs.x_fin, W + lnf_g_, W + lnf_b_, hs.xf, hs.meanf, hs.rstdf, T, h, 1e-5f, st), "lnf");
        }
        gemm(desc(T, c.vocab, h, mat(hs.xf, h), mat(W + w_head_, h), mat(hs.dlogits, c.vocab), PTK_EPI_BF16), st);
        const float scale = 1.f / (static_cast<float>(T) * c.micro_batches);
        kl(2, cross_entropy(hs.dlogits, labels, loss_rows_, loss_acc_, T, c.vocab, scale, scale, st), "xent");
    } else if (L_ == 0) {
        ck(cudaMemcpyAsync(x_out, cur, static_cast<size_t>(T) * h * 2, cudaMemcpyDeviceToDevice, st), "copy");
    }
}

void GptStage::backward(int slot, const int32_t* tok, const __nv_bfloat16* dy, __nv_bfloat16* dx, cudaStream_t st) {
    const ptk_gpt_config& c = cfg_;
    const int T = tokens(), h = c.hidden;
    auto& S = vstash_.at(static_cast<size_t>(slot));
    const __nv_bfloat16* W = wbf_;
    float* G = grad_;
    const __nv_bfloat16* g = dy;
    // Paired weight gradients, balanced: layers of even global index pair backwards (0,1), (2,3),
    // ... and layers of odd index (1,2), (3,4), ... (0 and an unpaired last one run alone), the head
    // counting as layer n_layer.  Every backward then defers about half of the weight gradients and
    // runs the other half as pairs, so consecutive backwards cost the same (1F1B's strict F/B
    // alternation would otherwise see alternating short and long backwards).  Pairs depend only on
    // the backward count, ascending for every plan: bit-identical across k and stage splits.
    const int n = wg_count_++;
    auto mode_of = [&](int global_layer) -> int {
        if (!pairs_on_) return 0;
        const bool odd = (global_layer & 1) != 0;
        if (odd ? (n & 1) != 0 : (n & 1) == 0) return 1;  // this backward defers the layer
        return (!odd || n >= 2) ? 2 : 0;                   // pair with the deferred one (odd layers: none at n = 0)
    };
    wg_mode_ = mode_of(c.n_layer);
    // the top layer's input gradient is an operand of its (deferred) FC2 weight gradient
    const bool top_defers = L_ > 0 && mode_of(c.layer_begin + L_ - 1) == 1;
    __nv_bfloat16* head_g = top_defers ? dhead_g_ : g_a_;
    if (wg_mode_ == 1) dy_ = dhead_dy_;  // the head's own deferred operand (BERT transform)
    if (c.has_head) {
        HeadStash& hs = vhead_.at(static_cast<size_t>(slot));
        // dxf = dlogits W_head ; dW_head += dlogitsᵀ xf
        gemm(desc(T, h, c.vocab, mat(hs.dlogits, c.vocab), mat(W + w_head_, h, 1), mat(d_ln_, h), PTK_EPI_BF16), st);
        wgrad(desc(c.vocab, h, T, mat(hs.dlogits, c.vocab, 1), mat(hs.xf, h, 1), mat(G + w_head_, h), PTK_EPI_ACC_F32), st);
        if (bert()) {
            // dt = LN_h'(dxf); d_tpre = dt * gelu'(t_pre); dx_fin = d_tpre Wt; dWt += d_tpreᵀ x_fin
            kl(1, layernorm_bwd(d_ln_, hs.t_act, hs.meanf, hs.rstdf, W + lnf_g_, nullptr, dx_mid_, vp(lnf_g_),
                                vp(lnf_b_), nullptr, T, h, st),
               "lnh bwd");
            kl(1, dgelu_mul(dx_mid_, hs.t_pre, dy_, static_cast<int64_t>(T) * h, st), "dgelu");
            gemm(desc(T, h, h, mat(dy_, h), mat(W + w_t_, h, 1), mat(head_g, h), PTK_EPI_BF16), st);
            wgrad(desc(h, h, T, mat(dy_, h, 1), mat(hs.x_fin, h, 1), mat(G + w_t_, h), PTK_EPI_ACC_F32), st);
            kl(1, colsum_partial(dy_, vp(b_t_), T, h, st), "dbt");
        } else {
            kl(1, layernorm_bwd(d_ln_, hs.x_fin, hs.meanf, hs.rstdf, W + lnf_g_, nullptr, head_g, vp(lnf_g_),
                                vp(lnf_b_), L_ > 0 ? vp(lw_[L_ - 1].b_fc2) : nullptr /* last layer's db2 */, T, h,
                                st),
               "lnf bwd");
        }
        g = head_g;
    }
    if (pairs_on_) use_scratch(-1);
    for (int i = L_ - 1; i >= 0; --i) {
        wg_mode_ = mode_of(c.layer_begin + i);
        // layer i's output gradient feeds layer i-1's FC2 weight gradient: persistent if that one defers
        const bool consumer_defers = i > 0 && mode_of(c.layer_begin + i - 1) == 1;
        __nv_bfloat16* out = (i == 0 && !c.has_embedding) ? dx
                             : consumer_defers              ? dbuf_[static_cast<size_t>(i)].out
                                                            : (g == g_a_ ? g_b_ : g_a_);
        if (pairs_on_) use_scratch(wg_mode_ == 1 ? i : -1);
        if (bert())
            bert_layer_backward(i, S[i], g, out, st);
        else
            layer_backward(i, S[i], g, out, st);
        g = out;
    }
    if (pairs_on_) use_scratch(-1);
    wg_mode_ = 0;
    if (c.has_embedding && bert()) {  // through the embedding LayerNorm
        EmbStash& e = vemb_.at(static_cast<size_t>(slot));
        __nv_bfloat16* dsum_bf = (g == g_a_) ? g_b_ : g_a_;
        kl(1, layernorm_bwd(g, e.sum, e.mean, e.rstd, W + lne_g_, nullptr, dsum_bf, vp(lne_g_), vp(lne_b_), nullptr, T,
                            h, st),
           "emb ln bwd");
        g = dsum_bf;
    }
    if (c.has_embedding) {
        kl(3, embedding_bwd(tok, g, G + wte_, G + wpe_, order_, T, c.seq, h, c.vocab, st), "embedding bwd");
    } else if (L_ == 0) {
        ck(cudaMemcpyAsync(dx, g, static_cast<size_t>(T) * h * 2, cudaMemcpyDeviceToDevice, st), "copy");
    }
}

float* GptStage::vp(int64_t offset) {
    auto it = vparts_.find(offset);
    if (it == vparts_.end()) throw std::logic_error("no gradient partials for a 1-D parameter");
    return it->second;
}

void GptStage::finalize_grads(cudaStream_t st) {
    flush_wgrads(st);
    kl(1, vec_grad_finalize(vsegs_, nvseg_, vseg_max_cols_, st), "finalize grads");
}

void GptStage::optimizer_step(float lr, float wd, cudaStream_t st) {
    finalize_grads(st);
    ++step_;
    kl(1, adamw_step(master_, grad_, adam_m_, adam_v_, wbf_, total_, lr, 0.9f, 0.95f, 1e-8f, wd, step_, st), "adamw");
}

void GptStage::collect_timing() {
    for (size_t i = 0; i + 1 < timing_.used; i += 2) {
        ck(cudaEventSynchronize(timing_.pool[i + 1]), "event sync");
        float ms = 0.f;
        ck(cudaEventElapsedTime(&ms, timing_.pool[i], timing_.pool[i + 1]), "elapsed");
        timing_.total_ms += ms;
        timing_.total_flops += timing_.flops[i / 2];
        ++timing_.launches;
    }
    timing_.used = 0;
    timing_.flops.clear();
}

void GptStage::zero_grads(cudaStream_t st) {
    wg_pending_.clear();
    wg_count_ = 0;
    ck(cudaMemsetAsync(grad_, 0, total_ * 4, st), "zero grads");
    for (const auto& kv : vparts_) {
        const ParamInfo* p = nullptr;
        for (const ParamInfo& q : params_)
            if (q.offset == kv.first) p = &q;
        ck(cudaMemsetAsync(kv.second, 0, static_cast<size_t>(kVecParts) * p->cols * 4, st), "zero partials");
    }
}

}  // namespace ptk
