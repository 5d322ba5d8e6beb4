// kFkB stage executor — see executor.h.
#include "executor.h"
#include "preload.h"

#include <cuda.h>

#include <algorithm>
#include <cstdlib>
#include <string>
#include <cstring>
#include <mutex>
#include <chrono>
#include <stdexcept>
#include <thread>

#include "pipetune/errors.hpp"

namespace ptk {

namespace {

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

using WaitValueFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
using WriteValueFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

struct StreamOps {
    WaitValueFn wait = nullptr;
    WriteValueFn write = nullptr;
};

const StreamOps& stream_ops() {
    static StreamOps ops;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            ops.wait = reinterpret_cast<WaitValueFn>(p);
        if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            ops.write = reinterpret_cast<WriteValueFn>(p);
    });
    if (!ops.wait || !ops.write) throw std::runtime_error("cuStreamWaitValue32/WriteValue32 unavailable");
    return ops;
}

void wait_flag(cudaStream_t st, const uint32_t* flag, uint32_t value) {
    const CUresult r = stream_ops().wait(reinterpret_cast<CUstream>(st), reinterpret_cast<CUdeviceptr>(flag), value,
                                         CU_STREAM_WAIT_VALUE_GEQ);
    if (r != CUDA_SUCCESS) throw std::runtime_error("cuStreamWaitValue32 failed: " + std::to_string(r));
}

void write_flag(cudaStream_t st, uint32_t* flag, uint32_t value) {
    const CUresult r = stream_ops().write(reinterpret_cast<CUstream>(st), reinterpret_cast<CUdeviceptr>(flag), value,
                                          CU_STREAM_WRITE_VALUE_DEFAULT);
    if (r != CUDA_SUCCESS) throw std::runtime_error("cuStreamWriteValue32 failed: " + std::to_string(r));
}

uint64_t mix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

constexpr size_t kHandle = sizeof(cudaIpcMemHandle_t);

}  // namespace

Executor::Executor(const ptk_exec_config& c) : cfg_(c) {
    if (c.stages < 1 || c.stage < 0 || c.stage >= c.stages || c.global_batch < 1)
        throw std::invalid_argument("Executor: bad stage / global batch");
    preload_all_kernels();  // no lazy module loading behind another stage's waiting streams
    int lo = 0, hi = 0;
    ck(cudaDeviceGetStreamPriorityRange(&lo, &hi), "priorities");
    if (std::getenv("PTK_FLAT_PRIORITY") != nullptr) hi = lo;  // diagnostics: all streams at one priority
    ck(cudaStreamCreateWithPriority(&comp_, cudaStreamNonBlocking, hi), "stream");
    // send streams at the highest priority: their only kernels are the emulator's one-thread trace
    // gates, which would otherwise wait behind every pending compute CTA for an SM slot
    ck(cudaStreamCreateWithPriority(&sendst_, cudaStreamNonBlocking, hi), "stream");
    ck(cudaStreamCreateWithPriority(&sendst_bwd_, cudaStreamNonBlocking, hi), "stream");
    if (const char* v = std::getenv("PTK_DEADLOCK_TIMEOUT_S")) deadlock_timeout_s_ = std::atof(v);
    if (const char* v = std::getenv("PTK_SEND_STREAMS")) per_link_send_ = std::string(v) == "per_link";
    ck(cudaStreamCreateWithPriority(&contend_[0], cudaStreamNonBlocking, lo), "stream");
    ck(cudaStreamCreateWithPriority(&contend_[1], cudaStreamNonBlocking, lo), "stream");
    stage_ = std::make_unique<GptStage>(c.gpt);
    ck(cudaEventCreate(&it_start_), "event");
    ck(cudaEventCreate(&it_end_), "event");
    ck(cudaEventCreateWithFlags(&h2d_done_, cudaEventDisableTiming), "event");
    ck(cudaEventRecord(h2d_done_, comp_), "event");
    alloc_comm();
    set_plan(1, c.gpt.micro_batch_size);
}

Executor::~Executor() {
    emu_.stop_contender();
    if (in_iteration_ || poisoned_) {  // half-enqueued or deadlocked: open this stage's flags so nothing waits forever
        poisoned_ = true;
        try {
            open_flags();
        } catch (...) {
        }
    }
    cudaStreamSynchronize(comp_);
    cudaStreamSynchronize(sendst_);
    cudaStreamSynchronize(sendst_bwd_);
    cudaStreamSynchronize(contend_[0]);
    cudaStreamSynchronize(contend_[1]);
    for (void* p : ipc_opened_) cudaIpcCloseMemHandle(p);
    for (cudaEvent_t e : pool_) cudaEventDestroy(e);
    for (cudaEvent_t e : act_sent_) cudaEventDestroy(e);
    for (cudaEvent_t e : grad_sent_) cudaEventDestroy(e);
    cudaEventDestroy(it_start_);
    cudaEventDestroy(it_end_);
    cudaEventDestroy(h2d_done_);
    for (void* p : allocs_) cudaFree(p);
    if (host_stage_) cudaFreeHost(host_stage_);
    cudaStreamDestroy(comp_);
    cudaStreamDestroy(sendst_);
    cudaStreamDestroy(sendst_bwd_);
    if (rescue_) cudaStreamDestroy(rescue_);
    cudaStreamDestroy(contend_[0]);
    cudaStreamDestroy(contend_[1]);
}

void Executor::alloc_comm() {
    const ptk_gpt_config& g = cfg_.gpt;
    const int64_t block = static_cast<int64_t>(cfg_.global_batch) * g.seq * g.hidden * 2;
    const int64_t tmax = static_cast<int64_t>(g.micro_batch_size) * g.seq;
    auto dalloc = [this](size_t n) {
        void* p = nullptr;
        ck(cudaMalloc(&p, n), "cudaMalloc comm");
        ck(cudaMemset(p, 0, n), "memset");
        allocs_.push_back(p);
        return p;
    };
    if (cfg_.stage > 0) {
        act_recv_ = static_cast<__nv_bfloat16*>(dalloc(block));
        act_flag_ = static_cast<uint32_t*>(dalloc(cfg_.global_batch * 4 + 256));
        for (int s = 0; s < g.slots; ++s) grad_send_.push_back(static_cast<__nv_bfloat16*>(dalloc(tmax * g.hidden * 2)));
        for (int s = 0; s < g.slots * g.micro_batch_size; ++s) {  // one per virtual slot at b = 1
            cudaEvent_t e;
            ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
            ck(cudaEventRecord(e, sendst_), "event");
            grad_sent_.push_back(e);
        }
    }
    if (cfg_.stage + 1 < cfg_.stages) {
        grad_recv_ = static_cast<__nv_bfloat16*>(dalloc(block));
        grad_flag_ = static_cast<uint32_t*>(dalloc(cfg_.global_batch * 4 + 256));
        for (int s = 0; s < g.slots; ++s) act_send_.push_back(static_cast<__nv_bfloat16*>(dalloc(tmax * g.hidden * 2)));
        for (int s = 0; s < g.slots * g.micro_batch_size; ++s) {
            cudaEvent_t e;
            ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
            ck(cudaEventRecord(e, sendst_), "event");
            act_sent_.push_back(e);
        }
    }
    if (cfg_.stages > 1) scratch_ = dalloc(kScratch);
    gt_start_ = static_cast<int64_t*>(dalloc(64));
    const int64_t toks = static_cast<int64_t>(cfg_.global_batch) * g.seq;
    tok_dev_ = static_cast<int32_t*>(dalloc(toks * 4));
    lab_dev_ = static_cast<int32_t*>(dalloc(toks * 4));
    ck(cudaHostAlloc(&host_stage_, toks * 2 * 4, cudaHostAllocDefault), "pinned");
}

std::vector<uint8_t> Executor::export_handles() const {
    std::vector<uint8_t> out(5 * (1 + kHandle), 0);
    const void* ptrs[5] = {act_recv_, act_flag_, grad_recv_, grad_flag_, scratch_};
    for (int i = 0; i < 5; ++i) {
        if (!ptrs[i]) continue;
        cudaIpcMemHandle_t h;
        ck(cudaIpcGetMemHandle(&h, const_cast<void*>(ptrs[i])), "ipc get");
        out[i * (1 + kHandle)] = 1;
        std::memcpy(&out[i * (1 + kHandle) + 1], &h, kHandle);
    }
    return out;
}

void Executor::import_peer(int peer, const uint8_t* bytes, size_t n) {
    if (n < 5 * (1 + kHandle)) throw std::invalid_argument("import_peer: short handle blob");
    auto open = [&](int i) -> void* {
        if (!bytes[i * (1 + kHandle)]) throw std::invalid_argument("import_peer: peer lacks the needed buffer");
        cudaIpcMemHandle_t h;
        std::memcpy(&h, bytes + i * (1 + kHandle) + 1, kHandle);
        void* p = nullptr;
        ck(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess), "ipc open");
        ipc_opened_.push_back(p);
        return p;
    };
    if (peer == cfg_.stage + 1) {
        peer_act_recv_ = static_cast<__nv_bfloat16*>(open(0));
        peer_act_flag_ = static_cast<uint32_t*>(open(1));
        peer_scratch_fwd_ = open(4);
    } else if (peer == cfg_.stage - 1) {
        peer_grad_recv_ = static_cast<__nv_bfloat16*>(open(2));
        peer_grad_flag_ = static_cast<uint32_t*>(open(3));
        peer_scratch_bwd_ = open(4);
    } else {
        throw std::invalid_argument("import_peer: not an adjacent stage");
    }
}

void Executor::connect_local(int peer, Executor& p) {
    if (peer == cfg_.stage + 1) {
        peer_act_recv_ = p.act_recv_;
        peer_act_flag_ = p.act_flag_;
        peer_scratch_fwd_ = p.scratch_;
    } else if (peer == cfg_.stage - 1) {
        peer_grad_recv_ = p.grad_recv_;
        peer_grad_flag_ = p.grad_flag_;
        peer_scratch_bwd_ = p.scratch_;
    } else {
        throw std::invalid_argument("connect_local: not an adjacent stage");
    }
}

void Executor::set_plan(int k, int b) {
    if (b < 1 || cfg_.global_batch % b) throw pipetune::ConfigError("set_plan: micro-batch size must divide the global batch");
    const int M = cfg_.global_batch / b;
    std::vector<int> sizes;
    for (int first = 0; first < M; first += k) sizes.push_back(std::min(k, M - first));
    install_plan(b, sizes, k);
}

void Executor::set_plan_groups(int b, const std::vector<int>& group_sizes) {
    int kmax = 0;
    for (int n : group_sizes) kmax = std::max(kmax, n);
    install_plan(b, group_sizes, kmax);
}

void Executor::install_plan(int b, const std::vector<int>& group_sizes, int k) {
    const ptk_gpt_config& g = cfg_.gpt;
    if (b < 1 || b > g.micro_batch_size || cfg_.global_batch % b)
        throw pipetune::ConfigError("set_plan: micro-batch size must divide the global batch and be <= b_max");
    if (k < 1) throw pipetune::ConfigError("set_plan: k must be >= 1");
    pipetune::ModelSpec spec;
    spec.global_batch = cfg_.global_batch;
    for (int s = 0; s < cfg_.stages; ++s) {
        pipetune::StageProfile p;
        p.stage_id = s;
        p.output_bytes_per_sample_fwd = static_cast<pipetune::Bytes>(g.seq) * g.hidden * 2;
        p.output_bytes_per_sample_bwd = p.output_bytes_per_sample_fwd;
        spec.stages.push_back(p);
    }
    pipetune::PlanConfig pc{1, b, cfg_.global_batch / b};
    graph_ = std::make_shared<const pipetune::TaskGraph>(pipetune::build_task_graph(spec, pc));
    std::vector<pipetune::MicroBatchGroup> groups;
    int first = 0;
    for (int n : group_sizes) {
        if (n < 1) throw pipetune::ConfigError("set_plan_groups: group sizes must be >= 1");
        groups.push_back({first, first + n - 1});
        first += n;
    }
    plan_ = pipetune::plan_groups(graph_, k, groups);  // throws PlanError unless the groups tile [0, M)
    // the stash must hold this stage's peak number of in-flight micro-batches
    int live = 0, peak = 0;
    for (int id : plan_.per_device[static_cast<size_t>(cfg_.stage)]) {
        const auto kind = graph_->node(id).kind;
        if (kind == pipetune::TaskKind::ForwardCompute) peak = std::max(peak, ++live);
        if (kind == pipetune::TaskKind::BackwardCompute) --live;
    }
    // paired weight gradients keep the previous micro-batch's slot live one backward longer
    if (g.wgrad_pairs) ++peak;
    // slots are b_max samples wide: at b | b_max each holds b_max / b micro-batches
    const int vslots = g.slots * ((g.micro_batch_size % b == 0) ? g.micro_batch_size / b : 1);
    if (peak > vslots)
        throw pipetune::InfeasibleModel("set_plan: k=" + std::to_string(k) + " b=" + std::to_string(b) + " needs " +
                                        std::to_string(peak) + " stash slots, stage has " + std::to_string(vslots));
    k_ = k;
    b_ = b;
    M_ = cfg_.global_batch / b;
    groups_ = group_sizes;
    stage_->set_micro_batch(b, M_);
}

void Executor::set_trace(int link, const EmuTrace& t) {
    const int slot = (link == 2 * cfg_.stage) ? 0 : (link == 2 * cfg_.stage - 1 ? 1 : -1);
    if (slot < 0) throw std::invalid_argument("set_trace: link is not outgoing from this stage");
    emu_.set_trace(slot, t);
}

void Executor::set_epoch(int64_t epoch_ns) { emu_.set_epoch(epoch_ns); }

cudaEvent_t Executor::ev() {
    if (pool_used_ == pool_.size()) {
        cudaEvent_t e;
        ck(cudaEventCreate(&e), "event");
        pool_.push_back(e);
    }
    return pool_[pool_used_++];
}

void Executor::synth_tokens(int iter, int32_t* dst) const {
    // Synthetic corpus: tokens uniform in [0, V) from a counter-based hash of
    // (seed, iteration, sample, position); labels are the next token.
    const ptk_gpt_config& g = cfg_.gpt;
    const int64_t gb = cfg_.global_batch, s = g.seq;
    int32_t* tok = dst;
    int32_t* lab = dst + gb * s;
    for (int64_t i = 0; i < gb; ++i) {
        uint64_t base = mix64(cfg_.data_seed ^ mix64(static_cast<uint64_t>(iter) * 0x10001ull + static_cast<uint64_t>(i)));
        int32_t prev = static_cast<int32_t>(mix64(base) % static_cast<uint64_t>(g.vocab));
        for (int64_t p = 0; p < s; ++p) {
            const int32_t next = static_cast<int32_t>(mix64(base + static_cast<uint64_t>(p) + 1) % static_cast<uint64_t>(g.vocab));
            tok[i * s + p] = prev;
            lab[i * s + p] = next;
            prev = next;
        }
    }
}

void Executor::send(bool fwd, int mb, const __nv_bfloat16* src, int64_t bytes, cudaEvent_t ready) {
    const ptk_gpt_config& g = cfg_.gpt;
    __nv_bfloat16* dst_block = fwd ? peer_act_recv_ : peer_grad_recv_;
    uint32_t* flag = fwd ? peer_act_flag_ : peer_grad_flag_;
    if (!dst_block || !flag) throw std::runtime_error("send: peer not connected");
    const int64_t off = static_cast<int64_t>(mb) * b_ * g.seq * g.hidden;
    cudaStream_t st = send_stream(fwd);
    ck(cudaStreamWaitEvent(st, ready, 0), "wait");
    XferRecord r{fwd ? 2 * cfg_.stage : 2 * cfg_.stage - 1, mb, bytes, ev(), ev()};
    ck(cudaEventRecord(r.start, st), "event");
    ck(emu_.paced_copy(fwd ? 0 : 1, dst_block + off, src, bytes, st), "peer copy");
    if (emu_.active(fwd ? 0 : 1)) emu_launches_ += 1;
    write_flag(st, flag + mb, epoch_);
    ck(cudaEventRecord(r.end, st), "event");
    xrec_.push_back(r);
}

void Executor::run_iteration(int iter, const int32_t* host_tokens) {
    begin_iteration(iter, host_tokens);
    while (enqueue_next()) {
    }
}

void Executor::begin_iteration(int iter, const int32_t* host_tokens) {
    if (poisoned_) throw pipetune::DeadlockDetected("executor poisoned by an earlier deadlock; destroy it");
    if (in_iteration_) throw std::logic_error("begin_iteration: the previous iteration is still being enqueued");
    const ptk_gpt_config& g = cfg_.gpt;
    const int S = cfg_.stages, s = cfg_.stage;
    const bool first = s == 0, last = s == S - 1;
    const int64_t toks = static_cast<int64_t>(cfg_.global_batch) * g.seq;
    validate_tokens(host_tokens);  // before any state changes
    iter_ = iter;
    ++epoch_;
    cursor_ = 0;
    in_iteration_ = true;
    pool_used_ = 0;
    crec_.clear();
    xrec_.clear();
    stage_->reset_launches();

    // data for this iteration (host -> device inside the iteration, e2e);
    // the pinned staging buffer is free once the previous iteration's H2D ran
    ck(cudaEventSynchronize(h2d_done_), "h2d wait");
    if (host_tokens)
        std::memcpy(host_stage_, host_tokens, static_cast<size_t>(toks) * 2 * 4);
    else
        synth_tokens(iter, host_stage_);
    ck(cudaEventRecord(it_start_, comp_), "event");
    ck(record_globaltimer(gt_start_, comp_), "globaltimer");  // the iteration start on the device clock
    ck(cudaStreamWaitEvent(sendst_, it_start_, 0), "wait");
    ck(cudaStreamWaitEvent(sendst_bwd_, it_start_, 0), "wait");
    h2d_bytes_ = 0;
    if (first) {
        ck(cudaMemcpyAsync(tok_dev_, host_stage_, toks * 4, cudaMemcpyHostToDevice, comp_), "h2d");
        h2d_bytes_ += toks * 4;
    }
    if (last) {
        ck(cudaMemcpyAsync(lab_dev_, host_stage_ + toks, toks * 4, cudaMemcpyHostToDevice, comp_), "h2d");
        h2d_bytes_ += toks * 4;
    }
    ck(cudaEventRecord(h2d_done_, comp_), "event");
    if (last) ck(cudaMemsetAsync(stage_->loss_accumulator(), 0, 4, comp_), "memset");
    if (contender_on_) {  // competing NVLink stores while a trace is in a preempted segment
        if (peer_scratch_fwd_) ck(emu_.start_contender(0, peer_scratch_fwd_, kScratch, contend_[0]), "contender");
        if (peer_scratch_bwd_) ck(emu_.start_contender(1, peer_scratch_bwd_, kScratch, contend_[1]), "contender");
    }
    emu_launches_ = 0;
}

void Executor::validate_tokens(const int32_t* host_tokens) const {
    // ids index the embedding / LM-head rows on the device: an out-of-range one is a ConfigError
    // here instead of a faulting kernel
    if (!host_tokens) return;
    const ptk_gpt_config& g = cfg_.gpt;
    const int64_t n = 2 * static_cast<int64_t>(cfg_.global_batch) * g.seq;
    for (int64_t i = 0; i < n; ++i)
        if (static_cast<uint32_t>(host_tokens[i]) >= static_cast<uint32_t>(g.vocab))
            throw pipetune::ConfigError("run_iteration: token/label id " + std::to_string(host_tokens[i]) + " at " +
                                        std::to_string(i) + " outside [0, vocab)");
}

void Executor::peek_next(int* kind, int* mb) const {
    const auto& order = plan_.per_device[static_cast<size_t>(cfg_.stage)];
    if (!in_iteration_ || cursor_ >= order.size()) {
        *kind = -1;
        *mb = -1;
        return;
    }
    const pipetune::TaskNode& n = graph_->node(order[cursor_]);
    *kind = n.kind == pipetune::TaskKind::ForwardCompute ? 0 : n.kind == pipetune::TaskKind::BackwardCompute ? 1 : 2;
    *mb = n.micro_batch;
}

bool Executor::enqueue_next() {
    if (!in_iteration_) return false;
    const auto& order = plan_.per_device[static_cast<size_t>(cfg_.stage)];
    if (cursor_ < order.size()) enqueue_node(order[cursor_++]);
    if (cursor_ < order.size()) return true;
    ck(cudaEventRecord(it_end_, comp_), "event");
    in_iteration_ = false;
    return false;
}

void Executor::enqueue_node(int id) {
    const ptk_gpt_config& g = cfg_.gpt;
    const int S = cfg_.stages, s = cfg_.stage;
    const bool first = s == 0, last = s == S - 1;
    const int64_t T = static_cast<int64_t>(b_) * g.seq;
    const int64_t act_bytes = T * g.hidden * 2;
    const pipetune::TaskNode& n = graph_->node(id);
    const int m = n.micro_batch;
    const int slot = m >= 0 ? m % stage_->virtual_slots() : 0;
    // this micro-batch's view of the b_max-wide send buffer of its physical slot
    const int split = stage_->slot_split();
    const int64_t sub = static_cast<int64_t>(slot % split) * T * g.hidden;
    GemmTiming& tm = stage_->gemm_timing();
    // one micro-batch in `stride`, rotating with the iteration so paired and unpaired weight-gradient
    // micro-batches (and PDL-overlapped ones) are all sampled over a run
    const int period = std::max(1, std::min(tm.stride, M_));
    tm.enabled = tm.armed && m >= 0 && m % tm.stride == static_cast<int>(epoch_ % static_cast<uint32_t>(period));
    if (n.kind == pipetune::TaskKind::ForwardCompute) {
        if (!first) wait_flag(comp_, act_flag_ + m, epoch_);
        __nv_bfloat16* out = last ? nullptr : act_send_[static_cast<size_t>(slot / split)] + sub;
        if (!last) ck(cudaStreamWaitEvent(comp_, act_sent_[static_cast<size_t>(slot)], 0), "wait");
        CompRecord r{id, 0, m, ev(), ev()};
        ck(cudaEventRecord(r.start, comp_), "event");
        stage_->forward(slot, tok_dev_ + m * T, first ? nullptr : act_recv_ + m * T * g.hidden, lab_dev_ + m * T,
                        out, comp_);
        ck(cudaEventRecord(r.end, comp_), "event");
        crec_.push_back(r);
        if (!last) {
            send(true, m, out, act_bytes, r.end);
            ck(cudaEventRecord(act_sent_[static_cast<size_t>(slot)], send_stream(true)), "event");
        }
    } else if (n.kind == pipetune::TaskKind::BackwardCompute) {
        if (!last) wait_flag(comp_, grad_flag_ + m, epoch_);
        __nv_bfloat16* dx = first ? nullptr : grad_send_[static_cast<size_t>(slot / split)] + sub;
        if (!first) ck(cudaStreamWaitEvent(comp_, grad_sent_[static_cast<size_t>(slot)], 0), "wait");
        CompRecord r{id, 1, m, ev(), ev()};
        ck(cudaEventRecord(r.start, comp_), "event");
        stage_->backward(slot, tok_dev_ + m * T, last ? nullptr : grad_recv_ + m * T * g.hidden, dx, comp_);
        ck(cudaEventRecord(r.end, comp_), "event");
        crec_.push_back(r);
        if (!first) {
            send(false, m, dx, act_bytes, r.end);
            ck(cudaEventRecord(grad_sent_[static_cast<size_t>(slot)], send_stream(false)), "event");
        }
    } else if (n.kind == pipetune::TaskKind::GradAccum) {
        CompRecord r{id, 2, -1, ev(), ev()};
        ck(cudaEventRecord(r.start, comp_), "event");
        if (defer_optimizer_)
            stage_->finalize_grads(comp_);  // the caller all-reduces, then steps the optimizer
        else
            stage_->optimizer_step(cfg_.lr, cfg_.weight_decay, comp_);
        ck(cudaEventRecord(r.end, comp_), "event");
        crec_.push_back(r);
    }
}

void run_local_pipeline(const std::vector<Executor*>& st, int iter, const int32_t* host_tokens) {
    const int S = static_cast<int>(st.size());
    for (int s = 0; s < S; ++s)
        if (!st[s] || st[s]->cfg().stage != s || st[s]->cfg().stages != S)
            throw std::invalid_argument("run_local_pipeline: stages[s] must be stage s of an S-stage pipeline");
    for (Executor* e : st) e->validate_tokens(host_tokens);  // all or none of the stages begin
    for (Executor* e : st) e->begin_iteration(iter, host_tokens);
    // enqueued forwards / backwards per stage (both ascending in every plan)
    std::vector<int> nf(static_cast<size_t>(S), 0), nb(static_cast<size_t>(S), 0);
    std::vector<bool> done(static_cast<size_t>(S), false);
    int left = S;
    while (left > 0) {
        bool progress = false;
        for (int s = 0; s < S; ++s) {
            for (;;) {
                if (done[s]) break;
                int kind = -1, mb = -1;
                st[s]->peek_next(&kind, &mb);
                const bool ready = kind == 2 || (kind == 0 && (s == 0 || nf[s - 1] > mb)) ||
                                   (kind == 1 && (s == S - 1 || nb[s + 1] > mb));
                if (!ready) break;
                if (kind == 0) ++nf[s];
                if (kind == 1) ++nb[s];
                if (!st[s]->enqueue_next()) {
                    done[s] = true;
                    --left;
                }
                progress = true;
            }
        }
        if (!progress)
            throw pipetune::DeadlockDetected("run_local_pipeline: no stage can enqueue its next node");
    }
}

double Executor::finish_iteration() {
    if (in_iteration_) throw std::logic_error("finish_iteration: the iteration is not fully enqueued");
    // Poll instead of blocking: a stage whose peer never sends waits forever in
    // cuStreamWaitValue32; SPEC's DeadlockDetected (errors.hpp) is raised instead.
    cudaEvent_t send_done = ev(), send_bwd_done = ev();
    ck(cudaEventRecord(send_done, sendst_), "event");
    ck(cudaEventRecord(send_bwd_done, sendst_bwd_), "event");
    const auto t0 = std::chrono::steady_clock::now();
    auto finished = [&] {
        for (cudaEvent_t e : {it_end_, send_done, send_bwd_done}) {
            const cudaError_t q = cudaEventQuery(e);
            if (q == cudaErrorNotReady) return false;
            ck(q, "event query");
        }
        return true;
    };
    int spins = 0;
    while (!finished()) {
        const double waited = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (waited > deadlock_timeout_s_) {
            poisoned_ = true;
            open_flags();  // this stage's streams drain (their inputs are garbage from here)
            emu_.stop_contender();
            throw pipetune::DeadlockDetected("stage " + std::to_string(cfg_.stage) + ": iteration not finished after " +
                                             std::to_string(deadlock_timeout_s_) + " s (a peer never delivered)");
        }
        if (++spins > 64) std::this_thread::sleep_for(std::chrono::microseconds(spins > 4096 ? 1000 : 50));
    }
    if (contender_on_) {
        emu_.stop_contender();
        ck(cudaStreamSynchronize(contend_[0]), "sync contender");
        ck(cudaStreamSynchronize(contend_[1]), "sync contender");
    }
    float ms = 0.f;
    ck(cudaEventElapsedTime(&ms, it_start_, it_end_), "elapsed");
    return ms;
}

void Executor::open_flags() {
    // cuStreamWaitValue32 GEQ is a cyclic comparison ((int32)(*flag - value) >= 0): a value half the
    // counter range ahead of the current epoch satisfies every wait of this and later epochs
    std::vector<uint32_t> v(static_cast<size_t>(cfg_.global_batch), epoch_ + (1u << 30));
    for (uint32_t* f : {act_flag_, grad_flag_})
        if (f) ck(cudaMemcpyAsync(f, v.data(), v.size() * 4, cudaMemcpyHostToDevice, rescue_stream()), "rescue");
    ck(cudaStreamSynchronize(rescue_stream()), "rescue sync");
}

cudaStream_t Executor::rescue_stream() {
    if (!rescue_) ck(cudaStreamCreateWithFlags(&rescue_, cudaStreamNonBlocking), "stream");
    return rescue_;
}

int64_t Executor::iteration_start_globaltimer() {
    int64_t v = 0;
    ck(cudaMemcpy(&v, gt_start_, 8, cudaMemcpyDeviceToHost), "d2h");
    return v;
}

float Executor::read_loss() {
    float v = 0.f;
    ck(cudaMemcpyAsync(&v, stage_->loss_accumulator(), 4, cudaMemcpyDeviceToHost, comp_), "d2h");
    ck(cudaStreamSynchronize(comp_), "sync");
    return v;
}

std::vector<int64_t> Executor::probe_link(int link, int64_t bytes, int repeats) {
    const bool fwd = link == 2 * cfg_.stage;
    if (!fwd && link != 2 * cfg_.stage - 1) throw std::invalid_argument("probe_link: not an outgoing link");
    // probes land in the peer's scratch block, never in its live receive slots
    void* dst = fwd ? peer_scratch_fwd_ : peer_scratch_bwd_;
    const __nv_bfloat16* src = fwd ? act_send_.at(0) : grad_send_.at(0);
    const int64_t cap = static_cast<int64_t>(cfg_.gpt.micro_batch_size) * cfg_.gpt.seq * cfg_.gpt.hidden * 2;
    if (!dst || bytes > cap || bytes > static_cast<int64_t>(kScratch))
        throw std::invalid_argument("probe_link: peer not connected or payload too large");
    cudaStream_t st = send_stream(fwd);
    std::vector<int64_t> out;
    cudaEvent_t a, b;
    ck(cudaEventCreate(&a), "event");
    ck(cudaEventCreate(&b), "event");
    for (int r = 0; r < repeats; ++r) {
        ck(cudaEventRecord(a, st), "event");
        ck(emu_.paced_copy(fwd ? 0 : 1, dst, src, bytes, st), "probe copy");
        ck(cudaEventRecord(b, st), "event");
        ck(cudaEventSynchronize(b), "sync");
        float ms = 0.f;
        ck(cudaEventElapsedTime(&ms, a, b), "elapsed");
        out.push_back(static_cast<int64_t>(static_cast<double>(ms) * 1e6 + 0.5));
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return out;
}

void Executor::profile_compute(int b, int repeats, int64_t* fwd_ns, int64_t* bwd_ns) {
    const ptk_gpt_config& g = cfg_.gpt;
    const int keep_b = b_, keep_k = k_;
    set_plan(1, b);
    const bool first = cfg_.stage == 0, last = cfg_.stage == cfg_.stages - 1;
    const int64_t T = static_cast<int64_t>(b) * g.seq;
    __nv_bfloat16* xin = first ? nullptr : act_recv_;
    __nv_bfloat16* xout = last ? nullptr : act_send_.at(0);
    __nv_bfloat16* dy = last ? nullptr : grad_recv_;
    __nv_bfloat16* dx = first ? nullptr : grad_send_.at(0);
    if (first || last) {  // deterministic data for the profile runs
        synth_tokens(0, host_stage_);
        const int64_t toks = static_cast<int64_t>(cfg_.global_batch) * g.seq;
        ck(cudaMemcpyAsync(tok_dev_, host_stage_, toks * 4, cudaMemcpyHostToDevice, comp_), "h2d");
        ck(cudaMemcpyAsync(lab_dev_, host_stage_ + toks, toks * 4, cudaMemcpyHostToDevice, comp_), "h2d");
    }
    cudaEvent_t e0, e1, e2;
    ck(cudaEventCreate(&e0), "event");
    ck(cudaEventCreate(&e1), "event");
    ck(cudaEventCreate(&e2), "event");
    double f = 0, bw = 0;
    // With paired weight gradients (as the pipeline runs them) a profile round is two micro-batches
    // in slots 0 and 1: the first backward defers its weight gradients, the second runs both as one
    // two-K-segment GEMM; the per-micro-batch figures are the pair's means.  (Profiling unpaired
    // weight gradients made small-b plans look cheaper than they run.)  Otherwise one micro-batch
    // in slot 0.
    const bool pairs = stage_->wgrad_pairs_on();
    stage_->flush_wgrads(comp_);
    const int per_round = pairs && g.slots >= 2 ? 2 : 1;
    if (per_round == 1) stage_->set_wgrad_pairs(false);
    for (int r = 0; r < repeats + 1; ++r) {  // first round is warm-up
        for (int m = 0; m < per_round; ++m) {
            ck(cudaEventRecord(e0, comp_), "event");
            stage_->forward(m, tok_dev_, xin, lab_dev_, xout, comp_);
            ck(cudaEventRecord(e1, comp_), "event");
            stage_->backward(m, tok_dev_, dy, dx, comp_);
            ck(cudaEventRecord(e2, comp_), "event");
            ck(cudaEventSynchronize(e2), "sync");
            float a = 0, c = 0;
            ck(cudaEventElapsedTime(&a, e0, e1), "elapsed");
            ck(cudaEventElapsedTime(&c, e1, e2), "elapsed");
            if (r > 0) {
                f += a / per_round;
                bw += c / per_round;
            }
        }
    }
    stage_->flush_wgrads(comp_);
    (void)T;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaEventDestroy(e2);
    stage_->zero_grads(comp_);
    stage_->set_wgrad_pairs(pairs);
    ck(cudaMemsetAsync(stage_->loss_accumulator(), 0, 4, comp_), "memset");
    ck(cudaStreamSynchronize(comp_), "sync");
    *fwd_ns = static_cast<int64_t>(f / repeats * 1e6 + 0.5);
    *bwd_ns = static_cast<int64_t>(bw / repeats * 1e6 + 0.5);
    set_plan(keep_k, keep_b);
}

}  // namespace ptk
