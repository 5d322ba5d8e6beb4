// kFkB stage executor: the hardware twin of the spec simulator.
//
// One Executor per process / GPU / pipeline stage.  run_iteration() walks
// plan.per_device[stage] (pipetune::plan_kfkb) and enqueues, in plan order:
//   F(m): [compute stream waits act_flag[m] >= iter+1]  stage.forward
//         -> send stream: waits F(m) done, copies the output into the next
//            stage's receive slot m over NVLink (peer copy engine), then
//            writes the peer's act_flag[m] = iter+1 (stream memory op)
//   B(m): same with grad_flag / the previous stage
//   GA:   AdamW step on the accumulated gradients
// Compute and transfers sit on separate streams and synchronise only through
// per-micro-batch flags, so a stage whose inputs have arrived keeps computing
// while a (possibly preempted) transfer drains — the overlap kFkB exploits.
// The preemption emulator paces every transfer against a LinkTrace on the
// device (globaltimer-gated chunks), and contender kernels add real competing
// NVLink traffic (emulator.cu).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <memory>
#include <string>
#include <vector>

#include "../../../include/ptk.h"
#include "emulator.h"
#include "gpt_stage.h"
#include "pipetune/plan.hpp"

namespace ptk {

struct CompRecord {
    int node;   // plan node id
    int kind;   // 0 F, 1 B, 2 GA
    int mb;
    cudaEvent_t start, end;
};

struct XferRecord {
    int link;
    int mb;
    int64_t bytes;
    cudaEvent_t start, end;
};

class Executor {
  public:
    explicit Executor(const ptk_exec_config& cfg);
    ~Executor();

    const ptk_exec_config& cfg() const { return cfg_; }
    GptStage& stage() { return *stage_; }

    // IPC: this stage's receive blocks and flags, and the peers' in return.
    std::vector<uint8_t> export_handles() const;
    void import_peer(int peer_stage, const uint8_t* handles, size_t n);
    // Same-process peers (tests): raw device pointers instead of IPC.
    void connect_local(int peer_stage, Executor& peer);

    void set_plan(int k, int micro_batch_size);
    // kFkB over an explicit list of consecutive group sizes (sum = global_batch / b):
    // group-boundary switching of k inside one iteration.
    void set_plan_groups(int micro_batch_size, const std::vector<int>& group_sizes);
    int plan_k() const { return k_; }
    // Data-parallel replicas: the GradAccum node leaves the
    // optimizer to the caller, who all-reduces the finalized gradients first.
    void set_defer_optimizer(bool on) { defer_optimizer_ = on; }
    cudaStream_t compute_stream() const { return comp_; }
    int plan_b() const { return b_; }
    const std::vector<int>& plan_groups() const { return groups_; }

    void set_trace(int link, const EmuTrace& trace);  // outgoing link pacing
    void set_contender(bool on) { contender_on_ = on; }
    void set_epoch(int64_t epoch_ns);

    // Enqueue one training iteration (non-blocking); host_tokens: pinned or
    // pageable int32 [2][global_batch*seq], the tokens then the labels
    // (NULL -> built-in synthetic data).  `iter` seeds the synthetic data only:
    // the arrival flags carry an internal epoch that advances once per
    // iteration, so a reused or restarted `iter` can never satisfy a wait with a
    // stale flag from an earlier iteration.
    void run_iteration(int iter, const int32_t* host_tokens);
    // The same, one plan node at a time: begin_iteration() stages the data,
    // enqueue_next() enqueues the next node of plan.per_device[stage] and
    // returns false once the iteration is fully enqueued.  Used to interleave
    // several same-process stages in a dependency-respecting global order.
    void begin_iteration(int iter, const int32_t* host_tokens);
    // ConfigError unless every token / label id of host_tokens is in [0, vocab).
    void validate_tokens(const int32_t* host_tokens) const;
    bool enqueue_next();
    // Next node of this stage's order (kind 0 F / 1 B / 2 GA, micro-batch), or
    // kind -1 once the iteration is fully enqueued.
    void peek_next(int* kind, int* mb) const;
    // Block until the iteration finished; fills records; returns device ms
    // from iteration start to the GA completion on this stage.  If it has not
    // finished after the deadlock timeout, the stage's own arrival flags are
    // forced open so its streams drain, the executor is poisoned (every later
    // run throws) and pipetune::DeadlockDetected is thrown (PTK_ERR_DEADLOCK).
    double finish_iteration();
    void set_deadlock_timeout(double seconds) { deadlock_timeout_s_ = seconds; }
    // One dedicated copy stream per outgoing link (true) or one send stream
    // for both directions (false, the spec simulator's model).
    void set_send_streams_per_link(bool on) { per_link_send_ = on; }
    bool poisoned() const { return poisoned_; }
    float read_loss();  // D2H of the iteration's loss (last stage only)

    // Timed probes on an outgoing link with the pipeline suspended.
    std::vector<int64_t> probe_link(int link, int64_t bytes, int repeats);
    // Measured compute durations (ns) of F and B at micro-batch size b.
    void profile_compute(int b, int repeats, int64_t* fwd_ns, int64_t* bwd_ns);

    const std::vector<CompRecord>& comp_records() const { return crec_; }
    const std::vector<XferRecord>& xfer_records() const { return xrec_; }
    cudaEvent_t iteration_start() const { return it_start_; }
    // %globaltimer (ns) when the last iteration started on this GPU: aligns the
    // records of several stages on one clock (hardware bubble_report).
    int64_t iteration_start_globaltimer();
    int64_t h2d_bytes() const { return h2d_bytes_; }
    int64_t d2h_bytes() const { return 4; }
    long kernel_launches() const { return stage_->launches() + emu_launches_; }

  private:
    void install_plan(int b, const std::vector<int>& group_sizes, int k);
    void enqueue_node(int id);
    cudaStream_t send_stream(bool fwd) const { return (per_link_send_ && !fwd) ? sendst_bwd_ : sendst_; }
    void alloc_comm();
    void send(bool forward, int mb, const __nv_bfloat16* src, int64_t bytes, cudaEvent_t ready);
    cudaEvent_t ev();
    cudaStream_t rescue_stream();
    void open_flags();
    cudaStream_t rescue_ = nullptr;
    void synth_tokens(int iter, int32_t* dst) const;

    ptk_exec_config cfg_;
    std::unique_ptr<GptStage> stage_;
    std::shared_ptr<const pipetune::TaskGraph> graph_;
    pipetune::SchedulePlan plan_;
    int k_ = 1, b_ = 1, M_ = 1;
    std::vector<int> groups_;
    int iter_ = 0;
    uint32_t epoch_ = 0;      // arrival-flag value of the current iteration (internal, monotone)
    size_t cursor_ = 0;       // next index into plan_.per_device[stage]
    bool in_iteration_ = false;
    bool poisoned_ = false;
    double deadlock_timeout_s_ = 600.0;
    bool per_link_send_ = false;

    cudaStream_t comp_ = nullptr, sendst_ = nullptr, sendst_bwd_ = nullptr, contend_[2] = {nullptr, nullptr};
    bool defer_optimizer_ = false;
    // receive blocks (owned; written by peers) and flags
    __nv_bfloat16 *act_recv_ = nullptr, *grad_recv_ = nullptr;
    uint32_t *act_flag_ = nullptr, *grad_flag_ = nullptr;
    // peers' blocks (IPC-mapped or same-process)
    __nv_bfloat16 *peer_act_recv_ = nullptr, *peer_grad_recv_ = nullptr;
    void* scratch_ = nullptr;                  // target of peers' contender traffic
    void *peer_scratch_fwd_ = nullptr, *peer_scratch_bwd_ = nullptr;
    static constexpr size_t kScratch = 64ull << 20;
    uint32_t *peer_act_flag_ = nullptr, *peer_grad_flag_ = nullptr;
    std::vector<void*> ipc_opened_;
    // send staging, one per stash slot, with WAR events
    std::vector<__nv_bfloat16*> act_send_, grad_send_;
    std::vector<cudaEvent_t> act_sent_, grad_sent_;
    // data
    int32_t *tok_dev_ = nullptr, *lab_dev_ = nullptr;
    int32_t* host_stage_ = nullptr;  // pinned [2][gb*seq]: tokens, then labels
    int64_t h2d_bytes_ = 0;
    long emu_launches_ = 0;
    cudaEvent_t h2d_done_ = nullptr;
    int64_t* gt_start_ = nullptr;

    // event pools and records
    std::vector<cudaEvent_t> pool_;
    size_t pool_used_ = 0;
    cudaEvent_t it_start_ = nullptr, it_end_ = nullptr;
    std::vector<CompRecord> crec_;
    std::vector<XferRecord> xrec_;

    // emulator
    Emulator emu_;
    bool contender_on_ = false;

    std::vector<void*> allocs_;
};

// Several stages of one pipeline in this process (same or different GPUs,
// wired with connect_local), `stages[s]` = stage s: enqueue one iteration of
// all of them in one global order where every node is enqueued after the
// nodes it receives from (F(m) after the previous stage's F(m), B(m) after
// the next stage's B(m)).  Any prefix of that order can run to completion, so
// the iteration also completes when kernel launches are serialised (ncu), and
// a plan whose orders cannot be merged raises pipetune::DeadlockDetected.
void run_local_pipeline(const std::vector<Executor*>& stages, int iter, const int32_t* host_tokens);

}  // namespace ptk
