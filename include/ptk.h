/*
 * ptk.h — the C ABI between the pipetune host layer (C++ / Python ctypes)
 * and the sm_100a stage runtime.  Plain pointers, sizes and ints only; no
 * torch or C++ types cross this boundary.  Every function returns an int
 * status (PTK_OK == 0) and never throws; ptk_last_error() describes the
 * most recent failure on the calling thread.
 *
 * Reference interfaces these entry points stand in for (paths relative to
 * /root/reference):
 *   - proj/src/model.cpp:43-47 compute_duration(): the reference models a
 *     stage's forward/backward as an affine duration.  ptk_stage_forward /
 *     ptk_stage_backward execute the real GPT stage for one micro-batch.
 *   - proj/src/taskgraph.cpp:68-76 Send/Recv node pairs: realised by the
 *     executor's P2P engine (ptk_exec_*), one copy stream per link.
 *   - proj/src/plan.cpp:75-81 plan_kfkb(): ptk_plan_* expose the planner over
 *     the ABI for FFI callers; the C++ API in include/pipetune/ is the
 *     source-compatible drop-in.
 *   - SPEC.md:342 simulate / :453 run_adaptive: ptk_sim_* and ptk_tuner_*.
 */
#ifndef PTK_H_
#define PTK_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------ status */
enum {
    PTK_OK = 0,
    PTK_ERR_ARG = 1,       /* invalid argument (maps to pipetune::ConfigError) */
    PTK_ERR_PLAN = 2,      /* plan parameters out of range (pipetune::PlanError) */
    PTK_ERR_CUDA = 3,      /* CUDA runtime / driver failure (pipetune::CudaError) */
    PTK_ERR_ALIGN = 4,     /* pointer or stride not 16-byte aligned */
    PTK_ERR_DEADLOCK = 5,  /* pipetune::DeadlockDetected */
    PTK_ERR_NOPROFILE = 6, /* pipetune::NoProfileData */
    PTK_ERR_INFEASIBLE = 7,/* pipetune::InfeasibleModel */
    PTK_ERR_UNKNOWN_CANDIDATE = 8,
    PTK_ERR_INTERNAL = 9,
    PTK_ERR_NOMEM = 10
};

const char* ptk_last_error(void);
const char* ptk_version(void);

/* ------------------------------------------------------------ GEMM */
enum { PTK_EPI_BF16 = 0, PTK_EPI_F32 = 1, PTK_EPI_ACC_F32 = 2, PTK_EPI_BIAS_GELU = 3, PTK_EPI_DGELU = 4 };
enum { PTK_CAUSAL_NONE = 0, PTK_CAUSAL_TILES = 1, PTK_CAUSAL_KHEAD = 2, PTK_CAUSAL_KTAIL = 3 };

/* A strided (optionally batched) matrix in device memory.  For operands,
 * mn_major = 0 means the reduction index k is contiguous: element (r, k) at
 * ptr[r*ld + k]; mn_major = 1 means element (r, k) at ptr[k*ld + r].
 * Batch index z = z1 + batch[0]*z2 adds z1*batch_stride[0] + z2*batch_stride[1]
 * (elements). */
typedef struct ptk_matrix {
    void* ptr;
    int mn_major;
    int64_t ld;
    int64_t batch_stride[2];
} ptk_matrix;

/* D[z] = A[z] (m x k) * B[z]^T (B is n x k), bf16 operands, fp32 accumulation,
 * epilogue selected by `epilogue` (see gemm_sm100.cu). */
typedef struct ptk_gemm_desc {
    int m, n, k;
    int batch[2];
    ptk_matrix a, b, c;
    void* c2;          /* PTK_EPI_BIAS_GELU: pre-activation output (same strides as c) */
    ptk_matrix aux;    /* residual (EPI_BF16) or pre-activation (EPI_DGELU) input */
    const void* bias;  /* bf16 [n] or NULL */
    int epilogue;
    int causal;
    int bn_hint;       /* 0 = auto, else 64 / 128 / 256 */
    int multicast;     /* dense BN=256 only: 1 = 2-CTA cluster with B-tile multicast (K-major B);
                          2 = CTA-pair tcgen05.mma.cta_group::2 (256x256 pair tile) */
    float* col_part;   /* optional, bf16 outputs, batch 1: fp32 [ceil(m/32)][n] += per-32-row-block column
                          sums of C as stored (fused bias-gradient partials) */
    /* optional second K segment (k2 > 0): D = A Bᵀ + A2 B2ᵀ, one fp32 accumulation over k + k2
     * (k % 64 == 0; same majors, batch 1, dense): the weight gradients of two micro-batches in one
     * launch, so the fp32 gradient is read and written once per pair */
    ptk_matrix a2, b2;
    int k2;
} ptk_gemm_desc;

int ptk_gemm(const ptk_gemm_desc* desc, void* stream);
/* The launch ptk_gemm would make for desc (no launch): info[0] tile width BN, info[1] grid
 * (CTAs), info[2] work items, info[3] 1 = 2-CTA cluster (B multicast or CTA pair). */
int ptk_gemm_plan_info(const ptk_gemm_desc* desc, int* info);

/* Fused attention forward (causal = 1: key <= query; 0: bidirectional): qkv bf16 [b][s][3][H][d] -> o bf16 [b*s][H*d],
 * lse fp32 [b][H][s] = log2(sum_k 2^(S_qk * log2(e)/sqrt(d))) (row max included). */
int ptk_flash_forward(const void* qkv, void* o, float* lse, int b, int s, int H, int d, int causal, void* stream);
/* Its backward: dqkv bf16 [b*s][3*H*d] (dQ | dK | dV sections) from qkv, o, dO = d(o),
 * lse; dsum: fp32 scratch [b][H][s] (holds tau*rowsum(dO*o)).  Deterministic (no atomics).
 * All pointers 16-byte aligned: the tensors are read / written by TMA and the per-block lse and
 * dsum rows (512 B) by bulk copies. */
int ptk_flash_backward(const void* qkv, const void* o, const void* dO, const float* lse, float* dsum, void* dqkv,
                       int b, int s, int H, int d, int causal, void* stream);

/* ------------------------------------------------------------ planner
 * Mirrors pipetune::StageProfile / ModelSpec (proj/include/pipetune/model.hpp:30-51). */
typedef struct ptk_stage_profile {
    int stage_id;
    double forward_fixed, forward_per_sample;
    double backward_fixed, backward_per_sample;
    int64_t weight_bytes;
    int64_t activation_bytes_per_sample;
    int64_t output_bytes_per_sample_fwd;
    int64_t output_bytes_per_sample_bwd;
} ptk_stage_profile;

typedef struct ptk_model {
    const ptk_stage_profile* stages;
    int stage_count;
    int global_batch;
} ptk_model;

enum { PTK_PLAN_1F1B = 0, PTK_PLAN_KFKB = 1, PTK_PLAN_GPIPE = 2 };

/* build_task_graph(model, b) + plan_1f1b / plan_kfkb(k) / plan_gpipe
 * (proj/src/taskgraph.cpp:35, proj/src/plan.cpp:70-104), dumped as JSON:
 * nodes, edges, lookup tables, per-device orders, units, sequences,
 * validate() violations, check_plan() count and topological_order().
 * On a pipetune::Error the JSON is {"error": "<type name>"} and the status
 * is the matching PTK_ERR_*.  *written receives the bytes needed (incl. NUL);
 * PTK_ERR_NOMEM if cap is too small. */
int ptk_plan_json(const ptk_model* model, int micro_batch_size, int plan_kind, int k, char* buf, size_t cap,
                  size_t* written);

/* ------------------------------------------------------------ spec modules
 * One JSON scenario in (schema_version 1, unknown keys rejected), one JSON
 * result out.  "op" selects: transfer | estimate | peak_memory | simulate |
 * enumerate | profile | compare | decide | tune — the memory, network,
 * simulator, costmodel and tuner operations of SPEC.md:203-491.  Errors:
 * {"error": "<pipetune type>", "message": ...} and the matching status. */
int ptk_scenario_json(const char* request, char* buf, size_t cap, size_t* written);

/* ------------------------------------------------------------ GPT stage
 * One pipeline stage of a GPT model on the current CUDA device: the real
 * compute behind compute_duration() (proj/src/model.cpp:43-47).  Layers
 * [layer_begin, layer_end) of an n_layer model; the embedding lives on the
 * stage with has_embedding, final LayerNorm + LM head + loss on has_head.
 * Weights are initialised on the device from `seed` per global tensor, so any
 * stage partition of the same model starts from identical weights. */
typedef struct ptk_gpt_config {
    int n_layer, hidden, heads, ffn, seq, vocab;
    int layer_begin, layer_end;
    int has_embedding, has_head;
    int micro_batch_size;  /* b */
    int slots;             /* activation-stash slots of micro_batch_size samples each; at a smaller b
                              that divides it, each slot holds micro_batch_size / b micro-batches
                              (virtual slots 0 .. slots * micro_batch_size / b - 1) */
    int micro_batches;     /* M: loss and gradients are the mean over M*b*seq tokens */
    int arch;              /* 0: GPT (pre-LN, causal, LM head); 1: BERT (post-LN, bidirectional,
                              embedding LayerNorm, MLM head = dense+GELU+LN+decoder over all positions) */
    uint64_t seed;
    /* half-layer stage boundaries (a layer = attention block + MLP block): */
    int skip_first_attn;   /* layer_begin's attention block is on the previous stage (input = its x_mid) */
    int skip_last_mlp;     /* layer_end-1's MLP block is on the next stage (output = its x_mid) */
    /* 1: weight gradients of consecutive backward micro-batches are computed in pairs, one GEMM with
     * two K segments per weight (the fp32 gradient is read and written once per pair).  The first
     * micro-batch of a pair keeps its gradient-side operands in per-layer buffers and its stash slot
     * stays live until the second one's backward, so the caller provides one more slot than the plan's
     * in-flight peak.  An unpaired last micro-batch is flushed by finalize (GradAccum). */
    int wgrad_pairs;
} ptk_gpt_config;

typedef struct ptk_stage ptk_stage;

int ptk_stage_create(const ptk_gpt_config* cfg, ptk_stage** out);
int ptk_stage_destroy(ptk_stage* st);
/* F(m) into stash slot `slot`: tok (int32 [b*seq], embedding stage), x_in (bf16
 * [b*seq, hidden], other stages), labels (int32, head stage), x_out (bf16, non-head). */
int ptk_stage_forward(ptk_stage* st, int slot, const int32_t* tok, const void* x_in, const int32_t* labels,
                      void* x_out, void* stream);
/* B(m) of stash slot `slot`: dy (bf16, non-head stages), dx (bf16, non-embedding).
 * Parameter gradients are accumulated (+=) and complete in stream order on return. */
int ptk_stage_backward(ptk_stage* st, int slot, const int32_t* tok, const void* dy, void* dx, void* stream);
/* GradAccum finalisation: AdamW on the accumulated gradients, then zero them. */
int ptk_stage_optimizer_step(ptk_stage* st, float lr, float weight_decay, void* stream);
int ptk_stage_zero_grads(ptk_stage* st, void* stream);
/* Flat device buffers (elements): fp32 master weights, bf16 weights, fp32 grads;
 * loss: device float accumulating the mean loss of the current iteration. */
int ptk_stage_buffers(ptk_stage* st, float** master, void** weights_bf16, float** grads, float** loss,
                      int64_t* numel);
/* Parameter i: name (copied into name_buf), element offset and shape; PTK_ERR_ARG past the end. */
int ptk_stage_param(ptk_stage* st, int i, char* name_buf, size_t cap, int64_t* offset, int64_t* rows, int64_t* cols);
/* GEMM event timing inside the stage's launches (roofline evidence). enable: -1 read only, 0 off,
   1 on (the executor samples one micro-batch in 8), > 1 on with that sampling stride. */
int ptk_stage_gemm_timing(ptk_stage* st, int enable, double* total_flops, double* total_ms, long* launches);
size_t ptk_stage_stash_bytes(ptk_stage* st);

/* ------------------------------------------------------------ executor
 * One pipeline stage per process/GPU walking plan_kfkb() orders
 * (proj/src/plan.cpp:20-59) with Send/Recv pairs (proj/src/taskgraph.cpp:68-76)
 * realised as NVLink peer copies on a dedicated copy stream plus
 * per-micro-batch arrival flags (stream memory ops).  gpt.micro_batch_size is
 * the largest b any plan will use; gpt.slots the largest in-flight count. */
typedef struct ptk_exec_config {
    ptk_gpt_config gpt;
    int stage, stages;
    int global_batch;
    float lr, weight_decay;
    uint64_t data_seed;
} ptk_exec_config;

typedef struct ptk_exec ptk_exec;

int ptk_exec_create(const ptk_exec_config* cfg, ptk_exec** out);
int ptk_exec_destroy(ptk_exec* ex);
/* IPC handles of this stage's receive blocks + arrival flags (opaque bytes). */
int ptk_exec_export(ptk_exec* ex, void* buf, size_t cap, size_t* written);
int ptk_exec_import(ptk_exec* ex, int peer_stage, const void* buf, size_t n);
int ptk_exec_connect_local(ptk_exec* ex, int peer_stage, ptk_exec* peer);
int ptk_exec_set_plan(ptk_exec* ex, int k, int micro_batch_size);
/* kFkB over explicit consecutive group sizes (sum = global_batch / micro_batch_size): k may change
 * at every group boundary inside one iteration (pipetune::plan_groups). */
int ptk_exec_set_plan_groups(ptk_exec* ex, int micro_batch_size, const int* group_sizes, int n_groups);
/* Emulated-preemption trace for an outgoing link (times relative to the epoch). */
int ptk_exec_set_trace(ptk_exec* ex, int link, double base_bytes_per_ns, int64_t latency_ns, int nseg,
                       const int64_t* start_ns, const int64_t* end_ns, const double* availability);
int ptk_exec_set_epoch(ptk_exec* ex, int64_t epoch_ns);
/* Contender kernels: real competing NVLink stores into the peer's scratch block
 * with duty cycle (1 - availability) while a link trace is preempted. */
int ptk_exec_set_contender(ptk_exec* ex, int on);
int64_t ptk_globaltimer(void);
/* Enqueue iteration `iter` (host_tokens: int32 [2][global_batch*seq] tokens then
 * labels, or NULL for the built-in synthetic corpus); finish blocks and
 * returns the stage's device milliseconds for it. */
int ptk_exec_run_iteration(ptk_exec* ex, int iter, const int32_t* host_tokens);
/* ptk_exec_run_iteration one plan node at a time: begin stages the data, each enqueue_next
 * enqueues the next node of the stage's order and sets *more = 0 once the iteration is fully
 * enqueued (then call finish).  `iter` only seeds the synthetic corpus: arrival flags carry an
 * internal per-executor epoch, so reusing or restarting `iter` is safe. */
int ptk_exec_begin_iteration(ptk_exec* ex, int iter, const int32_t* host_tokens);
int ptk_exec_enqueue_next(ptk_exec* ex, int* more);
/* All n stages of one pipeline in this process (stages[s] = stage s, wired with
 * ptk_exec_connect_local): one iteration enqueued in a global order where each node follows the
 * nodes it receives from, so it completes even when launches are serialised (ncu).  A plan whose
 * per-device orders cannot be merged returns PTK_ERR_DEADLOCK.  Finish each stage afterwards. */
int ptk_exec_run_local(ptk_exec* const* stages, int n, int iter, const int32_t* host_tokens);
/* Blocks until the stage's iteration (compute and sends) finished.  After the deadlock timeout
 * (default 600 s, env PTK_DEADLOCK_TIMEOUT_S) it returns PTK_ERR_DEADLOCK
 * (pipetune::DeadlockDetected, proj/include/pipetune/errors.hpp:38-40): the stage's arrival flags
 * are forced open so its streams drain, and the executor is poisoned (destroy it). */
int ptk_exec_finish_iteration(ptk_exec* ex, double* ms);
int ptk_exec_set_deadlock_timeout(ptk_exec* ex, double seconds);
/* 1: one dedicated copy stream per outgoing link (activations and gradients of a middle stage
 * never queue behind each other); 0 (default): one send stream per stage for both directions,
 * the spec simulator's model the cost model predicts.  Env PTK_SEND_STREAMS=per_link. */
int ptk_exec_set_send_streams(ptk_exec* ex, int per_link);
int ptk_exec_read_loss(ptk_exec* ex, float* loss);
/* Records of the last finished iteration, ns from its start:
 * {"compute": [[node, kind(0F/1B/2GA), mb, start, end]...], "xfer": [[link, mb, bytes, start, end]...],
 *  "launches": n, "h2d_bytes": n, "k": k, "b": b, "groups": [plan group sizes...],
 *  "t0_globaltimer": the iteration start on the GPU's %globaltimer (ns), "stage": s}.
 * Scenario op "hardware_report" turns several stages' records into a SimResult
 * (bubble_report / queue_analysis). */
int ptk_exec_timeline_json(ptk_exec* ex, char* buf, size_t cap, size_t* written);
int ptk_exec_probe_link(ptk_exec* ex, int link, int64_t bytes, int repeats, int64_t* out_ns);
int ptk_exec_profile_compute(ptk_exec* ex, int micro_batch_size, int repeats, int64_t* fwd_ns, int64_t* bwd_ns);
int ptk_exec_gemm_timing(ptk_exec* ex, int enable, double* total_flops, double* total_ms, long* launches);
/* Non-owning view of the executor's stage (weights, grads, parameter table). */
ptk_stage* ptk_exec_stage(ptk_exec* ex);
/* Data-parallel replicas: with defer != 0 the GradAccum node only finalizes the
 * stage gradients; the caller all-reduces them across replicas on ptk_exec_compute_stream() and then
 * calls ptk_stage_optimizer_step on that stream (ptk_exec_stage gives the stage). */
int ptk_exec_set_defer_optimizer(ptk_exec* ex, int defer);
int ptk_exec_compute_stream(ptk_exec* ex, void** stream);
/* Paired weight gradients on/off for the following iterations (the stage must have been created
 * with ptk_gpt_config.wgrad_pairs = 1; off = one weight-gradient GEMM per micro-batch). */
int ptk_exec_set_wgrad_pairs(ptk_exec* ex, int on);

#ifdef __cplusplus
}
#endif

#endif /* PTK_H_ */
