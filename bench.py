"""bench.py — samples/s of the B200 kFkB pipeline executor (GPT-1.3B, bf16).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N = 1: one GPU runs the whole model as a single stage (no pipeline), 32
micro-batches of b = 2 (global batch 64, seq 1024) — BASELINE.json configs[1]
at one GPU.  N > 1 (torchrun, one rank per GPU = one pipeline stage): the same
model split into N stages with emulated NVLink preemption on every link; the
timed steps run the Ada-Grouper plan (k chosen online by the C++ tuner from
live link/compute profiles), and 1F1B is timed beside it on the same kernels.
One JSON line on rank 0.  `--impl reference` times the CPU path (reference
planner from oracle/_ref + fp32 oracle model on the host cores).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "samples/sec under emulated preemption: Ada-Grouper kFkB vs 1F1B, 2/4/8 B200"
GLOBAL_BATCH, MICRO_B = 64, 2
JSON_OUT = sys.stdout  # rank 0's JSON line (main() points it at the original stdout)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--link-gbps", type=float, default=100.0, help="emulated link bandwidth (Gb/s)")
    p.add_argument("--availability", type=float, default=0.5, help="availability while preempted")
    p.add_argument("--trace", choices=["constant", "two-regime", "bursty", "square", "none"], default="constant")
    p.add_argument("--period-ms", type=float, default=1000.0,
                   help="square: preempted (availability) for period-ms, free for period-ms, repeating")
    p.add_argument("--regime-ms", type=float, default=2000.0, help="two-regime: preempted for the first X ms")
    p.add_argument("--on-ms", type=float, default=200.0, help="bursty: mean preempted (ON) burst")
    p.add_argument("--off-ms", type=float, default=300.0, help="bursty: mean idle (OFF) gap")
    p.add_argument("--trace-seed", type=int, default=1)
    p.add_argument("--retune", type=int, default=0, help="re-tune every N steps (0: once at start)")
    p.add_argument("--tuner-log", type=str, default="")
    p.add_argument("--contender", action="store_true", help="also launch competing NVLink traffic kernels")
    p.add_argument("--model", choices=["1.3b", "6.7b", "bert-large"], default="1.3b")
    p.add_argument("--global-batch", type=int, default=GLOBAL_BATCH)
    p.add_argument("--micro-batch", type=int, default=MICRO_B)
    p.add_argument("--mem-cap-gb", type=float, default=0.0,
                   help="imposed per-GPU memory limit: candidates = the (k, b) frontier under it (config 4)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-wgrad-pairs", action="store_true",
                   help="one weight-gradient GEMM per micro-batch (default: two-K-segment pairs, whose "
                        "buffers the --mem-cap-gb frontier budgets)")
    p.add_argument("--tuner-repeats", type=int, default=3, help="active link probes per payload (SPEC default 3)")
    p.add_argument("--probe-every", type=int, default=1,
                   help="with --passive-profile: re-probe other candidates' payloads every N tuning rounds "
                        "(1: every round, SPEC.md:294)")
    p.add_argument("--passive-profile", action="store_true",
                   help="feed every re-tuning round the last iteration's own transfers as link samples and probe "
                        "only the other candidates' payloads")
    p.add_argument("--ref-stages", type=int, default=1,
                   help="--impl reference: S > 1 runs the CPU-thread pipeline executor (S stage threads, "
                        "S micro-batches per step, oracle/cpu_pipeline.py); 1 = the whole model on all cores")
    p.add_argument("--timeline", type=str, default="")
    p.add_argument("--k-sweep", action="store_true",
                   help="configs[2]: also time a fixed-plan kFkB arm for every candidate k (1/2/4/8 ...), "
                        "reported under schedules.kfkb_sweep")
    return p.parse_args()


def peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text()), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu, self.rows, self.stop = gpu, [], threading.Event()
        self.t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self.stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self.stop.wait(0.2)

    def __enter__(self):
        self.t.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.t.join(timeout=6)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in self.rows for n, v in zip(names, r[4:8]) if v.strip().lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def gemm_traffic():
    """DRAM bytes per launch of the representative stage GEMM from the committed ncu capture
    (profiles/gemm_traffic.json), or None when no capture is committed."""
    try:
        t = json.loads((ROOT / "profiles" / "gemm_traffic.json").read_text())
        return {"bytes_per_launch": t["dram_read_bytes"] + t["dram_write_bytes"],
                "algorithmic_bytes_per_launch": t["algorithmic_read_bytes"] + t["algorithmic_write_bytes"],
                "kernel": t["kernel"], "source": t["source"]}
    except Exception:
        return None


def trace_segments(args, link: int):
    """LinkTrace availability segments (ns from the arm's epoch)."""
    H = 10**13
    a = args.availability
    if args.trace == "none" or a >= 1.0:
        return []
    if args.trace == "constant":
        return [(0, H, a)]
    if args.trace == "two-regime":
        return [(0, int(args.regime_ms * 1e6), a)]
    if args.trace == "square":  # regime changes every period: preempted, free, preempted, ...
        P = int(args.period_ms * 1e6)
        return [(2 * i * P, (2 * i + 1) * P, a) for i in range(int(600e9 // (2 * P)) + 1)]
    import random
    rng = random.Random(args.trace_seed * 1000 + link)  # seeded two-state Markov ON/OFF
    segs, t = [], 0.0
    while t < 120e9:
        t += rng.expovariate(1.0 / (args.off_ms * 1e6))
        on = rng.expovariate(1.0 / (args.on_ms * 1e6))
        segs.append((int(t), int(t + on), a))
        t += on
    return segs


def reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle.cpu_baseline import CpuTrainer
    from oracle.cpu_pipeline import CpuPipeline
    from paper_2303_01675_b200.stage import BERT_LARGE, GPT_1_3B, GPT_6_7B
    shape = {"6.7b": GPT_6_7B, "bert-large": BERT_LARGE}.get(args.model, GPT_1_3B)
    S = max(1, args.ref_stages)
    trainer = CpuTrainer(shape, 1, 1) if S == 1 else CpuPipeline(shape, S, 1, S, k=1)
    for _ in range(min(args.warmup, 1)):  # one untimed warm-up sample (allocator, thread pool)
        trainer.step()
    vals = []
    cb = None
    for i in range(max(1, args.steps)):
        cb = trainer.step()
        vals.append(cb["value"])
    v = statistics.median(vals)
    cb["value"] = v
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "samples/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 / v, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"{args.model} training step on the CPU path (fp32), bounded sample of "
                               f"{S} sample(s)/step",
                   "global_batch": args.global_batch, "seq_len": shape.seq,
                   "parallelism": "none (host cores)" if S == 1 else f"pp{S} stage threads (host cores)"},
        "cpu_baseline": cb,
        "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def spawn_ranks(args) -> int:
    """`python bench.py --gpus N` (N > 1) without torchrun: re-launch this script under
    torch.distributed.run, one rank per GPU / pipeline stage, and pass its exit code through."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        sys.exit(spawn_ranks(args))
    if args.impl == "reference":
        return reference_arm(args)

    # rank 0 prints exactly one JSON line on stdout: NCCL's communicator-init lines (which name
    # nRanks) go to stderr, nothing else of NCCL's is printed
    # Native libraries (NCCL's version banner and INIT lines, which name nRanks) print on fd 1; rank
    # 0 owes exactly one JSON line on stdout.  So fd 1 of this process is pointed at stderr and the
    # JSON line goes to a saved copy of the original stdout.
    global JSON_OUT
    sys.stdout.flush()
    JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    if os.environ.get("NCCL_DEBUG", "").upper() in ("", "VERSION", "WARN"):
        os.environ["NCCL_DEBUG"] = "INFO"
        os.environ["NCCL_DEBUG_SUBSYS"] = "INIT"
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:  # every link is paced (trace "none" = the base rate)
        # leave SMs free for the emulator's trace gates (and contender CTAs): persistent GEMM / attention
        # grids would otherwise hold every SM and delay each gate by a whole kernel (runtime/sm_budget.h)
        os.environ.setdefault("PTK_SM_RESERVE", str(1 + (int(os.environ.get("PTK_CONTENDER_CTAS", "4"))
                                                         if args.contender else 0)))
    import torch
    import torch.distributed as dist

    from paper_2303_01675_b200.executor import StageExecutor, partition_halves, stage_slots
    from paper_2303_01675_b200.stage import BERT_LARGE, GPT_1_3B, GPT_6_7B
    from paper_2303_01675_b200.tuning import OnlineTuner, candidate_set, outgoing_links

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE={world}; using {world}", file=sys.stderr)
    # PTK_OVERSUBSCRIBE=1 (dry runs only): more ranks than GPUs, rank -> GPU local % count, gloo only
    oversub = os.environ.get("PTK_OVERSUBSCRIBE") == "1"
    if oversub:
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    group = None
    if world > 1:
        if oversub:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
            dist.all_reduce(torch.ones(1, device="cuda"))  # creates the communicator now
            torch.cuda.synchronize()
        group = dist.new_group(backend="gloo")
    log = lambda msg: print(f"[bench rank {rank}] {msg}", file=sys.stderr, flush=True)  # noqa: E731
    log(f"world {world}, device {local}")

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier(group=group)

    shape = {"6.7b": GPT_6_7B, "bert-large": BERT_LARGE}.get(args.model, GPT_1_3B)
    GB = args.global_batch
    S = world
    # half-layer stage cuts (attention | MLP blocks), weights measured on B200
    halves = partition_halves(shape.n_layer, S, head_weight=2.3 if shape.arch == "bert" else 1.6,
                              attn_weight=0.42 if shape.arch == "bert" else 0.47)
    layers = halves
    cap = args.mem_cap_gb * 1e9 if args.mem_cap_gb > 0 else None
    wgrad_pairs = not args.no_wgrad_pairs
    cands = candidate_set(shape, halves, S, GB, cap, fixed_b=args.micro_batch, halves=True,
                          wgrad_pairs=wgrad_pairs) if S > 1 else [[1, args.micro_batch, GB // args.micro_batch]]
    # physical slots are b_max samples wide: enough of them for every candidate's in-flight samples
    slots, b_max = stage_slots(rank, S, cands)
    ex = StageExecutor(shape, rank, S, GB, b_max=b_max, slots=slots, halves=halves[rank], wgrad_pairs=wgrad_pairs)
    ks = [c[0] for c in cands]
    b = cands[0][1]  # plan micro-batch size before tuning (the k=1 candidate)
    M = GB // b
    act_bytes = b * shape.seq * shape.hidden * 2
    trace_desc = None
    if S > 1:
        ex.connect_dist(group)
        base = args.link_gbps * 1e9 / 8 / 1e9  # bytes per ns
        for link in outgoing_links(rank, S):
            ex.set_trace(link, base, 0, trace_segments(args, link))
        ex.set_contender(args.contender)
        trace_desc = {"emulated_link_gbps": args.link_gbps, "trace": args.trace, "availability": args.availability,
                      "regime_ms": args.regime_ms if args.trace == "two-regime" else None,
                      "period_ms": args.period_ms if args.trace == "square" else None,
                      "bursty_mean_on_off_ms": [args.on_ms, args.off_ms] if args.trace == "bursty" else None,
                      "seed": args.trace_seed, "retune_every": args.retune, "contender_kernels": args.contender,
                      "tuner_repeats": args.tuner_repeats, "passive_profile": args.passive_profile,
                      "probe_every": args.probe_every}

    sync_gt = [0]

    def arm_reset():
        """Every arm replays the trace from t=0 (per-rank globaltimer epoch after a barrier)."""
        barrier()
        if S > 1:
            sync_gt[0] = ex.globaltimer()
            ex.set_epoch(sync_gt[0])

    it = 0

    def run(n, cfg, groups=None):
        nonlocal it
        if groups:  # a mixed-k plan chosen by the tuner (remainder group first)
            ex.set_plan_groups(cfg[1], groups)
        else:
            ex.set_plan(cfg[0], cfg[1])
        ms = []
        for _ in range(n):
            ex.run_iteration(it)
            ms.append(ex.finish_iteration())
            it += 1
        return ms

    by_k = {c[0]: c for c in cands}
    log(f"candidates {cands}, slots {slots}, b_max {b_max}")
    arm_reset()
    run(args.warmup, cands[0])
    log("warm-up done")
    if S > 1:
        for c in cands[1:]:
            run(1, c)  # every candidate plan warmed (GEMM / attention plans cached)

    gemm_stride = int(os.environ.get("PTK_BENCH_GEMM_STRIDE", "32"))
    gemm_sampling = os.environ.get("PTK_BENCH_GEMM_TIMING", "1") != "0"  # 0: diagnostics, no per-GEMM events

    def run_arm(n, cfg):
        """A fixed-plan arm under the same GEMM event sampling as the timed Ada-Grouper arm (the events
        break the PDL overlap of the sampled micro-batch), so the arms compare like for like."""
        if gemm_sampling:
            ex.gemm_timing(gemm_stride)
        out = run(n, cfg)
        if gemm_sampling:
            ex.gemm_timing(0)  # discarded: the roofline is the Ada-Grouper arm's
        return out

    # ---- fixed-plan arms (same kernels, same trace from t=0)
    fixed = {}
    if S > 1:
        for k in (sorted(by_k) if args.k_sweep else (1, 2)):
            if k in by_k:
                arm_reset()
                fixed[k] = run_arm(args.steps, by_k[k])
                log(f"fixed arm k={k}: {sum(fixed[k]):.1f} ms")
        if wgrad_pairs and 1 in by_k:
            # 1F1B also with one weight-gradient GEMM per micro-batch: pairing alternates short and
            # long backwards, which 1F1B's strict F/B alternation cannot absorb; the arm reports the
            # faster of the two (decided on the max-over-ranks times below)
            ex.set_wgrad_pairs(False)
            arm_reset()
            fixed["1_unpaired"] = run_arm(args.steps, by_k[1])
            ex.set_wgrad_pairs(True)

    # ---- timed region: Ada-Grouper (tuning round at start, re-tune every `retune` steps)
    tuner = OnlineTuner(ex, rank, S, GB, [(c[0], c[1]) for c in cands], shape.seq * shape.hidden * 2,
                        group=group, repeats=args.tuner_repeats, passive=args.passive_profile,
                        probe_every=args.probe_every) if S > 1 else None
    if tuner is not None:
        tuner.profile_compute()  # once, before the timed region
    chosen, chosen_groups, decisions, tune_s = cands[0], [], [], 0.0
    arm_reset()
    with ClockSampler(local) as clk:
        if gemm_sampling:
            # one micro-batch in 32 per stage and step, rotating with the step: event records between GEMMs
            # break the PDL overlap of the sampled micro-batches (1 in 8 cost BERT-large 4.5 % of a step)
            ex.gemm_timing(gemm_stride)
        t0 = time.perf_counter()
        ms, plans_run = [], []
        # A re-tuning round whose candidates all share the running plan's micro-batch size needs no
        # probe (the passive samples of the last iteration cover every candidate payload on every
        # rank), so it runs on the host WHILE the GPU executes the step before the boundary, on the
        # timeline of the step before that; the decision applies from the boundary on.  Only the host
        # time the step did not cover is charged.  Rounds that must probe stay at the boundary with
        # the pipeline suspended.
        overlap_ok = tuner is not None and args.passive_profile and args.retune > 0 and \
            os.environ.get("PTK_BENCH_OVERLAP_TUNING", "1") != "0"
        pending, last_tl = None, None
        for step in range(args.steps):
            due = tuner is not None and (step == 0 or (args.retune > 0 and step % args.retune == 0))
            if pending is not None:  # decided during the previous step
                chosen, chosen_groups = pending
                pending = None
            elif due:
                tr0 = time.perf_counter()
                if step > 0 and args.passive_profile:
                    tuner.observe_iteration(ex.timeline(), clock=step)
                # the incumbent is the plan the executor ran last (the warm-up plan before the first
                # round), so the first round is already a switch decision
                d = tuner.round(list(chosen), clock=step, current_groups=chosen_groups)
                decisions.append(d)
                chosen = d["chosen"]
                chosen_groups = d.get("chosen_groups", [])
                barrier()
                tune_s += time.perf_counter() - tr0
            if chosen_groups:
                ex.set_plan_groups(chosen[1], chosen_groups)
            else:
                ex.set_plan(chosen[0], chosen[1])
            ex.run_iteration(it)
            nxt, host_s = step + 1, None
            if (overlap_ok and last_tl is not None and nxt < args.steps and nxt % args.retune == 0
                    and not tuner.needs_probes(chosen[1])):
                tr0 = time.perf_counter()
                tuner.observe_iteration(last_tl, clock=nxt)
                d = tuner.round(list(chosen), clock=nxt, current_groups=chosen_groups)
                decisions.append(d)
                pending = (d["chosen"], d.get("chosen_groups", []))
                barrier()
                host_s = time.perf_counter() - tr0
            dev_ms = ex.finish_iteration()
            it += 1
            ms.append(dev_ms)
            if host_s is not None:
                tune_s += max(0.0, host_s - dev_ms * 1e-3)
            plans_run.append([chosen[0], chosen[1]] + ([chosen_groups] if chosen_groups else []))
            last_tl = ex.timeline() if overlap_ok and (step + 2) % args.retune == 0 else None
        barrier()
        wall = time.perf_counter() - t0
        gemm_flops, gemm_ms, gemm_n = ex.gemm_timing(0)
    log("timed Ada-Grouper arm done")
    tl = ex.timeline()
    # achieved transfer / forward ratio of the last timed iteration (the paper's regime is ~0.5,
    # PAPER.md:102): mean paced transfer vs mean forward of this stage
    fwd_ns = [r[4] - r[3] for r in tl["compute"] if r[1] == 0]
    xfer_ns = [r[4] - r[3] for r in tl["xfer"]]
    xf_ratio = round(statistics.mean(xfer_ns) / statistics.mean(fwd_ns), 4) if fwd_ns and xfer_ns else None
    loss = ex.read_loss() if rank == S - 1 else None
    if tuner is not None and rank == 0 and args.tuner_log:
        Path(args.tuner_log).write_text(json.dumps({"trace": trace_desc, "candidates": cands, "rounds": tuner.log}))
    ms_1f1b = fixed.get(1, ms)
    b, M = chosen[1], chosen[2]

    # ---- e2e: host token buffers through the C ABI, H2D + loss D2H inside the timed steps
    import numpy as np
    rng = np.random.default_rng(7)
    host = rng.integers(0, shape.vocab, size=(2, GB * shape.seq), dtype=np.int32)
    if chosen_groups:
        ex.set_plan_groups(chosen[1], chosen_groups)
    else:
        ex.set_plan(chosen[0], chosen[1])
    arm_reset()  # the same trace window as the timed arm (time-varying traces replay from t=0)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        ex.run_iteration(it, host.ctypes.data)
        ex.finish_iteration()
        if rank == S - 1:
            ex.read_loss()
        it += 1
    barrier()
    e2e_s = time.perf_counter() - t0

    def gather(x):
        if world == 1:
            return [x]
        out = [None] * world
        dist.all_gather_object(out, x, group=group)
        return out

    all_ms = gather(sum(ms) + tune_s * 1e3)
    all_1f1b = gather(sum(ms_1f1b))
    all_1f1b_u = gather(sum(fixed["1_unpaired"])) if "1_unpaired" in fixed else None
    all_k2 = gather(sum(fixed.get(2, ms)))
    all_sweep = {k: gather(sum(fixed[k])) for k in sorted(by_k) if k in fixed} if args.k_sweep else None
    all_loss = gather(loss)
    all_e2e = gather(e2e_s)
    all_launch = gather(tl["launches"] * args.steps)
    all_h2d = gather(tl["h2d_bytes"])
    all_gemm = gather((gemm_flops, gemm_ms, gemm_n))
    all_clk = gather(clk.summary())
    all_xf = gather(xf_ratio)
    all_tl = gather(tl) if S > 1 else None
    all_sync = gather(sync_gt[0]) if S > 1 else None
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    T = max(all_ms) / 1e3
    value = GB * args.steps / T
    v1f1b = GB * args.steps / (max(all_1f1b) / 1e3)
    v1f1b_paired = v1f1b
    v1f1b_unpaired = GB * args.steps / (max(all_1f1b_u) / 1e3) if all_1f1b_u else None
    if v1f1b_unpaired is not None:
        v1f1b = max(v1f1b, v1f1b_unpaired)
    vk2 = GB * args.steps / (max(all_k2) / 1e3)
    loss = all_loss[-1]
    pk, pk_kind = peaks()
    peak_sus = pk.get("bf16_tflops_sustained", pk["bf16_tflops"])
    gf = sum(g[0] for g in all_gemm)
    gt = sum(g[1] for g in all_gemm) / 1e3
    achieved = gf / gt / 1e12 if gt > 0 else 0.0
    flops_sample = shape.flops_per_sample()
    # ideal pipeline roofline: T* = sum_s T_s + (M-1) max_s T_s, T_s = b*FLOPs_s/P
    Ts = [b * shape.flops_halves(s_, e, i == S - 1) / (peak_sus * 1e12) for i, (s_, e) in enumerate(halves)]
    t_star = sum(Ts) + (M - 1) * max(Ts)
    ideal = M * b / t_star
    out = {
        "metric": METRIC, "value": round(value, 3), "unit": "samples/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(T * 1e3 / args.steps, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": {"1.3b": "GPT-1.3B training step (configs[1]: 24L h2048 32 heads s1024 V50304)",
                                "6.7b": "GPT-6.7B training step (configs[3]: 32L h4096 32 heads s1024 V50304)",
                                "bert-large": "BERT-large MLM training step (configs[4]: 24L h1024 16 heads s512 "
                                              "V30528, post-LN, bidirectional)"}[args.model],
                   "global_batch": GB, "micro_batch": b, "micro_batches": M, "seq_len": shape.seq,
                   "candidates_kbM": cands, "memory_cap_gb": args.mem_cap_gb or None,
                   "stages": S, "layers_per_stage": [(e - s_) / 2 for s_, e in halves],
                   "half_layer_ranges": [list(x) for x in halves],
                   "parallelism": f"pp{S}" if S > 1 else "single stage (no pipeline)",
                   "wgrad_pairs": wgrad_pairs,
                   "sm_reserved_for_emulator": int(os.environ.get("PTK_SM_RESERVE", "0")),
                   "schedule": (f"Ada-Grouper adaptive kFkB ((k, b) per step {plans_run})" if S > 1 else "1F1B (S=1)"),
                   "emulated_preemption": trace_desc, "l2": "working set (weights + activations) >> 126 MB L2"},
        "schedules": {"ada_grouper": {"kb_per_step": plans_run, "samples_per_s": round(value, 3),
                                      "tuning_overhead_s": round(tune_s, 4)},
                      "1f1b": {"kbM": by_k.get(1), "samples_per_s": round(v1f1b, 3),
                               "paired_wgrads_samples_per_s": round(v1f1b_paired, 3),
                               "unpaired_wgrads_samples_per_s": round(v1f1b_unpaired, 3) if v1f1b_unpaired else None},
                      "kfkb_k2": {"kbM": by_k.get(2), "samples_per_s": round(vk2, 3)},
                      "speedup_vs_1f1b": round(value / v1f1b, 4)},
        **({"kfkb_sweep": {str(k): {"kbM": by_k[k], "samples_per_s": round(GB * args.steps / (max(v) / 1e3), 3)}
                            for k, v in all_sweep.items()}} if all_sweep else {}),
        "tuner_decisions": [{"chosen": d["chosen"], "chosen_groups": d.get("chosen_groups"), "switched": d["switched"],
                             "estimates_ns": [e[3] for e in d["estimates"]]} for d in decisions],
        "pipeline_roofline": {"ideal_samples_per_s": round(ideal, 2), "frac": round(value / ideal, 4),
                              "peak_tflops": peak_sus, "peak_kind": f"sustained bf16, {pk_kind}"},
        "roofline": {"bound": "tensor", "kernel": "gemm_bf16_kernel (tcgen05 + TMA, all stage GEMMs)",
                     "achieved": round(achieved, 1), "peak": peak_sus, "unit": "TFLOP/s",
                     "frac": round(achieved / peak_sus, 4),
                     "traffic": (gemm_traffic() or {}).get("bytes_per_launch"), "traffic_detail": gemm_traffic(),
                     "launches": sum(g[2] for g in all_gemm),
                     "note": f"algorithmic GEMM FLOPs / summed CUDA-event GEMM durations over the timed steps; "
                             f"peak = sustained bf16 of {pk_kind} MEASURED_PEAKS.json"},
        "e2e": {"value": round(GB * args.steps / max(all_e2e), 3), "unit": "samples/s",
                "h2d_bytes_per_step": int(sum(all_h2d)), "d2h_bytes_per_step": 4},
        "gpu_launches": int(sum(all_launch)),
        "transfer_forward_ratio": ({"per_stage": all_xf, "mean": round(statistics.mean(x for x in all_xf if x), 4),
                                    "what": "mean paced inter-stage transfer / mean stage forward, last timed "
                                            "iteration (paper regime ~0.5, PAPER.md:102)"}
                                   if world > 1 and any(all_xf) else None),
        "loss": loss,
        "clocks": all_clk[0],
        "wall_s_timed": round(wall, 3),
    }
    if S > 1:
        # bubble_report / queue_analysis of the last timed iteration from the GPU timestamps, and the
        # cost model's simulate() of the same plan fed that iteration's mean durations
        try:
            from paper_2303_01675_b200.report import pipeline_report
            from paper_2303_01675_b200.tuning import pipeline_model
            out["hardware_report"] = pipeline_report(all_tl, pipeline_model(S, GB, shape.seq * shape.hidden * 2),
                                                     [g - all_sync[0] for g in all_sync])
            out["hardware_report"].pop("queue_analysis", None)
        except Exception as e:
            out["hardware_report"] = {"error": str(e)[:300]}
    if not args.no_cpu_baseline and world == 1:
        from oracle.cpu_baseline import time_cpu_training
        torch.cuda.empty_cache()
        out["cpu_baseline"] = time_cpu_training(shape, 1, 1)
    try:
        from oracle.cpu_baseline import planner_cost_us
        out["reference_planner_cpu"] = planner_cost_us(S, M, b, chosen[0])
    except Exception as e:  # the compiled reference planner is test infrastructure; report, never fail
        out["reference_planner_cpu"] = {"error": str(e)[:200]}
    if args.timeline:
        Path(args.timeline).write_text(json.dumps(tl))
    JSON_OUT.write(json.dumps(out) + "\n")
    JSON_OUT.flush()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
