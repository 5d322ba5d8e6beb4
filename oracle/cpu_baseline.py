"""ORACLE TEST INFRASTRUCTURE — the CPU path timed as bench.py's baseline.

"The reference's CPU path" for this hot path:
  (i)   the reference planner, compiled unmodified from /root/reference into
        oracle/_ref/ref_dump (travels to the GPU box with the snapshot), gives
        the per-device kFkB order;
  (ii)  that order is executed on the host cores by the fp32 oracle model
        (oracle/gpt_oracle.py) — one fwd+bwd per scheduled micro-batch —
        over a BOUNDED sample of the workload.
Only bench.py's cpu_baseline leg and `--impl reference` call this.
"""
from __future__ import annotations

import os
import subprocess
import time
from pathlib import Path

import torch

from . import gpt_oracle as G

ROOT = Path(__file__).resolve().parents[1]
REF_BIN = ROOT / "oracle" / "_ref" / "ref_dump"


def reference_order(stages: int, micro_batches: int, b: int, k: int) -> tuple[list[str], str]:
    """Stage-0 order from the compiled reference planner, else the oracle restatement."""
    if REF_BIN.exists():
        out = subprocess.run([str(REF_BIN)], input=f"{stages} {micro_batches} {b} 1 {k} 1 1\n",
                             capture_output=True, text=True, check=True).stdout
        import json
        seq = json.loads(out)["sequences"][0].split()
        return seq, "reference"
    from . import spec_oracle as O
    g = O.Graph([{"output_bytes_per_sample_fwd": 1, "output_bytes_per_sample_bwd": 1}] * stages, b, micro_batches)
    orders = O.kfkb_orders(g, k)
    names = {0: "F", 1: "B", 4: "GA"}
    seq = [names[g.nodes[i][0]] + (str(g.nodes[i][2]) if g.nodes[i][0] != 4 else "") for i in orders[0]]
    return seq, "port"


class CpuTrainer:
    """The CPU path, weights initialised once; step() times one bounded sample."""

    def __init__(self, shape, b: int, micro_batches_to_run: int, k: int = 1, threads: int | None = None,
                 seed: int = 1234):
        self.shape, self.b, self.M, self.k, self.seed = shape, b, micro_batches_to_run, k, seed
        self.threads = threads or os.cpu_count() or 1
        torch.set_num_threads(self.threads)
        self.seq, self.kind = reference_order(1, micro_batches_to_run, b, k)
        self.w = init_weights(shape)

    def step(self) -> dict:
        shape, b = self.shape, self.b
        for t in self.w.values():
            t.grad = None
        stash = {}
        t0 = time.perf_counter()
        for tok_name in self.seq:
            if tok_name == "GA":
                continue
            m = int(tok_name[1:])
            if tok_name[0] == "F":
                tok, lab = G.synthetic_batch(self.seed, m, b, shape.seq, shape.vocab)
                _, loss = G.stage_forward(self.w, shape, 0, shape.n_layer, True, True, tok=tok, labels=lab,
                                          micro_batches=self.M)
                stash[m] = loss
            else:
                stash.pop(m).backward()
        dt = time.perf_counter() - t0
        samples = b * self.M
        return {"value": samples / dt, "unit": "samples/s", "cores": self.threads, "kind": "port",
                "order_source": self.kind, **host_info(),
                "sample": f"{shape.n_layer}-layer h={shape.hidden} s={shape.seq} {shape.arch.upper()} fp32 fwd+bwd "
                          f"of {samples} sample(s) (b={b}) by the oracle port (oracle/gpt_oracle.py) on the host "
                          f"cores, in the order of the {self.kind} planner; {dt:.1f} s"}


def host_info() -> dict:
    """CPU model and core count of the host the CPU path ran on."""
    model = "unknown"
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count()}


def planner_cost_us(stages: int, micro_batches: int, b: int, k: int, reps: int = 200) -> dict | None:
    """Mean µs of the COMPILED REFERENCE planner (build_task_graph + plan_kfkb, reference
    taskgraph.cpp:35 / plan.cpp:75) for this configuration, 1 core — the reference's own CPU cost
    of the path, timed beside the GPU run (oracle/ref_dump --time)."""
    if not REF_BIN.exists():
        return None
    out = subprocess.run([str(REF_BIN), "--time", str(reps)], input=f"{stages} {micro_batches} {b} 1 {k} 1 1\n",
                         capture_output=True, text=True, check=True).stdout.split()
    return {"us": float(out[0]), "config": [stages, micro_batches, b, k], "reps": reps,
            "what": "reference build_task_graph + plan_kfkb, g++ -O2, 1 core"}


def init_weights(shape):
    g = torch.Generator().manual_seed(42)
    h, f, V, s = shape.hidden, shape.ffn, shape.vocab, shape.seq
    w = {"wte": torch.randn(V, h, generator=g) * 0.02, "wpe": torch.randn(s, h, generator=g) * 0.02,
         "lnf_g": torch.ones(h), "lnf_b": torch.zeros(h), "w_head": torch.randn(V, h, generator=g) * 0.02}
    for l in range(shape.n_layer):
        p = f"h{l}."
        w.update({p + "ln1_g": torch.ones(h), p + "ln1_b": torch.zeros(h),
                  p + "w_qkv": torch.randn(3 * h, h, generator=g) * 0.02, p + "b_qkv": torch.zeros(3 * h),
                  p + "w_o": torch.randn(h, h, generator=g) * 0.02, p + "b_o": torch.zeros(h),
                  p + "ln2_g": torch.ones(h), p + "ln2_b": torch.zeros(h),
                  p + "w_fc1": torch.randn(f, h, generator=g) * 0.02, p + "b_fc1": torch.zeros(f),
                  p + "w_fc2": torch.randn(h, f, generator=g) * 0.02, p + "b_fc2": torch.zeros(h)})
    if shape.arch == "bert":
        w.update({"lne_g": torch.ones(h), "lne_b": torch.zeros(h), "w_t": torch.randn(h, h, generator=g) * 0.02,
                  "b_t": torch.zeros(h)})
    for t in w.values():
        t.requires_grad_(True)
    return w


def time_cpu_training(shape, b: int, micro_batches_to_run: int, k: int = 1, threads: int | None = None,
                      seed: int = 1234) -> dict:
    """One bounded sample: fwd+bwd of `micro_batches_to_run` micro-batches of size b."""
    return CpuTrainer(shape, b, micro_batches_to_run, k, threads, seed).step()
