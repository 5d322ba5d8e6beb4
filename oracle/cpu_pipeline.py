"""ORACLE TEST INFRASTRUCTURE — the CPU-thread pipeline executor.

The reference's own "execution" of a plan is the spec's discrete-event
simulator; SURVEY §8(d) asks for the CPU path that really runs it: one
`threading.Thread` per stage, the buffer queues of the simulator (SPEC.md:333:
one FIFO receive stream per device and link) as `queue.Queue`s, and the fp32
oracle math (oracle/gpt_oracle.py) for each scheduled F/B, with the host cores
split between the stages (torch's intra-op pool sized nproc / S; the stage
threads' ops run concurrently, PyTorch releases the GIL inside them).

Each stage walks the per-device order of the UNMODIFIED reference planner
(oracle/_ref/ref_dump, plan_kfkb — reference plan.cpp:70-104) or, when that
binary is absent, the oracle restatement (spec_oracle.kfkb_orders).  Stage s
holds layers [s·L/S, (s+1)·L/S), the embedding on stage 0 and the head + loss
on stage S-1 (the reference's contiguous layer stages, model.hpp:55).
Activations travel forward as detached tensors; the receiving stage makes them
autograd leaves and sends their .grad back, so gradients equal the
single-process model's (tests/test_cpu_pipeline.py).

Only tests/, bench.py's cpu_baseline leg and `--impl reference` use this.
"""
from __future__ import annotations

import json
import os
import queue
import subprocess
import threading
import time

import torch

from . import gpt_oracle as G
from .cpu_baseline import REF_BIN, init_weights


def reference_orders(stages: int, micro_batches: int, b: int, k: int) -> tuple[list[list[str]], str]:
    """Every stage's kFkB order ("F0", "B0", ..., "GA") from the compiled reference planner, else the port."""
    if REF_BIN.exists():
        out = subprocess.run([str(REF_BIN)], input=f"{stages} {micro_batches} {b} 1 {k} 1 1\n",
                             capture_output=True, text=True, check=True).stdout
        return [s.split() for s in json.loads(out)["sequences"]], "reference"
    from . import spec_oracle as O
    g = O.Graph([{"output_bytes_per_sample_fwd": 1, "output_bytes_per_sample_bwd": 1}] * stages, b, micro_batches)
    names = {0: "F", 1: "B", 4: "GA"}
    return [[names[g.nodes[i][0]] + (str(g.nodes[i][2]) if g.nodes[i][0] != 4 else "") for i in order]
            for order in O.kfkb_orders(g, k)], "port"


class CpuPipeline:
    """S stage threads executing the reference plan on the host cores; step() = one iteration."""

    def __init__(self, shape, stages: int, b: int, micro_batches: int, k: int = 1, threads: int | None = None,
                 seed: int = 1234, weights: dict | None = None):
        if not 1 <= stages <= shape.n_layer:
            raise ValueError("need 1 <= stages <= layers")
        self.shape, self.S, self.b, self.M, self.k, self.seed = shape, stages, b, micro_batches, k, seed
        self.threads = threads or os.cpu_count() or 1
        self.orders, self.kind = reference_orders(stages, micro_batches, b, k)
        self.bounds = [(s * shape.n_layer // stages, (s + 1) * shape.n_layer // stages) for s in range(stages)]
        self.w = weights if weights is not None else init_weights(shape)
        self.loss = 0.0

    def _stage(self, s: int, acts: list, grads: list, losses: list, errors: list):
        shape, S, b = self.shape, self.S, self.b
        l0, l1 = self.bounds[s]
        stash = {}
        try:
            for op in self.orders[s]:
                if op == "GA":
                    continue  # gradients accumulated in place, micro-batch order
                m = int(op[1:])
                if op[0] == "F":
                    tok, lab = G.synthetic_batch(self.seed, m, b, shape.seq, shape.vocab)
                    x_in = None if s == 0 else acts[s - 1].get().requires_grad_(True)
                    out, loss = G.stage_forward(self.w, shape, l0, l1, s == 0, s == S - 1, tok=tok, x_in=x_in,
                                                labels=lab, micro_batches=self.M)
                    if s < S - 1:
                        acts[s].put(out.detach())
                        stash[m] = (x_in, out)
                    else:
                        losses.append(loss.item())
                        stash[m] = (x_in, loss)
                elif op[0] == "B":
                    x_in, y = stash.pop(m)
                    if s == S - 1:
                        y.backward()
                    else:
                        y.backward(grads[s].get())
                    if s > 0:
                        grads[s - 1].put(x_in.grad)
                else:
                    raise ValueError(f"stage {s}: unknown plan op {op!r}")
        except BaseException as e:  # surface a stage failure instead of deadlocking its peers
            errors.append(e)
            for q in acts + grads:
                q.put(None)

    def step(self) -> dict:
        for t in self.w.values():
            t.grad = None
        S = self.S
        torch.set_num_threads(max(1, self.threads // S))
        acts = [queue.Queue() for _ in range(S - 1)]
        grads = [queue.Queue() for _ in range(S - 1)]
        losses, errors = [], []
        workers = [threading.Thread(target=self._stage, args=(s, acts, grads, losses, errors), daemon=True)
                   for s in range(S)]
        t0 = time.perf_counter()
        for t in workers:
            t.start()
        for t in workers:
            t.join()
        dt = time.perf_counter() - t0
        if errors:
            raise errors[0]
        self.loss = sum(losses)
        samples = self.b * self.M
        shape = self.shape
        from .cpu_baseline import host_info
        return {"value": samples / dt, "unit": "samples/s", "cores": self.threads, "kind": "port",
                "order_source": self.kind, **host_info(),
                "sample": f"{shape.n_layer}-layer h={shape.hidden} s={shape.seq} {shape.arch.upper()} fp32, "
                          f"{S} stage thread(s) x {max(1, self.threads // S)} intra-op threads, one iteration of "
                          f"{self.M} micro-batch(es) of b={self.b} in the reference planner's k={self.k} order; "
                          f"{dt:.1f} s"}
