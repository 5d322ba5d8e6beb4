"""Python handle over the kFkB stage executor (ptk_exec_* in include/ptk.h).

The host loop lives in C++ (executor.cu); this module only wires processes
together: one process per GPU/stage, IPC handles exchanged over a gloo group
(torch.distributed is plumbing), and the tuner's measurements gathered so
every rank feeds the same samples to the C++ decision function.
"""
from __future__ import annotations

import ctypes as C
import json
import math

from . import _lib as L
from .stage import GptConfig, ModelShape, _declare as _declare_stage


class ExecConfig(C.Structure):
    _fields_ = [("gpt", GptConfig), ("stage", C.c_int), ("stages", C.c_int), ("global_batch", C.c_int),
                ("lr", C.c_float), ("weight_decay", C.c_float), ("data_seed", C.c_uint64)]


def _declare(lib):
    if getattr(lib, "_exec_declared", False):
        return
    _declare_stage(lib)
    V, I, P = C.c_void_p, C.c_int, C.POINTER
    lib.ptk_exec_create.argtypes = [P(ExecConfig), P(V)]
    lib.ptk_exec_destroy.argtypes = [V]
    lib.ptk_exec_export.argtypes = [V, V, C.c_size_t, P(C.c_size_t)]
    lib.ptk_exec_import.argtypes = [V, I, V, C.c_size_t]
    lib.ptk_exec_connect_local.argtypes = [V, I, V]
    lib.ptk_exec_set_plan.argtypes = [V, I, I]
    lib.ptk_exec_set_plan_groups.argtypes = [V, I, C.POINTER(C.c_int), I]
    lib.ptk_exec_set_trace.argtypes = [V, I, C.c_double, C.c_int64, I, P(C.c_int64), P(C.c_int64), P(C.c_double)]
    lib.ptk_exec_set_epoch.argtypes = [V, C.c_int64]
    lib.ptk_exec_set_contender.argtypes = [V, I]
    lib.ptk_globaltimer.restype = C.c_int64
    lib.ptk_exec_run_iteration.argtypes = [V, I, V]
    lib.ptk_exec_finish_iteration.argtypes = [V, P(C.c_double)]
    lib.ptk_exec_begin_iteration.argtypes = [V, I, V]
    lib.ptk_exec_enqueue_next.argtypes = [V, P(I)]
    lib.ptk_exec_run_local.argtypes = [P(V), I, I, V]
    lib.ptk_exec_set_deadlock_timeout.argtypes = [V, C.c_double]
    lib.ptk_exec_set_send_streams.argtypes = [V, I]
    lib.ptk_exec_read_loss.argtypes = [V, P(C.c_float)]
    lib.ptk_exec_timeline_json.argtypes = [V, C.c_char_p, C.c_size_t, P(C.c_size_t)]
    lib.ptk_exec_probe_link.argtypes = [V, I, C.c_int64, I, P(C.c_int64)]
    lib.ptk_exec_profile_compute.argtypes = [V, I, I, P(C.c_int64), P(C.c_int64)]
    lib.ptk_exec_gemm_timing.argtypes = [V, I, P(C.c_double), P(C.c_double), P(C.c_long)]
    lib.ptk_exec_stage.argtypes = [V]
    lib.ptk_exec_stage.restype = C.c_void_p
    lib.ptk_exec_set_defer_optimizer.argtypes = [V, I]
    lib.ptk_exec_set_wgrad_pairs.argtypes = [V, I]
    lib.ptk_exec_compute_stream.argtypes = [V, P(V)]
    lib._exec_declared = True


def partition_layers(n_layer: int, stages: int, head_weight: float = 2.0) -> list[tuple[int, int]]:
    """Contiguous layer ranges minimising the bottleneck stage, counting the LM
    head (on the last stage) as `head_weight` layer-equivalents."""
    if stages == 1:
        return [(0, n_layer)]
    best = None
    # binary-search-free exhaustive DP over cut points (n_layer <= 64)
    from functools import lru_cache

    @lru_cache(None)
    def solve(start: int, k: int):
        if k == 1:
            cost = (n_layer - start) + head_weight
            return (cost, ((start, n_layer),))
        out = None
        for end in range(start + 1, n_layer - k + 2):
            rest = solve(end, k - 1)
            cost = max(end - start, rest[0])
            if out is None or cost < out[0] or (cost == out[0] and end - start > out[1][0][1] - out[1][0][0]):
                out = (cost, ((start, end),) + rest[1])
        return out

    best = solve(0, stages)
    return list(best[1])


def partition_halves(n_layer: int, stages: int, head_weight: float = 1.6, attn_weight: float = 0.47,
                     embed_weight: float = 0.05) -> list[tuple[int, int]]:
    """Contiguous HALF-layer ranges [hb, he) (2l = attention block, 2l+1 = MLP block of layer l)
    minimising the bottleneck stage cost, with the attention block at `attn_weight` of a layer
    (measured on B200: 322 vs 357 us per GPT-1.3B layer-micro-batch), the LM head at `head_weight`
    layers on the last stage and the embedding at `embed_weight` on the first.  Half-layer cuts let
    24 layers + head balance over 8 stages (bottleneck 3.3 instead of 4 layer-equivalents)."""
    n = 2 * n_layer
    w = [attn_weight if u % 2 == 0 else 1.0 - attn_weight for u in range(n)]
    pre = [0.0]
    for x in w:
        pre.append(pre[-1] + x)
    from functools import lru_cache

    @lru_cache(None)
    def solve(start: int, k: int):
        # minimise the bottleneck, then the sum of squared stage costs (spreads the slack)
        extra_first = embed_weight if start == 0 else 0.0
        if k == 1:
            c = pre[n] - pre[start] + head_weight + extra_first
            return (c, c * c, ((start, n),))
        best = None
        for end in range(start + 1, n - k + 2):
            rest = solve(end, k - 1)
            c = pre[end] - pre[start] + extra_first
            key = (round(max(c, rest[0]), 9), round(c * c + rest[1], 9))
            if best is None or key < (round(best[0], 9), round(best[1], 9)):
                best = (max(c, rest[0]), c * c + rest[1], ((start, end),) + rest[2])
        return best

    return list(solve(0, stages)[2])


def max_inflight(stage: int, stages: int, micro_batches: int, k: int) -> int:
    """Peak in-flight forwards of kFkB at a stage: min(M, min(S-s, ceil(M/k))*k)."""
    return min(micro_batches, min(stages - stage, math.ceil(micro_batches / k)) * k)


def stage_slots(stage: int, stages: int, candidates) -> tuple[int, int]:
    """(slots, b_max) the executor of `stage` needs to run every (k, b, M) candidate: physical stash
    slots are b_max samples wide and hold b_max / b micro-batches each (sample-granular stash), so the
    count covers the largest in-flight sample count over the candidates (SURVEY §4 closed form)."""
    b_max = max(c[1] for c in candidates)
    slots = -(-max(max_inflight(stage, stages, c[2], c[0]) * c[1] for c in candidates) // b_max)
    slots = max(slots, max(max_inflight(stage, stages, c[2], c[0]) for c in candidates if c[1] == b_max))
    return slots, b_max


def _tokens_ptr(host_tokens):
    """host_tokens: None, a raw pointer (int), or an int32 array of 2 * global_batch * seq ids
    (tokens then labels) — an array stays referenced by the caller's frame for the whole call."""
    if host_tokens is None or isinstance(host_tokens, int):
        return host_tokens
    import numpy as np
    if not (isinstance(host_tokens, np.ndarray) and host_tokens.dtype == np.int32 and host_tokens.flags.c_contiguous):
        raise TypeError("host_tokens must be a C-contiguous int32 numpy array or a pointer")
    return host_tokens.ctypes.data


class StageExecutor:
    def __init__(self, shape: ModelShape, stage: int, stages: int, global_batch: int, b_max: int, slots: int,
                 layers: tuple[int, int] | None = None, seed: int = 42, data_seed: int = 1234, lr: float = 1e-4,
                 weight_decay: float = 0.0, halves: tuple[int, int] | None = None, wgrad_pairs: bool = False):
        """`layers` = whole-layer range [lb, le); or `halves` = half-layer range [hb, he) (stage
        boundaries may fall between a layer's attention and MLP blocks).  `wgrad_pairs`: weight
        gradients of consecutive micro-batches in one two-segment GEMM (one more stash slot)."""
        self.lib = L.lib()
        _declare(self.lib)
        from .stage import halves_to_layers
        if halves is not None:
            lb, le, sfa, slm = halves_to_layers(*halves)
        else:
            lb, le = layers if layers is not None else partition_layers(shape.n_layer, stages)[stage]
            sfa = slm = 0
        if wgrad_pairs:
            slots += 1  # the deferred micro-batch's stash stays live until its partner's backward
        gpt = GptConfig(shape.n_layer, shape.hidden, shape.heads, shape.ffn, shape.seq, shape.vocab, lb, le,
                        int(stage == 0), int(stage == stages - 1), b_max, slots, global_batch // b_max,
                        shape.arch_id, seed, sfa, slm, int(wgrad_pairs))
        self.cfg = ExecConfig(gpt, stage, stages, global_batch, lr, weight_decay, data_seed)
        self.shape, self.stage, self.stages, self.global_batch = shape, stage, stages, global_batch
        h = C.c_void_p()
        L.check(self.lib.ptk_exec_create(C.byref(self.cfg), C.byref(h)))
        self.h = h

    # ---- wiring
    def export_handles(self) -> bytes:
        buf = C.create_string_buffer(4096)
        n = C.c_size_t()
        L.check(self.lib.ptk_exec_export(self.h, buf, len(buf), C.byref(n)))
        return buf.raw[:n.value]

    def import_peer(self, peer_stage: int, blob: bytes):
        L.check(self.lib.ptk_exec_import(self.h, peer_stage, blob, len(blob)))

    def connect_local(self, peer_stage: int, peer: "StageExecutor"):
        L.check(self.lib.ptk_exec_connect_local(self.h, peer_stage, peer.h))

    def connect_dist(self, group=None):
        """Exchange IPC handles with the neighbouring ranks (rank in `group` == stage)."""
        import torch.distributed as dist
        blobs = [None] * dist.get_world_size(group)
        dist.all_gather_object(blobs, self.export_handles(), group=group)
        if self.stage + 1 < self.stages:
            self.import_peer(self.stage + 1, blobs[self.stage + 1])
        if self.stage > 0:
            self.import_peer(self.stage - 1, blobs[self.stage - 1])

    # ---- data-parallel replicas
    def set_defer_optimizer(self, on: bool = True):
        """GradAccum only finalizes the gradients; data_parallel_step() all-reduces and steps."""
        L.check(self.lib.ptk_exec_set_defer_optimizer(self.h, int(bool(on))))

    def set_wgrad_pairs(self, on: bool):
        """Paired weight gradients on/off from the next iteration (needs wgrad_pairs=True at creation)."""
        L.check(self.lib.ptk_exec_set_wgrad_pairs(self.h, int(bool(on))))

    def compute_stream(self) -> int:
        s = C.c_void_p()
        L.check(self.lib.ptk_exec_compute_stream(self.h, C.byref(s)))
        return s.value or 0

    def data_parallel_step(self, dp_group, step: bool = True):
        """After run_iteration(): average this stage's gradients over its data-parallel replicas
        (NCCL all-reduce, ordered on the executor's compute stream) and run AdamW there.
        Replicas start from identical weights (same seed) and stay bit-identical."""
        import torch
        import torch.distributed as dist
        if not hasattr(self, "_dp_view"):
            self._dp_view = self.stage_view()
        stream = torch.cuda.ExternalStream(self.compute_stream())
        with torch.cuda.stream(stream):
            if dist.get_backend(dp_group) == "nccl":
                dist.all_reduce(self._dp_view.grads, op=dist.ReduceOp.AVG, group=dp_group)
            else:  # gloo (tests on one GPU): no AVG reduction; sum, then scale on the compute stream
                dist.all_reduce(self._dp_view.grads, op=dist.ReduceOp.SUM, group=dp_group)
                self._dp_view.grads.mul_(1.0 / dist.get_world_size(dp_group))
        if step:
            L.check(self.lib.ptk_stage_optimizer_step(self.lib.ptk_exec_stage(self.h), self.cfg.lr,
                                                      self.cfg.weight_decay, C.c_void_p(stream.cuda_stream)))

    # ---- schedule / emulator
    def set_plan(self, k: int, b: int):
        L.check(self.lib.ptk_exec_set_plan(self.h, k, b))

    def set_plan_groups(self, b: int, group_sizes):
        """kFkB over explicit group sizes (k switches at group boundaries inside an iteration)."""
        arr = (C.c_int * len(group_sizes))(*[int(x) for x in group_sizes])
        L.check(self.lib.ptk_exec_set_plan_groups(self.h, b, arr, len(group_sizes)))

    def set_trace(self, link: int, base_bytes_per_ns: float, latency_ns: int, segments):
        n = len(segments)
        s = (C.c_int64 * max(n, 1))(*[int(x[0]) for x in segments])
        e = (C.c_int64 * max(n, 1))(*[int(x[1]) for x in segments])
        a = (C.c_double * max(n, 1))(*[float(x[2]) for x in segments])
        L.check(self.lib.ptk_exec_set_trace(self.h, link, base_bytes_per_ns, latency_ns, n, s, e, a))

    def set_contender(self, on: bool):
        L.check(self.lib.ptk_exec_set_contender(self.h, int(on)))

    def set_epoch(self, epoch_ns: int):
        L.check(self.lib.ptk_exec_set_epoch(self.h, epoch_ns))

    def globaltimer(self) -> int:
        return self.lib.ptk_globaltimer()

    # ---- iterations
    def run_iteration(self, it: int, host_tokens=None):
        L.check(self.lib.ptk_exec_run_iteration(self.h, it, _tokens_ptr(host_tokens)))

    def begin_iteration(self, it: int, host_tokens=None):
        L.check(self.lib.ptk_exec_begin_iteration(self.h, it, _tokens_ptr(host_tokens)))

    def enqueue_next(self) -> bool:
        more = C.c_int()
        L.check(self.lib.ptk_exec_enqueue_next(self.h, C.byref(more)))
        return bool(more.value)

    def set_deadlock_timeout(self, seconds: float):
        L.check(self.lib.ptk_exec_set_deadlock_timeout(self.h, float(seconds)))

    def set_send_streams(self, per_link: bool):
        L.check(self.lib.ptk_exec_set_send_streams(self.h, int(bool(per_link))))

    def finish_iteration(self) -> float:
        ms = C.c_double()
        L.check(self.lib.ptk_exec_finish_iteration(self.h, C.byref(ms)))
        return ms.value

    def read_loss(self) -> float:
        v = C.c_float()
        L.check(self.lib.ptk_exec_read_loss(self.h, C.byref(v)))
        return v.value

    def timeline(self) -> dict:
        n = C.c_size_t()
        buf = C.create_string_buffer(1 << 22)
        L.check(self.lib.ptk_exec_timeline_json(self.h, buf, len(buf), C.byref(n)))
        return json.loads(buf.value.decode())

    def probe_link(self, link: int, nbytes: int, repeats: int) -> list[int]:
        out = (C.c_int64 * repeats)()
        L.check(self.lib.ptk_exec_probe_link(self.h, link, nbytes, repeats, out))
        return list(out)

    def profile_compute(self, b: int, repeats: int = 3) -> tuple[int, int]:
        f, bw = C.c_int64(), C.c_int64()
        L.check(self.lib.ptk_exec_profile_compute(self.h, b, repeats, C.byref(f), C.byref(bw)))
        return f.value, bw.value

    def gemm_timing(self, enable: int = -1):
        fl, ms, n = C.c_double(), C.c_double(), C.c_long()
        L.check(self.lib.ptk_exec_gemm_timing(self.h, enable, C.byref(fl), C.byref(ms), C.byref(n)))
        return fl.value, ms.value, n.value

    def stage_view(self):
        from .stage import GptStage
        return GptStage.view(self.lib, self.lib.ptk_exec_stage(self.h), self.shape, self.cfg.gpt.micro_batch_size)

    @staticmethod
    def run_local(stages: "list[StageExecutor]", it: int, host_tokens=None) -> list[float]:
        """One iteration of a whole same-process pipeline (stages[s] = stage s, connect_local-wired),
        enqueued in a global dependency-respecting order (ptk_exec_run_local), then finished stage by
        stage; returns each stage's device ms."""
        lib = stages[0].lib
        arr = (C.c_void_p * len(stages))(*[e.h.value for e in stages])
        L.check(lib.ptk_exec_run_local(arr, len(stages), it, _tokens_ptr(host_tokens)))
        return [e.finish_iteration() for e in stages]

    def close(self):
        if getattr(self, "h", None):
            self.lib.ptk_exec_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
