"""Ada-Grouper online tuning across pipeline ranks (SPEC.md:453-467 on hardware).

A tuning round runs with the pipeline suspended at an iteration boundary:
  1. compute profiles — measured once per candidate micro-batch size at
     startup with CUDA events on each rank's own stage;
  2. link profiles — every rank probes its outgoing links `repeats` times per
     candidate payload through the (emulated) link, int64 ns samples;
  3. everything is all-gathered, so every rank holds the same inputs, and each
     rank calls the C++ decision function (pipetune::tuning_round via
     ptk_scenario_json op "decide"); the decision is deterministic, so all
     ranks switch to the same plan at the same boundary.
The recorded inputs form a replay log: the CPU oracle fed the same samples
must reproduce the decision bit for bit (tests/test_tuning_replay.py).
"""
from __future__ import annotations

from . import pipetune as pt


def outgoing_links(stage: int, stages: int) -> list[int]:
    """2s carries activations s -> s+1, 2s-1 carries grads s -> s-1 (model.hpp:15-24)."""
    out = []
    if stage + 1 < stages:
        out.append(2 * stage)
    if stage > 0:
        out.append(2 * stage - 1)
    return out


def pipeline_model(stages: int, global_batch: int, act_bytes_per_sample: int) -> dict:
    """The pipetune ModelSpec the decision runs on: real per-sample transfer bytes."""
    return pt.model_dict(pt.ModelSpec([pt.StageProfile(stage_id=s, output_bytes_per_sample_fwd=act_bytes_per_sample,
                                                       output_bytes_per_sample_bwd=act_bytes_per_sample)
                                       for s in range(stages)], global_batch))


def all_gather(obj, group=None, world: int = 1):
    if world == 1:
        return [obj]
    import torch.distributed as dist
    out = [None] * world
    dist.all_gather_object(out, obj, group=group)
    return out


class OnlineTuner:
    def __init__(self, ex, rank: int, stages: int, global_batch: int, candidates: list[tuple[int, int]],
                 act_bytes_per_sample: int, hysteresis: float = 0.02, repeats: int = 3, window: int = 8,
                 group=None, passive: bool = False, mixed: bool = True, probe_every: int = 1):
        self.ex, self.rank, self.S = ex, rank, stages
        # with passive samples, re-probe the other candidates' payloads only every `probe_every`
        # rounds (1: every round); in between, their ProfileStore buckets keep serving
        # the last `window` samples
        self.probe_every = max(1, probe_every)
        self.rounds = 0
        self.gb = global_batch
        self.cands = [[k, b, global_batch // b] for k, b in candidates]
        self.act = act_bytes_per_sample
        self.h, self.repeats, self.window, self.group = hysteresis, repeats, window, group
        self.passive = passive  # use observe_iteration() samples for the current payload
        # mixed-k candidates: for every k that does not divide M, the remainder group first
        # (shorter warm-up than uniform kFkB's short last group; tests/test_mixed_plans.py)
        self.mixed = [[b, [M % k] + [k] * (M // k)] for k, b, M in self.cands if M % k] if mixed else []
        self.compute = None
        self.samples: list[list[int]] = []
        self.log: list[dict] = []
        self.model = pipeline_model(stages, global_batch, act_bytes_per_sample)

    def profile_compute(self):
        """Once, at startup: F/B durations per candidate b on this rank, gathered."""
        mine = []
        for b in sorted({c[1] for c in self.cands}):
            f, bw = self.ex.profile_compute(b, 3)
            mine += [[self.rank, b, 0, f], [self.rank, b, 1, bw]]
        self.compute = sorted(x for r in all_gather(mine, self.group, self.S) for x in r)

    def _add_samples(self, gathered):
        """Append in recording order, keeping only the last `window` per (link, payload) bucket —
        all the ProfileStore ever reads, so the request stays bounded."""
        self.samples += gathered
        keep, seen = [], {}
        for x in reversed(self.samples):
            key = (x[0], x[1])
            if seen.get(key, 0) < self.window:
                seen[key] = seen.get(key, 0) + 1
                keep.append(x)
        self.samples = keep[::-1]

    def observe_iteration(self, timeline: dict, clock: int = 0):
        """Passive link profile: every transfer the last iteration made on this rank's outgoing links
        is a sample of its exact payload under the live contention (no pipeline suspension).
        Collective: every rank calls it after the same iteration."""
        mine = [[int(link), int(nbytes), clock, int(end) - int(start)]
                for link, mb, nbytes, start, end in timeline.get("xfer", [])]
        self._add_samples(sorted(x for r in all_gather(mine, self.group, self.S) for x in r))
        self.passive_bytes = {x[1] for x in mine}

    def needs_probes(self, current_b: int) -> bool:
        """Whether the next round, observing an iteration that ran at micro-batch `current_b`, will
        probe any payload.  Computed from state every rank shares (candidates, gathered samples,
        round count), so all ranks agree without a collective."""
        payloads = {c[1] * self.act for c in self.cands}
        skip = {current_b * self.act} if self.passive else set()
        if self.passive and self.rounds % self.probe_every != 0:
            skip |= {x[1] for x in self.samples}
        return bool(payloads - skip)

    def profile_links(self, clock: int = 0):
        """Active probes (pipeline suspended): every candidate payload not already
        measured passively in the last iteration, `repeats` times per outgoing link (rounds between
        `probe_every` boundaries probe only payloads the store has never seen)."""
        mine = []
        skip = getattr(self, "passive_bytes", set()) if self.passive else set()
        if self.passive and self.rounds % self.probe_every != 0:
            skip = skip | {x[1] for x in self.samples}
        for b in sorted({c[1] for c in self.cands}):
            nbytes = b * self.act
            if nbytes in skip:
                continue
            for link in outgoing_links(self.rank, self.S):
                for d in self.ex.probe_link(link, nbytes, self.repeats):
                    mine.append([link, nbytes, clock, d])
        self._add_samples(sorted(x for r in all_gather(mine, self.group, self.S) for x in r))

    def decide(self, current, clock: int = 0, current_groups=None) -> dict:
        req = {"op": "decide", "model": self.model, "candidates": self.cands, "compute_profile": self.compute,
               "samples": [list(x) for x in self.samples], "hysteresis": self.h, "window": self.window,
               "clock": clock}
        if self.mixed:
            req["group_candidates"] = self.mixed
        if current is not None:
            req["current"] = list(current)[:3]
        if current_groups:
            req["current_groups"] = list(current_groups)
        d = pt.scenario(req)["decision"]
        self.log.append({"request": req, "decision": d})
        return d

    def round(self, current, clock: int = 0, current_groups=None) -> dict:
        if self.compute is None:
            self.profile_compute()
        self.profile_links(clock)
        self.rounds += 1
        return self.decide(current, clock, current_groups)


def pair_bytes_per_sample(shape, hb: int, he: int, has_head: bool) -> int:
    """Per-sample bytes of the paired-weight-gradient buffers GptStage allocates at b_max
    (gpt_stage.cu, `wgrad_pairs`: per layer of the stage out, d(x_mid), d_ln, dy [T,h], d_pre [T,f],
    dqkv [T,3h]; on the head stage the head's g and dy [T,h])."""
    from .stage import halves_to_layers
    lb, le, _, _ = halves_to_layers(hb, he)
    s, h, f = shape.seq, shape.hidden, shape.ffn
    return (le - lb) * (7 * s * h + s * f) * 2 + (2 * s * h * 2 if has_head else 0)


def memory_model(shape, layers, stages: int, global_batch: int, halves: bool = False,
                 pairs_b_max: int = 0) -> dict:
    """pipetune ModelSpec with the real per-stage byte model: weights = fp32 master +
    grad + AdamW m, v + bf16 copy (18 B/param); activations = the stash per sample.
    `layers`: per-stage layer ranges, or half-layer ranges when `halves`.  pairs_b_max > 0 budgets
    paired weight gradients allocated at that b_max as a fixed per-stage cost: their buffers plus
    the one extra stash slot of b_max samples the executor keeps (SPEC.md:218-226 liveness + it)."""
    st = []
    for s_, (lb, le) in enumerate(layers):
        first, last = s_ == 0, s_ == stages - 1
        params = shape.param_count_halves(lb, le, first, last) if halves else shape.param_count(le - lb, first, last)
        stash = shape.stash_bytes_halves(lb, le, last, first) if halves else \
            shape.stash_bytes_per_sample(le - lb, last, first)
        hb, he = (lb, le) if halves else (2 * lb, 2 * le)
        fixed = pairs_b_max * (stash + pair_bytes_per_sample(shape, hb, he, last)) if pairs_b_max else 0
        st.append(pt.StageProfile(
            stage_id=s_, weight_bytes=18 * params + fixed,
            activation_bytes_per_sample=stash,
            output_bytes_per_sample_fwd=shape.seq * shape.hidden * 2,
            output_bytes_per_sample_bwd=shape.seq * shape.hidden * 2))
    return pt.model_dict(pt.ModelSpec(st, global_batch))


def candidate_set(shape, layers, stages: int, global_batch: int, mem_cap_bytes: int | None, k_max: int = 8,
                  fixed_b: int = 2, halves: bool = False, wgrad_pairs: bool = False) -> list[list[int]]:
    """Ada-Grouper candidates: the (k, b) memory-limit frontier via the C++
    enumerate_candidates under an imposed per-GPU cap; without a cap, k in {1,2,4,8} at b.
    With wgrad_pairs the pairing buffers of the allocation (sized by the largest candidate b) are
    budgeted too: b_max is iterated to a fixed point (it can only shrink)."""
    if mem_cap_bytes is None:
        M = global_batch // fixed_b
        return [[k, fixed_b, M] for k in (1, 2, 4, 8) if k <= M]

    def frontier(pairs_b_max):
        model = memory_model(shape, layers, stages, global_batch, halves, pairs_b_max)
        out = pt.scenario({"op": "enumerate", "model": model, "k_max": k_max,
                           "cluster": {"device_memory_limit": int(mem_cap_bytes), "devices": stages}})
        return [e[:3] for e in out["entries"]]

    cands = frontier(0)
    if not wgrad_pairs:
        return cands
    # The pairing buffers are a fixed cost sized by the largest candidate b.  Take the largest b_max
    # (a divisor of the global batch, from the unpaired frontier's largest b down) that is
    # self-consistent: with the buffers budgeted at b_max the frontier still reaches b_max.  Budgets
    # that leave no frontier at all are skipped (they used to raise InfeasibleModel).
    divisors = [d for d in range(global_batch, 0, -1) if global_batch % d == 0]
    for b_max in [d for d in divisors if d <= max(c[1] for c in cands)]:
        try:
            paired = frontier(b_max)
        except pt.PipetuneError as e:
            if e.kind != "InfeasibleModel":
                raise
            continue
        if max(c[1] for c in paired) < b_max:
            continue
        out = []
        for k, b, _ in paired:  # a candidate above the budget runs at the largest divisor within it
            b = max(d for d in divisors if d <= min(b, b_max))
            if all(o[0] != k for o in out):
                out.append([k, b, global_batch // b])
        return out
    raise pt.PipetuneError("InfeasibleModel", "no (k, b) fits the memory cap with the paired weight-gradient buffers")
