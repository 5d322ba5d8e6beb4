"""Multi-GPU pipeline correctness (torchrun, one rank per GPU = one stage).

After 2 training iterations the master weights of every parameter must be
bit-identical between (a) 1F1B, (b) kFkB k=2, (c) kFkB k=2 under emulated
preemption (paced links), and (d) a single-GPU, single-stage run of the same
model — deterministic kernels + ascending micro-batch order on every device.
Prints one JSON line on rank 0.
"""
import hashlib
import json
import os
import sys
from pathlib import Path

import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2303_01675_b200.executor import StageExecutor, max_inflight  # noqa: E402
from paper_2303_01675_b200.stage import ModelShape  # noqa: E402
from paper_2303_01675_b200.tuning import outgoing_links  # noqa: E402

SHAPE = ModelShape(4, 1024, 16, 4096, 512, 8192)
GB, B = 16, 2


PAIRS = os.environ.get("PTK_WGRAD_PAIRS", "0") == "1"  # paired weight gradients on every arm


def digests(ex):
    st = ex.stage_view()
    torch.cuda.synchronize()
    return {n: hashlib.sha256(st.param(n, "master").cpu().numpy().tobytes()).hexdigest()[:16] for n in st.params}


def run_pipeline(rank, S, k, group, trace=False, iters=2, half_cuts=False):
    M = GB // B
    layers = [(0, 2), (2, 4)] if S == 2 else [(i, i + 1) for i in range(4)]
    # half-layer cuts (attention | MLP of a layer on adjacent stages)
    halves = [(0, 5), (5, 8)] if S == 2 else [(0, 3), (3, 4), (4, 7), (7, 8)]
    slots = max(max_inflight(rank, S, M, kk) for kk in (1, 2, 3, 4))
    if half_cuts:
        ex = StageExecutor(SHAPE, rank, S, GB, b_max=B, slots=slots, halves=halves[rank], lr=1e-3, wgrad_pairs=PAIRS)
    else:
        ex = StageExecutor(SHAPE, rank, S, GB, b_max=B, slots=slots, layers=layers[rank], lr=1e-3, wgrad_pairs=PAIRS)
    ex.connect_dist(group)
    if trace:
        for link in outgoing_links(rank, S):
            ex.set_trace(link, 12.5 * 0.5, 2000, [])  # 50 Gb/s effective, 2 us latency
        dist.barrier(group=group)
        ex.set_epoch(ex.globaltimer())
    if isinstance(k, list):
        ex.set_plan_groups(B, k)  # mixed group sizes: k switches at group boundaries
    else:
        ex.set_plan(k, B)
    ms, loss = [], None
    for it in range(iters):
        ex.run_iteration(it)
        ms.append(ex.finish_iteration())
        if rank == S - 1:
            loss = ex.read_loss()
    tl = ex.timeline()
    d = digests(ex)
    dist.barrier(group=group)
    ex.close()
    return d, loss, ms, tl


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("gloo")
    group = dist.group.WORLD
    res = {}
    for name, k, tr, hc in (("1f1b", 1, False, False), ("k2", 2, False, False), ("k2_paced", 2, True, False),
                            ("mixed", [1, 3, 2, 2], True, False), ("half_cuts", 2, False, True)):
        d, loss, ms, tl = run_pipeline(rank, world, k, group, tr, half_cuts=hc)
        allds = [None] * world
        dist.all_gather_object(allds, (d, loss, ms, len(tl["xfer"])), group=group)
        merged = {}
        for dd, _, _, _ in allds:
            merged.update(dd)
        res[name] = {"digest": merged, "loss": allds[-1][1], "ms": [x[2] for x in allds],
                     "xfers": [x[3] for x in allds]}
    if rank == 0:
        ref = StageExecutor(SHAPE, 0, 1, GB, b_max=B, slots=1, layers=(0, 4), lr=1e-3, wgrad_pairs=PAIRS)
        ref.set_plan(1, B)
        loss = None
        for it in range(2):
            ref.run_iteration(it)
            ref.finish_iteration()
            loss = ref.read_loss()
        single = digests(ref)
        out = {
            "k1_vs_k2_bit_identical": res["1f1b"]["digest"] == res["k2"]["digest"],
            "paced_bit_identical": res["k2"]["digest"] == res["k2_paced"]["digest"],
            "mixed_groups_bit_identical": res["k2"]["digest"] == res["mixed"]["digest"],
            "half_layer_cuts_bit_identical": res["k2"]["digest"] == res["half_cuts"]["digest"],
            "pipeline_vs_single_gpu_bit_identical": res["1f1b"]["digest"] == single,
            "loss": {"1f1b": res["1f1b"]["loss"], "k2": res["k2"]["loss"], "paced": res["k2_paced"]["loss"],
                     "mixed": res["mixed"]["loss"], "single": loss},
            "ms": {k: v["ms"] for k, v in res.items()}, "xfers": {k: v["xfers"] for k, v in res.items()},
            "n_params": len(single), "wgrad_pairs": PAIRS,
        }
        out["ok"] = all([out["k1_vs_k2_bit_identical"], out["paced_bit_identical"],
                         out["mixed_groups_bit_identical"], out["half_layer_cuts_bit_identical"],
                         out["pipeline_vs_single_gpu_bit_identical"]])
        print(json.dumps(out), flush=True)
    dist.barrier(group=group)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
