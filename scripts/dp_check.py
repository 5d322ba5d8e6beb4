"""Data-parallel replicas of the pipeline, torchrun on W GPUs.

W = S * R ranks: rank -> (replica r = rank // S, stage s = rank % S).  Each
replica runs the kFkB pipeline over its 1/R share of the global batch; at
GradAccum every stage all-reduces (NCCL, ReduceOp.AVG) its finalized gradients
with the same stage of the other replicas on the executor's compute stream,
then steps AdamW.  Checks, printed as one JSON line on rank 0:
  * replicas stay bit-identical (every parameter, every stage);
  * the DP run matches a single GPU training on the whole global batch
    (same micro-batch size and data; fp32 reduction order differs, so the
    master weights agree to a small relative tolerance, not bitwise).

    torchrun --nproc-per-node 2 scripts/dp_check.py --stages 1
    torchrun --nproc-per-node 4 scripts/dp_check.py --stages 2
"""
import argparse
import hashlib
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2303_01675_b200.executor import StageExecutor, max_inflight, partition_layers  # noqa: E402
from paper_2303_01675_b200.stage import ModelShape  # noqa: E402

SHAPE = ModelShape(4, 512, 8, 2048, 256, 4096)
GB, B, ITERS = 16, 2, 2


def host_batch(it, lo, hi):
    """Tokens + next-token labels of samples [lo, hi) of iteration `it` (int32, [tokens; labels])."""
    rng = np.random.default_rng(1000 + it)
    full = rng.integers(0, SHAPE.vocab, size=(GB, SHAPE.seq + 1), dtype=np.int32)
    part = full[lo:hi]
    return np.ascontiguousarray(np.concatenate([part[:, :-1].ravel(), part[:, 1:].ravel()]))


def run(ex, replica, replicas, dp_group, iters, step_last=True):
    """`iters` iterations; the last one stops after the gradient all-reduce unless step_last."""
    n = GB // replicas
    st = ex.stage_view()
    for it in range(iters):
        toks = host_batch(it, replica * n, (replica + 1) * n)
        ex.run_iteration(it, toks.ctypes.data)
        last = it == iters - 1
        if dp_group is not None:
            ex.data_parallel_step(dp_group, step=step_last or not last)
        ex.finish_iteration()
        torch.cuda.synchronize()
    return ({name: st.param(name, "grads").cpu().clone() for name in st.params},
            {name: st.param(name, "master").cpu().clone() for name in st.params})


def run_from(ex, replica, replicas, dp_group, first, last):
    n = GB // replicas
    st = ex.stage_view()
    for it in range(first, last):
        toks = host_batch(it, replica * n, (replica + 1) * n)  # keep the array alive across the call
        ex.run_iteration(it, toks.ctypes.data)
        ex.data_parallel_step(dp_group)
        ex.finish_iteration()
    torch.cuda.synchronize()
    return None, {name: st.param(name, "master").cpu().clone() for name in st.params}


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--stages", type=int, default=1)
    p.add_argument("--one-gpu", action="store_true",
                   help="every rank on cuda:0 with gloo gradient all-reduce (tests/test_dp_gpu.py)")
    a = p.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = 0 if a.one_gpu else int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(dev)
    if a.one_gpu:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
    S = a.stages
    R = world // S
    replica, stage = rank // S, rank % S
    pipe_groups = [dist.new_group([r * S + s for s in range(S)], backend="gloo") for r in range(R)]
    dp_groups = [dist.new_group([r * S + s for r in range(R)], backend="gloo" if a.one_gpu else "nccl")
                 for s in range(S)]
    layers = partition_layers(SHAPE.n_layer, S)
    M = (GB // R) // B
    slots = max(max_inflight(stage, S, M, k) for k in (1, 2))
    ex = StageExecutor(SHAPE, stage, S, GB // R, b_max=B, slots=slots, layers=layers[stage], lr=1e-3)
    if S > 1:
        ex.connect_dist(pipe_groups[replica])
    ex.set_plan(2, B)
    ex.set_defer_optimizer(True)
    # 1) the first iteration's averaged gradient vs a single GPU on the whole global batch
    #    (same weights, same data; only the fp32 reduction order differs)
    g, _ = run(ex, replica, R, dp_groups[stage], 1, step_last=False)
    import ctypes as C
    ex.lib.ptk_stage_optimizer_step(ex.lib.ptk_exec_stage(ex.h), ex.cfg.lr, ex.cfg.weight_decay,
                                    C.c_void_p(ex.compute_stream()))
    # 2) two more full DP steps: the replicas must stay bit-identical
    _, w = run_from(ex, replica, R, dp_groups[stage], 1, 1 + ITERS)
    ex.close()
    digest = hashlib.sha256(b"".join(w[n].numpy().tobytes() for n in sorted(w))).hexdigest()[:16]
    digests = [None] * world
    dist.all_gather_object(digests, (replica, stage, digest))
    gref = None
    if rank == 0:  # single-GPU reference: whole model, whole global batch, same data and updates
        ref = StageExecutor(SHAPE, 0, 1, GB, b_max=B, slots=1, layers=(0, SHAPE.n_layer), lr=1e-3)
        ref.set_plan(1, B)
        ref.set_defer_optimizer(True)
        n = GB
        st = ref.stage_view()
        toks = host_batch(0, 0, n)
        ref.run_iteration(0, toks.ctypes.data)
        ref.finish_iteration()
        torch.cuda.synchronize()
        gref = {name: st.param(name, "grads").cpu().clone() for name in st.params}
        ref.close()
    gathered = [None] * world
    dist.all_gather_object(gathered, g)
    if rank == 0:
        identical = all(len({d for (r, s, d) in digests if s == st}) == 1 for st in range(S))
        merged = {}
        for gg in gathered[:S]:  # replica 0's stages
            merged.update(gg)
        worst = max(((merged[n] - gref[n]).norm().item() / (gref[n].norm().item() + 1e-12), n) for n in gref)
        out = {"world": world, "stages": S, "replicas": R, "replicas_bit_identical_after_3_steps": identical,
               "max_rel_grad_diff_vs_single_gpu": worst[0], "worst_param": worst[1],
               "ok": identical and worst[0] < 1e-4}
        print(json.dumps(out), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
