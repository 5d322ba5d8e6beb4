"""Preemption emulator check on 2 GPUs (torchrun): paced transfers follow the
trace and contender kernels add real NVLink traffic without stalling compute.
Prints per-configuration iteration times and measured transfer durations."""
import json
import os
import sys
import time
from pathlib import Path

import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2303_01675_b200.executor import StageExecutor  # noqa: E402
from paper_2303_01675_b200.stage import ModelShape  # noqa: E402
from paper_2303_01675_b200.tuning import outgoing_links  # noqa: E402

SHAPE = ModelShape(4, 1024, 16, 4096, 512, 8192)


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo")
    ex = StageExecutor(SHAPE, rank, world, 16, b_max=2, slots=8, layers=[(0, 2), (2, 4)][rank])
    ex.connect_dist()
    base = 12.5  # 100 Gb/s in bytes/ns
    out = {}
    for name, segs, cont in (("ideal", [], False), ("half", [(0, 10**13, 0.5)], False),
                             ("half+contender", [(0, 10**13, 0.5)], True)):
        for link in outgoing_links(rank, world):
            ex.set_trace(link, base, 0, segs)
        ex.set_contender(cont)
        dist.barrier()
        ex.set_epoch(ex.globaltimer())
        ex.set_plan(2, 2)
        ms = []
        for it in range(3):
            t0 = time.time()
            ex.run_iteration(it)
            ms.append(round(ex.finish_iteration(), 3))
            print(f"rank {rank} {name} it {it} {ms[-1]} ms wall {time.time()-t0:.3f}s", flush=True)
        tl = ex.timeline()
        x = [e[4] - e[3] for e in tl["xfer"]]
        probe = ex.probe_link(outgoing_links(rank, world)[0], 2 * 512 * 1024 * 2, 3)
        out[name] = {"iter_ms": ms, "xfer_ns_mean": sum(x) / max(1, len(x)), "probe_ns": probe}
    allo = [None] * world
    dist.all_gather_object(allo, out)
    if rank == 0:
        print(json.dumps(allo))
    dist.barrier()
    ex.set_contender(False)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
