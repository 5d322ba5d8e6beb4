"""Contender calibration on 2 GPUs (torchrun): how much do the emulator's contender kernels (CTAs of
peer st.v4 stores into the neighbour's scratch block, duty PTK_CONTENDER_DUTY) slow an UNPACED
inter-stage NVLink copy (copy engine, 8 MiB), and how much do they slow the stage's own compute?

Run once per contender size (PTK_CONTENDER_CTAS is read once per process):
  for c in 0 4 16 32 64 132; do PTK_CONTENDER_CTAS=$c PTK_CONTENDER_DUTY=1.0 \\
      torchrun --nproc-per-node 2 scripts/contender_calibration.py $c; done
Prints one JSON line (rank 0).  Not part of the library.
"""
import json
import os
import statistics
import sys
from pathlib import Path

import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2303_01675_b200.executor import StageExecutor  # noqa: E402
from paper_2303_01675_b200.stage import ModelShape  # noqa: E402
from paper_2303_01675_b200.tuning import outgoing_links  # noqa: E402

SHAPE = ModelShape(4, 2048, 32, 8192, 1024, 50304)  # GPT-1.3B layers; 8 MiB activations at b=2


def main():
    ctas = int(sys.argv[1]) if len(sys.argv) > 1 else 0
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo")
    ex = StageExecutor(SHAPE, rank, world, 16, b_max=2, slots=8, layers=[(0, 2), (2, 4)][rank])
    ex.connect_dist()
    # a trace that is "preempted" (so the contender runs) but paces at 10 TB/s (i.e. not at all):
    # the copy runs at whatever NVLink bandwidth the contender leaves it
    for link in outgoing_links(rank, world):
        ex.set_trace(link, 1e4, 0, [(0, 10**13, 0.999)])
    ex.set_contender(ctas > 0)
    ex.set_plan(2, 2)
    fwd, bwd, xfer, it_ms = [], [], [], []
    for it in range(5):
        dist.barrier()
        ex.set_epoch(ex.globaltimer())
        ex.run_iteration(it)
        ms = ex.finish_iteration()
        if it < 2:
            continue  # warm-up
        it_ms.append(ms)
        tl = ex.timeline()
        fwd += [r[4] - r[3] for r in tl["compute"] if r[1] == 0]
        bwd += [r[4] - r[3] for r in tl["compute"] if r[1] == 1]
        xfer += [(r[2], r[4] - r[3]) for r in tl["xfer"]]
    mine = {"rank": rank, "fwd_us": statistics.mean(fwd) / 1e3, "bwd_us": statistics.mean(bwd) / 1e3,
            "xfer_us": statistics.mean(x[1] for x in xfer) / 1e3,
            "xfer_gbps": statistics.mean(x[0] / x[1] for x in xfer), "iter_ms": statistics.mean(it_ms)}
    allo = [None] * world
    dist.all_gather_object(allo, mine)
    if rank == 0:
        print(json.dumps({"contender_ctas": ctas, "duty": os.environ.get("PTK_CONTENDER_DUTY"),
                          "gated": os.environ.get("PTK_EMU_NO_GATE") is None,
                          "sm_reserve": int(os.environ.get("PTK_SM_RESERVE", "0")), "ranks": allo}))
    dist.barrier()
    ex.set_contender(False)
    ex.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
