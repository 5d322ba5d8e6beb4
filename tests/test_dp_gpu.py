"""Data-parallel replicas of the pipeline (SPEC.md:139 open question) under pytest:
two replicas of a 1-stage pipeline as two processes on cuda:0 (gloo all-reduce of the finalized
stage gradients, on the executor's compute stream; NCCL on real multi-GPU runs) — replicas stay
bit-identical over three steps, and the averaged first-iteration gradient equals one executor
training on the whole global batch to 1e-4 relative (only the fp32 reduction order differs).
scripts/dp_check.py is the program; profiles/r1_dp_check_n2_n4.json has its NCCL runs on 2/4 GPUs."""
import json
import socket
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
pytestmark = pytest.mark.gpu


@pytest.mark.timeout(300)
def test_two_replicas_one_gpu(cuda):
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", f"--master-port={port}", str(ROOT / "scripts" / "dp_check.py"),
                          "--stages", "1", "--one-gpu"], capture_output=True, text=True, timeout=280, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    line = [ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1]
    d = json.loads(line)
    assert d["replicas"] == 2 and d["replicas_bit_identical_after_3_steps"], d
    assert d["max_rel_grad_diff_vs_single_gpu"] < 1e-4, d
