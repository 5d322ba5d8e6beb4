"""Debug tool: one S=1 executor iteration of a small GPT (h=512, 8 heads, s=256, V=4096), b=2."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2303_01675_b200.executor import StageExecutor  # noqa: E402
from paper_2303_01675_b200.stage import ModelShape  # noqa: E402

shape = ModelShape(4, 512, 8, 2048, 256, 4096)
GB = int(sys.argv[1]) if len(sys.argv) > 1 else 16
ex = StageExecutor(shape, 0, 1, GB, b_max=2, slots=1, layers=(0, 4), lr=1e-3)
ex.set_plan(1, 2)
ex.set_defer_optimizer(True)
rng = np.random.default_rng(1000)
full = rng.integers(0, shape.vocab, size=(GB, shape.seq + 1), dtype=np.int32)
toks = np.ascontiguousarray(np.concatenate([full[:, :-1].ravel(), full[:, 1:].ravel()]))
ex.run_iteration(0, toks.ctypes.data)
print("ms", ex.finish_iteration(), "loss", ex.read_loss(), flush=True)
