"""One short GPT-1.3B-shaped training iteration for ncu launch lists / captures.

Same layer shapes as the bench (h2048, 32 heads, s1024, V50304, b=2) but
`--layers` layers and `--mb` micro-batches so a serialised ncu pass stays short.
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2303_01675_b200.executor import StageExecutor  # noqa: E402
from paper_2303_01675_b200.stage import ModelShape  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--layers", type=int, default=2)
p.add_argument("--mb", type=int, default=2)
p.add_argument("--iters", type=int, default=2)
a = p.parse_args()
shape = ModelShape(a.layers, 2048, 32, 8192, 1024, 50304)
ex = StageExecutor(shape, 0, 1, 2 * a.mb, b_max=2, slots=1, layers=(0, a.layers))
for i in range(a.iters):
    ex.run_iteration(i)
    print(f"iter {i}: {ex.finish_iteration():.2f} ms", flush=True)
