"""One short GPT-1.3B-shaped training iteration for ncu launch lists / captures.

Same layer shapes as the bench (h2048, 32 heads, s1024, V50304, b=2) but
`--layers` layers and `--mb` micro-batches so a serialised ncu pass stays short.
"""
import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2303_01675_b200.executor import StageExecutor  # noqa: E402
from paper_2303_01675_b200.stage import ModelShape  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--layers", type=int, default=2)
p.add_argument("--mb", type=int, default=2)
p.add_argument("--iters", type=int, default=2)
p.add_argument("--model", choices=["gpt", "bert"], default="gpt")
p.add_argument("--b", type=int, default=0, help="micro-batch size (default 2 GPT / 4 BERT)")
p.add_argument("--pairs", type=int, default=1, help="paired weight gradients (two-segment wgrad GEMMs)")
a = p.parse_args()
if a.model == "bert":
    shape, b = ModelShape(a.layers, 1024, 16, 4096, 512, 30528, "bert"), a.b or 4
else:
    shape, b = ModelShape(a.layers, 2048, 32, 8192, 1024, 50304), a.b or 2
ex = StageExecutor(shape, 0, 1, b * a.mb, b_max=b, slots=1, layers=(0, a.layers), wgrad_pairs=bool(a.pairs))
for i in range(a.iters):
    t0 = time.perf_counter()
    ex.run_iteration(i)
    host = (time.perf_counter() - t0) * 1e3
    print(f"iter {i}: {ex.finish_iteration():.2f} ms (host enqueue {host:.2f} ms)", flush=True)
