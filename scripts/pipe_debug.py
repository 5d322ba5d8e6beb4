"""Debug tool: an S-stage pipeline of the bench model in ONE process on cuda:0 (connect_local,
ptk_exec_run_local), with the bench's slot / b_max / pairing arithmetic, a short deadlock timeout,
and per-iteration timings.  Not part of the library.

    python scripts/pipe_debug.py --model 1.3b --stages 2 --cap-gb 24 --plans 1,4 2,2 4,1 [--no-pairs]
"""
import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2303_01675_b200.executor import StageExecutor, max_inflight, partition_halves  # noqa: E402
from paper_2303_01675_b200.stage import BERT_LARGE, GPT_1_3B, GPT_6_7B, TOY  # noqa: E402
from paper_2303_01675_b200.tuning import candidate_set  # noqa: E402


def main():
    import faulthandler
    faulthandler.dump_traceback_later(int(__import__("os").environ.get("PTK_DEBUG_DUMP_S", "120")), exit=True)
    p = argparse.ArgumentParser()
    p.add_argument("--model", default="1.3b")
    p.add_argument("--stages", type=int, default=2)
    p.add_argument("--gb", type=int, default=64)
    p.add_argument("--cap-gb", type=float, default=0)
    p.add_argument("--plans", nargs="*", default=[])
    p.add_argument("--no-pairs", action="store_true")
    p.add_argument("--iters", type=int, default=2)
    p.add_argument("--timeout", type=float, default=60)
    p.add_argument("--trace-gbps", type=float, default=0)
    a = p.parse_args()
    shape = {"1.3b": GPT_1_3B, "6.7b": GPT_6_7B, "bert-large": BERT_LARGE, "toy": TOY}[a.model]
    S = a.stages
    halves = partition_halves(shape.n_layer, S, head_weight=2.3 if shape.arch == "bert" else 1.6,
                              attn_weight=0.42 if shape.arch == "bert" else 0.47)
    pairs = not a.no_pairs
    cap = a.cap_gb * 1e9 if a.cap_gb else None
    cands = candidate_set(shape, halves, S, a.gb, cap, fixed_b=2, halves=True, wgrad_pairs=pairs)
    b_max = max(c[1] for c in cands)
    exs = []
    for r in range(S):
        slots = -(-max(max_inflight(r, S, c[2], c[0]) * c[1] for c in cands) // b_max)
        slots = max(slots, max(max_inflight(r, S, c[2], c[0]) for c in cands if c[1] == b_max))
        print(f"stage {r}: halves {halves[r]}, slots {slots}, b_max {b_max}, pairs {pairs}", flush=True)
        print(f"creating stage {r}", flush=True)
        exs.append(StageExecutor(shape, r, S, a.gb, b_max=b_max, slots=slots, halves=halves[r], wgrad_pairs=pairs))
    for r, e in enumerate(exs):
        if r + 1 < S:
            e.connect_local(r + 1, exs[r + 1])
        if r > 0:
            e.connect_local(r - 1, exs[r - 1])
        e.set_deadlock_timeout(a.timeout)
        if a.trace_gbps:
            from paper_2303_01675_b200.tuning import outgoing_links
            for link in outgoing_links(r, S):
                e.set_trace(link, a.trace_gbps / 8, 0, [])
    print("candidates", cands, flush=True)
    plans = [tuple(int(x) for x in s.split(",")) for s in a.plans] or [(c[0], c[1]) for c in cands]
    it = 0
    for k, b in plans:
        print(f"set_plan k={k} b={b}", flush=True)
        for e in exs:
            e.set_plan(k, b)
        for _ in range(a.iters):
            t0 = time.perf_counter()
            ms = StageExecutor.run_local(exs, it)
            it += 1
            print(f"plan k={k} b={b}: iteration {it} {time.perf_counter() - t0:.3f} s, stage ms "
                  f"{[round(x, 1) for x in ms]}, loss {exs[-1].read_loss():.4f}", flush=True)
    for e in exs:
        e.close()


if __name__ == "__main__":
    main()
