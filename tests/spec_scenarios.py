"""Scenario builders shared by the spec-oracle and spec-parity tests."""
import random


def stage(f=1.0, b=2.0, ff=0.0, bf=0.0, act=0, w=0, out_f=0, out_b=0):
    return {"forward_fixed": ff, "forward_per_sample": f, "backward_fixed": bf, "backward_per_sample": b,
            "weight_bytes": w, "activation_bytes_per_sample": act, "output_bytes_per_sample_fwd": out_f,
            "output_bytes_per_sample_bwd": out_b}


def const_traces(S, base=10.0, latency=0.0):
    return [{"link": l, "base_bandwidth": base, "latency": latency, "segments": []}
            for l in range(2 * (S - 1))]


def fig2(S=4, M=8, k=1, xfer_bytes=5, kind="kfkb"):
    """SPEC.md:56/63/350: f=1, b_dur=2, transfer = 0.5*f on a constant 10 B/u link."""
    return {"op": "simulate",
            "model": {"global_batch": M, "stages": [stage(out_f=xfer_bytes, out_b=xfer_bytes) for _ in range(S)]},
            "plan": {"kind": kind, "k": k, "micro_batch_size": 1}, "traces": const_traces(S)}


def zero_comm(S, M, kind="1f1b", k=1):
    return {"op": "simulate", "model": {"global_batch": M, "stages": [stage() for _ in range(S)]},
            "plan": {"kind": kind, "k": k, "micro_batch_size": 1}, "traces": const_traces(S)}


def random_scenario(rng: random.Random, op="simulate"):
    S = rng.randint(1, 5)
    gb = rng.choice([4, 6, 8, 12, 16, 24])
    stages = [stage(f=rng.choice([0.5, 1.0, 1.25]), b=rng.choice([1.0, 2.0, 2.5]), ff=rng.choice([0.0, 0.1, 0.3]),
                    bf=rng.choice([0.0, 0.2]), act=rng.randint(1, 50), w=rng.randint(0, 100),
                    out_f=rng.randint(0, 40), out_b=rng.randint(0, 40)) for _ in range(S)]
    traces = []
    for l in range(2 * (S - 1)):
        segs, t = [], 0.0
        for _ in range(rng.randint(0, 4)):
            t += rng.choice([0.5, 1.0, 2.5, 4.0])
            e = t + rng.choice([1.0, 3.0, 7.5])
            segs.append([t, e, rng.choice([0.1, 0.25, 0.5, 0.8])])
            t = e
        tr = {"link": l, "base_bandwidth": rng.choice([5.0, 10.0, 40.0]), "latency": rng.choice([0.0, 0.05, 0.2]),
              "segments": segs}
        if rng.random() < 0.3:
            tr["utilization_curve"] = [[rng.randint(0, 80), 0.5]]
        traces.append(tr)
    b = rng.choice([d for d in range(1, gb + 1) if gb % d == 0])
    M = gb // b
    req = {"op": op, "model": {"global_batch": gb, "stages": stages}, "traces": traces,
           "plan": {"kind": rng.choice(["1f1b", "kfkb", "gpipe"]), "k": rng.randint(1, M), "micro_batch_size": b},
           "start": rng.choice([0, 1_000_000_000, 2_500_000_000])}
    return req
