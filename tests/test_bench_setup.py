"""The bench's multi-stage set-up arithmetic on the CPU, for every stage count the driver may run
(2, 4, 8): half-layer partition, (k, b) candidates with and without a memory cap, and the stash
slots each rank allocates.  Every candidate plan from the C++ planner (reference plan.cpp:20-81)
must fit the slots its executor would have, exactly as Executor::install_plan checks on the GPU
(virtual slots = slots * b_max / b, one more with paired weight gradients) — so an 8-stage run on
an 8-GPU box cannot fail at set_plan even though no 8-GPU box was available to test on."""
import pytest

from paper_2303_01675_b200 import pipetune as pt
from paper_2303_01675_b200.executor import partition_halves, stage_slots
from paper_2303_01675_b200.stage import BERT_LARGE, GPT_1_3B, GPT_6_7B
from paper_2303_01675_b200.tuning import candidate_set

CASES = [(GPT_1_3B, 64, 2, None), (GPT_1_3B, 64, 2, 16e9), (GPT_1_3B, 64, 2, 24e9), (BERT_LARGE, 64, 4, None),
         (GPT_6_7B, 64, 1, 60e9)]


def _peak_inflight(plan: dict, device: int) -> int:
    live = peak = 0
    for nid in plan["per_device"][device]:
        kind = plan["nodes"][nid][0]
        if kind == 0:
            live += 1
            peak = max(peak, live)
        elif kind == 1:
            live -= 1
    return peak


@pytest.mark.parametrize("S", [2, 4, 8])
@pytest.mark.parametrize("shape,gb,b,cap", CASES, ids=lambda x: getattr(x, "hidden", x))
def test_every_candidate_fits_every_rank(S, shape, gb, b, cap):
    halves = partition_halves(shape.n_layer, S, head_weight=2.3 if shape.arch == "bert" else 1.6,
                              attn_weight=0.42 if shape.arch == "bert" else 0.47)
    assert halves[0][0] == 0 and halves[-1][1] == 2 * shape.n_layer
    assert all(h[0] < h[1] and h[1] == n[0] for h, n in zip(halves, halves[1:]))
    try:
        cands = candidate_set(shape, halves, S, gb, cap, fixed_b=b, halves=True, wgrad_pairs=True)
    except pt.PipetuneError as e:
        assert e.kind == "InfeasibleModel" and cap is not None
        return
    assert cands
    model = pt.ModelSpec([pt.StageProfile(stage_id=s, output_bytes_per_sample_fwd=1, output_bytes_per_sample_bwd=1)
                          for s in range(S)], gb)
    for rank in range(S):
        slots, b_max = stage_slots(rank, S, cands)
        slots += 1  # paired weight gradients (StageExecutor adds it)
        for k, cb, M in cands:
            plan = pt.plan_kfkb(model, cb, k)
            vslots = slots * (b_max // cb if b_max % cb == 0 else 1)
            assert _peak_inflight(plan, rank) + 1 <= vslots, (S, rank, k, cb)


@pytest.mark.parametrize("S", [2, 4, 8])
@pytest.mark.parametrize("shape,b,cap", [(GPT_1_3B, 2, 16e9), (GPT_1_3B, 2, 40e9), (GPT_1_3B, 2, 80e9),
                                         (BERT_LARGE, 4, 8e9), (BERT_LARGE, 4, 12e9), (GPT_6_7B, 1, 60e9),
                                         (GPT_6_7B, 1, 80e9)], ids=lambda x: getattr(x, "hidden", x))
def test_paired_candidates_fit_their_own_budget(S, shape, b, cap):
    """With paired weight gradients the pairing buffers are a fixed per-stage cost sized by the largest
    candidate b.  Every candidate (k, b) must fit the cap with those buffers charged at that b_max
    (the memory frontier under that budget reaches b for the same k), and budgets that leave no
    frontier are skipped instead of raising (round 2: 10/12 GB BERT and 40 GB GPT-1.3B raised)."""
    from paper_2303_01675_b200.tuning import memory_model
    halves = partition_halves(shape.n_layer, S, head_weight=2.3 if shape.arch == "bert" else 1.6,
                              attn_weight=0.42 if shape.arch == "bert" else 0.47)
    try:
        cands = candidate_set(shape, halves, S, 64, cap, fixed_b=b, halves=True, wgrad_pairs=True)
    except pt.PipetuneError as e:
        assert e.kind == "InfeasibleModel"
        return
    b_max = max(c[1] for c in cands)
    out = pt.scenario({"op": "enumerate", "model": memory_model(shape, halves, S, 64, True, b_max), "k_max": 8,
                       "cluster": {"device_memory_limit": int(cap), "devices": S}})
    best = {e[0]: e[1] for e in out["entries"]}
    for k, cb, M in cands:
        assert M * cb == 64
        assert k in best and best[k] >= cb, (k, cb, best)
