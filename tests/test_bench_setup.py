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
