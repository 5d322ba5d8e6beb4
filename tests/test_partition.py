"""Stage partitioning (CPU): whole-layer and half-layer cuts."""
import sys
from pathlib import Path

import pytest

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2303_01675_b200.executor import partition_halves, partition_layers  # noqa: E402
from paper_2303_01675_b200.stage import GPT_1_3B, halves_to_layers  # noqa: E402


def _cost(rng, attn=0.47, head=1.6, emb=0.05, first=False, last=False):
    c = sum(attn if u % 2 == 0 else 1 - attn for u in range(*rng))
    return c + (head if last else 0.0) + (emb if first else 0.0)


@pytest.mark.parametrize("stages", [1, 2, 3, 4, 6, 8])
def test_half_partition_tiles_and_balances(stages):
    parts = partition_halves(24, stages)
    assert parts[0][0] == 0 and parts[-1][1] == 48
    assert all(a[1] == b[0] and a[0] < a[1] for a, b in zip(parts, parts[1:]))
    costs = [_cost(r, first=i == 0, last=i == stages - 1) for i, r in enumerate(parts)]
    # never worse than the best whole-layer cut with the same cost model
    whole = partition_layers(24, stages, head_weight=1.6)
    wcost = max(_cost((2 * a, 2 * b), first=i == 0, last=i == stages - 1) for i, (a, b) in enumerate(whole))
    assert max(costs) <= wcost + 1e-9


def test_half_partition_beats_whole_layers_on_8_stages():
    parts = partition_halves(24, 8)
    costs = [_cost(r, first=i == 0, last=i == 7) for i, r in enumerate(parts)]
    assert max(costs) < 3.6  # whole layers: 4.05 (a 4-layer stage + embedding)


def test_halves_to_layers():
    assert halves_to_layers(0, 48) == (0, 24, 0, 0)
    assert halves_to_layers(13, 26) == (6, 13, 1, 0)   # MLP of layer 6 .. layer 12
    assert halves_to_layers(0, 13) == (0, 7, 0, 1)     # layers 0..5 + attention of layer 6
    assert halves_to_layers(3, 4) == (1, 2, 1, 0)      # only the MLP block of layer 1


def test_half_memory_model_matches_whole_layers():
    s = GPT_1_3B
    assert s.param_count_halves(0, 48, True, True) == s.param_count(24, True, True)
    assert s.stash_bytes_halves(4, 10, False) == s.stash_bytes_per_sample(3, False, has_embedding=False)
    assert s.stash_bytes_halves(0, 6, False) == s.stash_bytes_per_sample(3, False)
    assert abs(s.flops_halves(0, 48, True) - s.flops_per_sample()) < 1e-3 * s.flops_per_sample()
