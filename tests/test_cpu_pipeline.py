"""The CPU-thread pipeline executor (oracle/cpu_pipeline.py): S stage threads
walking the reference planner's kFkB orders with FIFO activation / gradient queues must train
exactly like the single-process model — same loss, same accumulated gradients."""
import pytest
import torch

from oracle.cpu_pipeline import CpuPipeline, reference_orders
from paper_2303_01675_b200.stage import ModelShape

TOY = ModelShape(4, 64, 4, 256, 32, 128)
TOY_BERT = ModelShape(4, 64, 4, 256, 32, 128, arch="bert")


def _grads(p):
    return {n: t.grad.clone() for n, t in p.w.items() if t.grad is not None}


@pytest.mark.parametrize("shape", [TOY, TOY_BERT], ids=["gpt", "bert"])
@pytest.mark.parametrize("stages,k", [(2, 1), (2, 2), (4, 1), (4, 4)])
def test_pipeline_matches_single_process(shape, stages, k):
    torch.manual_seed(0)
    ref = CpuPipeline(shape, 1, 2, 4, k=1, threads=2)
    ref.step()
    g_ref = _grads(ref)
    pipe = CpuPipeline(shape, stages, 2, 4, k=k, threads=4, weights=ref.w)
    pipe.step()
    g = _grads(pipe)
    assert set(g) == set(g_ref)
    assert pipe.loss == pytest.approx(ref.loss, rel=1e-6)
    for n in g_ref:
        torch.testing.assert_close(g[n], g_ref[n], rtol=1e-5, atol=1e-7, msg=n)


def test_orders_are_the_reference_kfkb_walk():
    orders, kind = reference_orders(2, 4, 1, 2)
    # S2M4 k=2
    assert [o for o in orders[0] if o != "GA"] == "F0 F1 F2 F3 B0 B1 B2 B3".split()
    assert [o for o in orders[1] if o != "GA"] == "F0 F1 B0 B1 F2 F3 B2 B3".split()


def test_stage_failure_does_not_hang():
    p = CpuPipeline(TOY, 2, 1, 2, threads=2)
    p.orders = [["F0", "B0"], ["F0", "X0"]]  # an unknown op on stage 1: stage 0 must not wait forever
    with pytest.raises(Exception):
        p.step()
