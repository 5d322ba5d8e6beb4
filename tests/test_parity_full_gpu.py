"""Parity at the benchmark configurations (VERDICT r1 "next" #2).

Oracle: oracle/gpt_oracle.py, plain-PyTorch fp32 (TF32 off) of exactly the stage libptk computes,
run on the GPU for these sizes.  The reference has no tensor math (it abstracts a
stage to compute_duration, proj/src/model.cpp:43-47), so the tolerances are ours:

  bf16 operands and bf16 activation stash, fp32 accumulation / statistics / gradients.
  * one transformer layer at full shape: output rel-err <= 1e-2, every gradient <= GRAD_TOL;
  * the whole 24-layer GPT-1.3B model (configs[1]) at b=2: loss |Δ| <= 5e-3·|loss| and every
    parameter gradient <= FULL_GRAD_TOL (24 layers of bf16 round-off compound);
  * AdamW (the GradAccum optimizer): master weights after two steps equal
    torch.optim.AdamW(betas=(0.9, 0.95), eps=1e-8) on the same gradients to fp32 round-off.
  * the stash byte model the memory-capped tuner uses (ModelShape.stash_bytes_halves) equals the
    stage's real allocation (ptk_stage_stash_bytes) exactly.
"""
import sys
from pathlib import Path

import pytest
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import gpt_oracle as G  # noqa: E402
from paper_2303_01675_b200.stage import (BERT_LARGE, GPT_1_3B, GPT_6_7B, TOY, TOY_BERT, GptStage,  # noqa: E402
                                         ModelShape, halves_to_layers)

pytestmark = pytest.mark.gpu

GRAD_TOL = 2e-2
FULL_GRAD_TOL = 2e-2
OUT_TOL = 1e-2


def _rel(a, b):
    return ((a.float() - b.float()).norm() / (b.float().norm() + 1e-12)).item()


def _layer_check(shape, b, layer_fn, dy_scale=1e-3):
    li = 5
    st = GptStage(shape, li, li + 1, False, False, b, slots=1, micro_batches=1)
    T, h = b * shape.seq, shape.hidden
    torch.manual_seed(0)
    x = torch.randn(T, h, device="cuda").bfloat16()
    dy = (torch.randn(T, h, device="cuda") * dy_scale).bfloat16()
    out, dx = torch.empty_like(x), torch.empty_like(x)
    st.forward(0, x_in=x, x_out=out)
    st.backward(0, dy=dy, dx=dx)
    torch.cuda.synchronize()
    w = {n: st.param(n).float().requires_grad_(True) for n in st.params}
    xr = x.float().view(b, shape.seq, h).requires_grad_(True)
    ref = layer_fn(xr, w, f"h{li}.", shape.heads)
    ref.backward(dy.float().view(b, shape.seq, h))
    errs = {"out": _rel(out.view(b, shape.seq, h), ref.detach()), "dx": _rel(dx.view(b, shape.seq, h), xr.grad)}
    for n in st.params:
        errs[n] = _rel(st.param(n, "grads"), w[n].grad)
    st.close()
    return errs


@pytest.mark.timeout(300)
def test_gpt67b_layer_full_shape(cuda):
    """One GPT-6.7B block (configs[3]: h=4096, 32 heads of d=128, s=1024) at b=1."""
    errs = _layer_check(GPT_6_7B, 1, G.layer_forward)
    assert errs.pop("out") <= OUT_TOL
    worst = max((v, n) for n, v in errs.items())
    assert worst[0] <= GRAD_TOL, worst


@pytest.mark.timeout(300)
def test_bert_large_layer_full_shape(cuda):
    """One BERT-large block (configs[4]: h=1024, 16 heads, s=512, post-LN, bidirectional) at b=4."""
    errs = _layer_check(BERT_LARGE, 4, G.bert_layer_forward)
    assert errs.pop("out") <= OUT_TOL
    worst = max((v, n) for n, v in errs.items())
    assert worst[0] <= GRAD_TOL, worst


@pytest.mark.timeout(300)
def test_gpt13b_layer_full_shape_tight(cuda):
    errs = _layer_check(GPT_1_3B, 2, G.layer_forward)
    assert errs.pop("out") <= OUT_TOL
    worst = max((v, n) for n, v in errs.items())
    assert worst[0] <= GRAD_TOL, worst


@pytest.mark.timeout(900)
def test_gpt13b_full_model_loss_and_grads(cuda):
    """configs[1]'s whole model (24 layers, embedding, LM head, V=50304) as one stage, b=2,
    two micro-batches of the global batch: loss and every gradient against fp32."""
    shape, b, M = GPT_1_3B, 2, 2
    st = GptStage(shape, 0, shape.n_layer, True, True, b, slots=1, micro_batches=M)
    batches = [G.synthetic_batch(1234, m, b, shape.seq, shape.vocab) for m in range(M)]
    st.loss.zero_()
    for tok, lab in batches:
        st.forward(0, tok=tok.int().cuda(), labels=lab.int().cuda())
        st.backward(0, tok=tok.int().cuda())
    torch.cuda.synchronize()
    loss = st.loss.item()
    grads = {n: st.param(n, "grads").float().clone() for n in st.params}
    w = {n: st.param(n).float().requires_grad_(True) for n in st.params}
    st.close()
    torch.cuda.empty_cache()
    ref = 0.0
    for tok, lab in batches:
        _, l_ = G.stage_forward(w, shape, 0, shape.n_layer, True, True, tok=tok.cuda(), labels=lab.cuda(),
                                micro_batches=M)
        l_.backward()
        ref += l_.item()
    assert abs(loss - ref) <= 5e-3 * abs(ref), (loss, ref)
    errs = {n: _rel(grads[n], w[n].grad) for n in grads}
    worst = max((v, n) for n, v in errs.items())
    print(f"GPT-1.3B full model: loss {loss:.5f} vs {ref:.5f}; worst grad rel-err {worst}")
    assert worst[0] <= FULL_GRAD_TOL, worst


@pytest.mark.timeout(300)
@pytest.mark.parametrize("shape", [TOY, TOY_BERT], ids=["gpt", "bert"])
def test_adamw_matches_torch_after_two_steps(cuda, shape):
    """The fused AdamW at GradAccum (adamw_kernel) vs torch.optim.AdamW over two steps on the
    gradients the stage itself accumulated (one micro-batch per step: the stage finalizes its
    1-D gradient partials at the iteration's last backward, so they are readable before the step)."""
    lr, wd = 1e-3, 0.1
    st = GptStage(shape, 0, shape.n_layer, True, True, 2, slots=1, micro_batches=1)
    names = list(st.params)
    params = [torch.nn.Parameter(st.param(n, "master").detach().clone()) for n in names]
    opt = torch.optim.AdamW(params, lr=lr, betas=(0.9, 0.95), eps=1e-8, weight_decay=wd, foreach=False)
    for step in range(2):
        tok, lab = G.synthetic_batch(77, step, 2, shape.seq, shape.vocab)
        st.forward(0, tok=tok.int().cuda(), labels=lab.int().cuda())
        st.backward(0, tok=tok.int().cuda())
        torch.cuda.synchronize()
        for p, n in zip(params, names):
            p.grad = st.param(n, "grads").detach().clone()
        assert any(float(p.grad.abs().max()) > 0 for p in params)
        st.optimizer_step(lr=lr, wd=wd)
        opt.step()
        torch.cuda.synchronize()
        for p, n in zip(params, names):
            got = st.param(n, "master")
            err = (got - p.detach()).abs().max().item()
            assert torch.allclose(got, p.detach(), rtol=1e-5, atol=1e-7), (step, n, err)
            assert torch.equal(st.param(n), got.bfloat16()), n
        assert float(st.grads.abs().max()) == 0.0
    st.close()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("shape,halves,b", [
    (GPT_1_3B, (0, 13), 2), (GPT_1_3B, (13, 26), 2), (GPT_1_3B, (39, 48), 1), (GPT_1_3B, (0, 48), 1),
    (BERT_LARGE, (0, 12), 4), (BERT_LARGE, (12, 37), 2), (BERT_LARGE, (37, 48), 4), (TOY, (2, 6), 2),
], ids=lambda x: str(x) if not isinstance(x, ModelShape) else x.arch + str(x.hidden))
def test_stash_byte_model_equals_allocation(cuda, shape, halves, b):
    hb, he = halves
    lb, le, sfa, slm = halves_to_layers(hb, he)
    first, last = hb == 0, he == 2 * shape.n_layer
    st = GptStage(shape, lb, le, first, last, b, slots=1, micro_batches=1, skip_first_attn=bool(sfa),
                  skip_last_mlp=bool(slm))
    real = st.stash_bytes()
    st.close()
    assert real == b * shape.stash_bytes_halves(hb, he, last, first), (real, b * shape.stash_bytes_halves(hb, he, last))
