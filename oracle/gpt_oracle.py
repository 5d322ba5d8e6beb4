"""ORACLE TEST INFRASTRUCTURE — fp32 reference of one GPT pipeline stage.

Not product code: only tests/, __graft_entry__.smoke() and bench.py's CPU
baseline may import this module.  The reference (/root/reference) has no
tensor math at all — it abstracts a stage to compute_duration()
(proj/src/model.cpp:43-47) — so loss/gradient parity is "unpinned by the
reference"; this is the builder's own plain-PyTorch fp32
model of exactly the stage libptk computes (same parameter names, GELU tanh
form, LayerNorm eps 1e-5, causal softmax(QKᵀ/√d), untied LM head, mean
cross-entropy over all M*b*seq tokens of the global batch).  It runs on CPU
threads (the CPU baseline) or, for large shapes in tests, on the GPU in fp32
with TF32 disabled.
"""
from __future__ import annotations

import math

import torch
import torch.nn.functional as F

torch.backends.cuda.matmul.allow_tf32 = False
torch.backends.cudnn.allow_tf32 = False


def layer_forward(x, w, p, heads):
    """One pre-LN transformer block; w: dict of fp32 tensors, p: name prefix."""
    B, S, h = x.shape
    d = h // heads
    a = F.layer_norm(x, (h,), w[p + "ln1_g"], w[p + "ln1_b"], 1e-5)
    qkv = a @ w[p + "w_qkv"].T + w[p + "b_qkv"]
    q, k, v = qkv.view(B, S, 3, heads, d).permute(2, 0, 3, 1, 4)
    att = (q @ k.transpose(-1, -2)) / math.sqrt(d)
    mask = torch.ones(S, S, dtype=torch.bool, device=x.device).tril()
    att = att.masked_fill(~mask, float("-inf")).softmax(-1)
    o = (att @ v).transpose(1, 2).reshape(B, S, h)
    x = x + o @ w[p + "w_o"].T + w[p + "b_o"]
    a = F.layer_norm(x, (h,), w[p + "ln2_g"], w[p + "ln2_b"], 1e-5)
    u = F.gelu(a @ w[p + "w_fc1"].T + w[p + "b_fc1"], approximate="tanh")
    return x + u @ w[p + "w_fc2"].T + w[p + "b_fc2"]


def bert_layer_forward(x, w, p, heads):
    """One post-LN BERT block (bidirectional attention, tanh-GELU as in the GPU epilogue)."""
    B, S, h = x.shape
    d = h // heads
    qkv = x @ w[p + "w_qkv"].T + w[p + "b_qkv"]
    q, k, v = qkv.view(B, S, 3, heads, d).permute(2, 0, 3, 1, 4)
    att = ((q @ k.transpose(-1, -2)) / math.sqrt(d)).softmax(-1)
    o = (att @ v).transpose(1, 2).reshape(B, S, h)
    x = F.layer_norm(x + o @ w[p + "w_o"].T + w[p + "b_o"], (h,), w[p + "ln1_g"], w[p + "ln1_b"], 1e-12)
    u = F.gelu(x @ w[p + "w_fc1"].T + w[p + "b_fc1"], approximate="tanh")
    return F.layer_norm(x + u @ w[p + "w_fc2"].T + w[p + "b_fc2"], (h,), w[p + "ln2_g"], w[p + "ln2_b"], 1e-12)


def stage_forward(w, shape, layer_begin, layer_end, has_embedding, has_head, tok=None, x_in=None, labels=None,
                  micro_batches=1):
    """Returns (x_out or None, loss contribution or None)."""
    bert = getattr(shape, "arch", "gpt") == "bert"
    if has_embedding:
        B, S = tok.shape
        x = w["wte"][tok] + w["wpe"][:S].unsqueeze(0)
        if bert:
            x = F.layer_norm(x, (shape.hidden,), w["lne_g"], w["lne_b"], 1e-12)
    else:
        x = x_in
    for l in range(layer_begin, layer_end):
        x = (bert_layer_forward if bert else layer_forward)(x, w, f"h{l}.", shape.heads)
    if not has_head:
        return x, None
    if bert:  # MLM head over all positions: dense + GELU + LN, then the decoder
        t = F.gelu(x @ w["w_t"].T + w["b_t"], approximate="tanh")
        xf = F.layer_norm(t, (shape.hidden,), w["lnf_g"], w["lnf_b"], 1e-12)
    else:
        xf = F.layer_norm(x, (shape.hidden,), w["lnf_g"], w["lnf_b"], 1e-5)
    logits = xf @ w["w_head"].T
    loss = F.cross_entropy(logits.reshape(-1, shape.vocab), labels.reshape(-1), reduction="sum")
    return None, loss / (labels.numel() * micro_batches)


def synthetic_batch(seed: int, micro_batch: int, b: int, seq: int, vocab: int):
    """Tokens uniform in [0, V); labels are the next token."""
    g = torch.Generator().manual_seed(seed * 1_000_003 + micro_batch)
    t = torch.randint(0, vocab, (b, seq + 1), generator=g, dtype=torch.int64)
    return t[:, :seq].contiguous(), t[:, 1:].contiguous()
