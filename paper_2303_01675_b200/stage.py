"""Python handle over one GPT pipeline stage (ptk_stage_* in include/ptk.h).

Device buffers owned by the C++ stage are exposed to torch zero-copy through
__cuda_array_interface__, so tests can read weights/grads without a copy and
feed torch-allocated activations in by pointer.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import torch

from . import _lib as L


class GptConfig(C.Structure):
    _fields_ = [
        ("n_layer", C.c_int), ("hidden", C.c_int), ("heads", C.c_int), ("ffn", C.c_int), ("seq", C.c_int),
        ("vocab", C.c_int), ("layer_begin", C.c_int), ("layer_end", C.c_int), ("has_embedding", C.c_int),
        ("has_head", C.c_int), ("micro_batch_size", C.c_int), ("slots", C.c_int), ("micro_batches", C.c_int),
        ("arch", C.c_int), ("seed", C.c_uint64), ("skip_first_attn", C.c_int), ("skip_last_mlp", C.c_int),
        ("wgrad_pairs", C.c_int),
    ]


def halves_to_layers(hb: int, he: int) -> tuple[int, int, int, int]:
    """Half-layer range [hb, he) (2l = attention block of layer l, 2l+1 = its MLP block) ->
    (layer_begin, layer_end, skip_first_attn, skip_last_mlp) of ptk_gpt_config."""
    return hb // 2, (he + 1) // 2, hb % 2, he % 2


@dataclass(frozen=True)
class ModelShape:
    n_layer: int
    hidden: int
    heads: int
    ffn: int
    seq: int
    vocab: int
    arch: str = "gpt"  # "gpt": pre-LN causal + LM head; "bert": post-LN bidirectional + MLM head

    @property
    def arch_id(self) -> int:
        return 1 if self.arch == "bert" else 0

    def params_per_layer(self) -> int:
        h, f = self.hidden, self.ffn
        return 3 * h * h + 3 * h + h * h + h + 2 * h * f + f + h + 4 * h

    def flops_per_sample(self) -> float:
        """Training FLOPs per sample (fwd + bwd = 3x fwd), causal attention at half."""
        h, f, s, l, V = self.hidden, self.ffn, self.seq, self.n_layer, self.vocab
        att = 2 * s * h if self.arch == "gpt" else 4 * s * h  # QKᵀ + PV, causal counted at half
        per_tok_layer = 2 * (3 * h * h + h * h + 2 * h * f) + att
        head = 2 * h * V + (2 * h * h if self.arch == "bert" else 0)  # BERT MLM transform
        return 3.0 * s * (l * per_tok_layer + head)


    def half_params(self) -> tuple[int, int]:
        """(attention block, MLP block) parameter counts of one layer."""
        h, f = self.hidden, self.ffn
        return 4 * h * h + 6 * h, 2 * h * f + f + 3 * h

    def param_count_halves(self, hb: int, he: int, has_embedding: bool, has_head: bool) -> int:
        pa, pm = self.half_params()
        n = sum(pa if u % 2 == 0 else pm for u in range(hb, he))
        return n + self.param_count(0, has_embedding, has_head)

    def stash_bytes_halves(self, hb: int, he: int, has_head: bool, has_embedding: bool | None = None) -> int:
        """Activation-stash bytes per in-flight sample of half-layer blocks [hb, he), exactly what
        GptStage allocates per slot divided by b (gpt_stage.cu, "activation stash"): per attention
        block x_in (not on a stage's first layer without the embedding: it reads the receive block),
        ln1, qkv, attn_o, its LayerNorm stats and lse; x_mid when the layer has both blocks; per MLP
        block ln2, fc1 pre-activation and activation and stats; the head's final LN input/output,
        bf16 dlogits and stats (+ BERT's transform), BERT's embedding sum and stats."""
        if has_embedding is None:
            has_embedding = hb == 0
        s, h, f, H = self.seq, self.hidden, self.ffn, self.heads
        lb, le, sfa, slm = halves_to_layers(hb, he)
        out = 0
        for i in range(lb, le):
            A = not (i == lb and sfa)
            M = not (i == le - 1 and slm)
            if A:
                out += (0 if (i == lb and not has_embedding) else s * h * 2)  # x_in
                out += (s * h + 3 * s * h + s * h) * 2 + 2 * s * 4 + H * s * 4  # ln1, qkv, attn_o; stats; lse
            if A and M:
                out += s * h * 2  # x_mid
            if M:
                out += (s * h + 2 * s * f) * 2 + 2 * s * 4  # ln2, fc1 pre/act; stats
        if has_head:
            out += 2 * s * h * 2 + s * self.vocab * 2 + 2 * s * 4 + (2 * s * h * 2 if self.arch == "bert" else 0)
        if has_embedding and self.arch == "bert":
            out += s * h * 2 + 2 * s * 4
        return out

    def flops_halves(self, hb: int, he: int, has_head: bool) -> float:
        """Training FLOPs per sample of half-layer blocks [hb, he) (+ the head)."""
        h, f, s, V = self.hidden, self.ffn, self.seq, self.vocab
        att = 2 * s * h if self.arch == "gpt" else 4 * s * h
        fa, fm = 2 * 4 * h * h + att, 2 * 2 * h * f
        n = sum(fa if u % 2 == 0 else fm for u in range(hb, he))
        if has_head:
            n += 2 * h * V + (2 * h * h if self.arch == "bert" else 0)
        return 3.0 * s * n

    def param_count(self, n_layers: int, has_embedding: bool, has_head: bool) -> int:
        h, V = self.hidden, self.vocab
        n = n_layers * self.params_per_layer()
        if has_embedding:
            n += V * h + self.seq * h + (2 * h if self.arch == "bert" else 0)
        if has_head:
            n += V * h + 2 * h + (h * h + h if self.arch == "bert" else 0)
        return n

    def stash_bytes_per_sample(self, n_layers: int, has_head: bool, has_embedding: bool = True) -> int:
        """Activation bytes one in-flight sample keeps on a stage of `n_layers` whole layers until
        its backward (stash_bytes_halves over whole layers; exact against ptk_stage_stash_bytes)."""
        return self.stash_bytes_halves(0, 2 * n_layers, has_head, has_embedding)


GPT_1_3B = ModelShape(24, 2048, 32, 8192, 1024, 50304)
GPT_6_7B = ModelShape(32, 4096, 32, 16384, 1024, 50304)
TOY = ModelShape(4, 256, 4, 1024, 128, 512)
BERT_LARGE = ModelShape(24, 1024, 16, 4096, 512, 30528, "bert")
TOY_BERT = ModelShape(4, 256, 4, 1024, 128, 512, "bert")


class _CAI:
    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None}


def device_view(ptr: int, numel: int, dtype: torch.dtype) -> torch.Tensor:
    if dtype == torch.float32:
        return torch.as_tensor(_CAI(ptr, (numel,), "<f4"), device="cuda")
    if dtype == torch.bfloat16:
        return torch.as_tensor(_CAI(ptr, (numel,), "<i2"), device="cuda").view(torch.bfloat16)
    raise TypeError(dtype)


def _declare(lib):
    if getattr(lib, "_stage_declared", False):
        return
    lib.ptk_stage_create.argtypes = [C.POINTER(GptConfig), C.POINTER(C.c_void_p)]
    lib.ptk_stage_destroy.argtypes = [C.c_void_p]
    lib.ptk_stage_forward.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    lib.ptk_stage_backward.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    lib.ptk_stage_optimizer_step.argtypes = [C.c_void_p, C.c_float, C.c_float, C.c_void_p]
    lib.ptk_stage_zero_grads.argtypes = [C.c_void_p, C.c_void_p]
    lib.ptk_stage_buffers.argtypes = [C.c_void_p] + [C.c_void_p] * 5
    lib.ptk_stage_param.argtypes = [C.c_void_p, C.c_int, C.c_char_p, C.c_size_t] + [C.POINTER(C.c_int64)] * 3
    lib.ptk_stage_gemm_timing.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                          C.POINTER(C.c_long)]
    lib.ptk_stage_stash_bytes.argtypes = [C.c_void_p]
    lib.ptk_stage_stash_bytes.restype = C.c_size_t
    lib._stage_declared = True


def _ptr(t) -> int:
    if t is None:
        return 0
    return t if isinstance(t, int) else t.data_ptr()


class GptStage:
    def __init__(self, shape: ModelShape, layer_begin: int, layer_end: int, has_embedding: bool, has_head: bool,
                 micro_batch_size: int, slots: int, micro_batches: int, seed: int = 42, skip_first_attn: bool = False,
                 skip_last_mlp: bool = False):
        self.lib = L.lib()
        _declare(self.lib)
        self.shape = shape
        self.cfg = GptConfig(shape.n_layer, shape.hidden, shape.heads, shape.ffn, shape.seq, shape.vocab,
                             layer_begin, layer_end, int(has_embedding), int(has_head), micro_batch_size, slots,
                             micro_batches, shape.arch_id, seed, int(skip_first_attn), int(skip_last_mlp))
        h = C.c_void_p()
        L.check(self.lib.ptk_stage_create(C.byref(self.cfg), C.byref(h)))
        self.h = h
        self.owned = True
        self._attach()

    @classmethod
    def view(cls, lib, handle: int, shape: ModelShape, micro_batch_size: int) -> "GptStage":
        """Non-owning wrapper of a stage that lives inside an executor."""
        self = cls.__new__(cls)
        self.lib, self.shape, self.owned = lib, shape, False
        _declare(lib)
        self.h = C.c_void_p(handle)
        self.cfg = GptConfig()
        self.cfg.micro_batch_size = micro_batch_size
        self._attach()
        return self

    def _attach(self):
        m, w, g, loss = C.c_void_p(), C.c_void_p(), C.c_void_p(), C.c_void_p()
        n = C.c_int64()
        L.check(self.lib.ptk_stage_buffers(self.h, C.byref(m), C.byref(w), C.byref(g), C.byref(loss), C.byref(n)))
        self.numel = n.value
        self.master = device_view(m.value, n.value, torch.float32)
        self.weights = device_view(w.value, n.value, torch.bfloat16)
        self.grads = device_view(g.value, n.value, torch.float32)
        self.loss = device_view(loss.value, 1, torch.float32)
        self.params = {}
        i = 0
        buf = C.create_string_buffer(128)
        while True:
            off, r, c = C.c_int64(), C.c_int64(), C.c_int64()
            if self.lib.ptk_stage_param(self.h, i, buf, 128, C.byref(off), C.byref(r), C.byref(c)) != 0:
                break
            self.params[buf.value.decode()] = (off.value, r.value, c.value)
            i += 1

    @property
    def tokens(self) -> int:
        return self.cfg.micro_batch_size * self.shape.seq

    def param(self, name: str, which: str = "weights") -> torch.Tensor:
        off, r, c = self.params[name]
        flat = {"weights": self.weights, "master": self.master, "grads": self.grads}[which]
        t = flat[off:off + r * c]
        return t.view(c) if r == 1 else t.view(r, c)

    def forward(self, slot, tok=None, x_in=None, labels=None, x_out=None, stream=None):
        s = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        L.check(self.lib.ptk_stage_forward(self.h, slot, _ptr(tok), _ptr(x_in), _ptr(labels), _ptr(x_out), s))

    def backward(self, slot, tok=None, dy=None, dx=None, stream=None):
        s = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        L.check(self.lib.ptk_stage_backward(self.h, slot, _ptr(tok), _ptr(dy), _ptr(dx), s))

    def optimizer_step(self, lr=1e-4, wd=0.0, stream=None):
        s = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        L.check(self.lib.ptk_stage_optimizer_step(self.h, lr, wd, s))

    def zero_grads(self, stream=None):
        s = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        L.check(self.lib.ptk_stage_zero_grads(self.h, s))

    def gemm_timing(self, enable: int = -1):
        fl, ms, n = C.c_double(), C.c_double(), C.c_long()
        L.check(self.lib.ptk_stage_gemm_timing(self.h, enable, C.byref(fl), C.byref(ms), C.byref(n)))
        return fl.value, ms.value, n.value

    def stash_bytes(self) -> int:
        return self.lib.ptk_stage_stash_bytes(self.h)

    def close(self):
        if self.h and self.owned:
            self.lib.ptk_stage_destroy(self.h)
        self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
