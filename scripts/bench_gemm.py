"""Time the tcgen05 GEMM on the GPT-1.3B stage shapes against cuBLAS (torch.matmul)."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2303_01675_b200 import _lib as L  # noqa: E402


MC = int(__import__("os").environ.get("PTK_MC", "2"))


def gemm_desc(m, n, k, A, a_mn, B, b_mn, Cm, epi):
    d = L.GemmDesc()
    d.m, d.n, d.k = m, n, k
    d.batch[0] = d.batch[1] = 1
    d.a = L.matrix(A.data_ptr(), m if a_mn else k, a_mn)
    d.b = L.matrix(B.data_ptr(), n if b_mn else k, b_mn)
    d.c = L.matrix(Cm.data_ptr(), n)
    d.aux = L.matrix(0, 0)
    d.epilogue = epi
    d.multicast = MC
    d.bn_hint = int(__import__("os").environ.get("PTK_BN", "0"))
    return d


FLUSH = __import__("os").environ.get("PTK_FLUSH", "0") == "1"
_flush_buf = None


def timeit(fn, iters=20):
    """Mean time per call. PTK_FLUSH=1: cold L2 — a 512 MB write between calls, each call timed alone."""
    global _flush_buf
    if FLUSH:
        if _flush_buf is None:
            _flush_buf = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
        for _ in range(2):
            fn()
        tot = 0.0
        for _ in range(iters):
            _flush_buf.fill_(1)
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            fn()
            e.record()
            torch.cuda.synchronize()
            tot += s.elapsed_time(e)
        return tot / iters * 1e-3
    for _ in range(3):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1e-3


def main():
    dev = torch.device("cuda:0")
    T, h, f, V = 2048, 2048, 8192, 50304
    B_ = L.EPI_BF16
    shapes = [  # (name, m, n, k, a_mn, b_mn, epi, bias, aux, c2)
        ("qkv_fwd", T, 3 * h, h, 0, 0, B_, 1, 0, 0),
        ("out_fwd", T, h, h, 0, 0, B_, 1, 1, 0),
        ("fc1_fwd", T, f, h, 0, 0, L.EPI_BIAS_GELU, 1, 0, 1),
        ("fc2_fwd", T, h, f, 0, 0, B_, 1, 1, 0),
        ("fc2_dgrad", T, f, h, 0, 1, L.EPI_DGELU, 0, 1, 0),
        ("fc2_wgrad", h, f, T, 1, 1, L.EPI_ACC_F32, 0, 0, 0),
        ("fc1_dgrad", T, h, f, 0, 1, B_, 0, 0, 0),
        ("fc1_wgrad", f, h, T, 1, 1, L.EPI_ACC_F32, 0, 0, 0),
        ("out_dgrad", T, h, h, 0, 1, B_, 0, 0, 0),
        ("out_wgrad", h, h, T, 1, 1, L.EPI_ACC_F32, 0, 0, 0),
        ("qkv_dgrad", T, h, 3 * h, 0, 1, B_, 0, 0, 0),
        ("qkv_wgrad", 3 * h, h, T, 1, 1, L.EPI_ACC_F32, 0, 0, 0),
        ("head_fwd", T, V, h, 0, 0, B_, 0, 0, 0),
        ("head_dgrad", T, h, V, 0, 1, B_, 0, 0, 0),
        ("head_wgrad", V, h, T, 1, 1, L.EPI_ACC_F32, 0, 0, 0),
        # epilogue isolation (same shapes, plain bf16 store)
        ("x_fc1_plain", T, f, h, 0, 0, B_, 0, 0, 0),
        ("x_fc1_bias", T, f, h, 0, 0, B_, 1, 0, 0),
        ("x_fc2dgrad_plain", T, f, h, 0, 1, B_, 0, 0, 0),
        ("x_out_plain", T, h, h, 0, 0, B_, 0, 0, 0),
        ("x_out_aux", T, h, h, 0, 0, B_, 0, 1, 0),
        ("x_fc2wgrad_f32", h, f, T, 1, 1, L.EPI_F32, 0, 0, 0),
        ("x_fc2wgrad_bf16", h, f, T, 1, 1, B_, 0, 0, 0),
        # BERT-large b=4 shapes (T=2048, h=1024, f=4096) under the GEMM modes (PTK_MC env: 0/1/2/3)
        ("bert_qkv", T, 3072, 1024, 0, 0, B_, 1, 0, 0),
        ("bert_out", T, 1024, 1024, 0, 0, B_, 1, 1, 0),
        ("bert_fc1", T, 4096, 1024, 0, 0, L.EPI_BIAS_GELU, 1, 0, 1),
        ("bert_fc2", T, 1024, 4096, 0, 0, B_, 1, 1, 0),
        ("bert_fc1_wgrad", 4096, 1024, T, 1, 1, L.EPI_ACC_F32, 0, 0, 0),
        ("bert_fc2_dgrad", T, 4096, 1024, 0, 1, L.EPI_DGELU, 0, 1, 0),
        ("bert_out_wgrad", 1024, 1024, T, 1, 1, L.EPI_ACC_F32, 0, 0, 0),
        ("x_kk", T, f, h, 0, 0, B_, 0, 0, 0),
        ("x_mk", T, f, h, 1, 0, B_, 0, 0, 0),
        ("x_km", T, f, h, 0, 1, B_, 0, 0, 0),
        ("x_mm", T, f, h, 1, 1, B_, 0, 0, 0),
        ("x_kk_f32", T, f, h, 0, 0, L.EPI_F32, 0, 0, 0),
        ("x_kk_acc", T, f, h, 0, 0, L.EPI_ACC_F32, 0, 0, 0),
        ("x_headw_f32", V, h, T, 1, 1, L.EPI_F32, 0, 0, 0),
        # wgrads of two micro-batches fused along K (K = 2T): vs 2x the K = T launches
        ("x_fc2_wgrad_2T", h, f, 2 * T, 1, 1, L.EPI_ACC_F32, 0, 0, 0),
        ("x_fc1_wgrad_2T", f, h, 2 * T, 1, 1, L.EPI_ACC_F32, 0, 0, 0),
        ("x_out_wgrad_2T", h, h, 2 * T, 1, 1, L.EPI_ACC_F32, 0, 0, 0),
        ("x_qkv_wgrad_2T", 3 * h, h, 2 * T, 1, 1, L.EPI_ACC_F32, 0, 0, 0),
        ("x_headw_bf16", V, h, T, 1, 1, B_, 0, 0, 0),
        ("x_headw_kk_acc", V, h, T, 0, 0, L.EPI_ACC_F32, 0, 0, 0),
    ]
    stream = torch.cuda.current_stream().cuda_stream
    out = []
    tot_ptk = tot_cub = tot_fl = 0.0
    only = __import__("os").environ.get("PTK_ONLY", "")
    for name, m, n, k, a_mn, b_mn, epi, bias, aux, c2 in shapes:
        if only and name not in only.split(","):
            continue
        A = torch.randn((k, m) if a_mn else (m, k), device=dev).bfloat16()
        B = torch.randn((k, n) if b_mn else (n, k), device=dev).bfloat16()
        Cm = torch.zeros(m, n, device=dev, dtype=torch.float32 if epi in (L.EPI_F32, L.EPI_ACC_F32) else torch.bfloat16)
        d = gemm_desc(m, n, k, A, a_mn, B, b_mn, Cm, epi)
        keep = []
        if bias:
            bv = torch.randn(n, device=dev).bfloat16()
            keep.append(bv)
            d.bias = bv.data_ptr()
        if aux:
            av = torch.randn(m, n, device=dev).bfloat16()
            keep.append(av)
            d.aux = L.matrix(av.data_ptr(), n)
        if c2:
            cv = torch.empty(m, n, device=dev, dtype=torch.bfloat16)
            keep.append(cv)
            d.c2 = cv.data_ptr()
        t = timeit(lambda: L.check(L.lib().ptk_gemm(d, stream)))
        Ab = A.T if a_mn else A
        Bb = B if b_mn else B.T
        tc = timeit(lambda: torch.matmul(Ab, Bb))
        fl = 2.0 * m * n * k
        if not name.startswith(("head", "x_", "bert_")):
            tot_ptk += t
            tot_cub += tc
            tot_fl += fl
        out.append({"gemm": name, "ptk_us": round(t * 1e6, 1), "ptk_tflops": round(fl / t / 1e12, 1),
                    "cublas_us": round(tc * 1e6, 1), "cublas_tflops": round(fl / tc / 1e12, 1)})
        print(json.dumps(out[-1]), flush=True)
    if only:
        return
    print(json.dumps({"layer_total_us": round(tot_ptk * 1e6, 1), "layer_tflops": round(tot_fl / tot_ptk / 1e12, 1),
                      "cublas_layer_us": round(tot_cub * 1e6, 1),
                      "cublas_layer_tflops": round(tot_fl / tot_cub / 1e12, 1)}), flush=True)


if __name__ == "__main__":
    main()
