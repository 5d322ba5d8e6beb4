"""Time the tcgen05 GEMM on the GPT-1.3B stage shapes against cuBLAS (torch.matmul)."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2303_01675_b200 import _lib as L  # noqa: E402


MC = int(__import__("os").environ.get("PTK_MC", "1"))


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
    return d


def timeit(fn, iters=20):
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
    T = 2048
    shapes = [  # (name, m, n, k, a_mn, b_mn, epi)
        ("qkv_fwd", T, 6144, 2048, 0, 0, L.EPI_BF16),
        ("fc1_fwd", T, 8192, 2048, 0, 0, L.EPI_BF16),
        ("fc2_fwd", T, 2048, 8192, 0, 0, L.EPI_BF16),
        ("out_fwd", T, 2048, 2048, 0, 0, L.EPI_BF16),
        ("fc1_dgrad", T, 2048, 8192, 0, 1, L.EPI_BF16),
        ("fc1_wgrad", 8192, 2048, T, 1, 1, L.EPI_ACC_F32),
        ("qkv_wgrad", 6144, 2048, T, 1, 1, L.EPI_ACC_F32),
        ("head_fwd", T, 50304, 2048, 0, 0, L.EPI_BF16),
    ]
    stream = torch.cuda.current_stream().cuda_stream
    out = []
    for name, m, n, k, a_mn, b_mn, epi in shapes:
        A = torch.randn((k, m) if a_mn else (m, k), device=dev).bfloat16()
        B = torch.randn((k, n) if b_mn else (n, k), device=dev).bfloat16()
        Cm = torch.zeros(m, n, device=dev, dtype=torch.float32 if epi == L.EPI_ACC_F32 else torch.bfloat16)
        d = gemm_desc(m, n, k, A, a_mn, B, b_mn, Cm, epi)
        t = timeit(lambda: L.check(L.lib().ptk_gemm(d, stream)))
        Ab = A.T if a_mn else A
        Bb = B if b_mn else B.T
        tc = timeit(lambda: torch.matmul(Ab, Bb))
        fl = 2.0 * m * n * k
        out.append({"gemm": name, "ptk_us": round(t * 1e6, 1), "ptk_tflops": round(fl / t / 1e12, 1),
                    "cublas_us": round(tc * 1e6, 1), "cublas_tflops": round(fl / tc / 1e12, 1)})
        print(json.dumps(out[-1]), flush=True)


if __name__ == "__main__":
    main()
