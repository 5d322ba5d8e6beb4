"""Repro harness: one GEMM launch on given shape/majors/epilogue with optional spacer allocations."""
import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2303_01675_b200 import _lib as L  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--m", type=int, default=50304)
p.add_argument("--n", type=int, default=2048)
p.add_argument("--k", type=int, default=2048)
p.add_argument("--amn", type=int, default=1)
p.add_argument("--bmn", type=int, default=1)
p.add_argument("--epi", type=int, default=1)
p.add_argument("--mc", type=int, default=2)
p.add_argument("--spacer-mb", type=int, default=0, help="allocate this many MB after the operands")
p.add_argument("--pre-spacer-mb", type=int, default=0, help="allocate this many MB before the operands")
p.add_argument("--reps", type=int, default=3)
a = p.parse_args()
dev = torch.device("cuda:0")
pre = torch.empty(a.pre_spacer_mb << 20, dtype=torch.uint8, device=dev) if a.pre_spacer_mb else None
m, n, k = a.m, a.n, a.k
A = torch.randn((k, m) if a.amn else (m, k), device=dev).bfloat16()
B = torch.randn((k, n) if a.bmn else (n, k), device=dev).bfloat16()
f32 = a.epi in (1, 2)
Cm = torch.zeros(m, n, device=dev, dtype=torch.float32 if f32 else torch.bfloat16)
sp = torch.empty(a.spacer_mb << 20, dtype=torch.uint8, device=dev) if a.spacer_mb else None
print("A", hex(A.data_ptr()), A.numel() * 2, "B", hex(B.data_ptr()), "C", hex(Cm.data_ptr()), Cm.numel() * Cm.element_size(),
      flush=True)
d = L.GemmDesc()
d.m, d.n, d.k = m, n, k
d.batch[0] = d.batch[1] = 1
d.a = L.matrix(A.data_ptr(), m if a.amn else k, a.amn)
d.b = L.matrix(B.data_ptr(), n if a.bmn else k, a.bmn)
d.c = L.matrix(Cm.data_ptr(), n)
d.aux = L.matrix(0, 0)
d.epilogue = a.epi
d.multicast = a.mc
info = (__import__("ctypes").c_int * 4)()
L.check(L.lib().ptk_gemm_plan_info(d, info))
print("plan", list(info), flush=True)
st = torch.cuda.current_stream().cuda_stream
for i in range(a.reps):
    L.check(L.lib().ptk_gemm(d, st))
    torch.cuda.synchronize()
ref = (A.float().T if a.amn else A.float()) @ (B.float() if a.bmn else B.float().T)
err = (Cm.float() - ref).abs().max().item() / ref.abs().max().item()
print("ok rel err", err, flush=True)
