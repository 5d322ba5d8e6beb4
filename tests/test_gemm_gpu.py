"""tcgen05 GEMM parity against a plain PyTorch fp32 reference (CPU, fp64 accumulate).

Covers every operand-major combination the GPT stage uses, batched strided
operands (the attention head layout), all epilogues and the causal modes.
Tolerance: bf16 output rounding (rel 1e-2 of the row scale) on top of fp32
accumulation order differences.
"""

import pytest
import torch

from paper_2303_01675_b200 import _lib as L

pytestmark = pytest.mark.gpu


def _ref_mm(a, b):
    return (a.double() @ b.double().T).float()


def _run(desc):
    L.check(L.lib().ptk_gemm(desc, torch.cuda.current_stream().cuda_stream))


def _desc(m, n, k, a, b, c, epi=L.EPI_BF16, bias=None, aux=None, c2=None, causal=0, batch=(1, 1), bn=0, mc=0):
    d = L.GemmDesc()
    d.m, d.n, d.k = m, n, k
    d.batch[0], d.batch[1] = batch
    d.a, d.b, d.c = a, b, c
    d.aux = aux if aux is not None else L.matrix(0, 0)
    d.c2 = c2 or 0
    d.bias = bias or 0
    d.epilogue, d.causal, d.bn_hint, d.multicast = epi, causal, bn, mc
    return d


def _close(out, ref, tol=1.5e-2):
    scale = ref.abs().max().item() + 1e-6
    err = (out.float().cpu() - ref).abs().max().item()
    assert err <= tol * scale, f"max err {err} vs scale {scale}"


@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("shape", [(128, 64, 64), (300, 520, 200), (256, 384, 1024), (640, 768, 320)])
@pytest.mark.parametrize("bn,mc", [(0, 0), (64, 0), (128, 0), (256, 0), (256, 1), (256, 2)])
def test_gemm_majors(cuda, a_mn, b_mn, shape, bn, mc):
    m, n, k = shape
    if a_mn and m % 8:
        m += 8 - m % 8
    torch.manual_seed(m * 7 + n * 3 + k + a_mn * 2 + b_mn)
    A = torch.randn(m, k).bfloat16()
    B = torch.randn(n, k).bfloat16()
    ref = _ref_mm(A.float(), B.float())
    As = (A.T.contiguous() if a_mn else A).to(cuda)
    Bs = (B.T.contiguous() if b_mn else B).to(cuda)
    Cd = torch.zeros(m, n, dtype=torch.bfloat16, device=cuda)
    d = _desc(m, n, k, L.matrix(As.data_ptr(), m if a_mn else k, a_mn),
              L.matrix(Bs.data_ptr(), n if b_mn else k, b_mn), L.matrix(Cd.data_ptr(), n), bn=bn, mc=mc)
    _run(d)
    torch.cuda.synchronize()
    _close(Cd, ref)


def test_gemm_epilogues(cuda):
    m, n, k = 256, 512, 384
    torch.manual_seed(0)
    A = torch.randn(m, k).bfloat16()
    B = (torch.randn(n, k) * 0.05).bfloat16()
    bias = torch.randn(n).bfloat16()
    res = torch.randn(m, n).bfloat16()
    acc = A.double() @ B.double().T
    Ad, Bd = A.to(cuda), B.to(cuda)
    bd, rd = bias.to(cuda), res.to(cuda)
    a, b = L.matrix(Ad.data_ptr(), k), L.matrix(Bd.data_ptr(), k)

    # bias + residual
    C = torch.empty(m, n, dtype=torch.bfloat16, device=cuda)
    _run(_desc(m, n, k, a, b, L.matrix(C.data_ptr(), n), bias=bd.data_ptr(), aux=L.matrix(rd.data_ptr(), n)))
    _close(C, (acc + bias.double() + res.double()).float())

    # fp32 store and fp32 accumulate
    F = torch.ones(m, n, dtype=torch.float32, device=cuda)
    _run(_desc(m, n, k, a, b, L.matrix(F.data_ptr(), n), epi=L.EPI_F32))
    _close(F, acc.float(), tol=1e-4)
    _run(_desc(m, n, k, a, b, L.matrix(F.data_ptr(), n), epi=L.EPI_ACC_F32))
    _close(F, (2 * acc).float(), tol=1e-4)

    # bias + gelu (tanh form) with pre-activation side output
    G = torch.empty(m, n, dtype=torch.bfloat16, device=cuda)
    P = torch.empty(m, n, dtype=torch.bfloat16, device=cuda)
    _run(_desc(m, n, k, a, b, L.matrix(G.data_ptr(), n), epi=L.EPI_BIAS_GELU, bias=bd.data_ptr(),
               c2=P.data_ptr()))
    pre = (acc + bias.double()).float()
    _close(P, pre)
    _close(G, torch.nn.functional.gelu(P.float().cpu(), approximate="tanh"))

    # dgelu: C = acc * gelu'(pre)
    D = torch.empty(m, n, dtype=torch.bfloat16, device=cuda)
    _run(_desc(m, n, k, a, b, L.matrix(D.data_ptr(), n), epi=L.EPI_DGELU, aux=L.matrix(rd.data_ptr(), n)))
    x = res.float().requires_grad_(True)
    torch.nn.functional.gelu(x, approximate="tanh").backward(torch.ones_like(x))
    _close(D, acc.float() * x.grad)


def _attn_layout(cuda, b, s, h, d, seed):
    """qkv [b, s, 3, h, d] as one [b*s, 3*h*d] buffer, like the QKV projection output."""
    torch.manual_seed(seed)
    qkv = torch.randn(b, s, 3, h, d).bfloat16()
    return qkv, qkv.to(cuda)


def test_gemm_batched_attention_scores(cuda):
    b, s, h, d = 2, 256, 4, 64
    qkv, qkvd = _attn_layout(cuda, b, s, h, d, 1)
    row = 3 * h * d
    S = torch.full((b, h, s, s), float("nan"), dtype=torch.float32, device=cuda)
    # batch z1 = head, z2 = sample
    qa = L.matrix(qkvd.data_ptr(), row, 0, d, s * row)
    kb = L.matrix(qkvd.data_ptr() + h * d * 2, row, 0, d, s * row)
    c = L.matrix(S.data_ptr(), s, 0, s * s, h * s * s)
    _run(_desc(s, s, d, qa, kb, c, epi=L.EPI_F32, causal=L.CAUSAL_TILES, batch=(h, b)))
    torch.cuda.synchronize()
    q = qkv[:, :, 0].permute(0, 2, 1, 3).double()
    k = qkv[:, :, 1].permute(0, 2, 1, 3).double()
    ref = (q @ k.transpose(-1, -2)).float()
    mask = torch.tril(torch.ones(s, s, dtype=torch.bool))
    out = S.cpu()
    assert torch.allclose(out[..., mask], ref[..., mask], atol=1e-3, rtol=1e-3)


def test_gemm_batched_pv_and_grads(cuda):
    """P·V (K-head), dSᵀ·Q style (K-tail, both operands MN-major) on a causal P."""
    b, s, h, d = 2, 256, 4, 64
    qkv, qkvd = _attn_layout(cuda, b, s, h, d, 2)
    row = 3 * h * d
    torch.manual_seed(3)
    P = torch.rand(b, h, s, s).tril().bfloat16()
    Pd = P.to(cuda)
    v = qkv[:, :, 2].permute(0, 2, 1, 3).double()
    # O[z] = P[z] · V[z]: A = P (K-major), B[n=d][k=kv] = V stored [kv][d] → MN-major
    O = torch.empty(b, s, h, d, dtype=torch.bfloat16, device=cuda)
    pa = L.matrix(Pd.data_ptr(), s, 0, s * s, h * s * s)
    vb = L.matrix(qkvd.data_ptr() + 2 * h * d * 2, row, 1, d, s * row)
    oc = L.matrix(O.data_ptr(), h * d, 0, d, s * h * d)
    _run(_desc(s, d, s, pa, vb, oc, causal=L.CAUSAL_KHEAD, batch=(h, b)))
    ref = (P.double() @ v).float().permute(0, 2, 1, 3)
    _close(O, ref)

    # dV[z] = P[z]^T · dO[z]: A[m=kv][k=q] = P stored [q][kv] → MN-major; B[n=d][k=q] = dO [q][d] → MN-major
    torch.manual_seed(4)
    dO = torch.randn(b, s, h, d).bfloat16()
    dOd = dO.to(cuda)
    dV = torch.empty(b, s, h, d, dtype=torch.bfloat16, device=cuda)
    pa_t = L.matrix(Pd.data_ptr(), s, 1, s * s, h * s * s)
    dob = L.matrix(dOd.data_ptr(), h * d, 1, d, s * h * d)
    dvc = L.matrix(dV.data_ptr(), h * d, 0, d, s * h * d)
    _run(_desc(s, d, s, pa_t, dob, dvc, causal=L.CAUSAL_KTAIL, batch=(h, b)))
    ref = (P.double().transpose(-1, -2) @ dO.permute(0, 2, 1, 3).double()).float().permute(0, 2, 1, 3)
    _close(dV, ref)


@pytest.mark.parametrize("mc", [1, 2])
def test_gemm_large_dense(cuda, mc):
    m, n, k = 2048, 6144, 2048
    torch.manual_seed(5)
    A = (torch.randn(m, k) * 0.5).bfloat16().to(cuda)
    B = (torch.randn(n, k) * 0.02).bfloat16().to(cuda)
    C = torch.empty(m, n, dtype=torch.bfloat16, device=cuda)
    _run(_desc(m, n, k, L.matrix(A.data_ptr(), k), L.matrix(B.data_ptr(), k), L.matrix(C.data_ptr(), n), mc=mc))
    ref = (A.float() @ B.float().T)  # fp32 on the GPU (TF32 disabled by default for matmul)
    torch.cuda.synchronize()
    err = (C.float() - ref).abs().max().item()
    assert err <= 1e-2 * ref.abs().max().item()


@pytest.mark.parametrize("mc", [0, 2])
def test_gemm_pair_epilogues_and_wgrad(cuda, mc):
    """The CTA-pair kernel with the fused epilogues and MN-major (wgrad) operands."""
    m, n, k = 768, 1280, 512
    torch.manual_seed(11)
    A = torch.randn(k, m).bfloat16()  # MN-major A (stored [k][m])
    B = torch.randn(k, n).bfloat16()  # MN-major B (stored [k][n])
    acc = A.double().T @ B.double()
    Ad, Bd = A.to(cuda), B.to(cuda)
    F = torch.ones(m, n, dtype=torch.float32, device=cuda)
    _run(_desc(m, n, k, L.matrix(Ad.data_ptr(), m, 1), L.matrix(Bd.data_ptr(), n, 1), L.matrix(F.data_ptr(), n),
               epi=L.EPI_ACC_F32, mc=mc))
    _close(F, (acc + 1.0).float(), tol=1e-4)
    bias = torch.randn(n).bfloat16().to(cuda)
    G = torch.empty(m, n, dtype=torch.bfloat16, device=cuda)
    P = torch.empty(m, n, dtype=torch.bfloat16, device=cuda)
    _run(_desc(m, n, k, L.matrix(Ad.data_ptr(), m, 1), L.matrix(Bd.data_ptr(), n, 1), L.matrix(G.data_ptr(), n),
               epi=L.EPI_BIAS_GELU, bias=bias.data_ptr(), c2=P.data_ptr(), mc=mc))
    _close(P, (acc + bias.double().cpu()).float())


@pytest.mark.parametrize("epi,mc", [(L.EPI_BF16, 2), (L.EPI_DGELU, 2), (L.EPI_BF16, 0)])
def test_gemm_fused_column_partials(cuda, epi, mc):
    """col_part: per-32-row-block column sums of C as stored (the fused bias gradient)."""
    m, n, k = 1024, 1536, 256
    torch.manual_seed(21)
    A = torch.randn(m, k).bfloat16().to(cuda)
    B = (torch.randn(n, k) * 0.1).bfloat16().to(cuda)
    aux = torch.randn(m, n).bfloat16().to(cuda)
    C = torch.empty(m, n, dtype=torch.bfloat16, device=cuda)
    part = torch.ones(m // 32 + 3, n, dtype=torch.float32, device=cuda)  # += semantics; spare rows untouched
    d = _desc(m, n, k, L.matrix(A.data_ptr(), k), L.matrix(B.data_ptr(), k), L.matrix(C.data_ptr(), n), epi=epi,
              aux=L.matrix(aux.data_ptr(), n) if epi == L.EPI_DGELU else None, mc=mc)
    d.col_part = part.data_ptr()
    _run(d)
    torch.cuda.synchronize()
    ref = C.float().view(m // 32, 32, n).sum(1) + 1.0
    assert torch.allclose(part[: m // 32], ref, rtol=1e-5, atol=1e-4)
    assert torch.equal(part[m // 32:], torch.ones(3, n, device=cuda))


def test_gemm_plan_info(cuda):
    """ptk_gemm_plan_info reports the launch ptk_gemm makes: the CTA-pair kernel for the wide dense
    stage GEMMs, a partial last wave split into half tiles, plain 1-CTA tiles for narrow outputs."""
    import ctypes
    A = torch.empty(2048, 8192, dtype=torch.bfloat16, device=cuda)
    B = torch.empty(8192, 8192, dtype=torch.bfloat16, device=cuda)
    C = torch.empty(2048, 8192, dtype=torch.bfloat16, device=cuda)
    info = (ctypes.c_int * 4)()

    def plan(m, n, k, mc):
        d = _desc(m, n, k, L.matrix(A.data_ptr(), k), L.matrix(B.data_ptr(), k), L.matrix(C.data_ptr(), n), mc=mc)
        L.check(L.lib().ptk_gemm_plan_info(d, info))
        return list(info)
    bn, grid, items, pair = plan(2048, 8192, 2048, 2)  # fc1 fwd: 8 x 32 = 256 pair tiles
    sms = torch.cuda.get_device_properties(cuda).multi_processor_count
    assert (bn, pair) == (256, 1) and grid == 2 * (sms // 2)
    tiles = 256
    rem = tiles % (sms // 2)
    assert items == (tiles - rem + 2 * rem if 2 * rem <= sms // 2 else tiles)
    assert plan(2048, 64, 512, 0)[0] == 64
    assert plan(256, 128, 512, 0)[:2] == [128, 2]


@pytest.mark.parametrize("a_mn,b_mn", [(1, 1), (0, 0), (0, 1)])
@pytest.mark.parametrize("epi", [L.EPI_ACC_F32, L.EPI_BF16])
def test_gemm_two_k_segments(cuda, a_mn, b_mn, epi):
    """k2 > 0: D = A Bᵀ + A2 B2ᵀ in one fp32 accumulation (the paired weight gradients of two
    micro-batches: MN-major [T][m] / [T][n] operands from two separate buffers)."""
    m, n, k, k2 = 1024, 1536, 512, 768
    torch.manual_seed(a_mn * 4 + b_mn + epi)
    mats = []
    for kk in (k, k2):
        A = torch.randn(m, kk).bfloat16()
        B = torch.randn(n, kk).bfloat16()
        mats.append((A, B, (A.T.contiguous() if a_mn else A).to(cuda), (B.T.contiguous() if b_mn else B).to(cuda)))
    ref = sum(A.double() @ B.double().T for A, B, _, _ in mats).float()
    f32 = epi == L.EPI_ACC_F32
    C = torch.ones(m, n, device=cuda) if f32 else torch.empty(m, n, dtype=torch.bfloat16, device=cuda)
    (_, _, A1, B1), (_, _, A2, B2) = mats
    d = _desc(m, n, k, L.matrix(A1.data_ptr(), m if a_mn else k, a_mn), L.matrix(B1.data_ptr(), n if b_mn else k, b_mn),
              L.matrix(C.data_ptr(), n), epi=epi, mc=2)
    d.a2 = L.matrix(A2.data_ptr(), m if a_mn else k2, a_mn)
    d.b2 = L.matrix(B2.data_ptr(), n if b_mn else k2, b_mn)
    d.k2 = k2
    _run(d)
    torch.cuda.synchronize()
    _close(C, ref + 1.0 if f32 else ref, tol=1e-4 if f32 else 1.5e-2)
