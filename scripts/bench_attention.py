"""Time the tcgen05 flash attention (forward, backward) on the bench shapes.

Algorithmic FLOPs: forward 4·b·H·s²·d (halved when causal), backward 2.5x the
forward (S recompute, dP, dV, dK, dQ).  CUDA events on the launching stream.
"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2303_01675_b200 import _lib as L  # noqa: E402


def timeit(fn, iters=50):
    for _ in range(5):
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
    lib = L.lib()
    st = torch.cuda.current_stream().cuda_stream
    only = sys.argv[1] if len(sys.argv) > 1 else None
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 50
    for name, b, s, H, d, causal in [("gpt-1.3b", 2, 1024, 32, 64, 1), ("bert-large", 4, 512, 16, 64, 0),
                                     ("bert-large b16", 16, 512, 16, 64, 0), ("gpt-6.7b", 2, 1024, 32, 128, 1),
                                     ("gpt-1.3b b4", 4, 1024, 32, 64, 1), ("gpt-1.3b b1", 1, 1024, 32, 64, 1)]:
        h = H * d
        qkv = (torch.randn(b * s, 3 * h, device=dev) * 0.5).bfloat16()
        o = torch.empty(b * s, h, device=dev, dtype=torch.bfloat16)
        lse = torch.empty(b * H * s, device=dev)
        dO = torch.randn(b * s, h, device=dev).bfloat16()
        dsum = torch.empty(b * H * s, device=dev)
        dqkv = torch.empty_like(qkv)

        def fwd():
            L.check(lib.ptk_flash_forward(qkv.data_ptr(), o.data_ptr(), lse.data_ptr(), b, s, H, d, causal, st))

        def bwd():
            L.check(lib.ptk_flash_backward(qkv.data_ptr(), o.data_ptr(), dO.data_ptr(), lse.data_ptr(),
                                           dsum.data_ptr(), dqkv.data_ptr(), b, s, H, d, causal, st))
        if only and name != only:
            continue
        tf = timeit(fwd, iters)
        tb = timeit(bwd, iters)
        flops = 4.0 * b * H * s * s * d * (0.5 if causal else 1.0)
        print(f"{name:16s} fwd {tf * 1e6:7.1f} us {flops / tf / 1e12:6.0f} TF/s   "
              f"bwd {tb * 1e6:7.1f} us {2.5 * flops / tb / 1e12:6.0f} TF/s", flush=True)


if __name__ == "__main__":
    main()
