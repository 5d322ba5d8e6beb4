"""Is a GEMM's last partial wave worth filling under the power cap?  Runs two shapes whose pair
tiles are all in one wave with the SAME per-pair work (one 256x256 tile, K=8192): 64 tiles (128 of
148 SMs busy) and 74 tiles (all SMs).  Each loops for ~4 s so the clocks settle at the power
cap; prints TFLOP/s over the last half and the median SM clock sampled meanwhile.  If the 74-tile
shape is ~74/64 faster per FLOP the idle SMs are pure waste (stream-K pays); if ~1.0 the chip is
power-bound and the idle SMs save clock.  Debug tool, not part of the library."""
import subprocess
import sys
import threading
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parent))
from bench_gemm import gemm_desc  # noqa: E402
from paper_2303_01675_b200 import _lib as L  # noqa: E402


def clocks(stop, out):
    while not stop.is_set():
        r = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits",
                            "-i", "0"], capture_output=True, text=True)
        try:
            c, p = r.stdout.strip().split(",")
            out.append((float(c), float(p)))
        except ValueError:
            pass
        time.sleep(0.1)


def run(name, m, n, k, seconds=4.0):
    A = torch.randn(m, k, device="cuda").bfloat16()
    B = torch.randn(n, k, device="cuda").bfloat16()
    C = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    d = gemm_desc(m, n, k, A, 0, B, 0, C, L.EPI_BF16)
    st = torch.cuda.current_stream().cuda_stream
    lib = L.lib()
    for _ in range(5):
        L.check(lib.ptk_gemm(d, st))
    torch.cuda.synchronize()
    stop, samp = threading.Event(), []
    th = threading.Thread(target=clocks, args=(stop, samp))
    th.start()
    t0 = time.time()
    times = []
    while time.time() - t0 < seconds:
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(50):
            L.check(lib.ptk_gemm(d, st))
        e.record()
        e.synchronize()
        times.append(s.elapsed_time(e) / 50 * 1e-3)
    stop.set()
    th.join()
    tail = times[len(times) // 2:]
    t = sum(tail) / len(tail)
    half = samp[len(samp) // 2:] or samp
    clk = sorted(x[0] for x in half)[len(half) // 2] if half else 0
    pw = sorted(x[1] for x in half)[len(half) // 2] if half else 0
    tf = 2.0 * m * n * k / t / 1e12
    print(f"{name:28s} {t * 1e6:8.1f} us/launch {tf:7.1f} TFLOP/s  sm {clk:.0f} MHz  {pw:.0f} W")
    return tf


if __name__ == "__main__":
    a = run("64 tiles 2048x2048x8192", 2048, 2048, 8192)
    b = run("74 tiles 512x9472x8192", 512, 9472, 8192)
    a2 = run("64 tiles again", 2048, 2048, 8192)
    print(f"ratio 74/64 tiles: {b / ((a + a2) / 2):.3f} (74/64 = {74 / 64:.3f})")
