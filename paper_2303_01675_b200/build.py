"""In-tree build of libptk.so (host planner C++ + sm_100a CUDA kernels).

Every translation unit under csrc/ is compiled with nvcc for
`-gencode arch=compute_100a,code=sm_100a` (host-only .cpp files go through
nvcc too, which forwards them to g++), then linked into
paper_2303_01675_b200/libptk.so.  The .so is git-ignored but travels to the
GPU box with the gpurun snapshot.  Object files are cached by content hash
in build/ so a rebuild only recompiles what changed.
"""
from __future__ import annotations

import concurrent.futures as cf
import hashlib
import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OBJ = ROOT / "build" / "obj"
LIB = PKG / "libptk.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++20", "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off",
          f"-I{ROOT / 'include'}", f"-I{CSRC}"]
# PTK_EXTRA_NVCC_FLAGS: extra -D switches for experiments (part of the object cache key)
CUDA_FLAGS = ARCH + ["-lineinfo", "--expt-relaxed-constexpr", "-Xptxas", "-v"] + COMMON + \
    os.environ.get("PTK_EXTRA_NVCC_FLAGS", "").split()
CXX_FLAGS = COMMON + ["-x", "c++"]


def _sources() -> list[Path]:
    out = []
    for p in sorted(CSRC.rglob("*")):
        if p.suffix in (".cu", ".cpp"):
            out.append(p)
    return out


def _headers_digest() -> str:
    h = hashlib.sha256()
    for d in (CSRC, ROOT / "include"):
        for p in sorted(d.rglob("*")):
            if p.suffix in (".h", ".hpp", ".cuh"):
                h.update(p.read_bytes())
    return h.hexdigest()


def _compile(src: Path, hdr: str, verbose: bool) -> Path:
    flags = CUDA_FLAGS if src.suffix == ".cu" else CXX_FLAGS
    key = hashlib.sha256(src.read_bytes() + hdr.encode() + " ".join(flags).encode()).hexdigest()[:16]
    obj = OBJ / f"{src.stem}.{key}.o"
    if obj.exists():
        return obj
    OBJ.mkdir(parents=True, exist_ok=True)
    cmd = [NVCC, *flags, "-c", str(src), "-o", str(obj) + ".tmp"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {src}\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    if verbose and src.suffix == ".cu":
        log = OBJ / f"{src.stem}.ptxas.log"
        log.write_text(r.stderr)
    os.replace(str(obj) + ".tmp", obj)
    return obj


def build(verbose: bool = False, jobs: int | None = None) -> Path:
    srcs = _sources()
    hdr = _headers_digest()
    jobs = jobs or max(1, min(len(srcs), os.cpu_count() or 4))
    with cf.ThreadPoolExecutor(jobs) as ex:
        objs = list(ex.map(lambda s: _compile(s, hdr, verbose), srcs))
    stamp = hashlib.sha256("".join(str(o) for o in objs).encode()).hexdigest()
    stamp_file = ROOT / "build" / "libptk.stamp"
    if LIB.exists() and stamp_file.exists() and stamp_file.read_text() == stamp:
        return LIB
    cmd = [NVCC, *ARCH, "-shared", "-o", str(LIB) + ".tmp", *map(str, objs), "-lcudart", "-ldl", "-lpthread"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    os.replace(str(LIB) + ".tmp", LIB)
    stamp_file.write_text(stamp)
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
