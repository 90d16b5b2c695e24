"""In-tree build of the native libraries (nvcc for sm_100a, g++ for host code).

Outputs (git-ignored, travel to the GPU box with the repo snapshot):
  paper_2209_03883_b200/libofdmr_b200.so  -- CUDA kernels + C-ABI (include/ofdmr_b200.h)
  paper_2209_03883_b200/libofdmr_gen.so   -- seeded synthetic frame generator (input side)
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
ROOT = PKG.parent
BUILD = PKG / "_build"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr", *ARCH]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _run(cmd: list[str]) -> None:
    print("+", " ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)


def _stale(out: Path, deps: list[Path]) -> bool:
    if not out.exists():
        return True
    t = out.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build_cuda(force: bool = False, verbose_ptxas: bool = False) -> Path:
    out = PKG / "libofdmr_b200.so"
    headers = list(CSRC.glob("*.cuh")) + [ROOT / "include" / "ofdmr_b200.h", ROOT / "include" / "ofdmr_gen.h"]
    units = {
        "radar_kernels": [],
        "mixed_kernels": [],
        "colpass2048": [],
        "fast_kernels": [],
        "fused_ce": [],
        "fused_pg2": [],
        "fused_pg3": [],
        "rowpass_zp": [],
        "noise_kernels": [],
        "ofdm_kernels": [],
        "io_kernels": [],
        "capi": [],
        "multi": [],
        # exact fp64 rounding order (no FMA contraction) for bit-parity of SFT decisions
        "sft_kernels": ["-fmad=false"],
        # GPU frame generator: the CPU generator's fp64 operation order (no FMA contraction)
        "gen_kernels": ["-fmad=false"],
    }
    deps = [CSRC / f"{u}.cu" for u in units] + headers
    if not force and not _stale(out, deps):
        return out
    BUILD.mkdir(exist_ok=True)
    nvcc = _nvcc()
    objs = []
    for unit, extra in units.items():
        obj = BUILD / f"{unit}.o"
        cmd = [nvcc, *NVFLAGS, *extra, "-c", str(CSRC / f"{unit}.cu"), "-o", str(obj)]
        if verbose_ptxas:
            cmd.insert(1, "-Xptxas=-v")
        _run(cmd)
        objs.append(str(obj))
    _run([nvcc, *ARCH, "-shared", "-o", str(out), *objs, "-lcudart"])
    return out


def build_gen(force: bool = False) -> Path:
    out = PKG / "libofdmr_gen.so"
    src = CSRC / "gen.cpp"
    if force or _stale(out, [src, ROOT / "include" / "ofdmr_gen.h"]):
        # default x86-64 codegen (no FMA) like the reference's Release build
        _run(["g++", "-O3", "-DNDEBUG", "-std=c++17", "-fPIC", "-shared", "-o", str(out), str(src), "-lpthread"])
    return out


def build_oracle(with_ref: bool = True) -> None:
    """Test-infrastructure libraries: oracle/liboracle.so and, when the reference tree is
    present (this container, not the GPU box), oracle/_ref/libofdmref.so."""
    mk = ROOT / "oracle" / "Makefile"
    _run(["make", "-s", "-f", str(mk), "all"])
    if with_ref and Path("/root/reference/proj/src").is_dir():
        _run(["make", "-s", "-f", str(mk), "ref"])


def build_examples() -> None:
    """C++ integration example against the reference headers (needs /root/reference)."""
    if Path("/root/reference/proj/include").is_dir() and (ROOT / "oracle" / "_ref" / "libofdmref.so").exists():
        _run(["make", "-s", "-f", str(ROOT / "examples" / "Makefile"), "all"])


def build_all(force: bool = False) -> None:
    build_gen(force)
    build_cuda(force)
    build_oracle()
    build_examples()


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
