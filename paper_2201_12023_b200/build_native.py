"""Build libmpexec.so (the C-ABI of include/mp_exec.h) in-tree for sm_100a.

Plain nvcc, no torch extension machinery: the library exports only extern "C"
symbols and is loaded with ctypes (see native.py).  Used by
__graft_entry__.build() and runnable as `python -m paper_2201_12023_b200.build_native`.
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB = PKG / "libmpexec.so"
SOURCES = ["gemm_sm100.cu", "attention.cu", "ops.cu", "moe.cu", "conv.cu", "comm.cu", "ilp.cpp"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def _nccl_dir() -> Path:
    """The NCCL torch ships (the one already loaded in-process when the library
    is used), so both sides agree on one libnccl.so.2."""
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for base in (spec.submodule_search_locations if spec else []):
        d = Path(base) / "nccl"
        if (d / "include" / "nccl.h").exists():
            return d
    return Path("/usr")


NCCL = _nccl_dir()
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "-Xptxas", "-v",
    "-I", str(PKG.parent / "include"),
    "-I", str(NCCL / "include"),
]


def needs_build() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES] + list(CSRC.glob("*.cuh")) + [PKG.parent / "include" / "mp_exec.h"]
    return any(d.stat().st_mtime > t for d in deps if d.exists())


def build(force: bool = False, verbose: bool = False) -> Path:
    # experiment hooks: extra -D flags and an alternative output path (the
    # product library is always built without them)
    extra = os.environ.get("MPEXEC_NVCC_EXTRA", "").split()
    out = Path(os.environ.get("MPEXEC_LIB_OUT", LIB))
    if not force and not extra and out == LIB and not needs_build():
        return LIB
    nccl_lib = NCCL / "lib"
    cmd = [NVCC, *FLAGS, *extra, *[str(CSRC / s) for s in SOURCES], "-o", str(out) + ".tmp",
           "-L", str(nccl_lib), "-l:libnccl.so.2", "-Xlinker", f"-rpath={nccl_lib}", "-lcuda"]
    # libcuda is resolved at run time through cudaGetDriverEntryPoint; link the stub
    # only so the symbol table is complete when a driver is absent (CPU container).
    stub = Path("/usr/local/cuda/lib64/stubs")
    if stub.exists():
        cmd[-1:-1] = ["-L", str(stub)]
    cmd.remove("-lcuda")
    res = subprocess.run(cmd, capture_output=True, text=True)
    log = (res.stdout or "") + (res.stderr or "")
    (out.parent / (out.stem + ".build.log")).write_text(" ".join(cmd) + "\n" + log)
    if res.returncode != 0:
        sys.stderr.write(log)
        raise RuntimeError(f"nvcc failed ({res.returncode}); see {out.parent / (out.stem + ".build.log")}")
    os.replace(str(out) + ".tmp", out)
    if verbose:
        sys.stdout.write(log)
    return out


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
