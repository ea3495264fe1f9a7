"""In-tree build of libiwpp_b200.so (nvcc, sm_100a).

No JIT cache: the shared object is written next to this file so it travels
with the repository snapshot to the GPU box.
"""

from __future__ import annotations

import os
import shutil
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libiwpp_b200.so")
SOURCES = ["capi.cu", "recon_tiles.cu", "recon_sweeps.cu", "recon_passes.cu", "edt.cu", "edt_block.cu", "edt_slab.cu", "edt_aux.cu", "imgio.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(HERE, "..", "include", "iwpp_b200.h"))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False, out: str | None = None,
          defines: tuple = ()) -> str:
    """Compile libiwpp_b200.so (or, for development variants, ``out`` with
    extra ``-D`` ``defines``)."""
    if out is None and not force and not _stale():
        return LIB
    target = out or LIB
    cmd = [_nvcc(), "-shared", "-Xcompiler", "-fPIC", "-O3", "-lineinfo", "-std=c++17",
           *ARCH, *[f"-D{d}" for d in defines], "-o", target + ".tmp",
           *[os.path.join(CSRC, s) for s in SOURCES]]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd))
    subprocess.run(cmd, check=True, cwd=CSRC)
    os.replace(target + ".tmp", target)
    return target


if __name__ == "__main__":
    import sys
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
