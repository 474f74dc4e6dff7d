"""Build libsfb.so in-tree with nvcc for sm_100a (no JIT cache: the .so travels
with the repo snapshot to the GPU box)."""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRC = os.path.join(HERE, "csrc", "sfb.cu")
DEPS = [SRC, os.path.join(HERE, "csrc", "sfb_kernel.cuh"), os.path.join(ROOT, "include", "sfb.h")]
OUT = os.path.join(HERE, "libsfb.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v", f"-I{os.path.join(ROOT, 'include')}"]


def up_to_date() -> bool:
    if not os.path.exists(OUT):
        return False
    t = os.path.getmtime(OUT)
    return all(os.path.getmtime(p) <= t for p in DEPS)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return OUT
    cmd = [NVCC, *FLAGS, "-o", OUT + ".tmp", SRC]
    proc = subprocess.run(cmd, capture_output=True, text=True)
    log = os.path.join(HERE, "csrc", "ptxas.log")
    with open(log, "w") as fh:
        fh.write(proc.stdout + proc.stderr)
    if proc.returncode != 0:
        sys.stderr.write(proc.stderr[-4000:])
        raise RuntimeError(f"nvcc failed ({proc.returncode}); see {log}")
    os.replace(OUT + ".tmp", OUT)
    if verbose:
        print(f"built {OUT}")
    return OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
