"""Build the native library in-tree for sm_100a.

    python -m paper_2502_02721_b200.build

produces ``paper_2502_02721_b200/_build/libhessketch_b200.so`` from
``csrc/hs_api.cu`` with explicit ``-gencode arch=compute_100a,code=sm_100a``.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "_build")
LIB = os.path.join(OUT_DIR, "libhessketch_b200.so")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "-Xptxas", "-warn-spills",
]


def _nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def sources():
    return sorted(
        os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cu", ".cuh", ".inc"))
    )


def up_to_date():
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    hdr = os.path.join(os.path.dirname(HERE), "include", "hessketch_b200.h")
    return all(os.path.getmtime(s) <= t for s in sources() + [hdr])


def build(force=False, verbose=True):
    if not force and up_to_date():
        return LIB
    os.makedirs(OUT_DIR, exist_ok=True)
    tmp = LIB + ".tmp"
    # HS_NVCC_DEFS: extra -D switches for compile-time experiments (e.g. "-DHS_ELIM_CS")
    extra = os.environ.get("HS_NVCC_DEFS", "").split()
    cmd = [_nvcc(), *NVCC_FLAGS, *extra, "-o", tmp, os.path.join(CSRC, "hs_api.cu")]
    if verbose:
        print(" ".join(cmd), flush=True)
    proc = subprocess.run(cmd, capture_output=True, text=True)
    out = (proc.stdout or "") + (proc.stderr or "")
    out = "\n".join(l for l in out.splitlines() if "Wno-deprecated-gpu-targets" not in l)
    if proc.returncode != 0:
        raise RuntimeError(f"nvcc failed ({proc.returncode}):\n{out}")
    if verbose and out.strip():
        print(out)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv)
