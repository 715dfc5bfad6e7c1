"""Build libckks_b200.so in-tree with nvcc for sm_100a (no JIT, no torch extension).

The library is a plain C-ABI shared object (include/ckks_b200.h) loaded with
ctypes; it travels to the GPU box with the repo snapshot.
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libckks_b200.so")
SOURCES = ["ntt.cu", "ntt_tc.cu", "bconv.cu", "kskip.cu", "ew.cu", "fused.cu", "bsgs.cu", "xof.cu", "capi.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC,-O2", "--expt-relaxed-constexpr", "-Xptxas", "-v"]


def _source_hash(extra=()) -> str:
    """sha256 over every CUDA source/header, the C-ABI header, the flags and nvcc's path."""
    import hashlib
    h = hashlib.sha256()
    deps = sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC)
                  if f.endswith((".cu", ".cuh", ".h")))
    deps.append(os.path.join(os.path.dirname(HERE), "include", "ckks_b200.h"))
    for d in deps:
        h.update(os.path.basename(d).encode())
        h.update(open(d, "rb").read())
    h.update(" ".join([NVCC, *FLAGS, *extra]).encode())
    return h.hexdigest()


def _stamp(out: str) -> str:
    return out + ".srchash"


def _stale() -> bool:
    """Rebuild unless the library exists AND was built from exactly these sources
    (a content hash, not mtimes: a shipped prebuilt .so newer than edited sources
    would otherwise be reused)."""
    if not os.path.exists(LIB) or not os.path.exists(_stamp(LIB)):
        return True
    return open(_stamp(LIB)).read().strip() != _source_hash()


def build(force: bool = False, verbose: bool = False, extra=(), out: str = LIB) -> str:
    """Compile every source and link `out`.  `extra` nvcc flags build A/B
    variants (e.g. -DCKB200_EXACT_SHOUP into another .so, selected at run time
    with CKB200_LIB=<path>)."""
    if out == LIB and not extra and not force and not _stale():
        return LIB
    from concurrent.futures import ThreadPoolExecutor

    def compile_one(src):
        tag = os.path.basename(out).replace(".so", "")
        obj = os.path.join(CSRC, src.replace(".cu", f".{tag}.o"))
        cmd = [NVCC, *FLAGS, *extra, "-c", os.path.join(CSRC, src), "-o", obj]
        return src, obj, subprocess.run(cmd, capture_output=True, text=True)

    objs = []
    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 1)) as ex:
        for src, obj, r in ex.map(compile_one, SOURCES):
            if r.returncode != 0:
                sys.stderr.write(r.stdout + r.stderr)
                raise RuntimeError(f"nvcc failed on {src}")
            if verbose:
                sys.stderr.write(r.stderr)
            objs.append(obj)
    cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *objs, "-o", out,
           "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("link failed")
    for o in objs:
        os.remove(o)
    with open(_stamp(out), "w") as f:
        f.write(_source_hash(extra) + "\n")
    return out


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if a not in ("--force", "-v")]
    flags = [a for a in args if a.startswith("-D")]
    outs = [a for a in args if a.endswith(".so")]
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, extra=flags,
                out=os.path.abspath(outs[0]) if outs else LIB))
