"""Build libpgk.so (the C-ABI CUDA library) in-tree for sm_100a with nvcc."""

from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB = PKG / "libpgk.so"
SOURCES = ["api.cu", "prune.cu", "reverse.cu", "pool_simt.cu", "pool_tc.cu", "pool_tc_f32.cu",
           "pool_tiles.cu",
           "prune_gram.cu", "prune_gram_f32.cu", "search.cu", "nnd.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3",
         "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-Xptxas", "-v"]


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES] + list(CSRC.glob("*.cuh")) + \
        [PKG.parent / "include" / "pgk.h"]
    return any(p.stat().st_mtime > t for p in deps if p.exists())


def build(force: bool = False, verbose: bool = False, out: Path | None = None,
          defines: tuple[str, ...] = ()) -> Path:
    """Compile every source for sm_100a and link libpgk.so (or `out`, with
    extra -D `defines`: kernel-variant builds for A/B timing)."""
    lib = Path(out) if out else LIB
    if not force and not defines and out is None and not _stale():
        return LIB
    tag = lib.stem if (defines or out) else ""
    dflags = [f"-D{d}" for d in defines]

    def compile_one(s):
        obj = CSRC / (s[:-3] + (f".{tag}.o" if tag else ".o"))
        cmd = [NVCC, *FLAGS, *dflags, "-c", str(CSRC / s), "-o", str(obj)]
        return s, str(obj), subprocess.run(cmd, capture_output=True, text=True)

    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 1)) as ex:
        results = list(ex.map(compile_one, SOURCES))
    objs, logs = [], []
    for s, obj, r in results:
        logs.append(r.stderr)
        if r.returncode != 0:
            sys.stderr.write(r.stderr)
            raise RuntimeError(f"nvcc failed on {s}")
        objs.append(obj)
    tmp = lib.with_suffix(".so.tmp")
    cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-Xlinker", "--no-undefined", *objs,
           "-o", str(tmp)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stderr)
        raise RuntimeError("nvcc link failed")
    os.replace(tmp, lib)
    (CSRC / (f"ptxas.{tag}.log" if tag else "ptxas.log")).write_text("".join(logs))
    if verbose:
        print("".join(logs))
    return lib


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
