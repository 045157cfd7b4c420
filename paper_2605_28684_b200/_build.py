"""Build ``lib/libadrom_b200.so`` from ``csrc/*.cu`` with nvcc for sm_100a.

Per-file flags: the translation units that evaluate the full-order residual
are compiled with ``--fmad=false`` so they reproduce numpy's (unfused)
arithmetic bit for bit; the linear-algebra units keep FMA contraction.

    python -m paper_2605_28684_b200._build [--force] [--verbose]
"""

from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OBJ = ROOT / "build" / "obj"
LIB = PKG / "lib" / "libadrom_b200.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                 "--expt-relaxed-constexpr", f"-I{ROOT / 'include'}", f"-I{CSRC}"]

#: per-translation-unit extra flags
UNITS = {
    "context.cu": [],
    "fom.cu": ["--fmad=false"],      # bitwise numpy parity of residual / Jacobian
    "sampled.cu": ["--fmad=false"],  # LSPG/Galerkin evaluate the residual too
    "reacting.cu": ["--fmad=false"], # configuration-4 residual (mirrors oracle/reacting.py)
    "btsolve.cu": [],
    "linalg.cu": [],
    "sampling.cu": [],
    "qdeim.cu": [],
    "factored.cu": [],
    "session.cu": [],
    "capi.cu": [],
    "bigsample.cu": ["--fmad=false"],  # large sampled sets (sampled residual bitwise)
    "diag.cu": ["--fmad=false"],       # error diagnostics (primitive fields as numpy)
    "dgemm.cu": [],                    # FP64 tensor-core GEMMs of the large-sample operator
    "hhqr.cu": [],                     # Householder QR / Q application (offline POD, orth, lstsq)
    "offline.cu": [],                  # fit_scaling, POD, orth, least_squares
}


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def _headers_mtime() -> float:
    hs = list(CSRC.glob("*.cuh")) + list((ROOT / "include").glob("*.h")) + [Path(__file__)]
    return max(h.stat().st_mtime for h in hs)


def _compile(src: Path, extra: list[str], verbose: bool) -> tuple[Path, str]:
    obj = OBJ / (src.stem + ".o")
    cmd = [nvcc(), *COMMON, *extra, "-Xptxas", "-v", "-c", str(src), "-o", str(obj)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    log = res.stdout + res.stderr
    (OBJ / (src.stem + ".ptxas.log")).write_text(log)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src.name}:\n{' '.join(cmd)}\n{log}")
    if verbose:
        print(log)
    return obj, log


def build(force: bool = False, verbose: bool = False) -> Path:
    OBJ.mkdir(parents=True, exist_ok=True)
    LIB.parent.mkdir(parents=True, exist_ok=True)
    hdr = _headers_mtime()
    srcs = [CSRC / u for u in UNITS if (CSRC / u).exists()]
    todo = []
    for s in srcs:
        obj = OBJ / (s.stem + ".o")
        if force or not obj.exists() or obj.stat().st_mtime < max(s.stat().st_mtime, hdr):
            todo.append(s)
    if todo:
        with cf.ThreadPoolExecutor(max_workers=min(8, len(todo))) as ex:
            list(ex.map(lambda s: _compile(s, UNITS[s.name], verbose), todo))
    objs = [OBJ / (s.stem + ".o") for s in srcs]
    if force or todo or not LIB.exists() or LIB.stat().st_mtime < max(o.stat().st_mtime for o in objs):
        cmd = [nvcc(), *ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-cudart", "static"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link failed:\n{' '.join(cmd)}\n{res.stdout}{res.stderr}")
    return LIB


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    args = ap.parse_args(argv)
    lib = build(force=args.force, verbose=args.verbose)
    print(lib)


if __name__ == "__main__":
    sys.exit(main())
