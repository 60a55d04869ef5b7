"""Build libcbessfm.so in-tree for sm_100a (no JIT cache, no torch headers).

One object per (real type, n_subbands) instantiation of the fused block
kernel (csrc/cbessfm_inst.cu) plus the C ABI (csrc/cbessfm_api.cu), compiled
in parallel with nvcc and linked into ``paper_2409_14489_b200/libcbessfm.so``.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
BUILD = PKG.parent / "build" / "cbessfm"
LIB = PKG / "libcbessfm.so"
HEADERS = [CSRC / "cbessfm_kernel.cuh", CSRC / "cbessfm_launch.cuh", CSRC / "cbessfm_ip.cuh",
           PKG.parent / "include" / "cbessfm.h",
           PKG.parent / "include" / "cbessfm_peaks.h",
           PKG.parent / "include" / "cbessfm_ssfm.h",
           PKG.parent / "include" / "cbessfm_coeff.h",
           PKG.parent / "include" / "cbessfm_rx.h", CSRC / "cbessfm_fft4.cuh"]
REALS = ("float", "double")
SUBBANDS = tuple(range(1, 10))
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
         "-Xptxas", "-v", "--expt-relaxed-constexpr"]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"),
                 "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found: cannot build the sm_100a extension")


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(Path(d).stat().st_mtime > t for d in deps)


def _compile(args):
    src, obj, defs, deps, log = args
    if not _stale(obj, [src, *deps]):
        return obj, None
    cmd = [_nvcc(), *ARCH, *FLAGS, *defs, "-c", str(src), "-o", str(obj)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    log.write_text(res.stdout + res.stderr)
    if res.returncode != 0:
        return obj, f"{' '.join(cmd)}\n{res.stderr[-4000:]}"
    return obj, None


def build(jobs: int | None = None, verbose: bool = False, profile: bool = False,
          variant: str | None = None, defines=()) -> Path:
    """Compile (incrementally) and link libcbessfm.so; returns its path.
    profile=True builds the phase-clock debug variant libcbessfm_prof.so;
    variant="x" with defines=("FOO",) builds an experiment variant
    libcbessfm_x.so (load it with CBESSFM_LIB)."""
    global BUILD, LIB
    if profile:
        variant, defines = "prof", (*defines, "CB_PHASE_PROFILE")
    if variant:
        BUILD = BUILD.parent / f"cbessfm_{variant}"
        LIB = PKG / f"libcbessfm_{variant}.so"
        FLAGS.extend(f"-D{d}" for d in defines)
    BUILD.mkdir(parents=True, exist_ok=True)
    jobs = jobs or max(1, min(len(REALS) * len(SUBBANDS) + 1, os.cpu_count() or 1))
    tasks = []
    for real in REALS:
        for p in SUBBANDS:
            obj = BUILD / f"inst_{real}_{p}.o"
            tasks.append((CSRC / "cbessfm_inst.cu", obj,
                          [f"-DCB_REAL={real}", f"-DCB_P={p}"], HEADERS,
                          BUILD / f"inst_{real}_{p}.log"))
    tasks.append((CSRC / "cbessfm_api.cu", BUILD / "api.o", [], HEADERS,
                  BUILD / "api.log"))
    tasks.append((CSRC / "cbessfm_peaks.cu", BUILD / "peaks.o", [], HEADERS,
                  BUILD / "peaks.log"))
    tasks.append((CSRC / "cbessfm_nlpr.cu", BUILD / "nlpr.o", [], HEADERS,
                  BUILD / "nlpr.log"))
    tasks.append((CSRC / "cbessfm_ssfm.cu", BUILD / "ssfm.o", [], HEADERS,
                  BUILD / "ssfm.log"))
    tasks.append((CSRC / "cbessfm_coeff.cu", BUILD / "coeff.o", [], HEADERS,
                  BUILD / "coeff.log"))
    tasks.append((CSRC / "cbessfm_rx.cu", BUILD / "rx.o", [], HEADERS,
                  BUILD / "rx.log"))
    tasks.append((CSRC / "cbessfm_wide.cu", BUILD / "wide.o", [], HEADERS,
                  BUILD / "wide.log"))
    with ThreadPoolExecutor(jobs) as ex:
        results = list(ex.map(_compile, tasks))
    errors = [e for _, e in results if e]
    if errors:
        raise RuntimeError("nvcc failed:\n" + "\n\n".join(errors))
    objs = [o for o, _ in results]
    if _stale(LIB, objs):
        cmd = [_nvcc(), *ARCH, "-shared", "-o", str(LIB), *map(str, objs),
               "-lcudart"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link failed:\n{res.stderr}")
    if verbose:
        print(f"built {LIB}")
    return LIB


if __name__ == "__main__":
    argv = sys.argv[1:]
    var = argv[argv.index("--variant") + 1] if "--variant" in argv else None
    defs = [argv[i + 1] for i, a in enumerate(argv) if a == "--define"]
    build(verbose=True, profile="--profile" in argv, variant=var, defines=defs)
    sys.exit(0)
