"""Build libadaptsolve.so (all CUDA sources, sm_100a) in-tree with nvcc."""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libadaptsolve.so")
# the same sources with -DAS_DEBUG: adds the test-only / diagnostic exports (as_debug_*) of
# include/adaptsolve.h; loaded only by tests and tools, never by the solve, the bench or smoke()
OUT_DEBUG = os.path.join(HERE, "libadaptsolve_debug.so")
DEBUG_ONLY = {"api.cu"}   # the only translation unit whose exports change under AS_DEBUG
BUILD = os.path.join(HERE, "build_obj")

NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
                 "-I", os.path.join(HERE, "..", "include")]
# detection decides booleans from floating-point compares: no contraction there
PER_FILE = {"detect.cu": ["-fmad=false"]}


def sources():
    return sorted(f for f in os.listdir(CSRC) if f.endswith(".cu"))


def _deps_mtime():
    return max(os.path.getmtime(os.path.join(CSRC, f)) for f in os.listdir(CSRC)) if os.path.isdir(CSRC) else 0


def _obj(src: str, debug: bool = False) -> str:
    return os.path.join(BUILD, src.replace(".cu", "_debug.o" if debug else ".o"))


def _compile(src: str, verbose: bool, debug: bool = False) -> str:
    obj = _obj(src, debug)
    cmd = [NVCC] + COMMON + PER_FILE.get(src, []) + (["-DAS_DEBUG"] if debug else []) + \
        ["-c", os.path.join(CSRC, src), "-o", obj]
    if verbose:
        cmd += ["-Xptxas", "-v"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return obj


def build(force: bool = False, verbose: bool = False) -> str:
    hdr = os.path.join(HERE, "..", "include", "adaptsolve.h")
    newest = max(_deps_mtime(), os.path.getmtime(hdr))
    if not force and all(os.path.exists(o) and os.path.getmtime(o) >= newest for o in (OUT, OUT_DEBUG)):
        return OUT
    os.makedirs(BUILD, exist_ok=True)
    # a source is recompiled when it, or any header, is newer than its object
    hdrs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))] + [hdr]
    newest_hdr = max(os.path.getmtime(h) for h in hdrs)

    def need(src: str, debug: bool) -> bool:
        obj = _obj(src, debug)
        if force or verbose or not os.path.exists(obj):
            return True
        return os.path.getmtime(obj) < max(newest_hdr, os.path.getmtime(os.path.join(CSRC, src)))

    def one(job) -> str:
        src, debug = job
        return _compile(src, verbose, debug) if need(src, debug) else _obj(src, debug)

    jobs = [(s, False) for s in sources()] + [(s, True) for s in sources() if s in DEBUG_ONLY]
    # the largest translation units first (they bound the wall time)
    jobs.sort(key=lambda j: -os.path.getsize(os.path.join(CSRC, j[0])))
    with cf.ThreadPoolExecutor(max_workers=min(10, (os.cpu_count() or 4) + 2)) as ex:
        objs = dict(zip(jobs, ex.map(one, jobs)))
    for out, debug in ((OUT, False), (OUT_DEBUG, True)):
        lst = [objs[(s, debug and s in DEBUG_ONLY)] for s in sources()]
        tmp = out + ".tmp"
        cmd = [NVCC] + ARCH + ["-shared", "-o", tmp] + lst + ["-lcudart", "-lcuda"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
        os.replace(tmp, out)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
