#!/usr/bin/env python
"""Full-size oracle references for the configs the GPU parity tests cannot re-solve on the fly.

TEST INFRASTRUCTURE.  Calls only ``oracle/`` (the plain CPU implementation) and ``workloads``
(seeded input generation); nothing here touches the CUDA path.  For each config it writes
``tests/golden/refs/<tag>.npz`` holding the SHA-256 of the input bytes, the oracle's X (or the
fp64 reference of Z21 for C5f), its flags / rcond / anorm / method and, for C4, the oracle's
singular values and rank.  ``tests/test_gpu_r02.py`` regenerates the inputs, checks the
hash and grades the GPU solve against these files (Z18-Z21).

    python tools/oracle_refs.py C5 C5f [--threads N]

(C4 is not stored: its Haar factors come from a LAPACK QR whose rounding differs between machines,
so its input bytes are not portable; its oracle takes seconds and runs inside the test.)

C5 and C5f are the long ones (an unblocked right-looking LU of n = 16384, ~4 n^3 bytes of
traffic each); they are computed once per input hash and committed.
"""
from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import workloads as W  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "refs")


def _save(tag, **kw):
    os.makedirs(OUT, exist_ok=True)
    p = os.path.join(OUT, f"{tag}.npz")
    np.savez(p, **kw)
    print(f"{tag}: wrote {p}", flush=True)


def _rep_fields(rep):
    return dict(flags=np.int64(rep["flags"]), method=np.int64(rep["method"]),
                primary_method=np.int64(rep["primary_method"]), rcond=np.float64(rep["rcond"]),
                anorm=np.float64(rep["anorm"]), rank=np.int64(rep["rank"]), sweeps=np.int64(rep["sweeps"]),
                info=np.int64(rep["info"]))


def ref_c4():
    A, B = W.make("C4")
    t0 = time.time()
    ret, X, rep, sig = oracle.solve(A, B)
    dt = time.time() - t0
    print(f"C4: ret={ret} flags={rep['flags']:#x} rank={rep['rank']} sweeps={rep['sweeps']} {dt:.1f}s", flush=True)
    _save("C4", sha256=W.sha256(A, B), ret=np.int64(ret), X=X, sigma=sig, seconds=dt, **_rep_fields(rep))


def ref_c5():
    A, B = W.make("C5")
    sha = W.sha256(A, B)
    t0 = time.time()
    ret, X, rep, _ = oracle.solve(A, B)
    dt = time.time() - t0
    print(f"C5: ret={ret} flags={rep['flags']:#x} rcond={rep['rcond']:.3e} {dt:.1f}s", flush=True)
    _save("C5", sha256=sha, ret=np.int64(ret), X=X, seconds=dt, **_rep_fields(rep))


def ref_c5f():
    """Z21: the fp32 oracle (NO_FALLBACK) gives the gate bit and rcond in fp32; the solution
    reference is the fp64 oracle on the exactly promoted A32 / B32 (forced LU, as the fp32 run)."""
    A32, B32 = W.make("C5f")
    sha = W.sha256(A32, B32)
    t0 = time.time()
    ret32, _, rep32, _ = oracle.solve(A32, B32, no_fallback=True)
    dt32 = time.time() - t0
    print(f"C5f fp32: ret={ret32} flags={rep32['flags']:#x} rcond={rep32['rcond']:.3e} {dt32:.1f}s", flush=True)
    A64 = np.asfortranarray(A32.astype(np.float64))
    B64 = np.asfortranarray(B32.astype(np.float64))
    del A32
    t0 = time.time()
    ret64, X64, rep64, _ = oracle.solve(A64, B64, no_fallback=True)
    dt64 = time.time() - t0
    print(f"C5f fp64-ref: ret={ret64} flags={rep64['flags']:#x} rcond={rep64['rcond']:.3e} {dt64:.1f}s", flush=True)
    f32 = {k + "32": v for k, v in _rep_fields(rep32).items()}
    _save("C5f", sha256=sha, ret32=np.int64(ret32), ret=np.int64(ret64), X=X64, seconds32=dt32, seconds=dt64,
          **f32, **_rep_fields(rep64))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("tags", nargs="+", choices=["C4", "C5", "C5f"])
    ap.add_argument("--threads", type=int, default=len(os.sched_getaffinity(0)))
    a = ap.parse_args()
    oracle.set_threads(a.threads)
    print(f"oracle threads: {oracle.get_threads()}", flush=True)
    for t in a.tags:
        {"C4": ref_c4, "C5": ref_c5, "C5f": ref_c5f}[t]()


if __name__ == "__main__":
    main()
