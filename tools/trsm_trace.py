"""Per-CTA timeline of the multi-RHS triangular solve of one C3b / C3a solve (AS_LU_TRACE=1 AS_TS_TRACE=1):
ticket t = step s * tiles + tile; prints, per block step, the tile-0 CTA's start / end (us)."""
import ctypes as C
import os
import sys
os.environ["AS_LU_TRACE"] = "1"
os.environ["AS_TS_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2007_11208_b200 as AS  # noqa: E402
import workloads as W  # noqa: E402
tag = sys.argv[1] if len(sys.argv) > 1 else "C3b"
tiles = int(sys.argv[2]) if len(sys.argv) > 2 else 8
nrhs = int(sys.argv[3]) if len(sys.argv) > 3 else 0
A, B = W.make(tag, nrhs=nrhs) if nrhs else W.make(tag)
dA, dB = AS.to_device(A), AS.to_device(B)
for _ in range(2):
    AS.as_solve_ex(dA, dB)
    torch.cuda.synchronize()
cap = 2048
lo, hi = (C.c_ulonglong * cap)(), (C.c_ulonglong * cap)()
cnt = AS.lib().as_debug_lu_trace(lo, hi, cap)
nblk = (A.shape[0] + 63) // 64
n_t = nblk * tiles
t0 = min(lo[i] for i in range(n_t))
ends = [(hi[i] - t0) / 1e3 for i in range(n_t)]
starts = [(lo[i] - t0) / 1e3 for i in range(n_t)]
print(f"{tag}: {n_t} CTAs, span {max(ends):.1f} us")
for s in list(range(0, nblk, max(1, nblk // 16))) + [nblk - 1]:
    row = [f"{ends[s * tiles + r]:7.1f}" for r in range(tiles)]
    print(f"step {s:3d} start {starts[s * tiles]:7.1f}  ends " + " ".join(row))
ph = [(hi[1024 + k] - t0) / 1e3 for k in range(6)]
print("step-32 tile-0 last step: spin-start %.1f  X-ready %.1f  stage-ready %.1f  product-done %.1f  dinv-ready %.1f  published %.1f" % tuple(ph))
print("X_31 published (tile 0 of step 31) at %.1f" % ends[31 * tiles])
