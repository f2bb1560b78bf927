"""Run a few adaptive solves of one BASELINE config (for ncu launch lists / captures).

--eager launches the identical kernels without the CUDA graph (ncu cannot profile
kernel nodes of graphs that contain conditional nodes)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2007_11208_b200 as AS  # noqa: E402
import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--calls", type=int, default=2)
ap.add_argument("--n", type=int, default=0)
ap.add_argument("--eager", action="store_true")
a = ap.parse_args()
if a.eager:
    AS.set_exec_mode(True)
kw = {"n": a.n} if a.n else {}
A, B = W.make(a.config, **kw)
dA, dB = AS.to_device(A), AS.to_device(B)
X = AS.empty_colmajor(B.shape[0], B.shape[1], dB.dtype)
for i in range(a.calls):
    ret, _, rep = AS.as_solve_ex(dA, dB, X=X)
    torch.cuda.synchronize()
    print(i, ret, rep["method"], hex(rep["flags"]), rep["rcond"], AS.last_kernel_nodes(), flush=True)
ts = AS.debug_timestamps() if os.environ.get("AS_USE_DEBUG_LIB") else None
if ts and ts[0] is not None:
    print("stamps_us", [round(x, 1) if x is not None else None for x in ts])
