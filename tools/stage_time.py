"""Stage timing (detect / factor+rcond / solve) of one config, graph or eager mode."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2007_11208_b200 as AS  # noqa: E402
import workloads as W  # noqa: E402
ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C5")
ap.add_argument("--eager", action="store_true")
ap.add_argument("--calls", type=int, default=3)
ap.add_argument("--n", type=int, default=0, help="override the config's n (e.g. C3a at 16384)")
a = ap.parse_args()
AS.set_instrumentation(True)
if a.eager:
    AS.set_exec_mode(True)
A, B = W.make(a.config, **({"n": a.n} if a.n else {}))
n = A.shape[0]
flops = {"C3a": n ** 3 / 3, "C5": 2 * n ** 3 / 3, "C5f": 2 * n ** 3 / 3, "C1": 2 * n ** 3 / 3}.get(a.config)
dA, dB = AS.to_device(A), AS.to_device(B)
X = AS.empty_colmajor(B.shape[0], B.shape[1], dB.dtype)
for i in range(a.calls):
    ret, _, rep = AS.as_solve_ex(dA, dB, X=X)
    torch.cuda.synchronize()
    st = AS.last_stage_ms()
    print(i, ret, hex(rep["flags"]), rep["method"], [round(x, 3) for x in st],
          f"factor stage {flops / (st[1] * 1e-3) / 1e12:.2f} TFLOP/s (factorization flops only)" if flops else "", flush=True)
if n <= 16384:
    import numpy as np
    Xh = AS.to_host(X)
    R = A @ Xh - B
    print("eta", float((np.abs(R).max(axis=0) / (np.abs(A).sum(axis=1).max() * np.abs(Xh).max(axis=0))).max()))
