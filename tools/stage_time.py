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
a = ap.parse_args()
AS.set_instrumentation(True)
if a.eager:
    AS.set_exec_mode(True)
A, B = W.make(a.config)
dA, dB = AS.to_device(A), AS.to_device(B)
X = AS.empty_colmajor(B.shape[0], B.shape[1], dB.dtype)
for i in range(a.calls):
    ret, _, rep = AS.as_solve_ex(dA, dB, X=X)
    torch.cuda.synchronize()
    print(i, ret, hex(rep["flags"]), [round(x, 3) for x in AS.last_stage_ms()])
