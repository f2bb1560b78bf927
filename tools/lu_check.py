"""Backward error of the dense LU path over sizes and dtypes (diagnostic; residual in fp64 on the GPU)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2007_11208_b200 as AS  # noqa: E402

sizes = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "256,1000,2048,4096,8192,16384").split(",")]
if os.environ.get("EAGER"):
    AS.set_exec_mode(True)
dts = (torch.float32,) if os.environ.get("F32ONLY") else (torch.float32, torch.float64)
g = torch.Generator(device="cuda").manual_seed(0)
for dt in dts:
    for n in sizes:
        A = torch.randn(n, n, generator=g, device="cuda", dtype=torch.float64)
        B = torch.randn(n, 4, generator=g, device="cuda", dtype=torch.float64)
        dA = A.to(dt).t().contiguous().t()
        dB = B.to(dt).t().contiguous().t()
        o = AS.make_options(no_fallback=True)
        ret, X, rep = AS.as_solve_ex(dA, dB, options=o)
        torch.cuda.synchronize()
        A64, X64, B64 = dA.double(), X.double(), dB.double()
        R = A64 @ X64 - B64
        eta = (R.abs().amax(0) / (A64.abs().sum(1).max() * X64.abs().amax(0))).max().item()
        print(f"{str(dt):14s} n={n:6d} ret={ret} flags={rep['flags']:#x} rcond={rep['rcond']:.3e} eta={eta:.3e}", flush=True)
