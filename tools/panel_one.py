"""One panel timing call (isolates a failing configuration): python tools/panel_one.py m kind dbg"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2007_11208_b200 as AS  # noqa: E402
m, kind, dbg = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]) if len(sys.argv) > 3 else 0
g = torch.Generator(device="cuda").manual_seed(0)
A = torch.randn(m, m, generator=g, device="cuda", dtype=torch.float64).t().contiguous().t()
t = AS.debug_panel_time(A, 0, min(128, m), kind=kind, iters=3, dbg=dbg)
torch.cuda.synchronize()
print(f"m={m} kind={kind} dbg={dbg}: {t:.1f} us", flush=True)
