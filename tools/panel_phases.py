import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2007_11208_b200 as AS
g = torch.Generator(device="cuda").manual_seed(0)
m = int(sys.argv[1]); kind = int(sys.argv[2]) if len(sys.argv) > 2 else 0
A = torch.randn(m, m, generator=g, device="cuda", dtype=torch.float64).t().contiguous().t()
t = AS.debug_panel_time(A, 0, min(128, m), kind=kind, iters=2, dbg=256)
torch.cuda.synchronize()
print("m", m, "kind", kind, "us", t, flush=True)
