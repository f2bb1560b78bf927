"""Cholesky diagonal-block timing (diagnostics): POTF2 + L21 and POTF2 alone, for the first block
column of an n x n SPD matrix, with the whole matrix restored before each launch (cold L2) or
only the panel columns (warm L2)."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2007_11208_b200 as AS
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
g = torch.Generator(device="cuda").manual_seed(0)
for dt in (torch.float64, torch.float32):
    M = torch.randn(n, n, generator=g, device="cuda", dtype=dt)
    A = (M @ M.t() / n + torch.eye(n, device="cuda", dtype=dt)).t().contiguous().t()
    for warm in (0, 4):
        for dbg, name in ((0, "potf2+l21"), (2, "potf2")):
            t = AS.debug_panel_time(A, 0, 64, kind=3, iters=20, dbg=dbg | warm)
            print(f"{dt} n={n} {'warm' if warm else 'cold'} L2 {name:10s} {t:8.2f} us", flush=True)
