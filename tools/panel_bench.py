"""Panel-kernel timing study: one LU / Cholesky panel in isolation (as_debug_panel_time), with
the register panel's ablation bits, over the row counts the C1 / C5 factorizations see."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2007_11208_b200 as AS  # noqa: E402

ms = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "128,256,512,1024,2048,4096,8192,16384").split(",")]
lu_only = os.environ.get("LU_ONLY")
g = torch.Generator(device="cuda").manual_seed(0)
dt = torch.float64
for m in ms:
    A = torch.randn(m, m, generator=g, device="cuda", dtype=dt).t().contiguous().t()
    row = [f"LU m={m:6d}"]
    for kind, dbg, tag in [(0, 0, "fast"), (0, 1, "noswap"), (0, 2, "nodefer"), (0, 8, "nocols"), (0, 11, "empty"),
                           (1, 0, "coop")]:
        t = AS.debug_panel_time(A, 0, min(128, m), kind=kind, iters=4, dbg=dbg)
        torch.cuda.synchronize()
        row.append(f"{tag} {t:8.1f}")
    print(" | ".join(row), flush=True)
if not lu_only:
    for m in [256, 1024, 4096]:
        G = torch.randn(m, m, generator=g, device="cuda", dtype=dt)
        A = (G @ G.t() / m + torch.eye(m, device="cuda", dtype=dt)).t().contiguous().t()
        row = [f"CH m={m:6d}"]
        for kind, tag in [(2, "cluster"), (3, "potf2+l21")]:
            t = AS.debug_panel_time(A, 0, 64, kind=kind, iters=4)
            torch.cuda.synchronize()
            row.append(f"{tag} {t:8.1f}")
        print(" | ".join(row), flush=True)
