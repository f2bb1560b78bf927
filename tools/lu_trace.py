"""Timeline of one C5-size LU factorization (AS_LU_TRACE=1): per 128-column block the trailing
GEMM (main stream), both panels and the look-ahead GEMM (high-priority stream)."""
import os, sys
os.environ["AS_LU_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2007_11208_b200 as AS  # noqa: E402
import workloads as W  # noqa: E402
tag = sys.argv[1] if len(sys.argv) > 1 else "C5"
A, B = W.make(tag)
dA, dB = AS.to_device(A), AS.to_device(B)
for _ in range(2):
    AS.as_solve_ex(dA, dB)
    torch.cuda.synchronize()
tr = AS.debug_lu_trace()
blocks = {}
for kind, k, s, e in tr:
    blocks.setdefault(k, {})[kind] = (s, e)
tot_p = tot_g = 0.0
prev_end = 0.0
for k in sorted(blocks):
    b = blocks[k]
    g = b.get("gemm"); p1 = b.get("panel1"); p2 = b.get("panel2"); la = b.get("gemm_la")
    if g: tot_g += g[1] - g[0]
    for p in (p1, p2):
        if p: tot_p += p[1] - p[0]
    show = os.environ.get("SHOW")
    if (show and int(show.split(",")[0]) <= k <= int(show.split(",")[1])) or (not show and (k % 8 == 0 or k > max(blocks) - 4)):
        fmt = lambda x: f"{x[0]:9.1f}-{x[1]:9.1f} ({x[1]-x[0]:7.1f})" if x else " " * 29
        print(f"blk {k:3d} gemm {fmt(g)} | p1 {fmt(p1)} | p2 {fmt(p2)} | la {fmt(la)}")
gaps = []
for k in sorted(blocks):
    if k + 1 in blocks and "gemm" in blocks[k] and "gemm" in blocks[k + 1]:
        gaps.append(blocks[k + 1]["gemm"][0] - blocks[k]["gemm"][1])
if gaps:
    print(f"gap GEMM_k end -> GEMM_k+1 start: mean {sum(gaps)/len(gaps):.1f} us, total {sum(gaps):.1f} us")
end = max(e for _, _, _, e in tr)
print(f"span {end:.1f} us, sum(main gemm) {tot_g:.1f} us, sum(panels) {tot_p:.1f} us")
