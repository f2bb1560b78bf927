""""standard vs adaptive" on B200 -- the GPU analogue of the paper's Tables 1-4
(P:535-615).  For each structure class of the paper's experiments (5-diagonal band, lower
triangular, sympd by the Fig. 3 recipe, dense) and size, the same seeded system is solved by
  adaptive : as_solve_ex with default options (detection -> dispatch -> structured solver)
  standard : AS_OPT_FORCE_METHOD(LU) | AS_OPT_SKIP_DETECT (dense LU, no detection: the paper's
             "standard solver")
through the public C-ABI, device-resident inputs, CUDA-event timing of R calls after warm-up.
Reported: mean ms per solve, reduction % = (standard - adaptive) / standard (Tables 1-3) and, for
dense input, the detection overhead % = (adaptive - standard) / standard (Table 4).  The paper's
CPU numbers (i5-5200U + OpenBLAS) are printed beside as context only.

    python tools/std_vs_adaptive.py [--sizes 100,250,500,1000,4096] [--reps 50] [--out profiles/r01/std_vs_adaptive.json]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2007_11208_b200 as AS  # noqa: E402
import workloads as W  # noqa: E402

# Tables 1-4: (standard s, adaptive s), CPU context only
PAPER = {
    "banded": {100: (1.48e-4, 4.76e-5), 250: (1.00e-3, 1.66e-4), 500: (5.41e-3, 5.94e-4), 1000: (3.27e-2, 2.89e-3)},
    "lower": {100: (1.40e-4, 3.82e-5), 250: (1.05e-3, 2.78e-4), 500: (5.48e-3, 1.12e-3), 1000: (3.26e-2, 5.19e-3)},
    "sympd": {100: (1.44e-4, 1.19e-4), 250: (1.03e-3, 7.66e-4), 500: (5.63e-3, 4.27e-3), 1000: (3.31e-2, 2.40e-2)},
    "dense": {100: (1.486e-4, 1.511e-4), 250: (1.220e-3, 1.223e-3), 500: (6.056e-3, 6.063e-3), 1000: (3.598e-2, 3.605e-2)},
}


def make(kind, n, seed):
    if kind == "banded":
        return W.random_banded(n, 2, 2, seed=seed)              # 5 diagonals (Table 1)
    if kind == "lower":
        return W.random_triangular(n, False, seed=seed)
    if kind == "sympd":
        return W.random_spd_fig3(n, seed=seed)
    return W.random_dense(n, seed=seed)


def time_solve(dA, dB, X, opts, reps):
    for _ in range(3):
        ret, _, rep = AS.as_solve_ex(dA, dB, X=X, options=opts)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        AS.as_solve_ex(dA, dB, X=X, options=opts)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, ret, rep


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="100,250,500,1000,4096")
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    std = AS.make_options(force_method=AS.METHOD_LU, skip_detect=True)
    rows = []
    for kind in ("banded", "lower", "sympd", "dense"):
        for n in [int(x) for x in a.sizes.split(",")]:
            A = make(kind, n, seed=n)
            B = np.asfortranarray(np.random.default_rng(n).standard_normal((n, 1)))
            dA, dB = AS.to_device(A), AS.to_device(B)
            X = AS.empty_colmajor(n, 1, dB.dtype)
            reps = a.reps if n <= 1000 else max(5, a.reps // 5)
            t_ad, r_ad, rep_ad = time_solve(dA, dB, X, None, reps)
            t_st, r_st, rep_st = time_solve(dA, dB, X, std, reps)
            row = {"kind": kind, "n": n, "adaptive_ms": t_ad, "standard_ms": t_st,
                   "adaptive_method": rep_ad["method"], "standard_method": rep_st["method"],
                   "ret": [r_ad, r_st]}
            if kind == "dense":
                row["overhead_pct"] = 100.0 * (t_ad - t_st) / t_st
            else:
                row["reduction_pct"] = 100.0 * (t_st - t_ad) / t_st
            if n in PAPER[kind]:
                ps, pa = PAPER[kind][n]
                row["paper_cpu_s"] = {"standard": ps, "adaptive": pa}
            rows.append(row)
            pct = row.get("reduction_pct", row.get("overhead_pct"))
            tag = "overhead" if kind == "dense" else "reduction"
            print(f"{kind:7s} n={n:5d}  adaptive {t_ad:8.3f} ms (method {rep_ad['method']})  standard {t_st:8.3f} ms"
                  f"  {tag} {pct:6.1f}%", flush=True)
    out = {"what": "standard (forced LU, no detection) vs adaptive solve on one B200, 1 RHS, fp64",
           "timing": "CUDA events over reps calls after 3 warm-up calls, inputs resident in HBM", "rows": rows}
    if a.out:
        os.makedirs(os.path.dirname(a.out), exist_ok=True)
        json.dump(out, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
