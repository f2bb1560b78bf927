"""Small solves of every path for compute-sanitizer (memcheck / racecheck / synccheck / initcheck).

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py [--eager]

Each case is checked against the oracle's method bits so a sanitizer run also exercises the path it
claims to (the sanitizer itself reports the hazards).  Sizes are small (the tools slow kernels down
10-100x) but cross every structural boundary: one-cluster LU (n <= 256), cluster panel, leaf panel
(m > 1536, several CTAs), band SPIKE and register chain, TRSM, Cholesky (+failure), SVD fallback,
batched one-block solver incl. LDL^T.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2007_11208_b200 as AS  # noqa: E402
import workloads as W  # noqa: E402

if "--eager" in sys.argv:
    AS.set_exec_mode(True)
rng = np.random.default_rng(0)
cases = [
    ("lu_small", W.random_dense(200, seed=1, shift=4.0)),
    ("lu_cluster", W.random_dense(700, seed=2)),
    ("lu_leaf", W.random_dense(1700, seed=3)),
    ("band_spike", W.random_banded(3000, 4, 3, seed=4, dominant=True)),
    ("band_chain", W.random_banded(900, 2, 2, seed=5)),
    ("band_seq", W.random_banded(600, 6, 5, seed=6)),
    ("upper", W.random_triangular(500, upper=True, seed=7)),
    ("spd", W.random_spd_fig3(400, seed=8)),
    ("illcond", W.illcond_c4(n=96, seed=9)[0]),
]
M = np.full((150, 150), -0.45)
np.fill_diagonal(M, 1.0)
cases.append(("chol_fail", np.asfortranarray(M)))
bad = 0
for name, A in cases:
    n = A.shape[0]
    B = np.asfortranarray(rng.standard_normal((n, 3)))
    ret, X, rep = AS.as_solve_ex(AS.to_device(A), AS.to_device(B))
    torch.cuda.synchronize()
    oret, Xo, orep, _ = oracle.solve(A, B)
    ok = ret == oret and (rep["flags"] & 0xFF) == (orep["flags"] & 0xFF)
    bad += not ok
    print(f"{name:12s} n={n:5d} ret={ret} method={rep['method']} flags={rep['flags']:#x} {'ok' if ok else 'MISMATCH'}",
          flush=True)
# batched one-block solver, incl. the symmetric-indefinite path
sysA = np.stack([W.random_dense(64, seed=s, shift=3.0) for s in range(6)] +
                [np.asfortranarray((lambda m: (m + m.T) / 2)(rng.standard_normal((64, 64)))) for _ in range(2)])
sysB = rng.standard_normal((8, 64, 2))
ret, X, rep, rets = AS.as_solve_batched(AS.to_device_batched(sysA), AS.to_device_batched(sysB),
                                        options=AS.make_options(sym_indef=True))
torch.cuda.synchronize()
print("batched ret", ret, rets.cpu().numpy().tolist(), [r["method"] for r in AS.reports_to_host(rep)], flush=True)
print("mismatches", bad)
sys.exit(1 if bad or ret else 0)
