"""A few eager-mode solves of one structure class / size (ncu launch lists): kind in banded, lower, sympd, dense."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_2007_11208_b200 as AS  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from std_vs_adaptive import make  # noqa: E402
kind, n = sys.argv[1], int(sys.argv[2])
AS.set_exec_mode(True)
A = make(kind, n, seed=n)
B = np.asfortranarray(np.random.default_rng(n).standard_normal((n, 1)))
dA, dB = AS.to_device(A), AS.to_device(B)
for _ in range(2):
    ret, X, rep = AS.as_solve_ex(dA, dB)
    torch.cuda.synchronize()
print(kind, n, ret, rep["method"], hex(rep["flags"]))
