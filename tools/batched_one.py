"""One as_solve_batched call of the bench's batched workload (1000 C1-recipe systems, n = 100) for ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2007_11208_b200 as AS  # noqa: E402
import workloads as W  # noqa: E402

n, cnt = 100, int(sys.argv[1]) if len(sys.argv) > 1 else 1000
pairs = [W.dense_c1(n=n, nrhs=1, seed=s) for s in range(cnt)]
dA = AS.to_device_batched(np.stack([p[0] for p in pairs]))
dB = AS.to_device_batched(np.stack([p[1] for p in pairs]))
for _ in range(2):
    ret, X, rep, rets = AS.as_solve_batched(dA, dB)
    torch.cuda.synchronize()
print("batched", ret, int(rets.abs().sum()))
