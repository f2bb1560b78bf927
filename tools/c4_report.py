import os, sys
sys.path.insert(0, os.getcwd())
import torch, paper_2007_11208_b200 as AS, workloads as W
A, B = W.make("C4")
ret, X, rep = AS.as_solve_ex(AS.to_device(A), AS.to_device(B)); torch.cuda.synchronize()
print(rep)
