"""TFLOP/s of the library GEMM (LU trailing-update shapes) vs the DMMA register-loop peak."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2007_11208_b200 as AS  # noqa: E402

peak = AS.measure_fp64_peak(40000)
print(f"fp64 DMMA peak {peak:.2f} TF")
for (M, N, K) in [(16384, 16384, 64), (16384, 16384, 128), (16384, 16384, 256), (8192, 8192, 128), (4096, 4096, 64)]:
    t = AS.bench_gemm(M, N, K, AS.AS_F64, False, 5)
    print(f"NN {M}x{N}x{K}: {t:.2f} TF ({100 * t / peak:.1f}%)")
t = AS.bench_gemm(4096, 4096, 64, AS.AS_F64, True, 5)
print(f"NT 4096x4096x64: {t:.2f} TF")
for (M, N, K) in [(16384, 16384, 64), (16384, 16384, 128)]:
    t = AS.bench_gemm(M, N, K, AS.AS_F32, False, 5)
    print(f"fp32 NN {M}x{N}x{K}: {t:.2f} TF")
