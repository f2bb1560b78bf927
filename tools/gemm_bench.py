"""TFLOP/s of the library's trailing-update GEMMs (fp64 DMMA, fp32 SIMT) at LU shapes vs the DMMA peak."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2007_11208_b200 as AS  # noqa: E402

peak = AS.measure_fp64_peak(40000)
print(f"fp64 DMMA peak {peak:.2f} TF")
for (M, N, K) in [(16384, 16384, 128), (16384, 16384, 256), (12288, 12288, 128), (8192, 8192, 128), (4096, 4096, 128),
                  (2048, 2048, 128)]:
    t = AS.bench_gemm(M, N, K, AS.AS_F64, False, 5)
    print(f"fp64 NN {M}x{N}x{K}: {t:.2f} TF ({100 * t / peak:.1f}%)", flush=True)
for (M, N, K) in [(16384, 16384, 64), (16384, 16384, 128), (16384, 16384, 256)]:
    t = AS.bench_gemm(M, N, K, AS.AS_F32, False, 5)
    print(f"fp32 NN {M}x{N}x{K}: {t:.2f} TF")
