"""TFLOP/s of the library's fp64 DMMA GEMM (LU trailing-update shapes) per tile configuration
(AS_GEMM_CFG: 0 BK16 x 2 stages, 1 BK16 x 3, 2 BK32 x 2, 3 BK32 x 3, 4 persistent 128x128 NN) vs the DMMA peak."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2007_11208_b200 as AS  # noqa: E402

peak = AS.measure_fp64_peak(40000)
print(f"fp64 DMMA peak {peak:.2f} TF")
for cfg in (0,):
    os.environ["AS_GEMM_CFG"] = str(cfg)
    for (M, N, K) in [(16384, 16384, 128), (16384, 16384, 256), (8192, 8192, 128), (4096, 4096, 128), (2048, 2048, 128)]:
        t = AS.bench_gemm(M, N, K, AS.AS_F64, False, 5)
        print(f"cfg {cfg} NN {M}x{N}x{K}: {t:.2f} TF ({100 * t / peak:.1f}%)", flush=True)
os.environ.pop("AS_GEMM_CFG")
for (M, N, K) in [(16384, 16384, 64), (16384, 16384, 128)]:
    t = AS.bench_gemm(M, N, K, AS.AS_F32, False, 5)
    print(f"fp32 NN {M}x{N}x{K}: {t:.2f} TF")
