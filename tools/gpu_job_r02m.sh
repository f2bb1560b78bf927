# r02m: DMMA GEMM with pointer-increment staging + 16-byte C access: gemm_bench per config,
# LU/Cholesky parity subset, C5 timeline and bench
set -x
O=gpurun_out/r02m
mkdir -p $O
timeout 600 python tools/gemm_bench.py > $O/gemm_bench.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_r02.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x -k "(lu or LU or debug_factor or spd or chol) and not c5 and not C5 and not narrow" > $O/pytest_lu.txt 2>&1; echo "rc=$?"
AS_USE_DEBUG_LIB=1 timeout 600 python tools/lu_trace.py C5 > $O/lu_trace_C5.txt 2>&1
timeout 600 python bench.py --config C5 --only --steps 5 --no-cpu-baseline > $O/bench_C5.json 2> $O/bench_C5.err
for cfg in 2 4; do
AS_GEMM_CFG=$cfg timeout 600 python bench.py --config C5 --only --steps 5 --no-cpu-baseline > $O/bench_C5_cfg$cfg.json 2> $O/bench_C5_cfg$cfg.err
done
timeout 600 python bench.py --config C3a --only --steps 10 --no-cpu-baseline > $O/bench_C3a.json 2> $O/bench_C3a.err
