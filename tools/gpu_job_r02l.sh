# r02l: persistent NN DMMA GEMM (AS_GEMM_CFG=4)
set -x
O=gpurun_out/r02l
mkdir -p $O
timeout 600 python tools/gemm_bench.py > $O/gemm_bench.txt 2>&1
AS_GEMM_CFG=4 timeout 600 python bench.py --config C5 --only --steps 5 --no-cpu-baseline > $O/bench_C5_cfg4.json 2> $O/bench_C5_cfg4.err
AS_GEMM_CFG=4 timeout 900 python -m pytest tests/test_gpu_r02.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "(lu or LU or debug_factor or c5 or spd or chol) and not c5f and not narrow" > $O/pytest_cfg4.txt 2>&1; echo "rc=$?"
