# r02i: DMMA GEMM tile configurations, C5 with the best
set -x
O=gpurun_out/r02i
mkdir -p $O
timeout 600 python tools/gemm_bench.py > $O/gemm_bench.txt 2>&1
for c in 1 2 3; do AS_GEMM_CFG=$c timeout 600 python bench.py --config C5 --only --steps 3 --no-cpu-baseline > $O/bench_C5_cfg$c.json 2>/dev/null; done
