# r02t: 512-thread panels, cluster-panel header inbox, GEMM C-tile L2 prefetch
set -x
O=gpurun_out/r02t
mkdir -p $O
timeout 600 python tools/gemm_bench.py > $O/gemm_bench.txt 2>&1
AS_GEMM_PREFETCH=0 timeout 600 python tools/gemm_bench.py > $O/gemm_bench_nopf.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_r02.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x -k "(lu or LU or debug_factor or determin or c4 or C4 or singular or spd or chol) and not narrow" > $O/pytest_lu.txt 2>&1; echo "rc=$?"
AS_USE_DEBUG_LIB=1 LU_ONLY=1 timeout 600 python tools/panel_bench.py 128,1536,2048,4096,8192 > $O/panel_bench.txt 2>&1
for m in 128 1536; do AS_USE_DEBUG_LIB=1 timeout 300 python tools/panel_phases.py $m 0 >> $O/panel_phases.txt 2>&1; done
b() { cfg=$1; name=$2; shift 2; env "$@" timeout 600 python bench.py --config $cfg --only --steps 5 --no-cpu-baseline > $O/bench_${cfg}_$name.json 2> $O/bench_${cfg}_$name.err; }
b C5 a AS_X=0
b C5 nopf AS_GEMM_PREFETCH=0
b C5 lf12288 AS_LU_LF_MIN_M=12288
b C5 lf14336 AS_LU_LF_MIN_M=14336
b C5 lf99999 AS_LU_LF_MIN_M=99999
b C5 b AS_X=0
b C5f a AS_X=0
b C5f nopf AS_GEMM_PREFETCH=0
b C3a a AS_X=0
b C4 a AS_X=0
python tools/std_vs_adaptive.py --out $O/std_vs_adaptive.json > $O/std_vs_adaptive.txt 2>&1
