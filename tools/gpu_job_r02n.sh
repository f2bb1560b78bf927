# r02n: LU dataflow schedule (fixed column chunks), swap+U12 v3, TRSM DMMA block product
set -x
O=gpurun_out/r02n
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_r02.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x -k "(lu or LU or debug_factor or spd or chol or triang or determin) and not c5 and not C5 and not narrow" > $O/pytest_lu.txt 2>&1; echo "rc=$?"
timeout 600 python bench.py --config C5 --only --steps 5 --no-cpu-baseline > $O/bench_C5.json 2> $O/bench_C5.err
AS_LU_SWAP_V2=1 timeout 600 python bench.py --config C5 --only --steps 5 --no-cpu-baseline > $O/bench_C5_swapv2.json 2> $O/bench_C5_swapv2.err
AS_LU_OLD_SCHED=1 timeout 600 python bench.py --config C5 --only --steps 5 --no-cpu-baseline > $O/bench_C5_oldsched.json 2> $O/bench_C5_oldsched.err
for m in 8192 12288; do
AS_LU_LF_MIN_M=$m timeout 600 python bench.py --config C5 --only --steps 5 --no-cpu-baseline > $O/bench_C5_lf$m.json 2> $O/bench_C5_lf$m.err
done
AS_USE_DEBUG_LIB=1 timeout 600 python tools/lu_trace.py C5 > $O/lu_trace_C5.txt 2>&1
for c in C5f C3a C3b C4 C1; do
timeout 600 python bench.py --config $c --only --steps 10 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 900 python -m pytest tests/test_gpu_r02.py -m gpu -q -p no:cacheprovider -x -k "c5 or C5" > $O/pytest_c5.txt 2>&1; echo "rc=$?"
