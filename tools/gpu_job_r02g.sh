# r02g: LU panel policy (leaf above 10240 rows, cooperative below), band chain reciprocals, LDL^T tests
set -x
O=gpurun_out/r02g
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_r02.py tests/test_gpu_batched.py -m gpu -q -p no:cacheprovider -k "narrow or ldlt" > $O/pytest_new.txt 2>&1; echo "new rc=$?"
timeout 600 python bench.py --config C5 --only --steps 5 --no-cpu-baseline > $O/bench_C5.json 2> $O/bench_C5.err
for m in 6144 8192 12288; do AS_LU_LF_MIN_M=$m timeout 600 python bench.py --config C5 --only --steps 3 --no-cpu-baseline > $O/bench_C5_lf$m.json 2>/dev/null; done
AS_LU_TRACE=1 AS_USE_DEBUG_LIB=1 timeout 300 python tools/lu_trace.py > $O/lu_trace_C5.txt 2>&1
python tools/std_vs_adaptive.py --out $O/std_vs_adaptive.json > $O/std_vs_adaptive.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_r02.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "(lu or LU or debug_factor or c5 or C5) and not narrow" > $O/pytest_lu.txt 2>&1; echo "lu rc=$?"
