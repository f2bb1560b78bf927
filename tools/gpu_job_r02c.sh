# r02c: leaf panel v2 (512 rows/CTA, co-resident with GEMM CTAs) + split swap/U12
set -x
O=gpurun_out/r02c
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_r02.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "(lu or LU or debug_factor or c5 or C5) and not c5f" > $O/pytest_lu.txt 2>&1; echo "pytest rc=$?"
timeout 600 python bench.py --config C5 --only --steps 5 --no-cpu-baseline > $O/bench_C5.json 2> $O/bench_C5.err; echo "bench rc=$?"
timeout 600 python bench.py --config C5f --only --steps 5 --no-cpu-baseline > $O/bench_C5f.json 2> $O/bench_C5f.err
AS_LU_TRACE=1 AS_USE_DEBUG_LIB=1 timeout 300 python tools/lu_trace.py > $O/lu_trace_C5.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C5_eager.csv \
    python tools/profile_one.py --config C5 --eager --calls 1 > /dev/null 2>&1
python tools/launches.py $O/launches_C5_eager.csv > $O/launches_C5_eager.txt 2>&1
