# r02o: schedule / swap kernel A-B on C5, 8-warp GEMM configs, fused small-n estimator
set -x
O=gpurun_out/r02o
mkdir -p $O
timeout 600 python tools/gemm_bench.py > $O/gemm_bench.txt 2>&1
b() { name=$1; shift; env "$@" timeout 600 python bench.py --config C5 --only --steps 5 --no-cpu-baseline > $O/bench_C5_$name.json 2> $O/bench_C5_$name.err; }
b default AS_X=0
b v3all AS_LU_SWAP_V3_MAXC=100000
b v2all AS_LU_SWAP_V3_MAXC=0
b sched1 AS_LU_SCHED=1
b sched1_v2all AS_LU_SCHED=1 AS_LU_SWAP_V3_MAXC=0
b gemm5 AS_GEMM_CFG=5
AS_USE_DEBUG_LIB=1 timeout 600 python tools/lu_trace.py C5 > $O/lu_trace_C5.txt 2>&1
AS_LU_SCHED=1 AS_USE_DEBUG_LIB=1 timeout 600 python tools/lu_trace.py C5 > $O/lu_trace_C5_sched1.txt 2>&1
AS_LU_SWAP_V3_MAXC=100000 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C5_v3all.csv python tools/profile_one.py --config C5 --eager --calls 1 > /dev/null 2>&1
python tools/launches.py $O/launches_C5_v3all.csv > $O/launches_C5_v3all.txt 2>&1; gzip -f $O/launches_C5_v3all.csv
timeout 600 python bench.py --config C1 --only --steps 200 --no-cpu-baseline > $O/bench_C1.json 2> $O/bench_C1.err
AS_EST_FUSED_OFF=1 timeout 600 python bench.py --config C1 --only --steps 200 --no-cpu-baseline > $O/bench_C1_nofuse.json 2> $O/bench_C1_nofuse.err
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?"
python tools/std_vs_adaptive.py --out $O/std_vs_adaptive.json > $O/std_vs_adaptive.txt 2>&1
