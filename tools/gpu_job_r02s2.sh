# r02s2: cooperative panel with self-validating exchange words
set -x
O=gpurun_out/r02s2
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_r02.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x -k "(lu or LU or debug_factor or determin or c4 or C4 or singular) and not narrow" > $O/pytest_lu.txt 2>&1; echo "rc=$?"
AS_USE_DEBUG_LIB=1 LU_ONLY=1 timeout 600 python tools/panel_bench.py 128,1536,2048,4096,8192 > $O/panel_bench.txt 2>&1
b() { cfg=$1; name=$2; shift 2; env "$@" timeout 600 python bench.py --config $cfg --only --steps 5 --no-cpu-baseline > $O/bench_${cfg}_$name.json 2> $O/bench_${cfg}_$name.err; }
b C5 a AS_X=0
b C5 lf8192 AS_LU_LF_MIN_M=8192
b C5 lf12288 AS_LU_LF_MIN_M=12288
b C5f a AS_X=0
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C5.csv python tools/profile_one.py --config C5 --eager --calls 1 > /dev/null 2>&1
python tools/launches.py $O/launches_C5.csv > $O/launches_C5.txt 2>&1; gzip -f $O/launches_C5.csv
python tools/std_vs_adaptive.py --out $O/std_vs_adaptive.json > $O/std_vs_adaptive.txt 2>&1
