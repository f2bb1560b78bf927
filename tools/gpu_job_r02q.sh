# r02q: panel phase counters, estimator test, C5 repeatability
set -x
O=gpurun_out/r02q
mkdir -p $O
for m in 128 1024 1536; do AS_USE_DEBUG_LIB=1 timeout 300 python tools/panel_phases.py $m 0 >> $O/panel_phases.txt 2>&1; done
AS_USE_DEBUG_LIB=1 LU_ONLY=1 timeout 600 python tools/panel_bench.py 128,512,1536,2048,4096,8192 > $O/panel_bench.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_r02.py -m gpu -q -p no:cacheprovider -k "small_estimator" > $O/pytest_est.txt 2>&1; echo "rc=$?"
b() { cfg=$1; name=$2; shift 2; env "$@" timeout 600 python bench.py --config $cfg --only --steps 5 --no-cpu-baseline > $O/bench_${cfg}_$name.json 2> $O/bench_${cfg}_$name.err; }
b C5 a AS_X=0
b C5 b AS_X=0
b C5 v3la AS_LU_SWAP_V3_MAXC=256
b C5 c AS_X=0
b C3b a AS_X=0
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C3b.csv python tools/profile_one.py --config C3b --eager --calls 1 > /dev/null 2>&1
python tools/launches.py $O/launches_C3b.csv > $O/launches_C3b.txt 2>&1
