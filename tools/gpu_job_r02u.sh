# r02u: left-looking one-CTA estimator with register prefetch; reverted GEMM prefetch / 512-thread panels
set -x
O=gpurun_out/r02u
mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?"
b() { cfg=$1; name=$2; shift 2; env "$@" timeout 600 python bench.py --config $cfg --only --steps $ST --no-cpu-baseline > $O/bench_${cfg}_$name.json 2> $O/bench_${cfg}_$name.err; }
ST=200 b C1 a AS_X=0
ST=200 b C1 nofuse AS_EST_FUSED_OFF=1
ST=5 b C5 a AS_X=0
ST=5 b C5 b AS_X=0
python tools/std_vs_adaptive.py --out $O/std_vs_adaptive.json > $O/std_vs_adaptive.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C1.csv python tools/profile_one.py --config C1 --eager --calls 1 > /dev/null 2>&1
python tools/launches.py $O/launches_C1.csv > $O/launches_C1.txt 2>&1
