# r02r: QR with one grid barrier per column (C4), TRSM back to SIMT products
set -x
O=gpurun_out/r02r
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_r02.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x -k "c4 or C4 or fallback or svd or singular or sweep or rank or triang or spd" > $O/pytest.txt 2>&1; echo "rc=$?"
b() { cfg=$1; name=$2; shift 2; env "$@" timeout 600 python bench.py --config $cfg --only --steps 10 --no-cpu-baseline > $O/bench_${cfg}_$name.json 2> $O/bench_${cfg}_$name.err; }
b C4 a AS_X=0
b C3b a AS_X=0
b C3a a AS_X=0
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C4.csv python tools/profile_one.py --config C4 --eager --calls 1 > /dev/null 2>&1
python tools/launches.py $O/launches_C4.csv > $O/launches_C4.txt 2>&1
