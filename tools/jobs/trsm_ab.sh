# TRSM staging rewrite: parity on every path that solves, then bench lines
set -x
O=${1:-gpurun_out/trsm_ab}
mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "not detect and not batched" > $O/pytest.txt 2>&1; echo "pytest rc=$?"
tail -4 $O/pytest.txt
b() { cfg=$1; name=$2; st=$3; shift 3; env "$@" timeout 600 python bench.py --config $cfg --only --steps $st --no-cpu-baseline > $O/bench_${cfg}_$name.json 2> $O/bench_${cfg}_$name.err; }
b C3b a 30 AS_X=0
b C3a a 20 AS_X=0
b C1 a 50 AS_X=0
b C4 a 5 AS_X=0
b C5 a 5 AS_X=0
b C5f a 5 AS_X=0
timeout 900 python tools/stage_time.py --config C3a --n 16384 --calls 3 > $O/chol16k.txt 2>&1
tail -n 3 $O/chol16k.txt
AS_TEST_PAIRS=1 AS_CHOL_PAIRS_MIN_N=512 timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "spd or chol or C3a or c3a" > $O/pytest_pairs512.txt 2>&1; tail -n 2 $O/pytest_pairs512.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C3b.csv python tools/profile_one.py --config C3b --eager --calls 1 > /dev/null 2>&1
python tools/launches.py $O/launches_C3b.csv > $O/launches_C3b.txt 2>&1; head -12 $O/launches_C3b.txt
