# tri_prep rewrite + alignment test: triangular / detect tests, C3b bench and launch list
set -x
O=${1:-gpurun_out/final_check}
mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "triang or detect or determin or estimator or config or force or skip or fp32 or chol_paired" > $O/pytest.txt 2>&1; echo "pytest rc=$?"
tail -4 $O/pytest.txt
b() { cfg=$1; name=$2; st=$3; shift 3; env "$@" timeout 600 python bench.py --config $cfg --only --steps $st --no-cpu-baseline > $O/bench_${cfg}_$name.json 2> $O/bench_${cfg}_$name.err; }
b C3b a 30 AS_X=0
b C3b b 30 AS_X=0
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C3b.csv python tools/profile_one.py --config C3b --eager --calls 1 > /dev/null 2>&1
python tools/launches.py $O/launches_C3b.csv > $O/launches_C3b.txt 2>&1; head -8 $O/launches_C3b.txt
