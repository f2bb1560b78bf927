set -x
O=${1:-gpurun_out/detect_check}
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "detect or smallcluster or lu_small or spd or triang or banded" > $O/pytest.txt 2>&1; echo "pytest rc=$?"
tail -4 $O/pytest.txt
b() { cfg=$1; name=$2; st=$3; shift 3; env "$@" timeout 600 python bench.py --config $cfg --only --steps $st --no-cpu-baseline > $O/bench_${cfg}_$name.json 2> $O/bench_${cfg}_$name.err; }
b C3b a 30 AS_X=0
b C3a a 20 AS_X=0
b C2 a 30 AS_X=0
b C1 a 50 AS_X=0
for c in C3b; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:detect --log-file $O/launches_$c.csv python tools/profile_one.py --config $c --eager --calls 1 > /dev/null 2>&1
python tools/launches.py $O/launches_$c.csv > $O/launches_$c.txt 2>&1; head -5 $O/launches_$c.txt
done
