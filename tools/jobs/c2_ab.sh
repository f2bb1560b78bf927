# C2: where the factor stage's +38 us after the TMA detection pass comes from
set -x
O=${1:-gpurun_out/c2_ab}
mkdir -p $O
b() { cfg=$1; name=$2; shift 2; env "$@" timeout 600 python bench.py --config $cfg --only --steps 30 --no-cpu-baseline > $O/bench_${cfg}_$name.json 2> $O/bench_${cfg}_$name.err; }
b C2 hint1 AS_DET_TMA_HINT=1
b C2 hint0 AS_DET_TMA_HINT=0
b C2 notma AS_DET_TMA=0
b C3a hint1 AS_DET_TMA_HINT=1
b C3b hint1 AS_DET_TMA_HINT=1
for m in 1 0; do
  AS_DET_TMA=$m AS_USE_DEBUG_LIB=1 python tools/profile_one.py --config C2 --calls 4 > $O/stamps_tma$m.txt 2>&1
  AS_DET_TMA=$m timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/l_C2_tma$m.csv \
      python tools/profile_one.py --config C2 --eager --calls 1 > /dev/null 2>&1
  python tools/launches.py $O/l_C2_tma$m.csv > $O/l_C2_tma$m.txt 2>&1
done
