# TMA detection pass: parity tests, A/B bench lines (AS_DET_TMA=0 is the register-direct path), launch lists
set -x
O=${1:-gpurun_out/tma}
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_r02.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x -k "detect" > $O/pytest.txt 2>&1; echo "pytest rc=$?"
tail -15 $O/pytest.txt
b() { cfg=$1; name=$2; shift 2; env "$@" timeout 600 python bench.py --config $cfg --only --steps 20 --no-cpu-baseline > $O/bench_${cfg}_$name.json 2> $O/bench_${cfg}_$name.err; }
for c in C2 C3a C3b; do
  b $c tma AS_X=0
  b $c notma AS_DET_TMA=0
  for m in 1 0; do
    AS_DET_TMA=$m timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:detect --csv --log-file $O/launches_${c}_tma$m.csv \
      python tools/profile_one.py --config $c --eager --calls 1 > /dev/null 2>&1
    grep -v "^==" $O/launches_${c}_tma$m.csv | cut -d, -f5,13- | head -20
  done
done
