# Round-1 final measurement job (r01i): full GPU suite, bench lines for every config, the reference
# arm, launch lists, and an ncu --set full capture of the new one-cluster LU (C1's dominant kernel)
set -x
O=gpurun_out/r01i
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?"
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?"
python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench default rc=$?"
for c in C1 C3a C3b C4 C5 C5f; do
  timeout 400 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; echo "$c rc=$?"
done
timeout 300 python bench.py --config C1 --steps 200 --warmup 10 --no-cpu-baseline > $O/bench_C1_200.json 2> $O/bench_C1_200.err; echo "C1x200 rc=$?"
python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err; echo "ref rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C2_bench.csv \
  python bench.py --eager --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1; echo "launch list rc=$?"
python tools/launches.py $O/launches_C2_bench.csv > $O/launches_C2_bench.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C1_eager.csv python tools/profile_one.py --config C1 --eager --calls 1 > /dev/null 2>&1; python tools/launches.py $O/launches_C1_eager.csv > $O/launches_C1_eager.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C4_eager.csv python tools/profile_one.py --config C4 --eager --calls 1 > /dev/null 2>&1; python tools/launches.py $O/launches_C4_eager.csv > $O/launches_C4_eager.txt
timeout 600 ncu --set full --import-source on --clock-control none -k regex:lu_small_kernel --launch-count 1 \
    -o $O/lu_small_C1 python tools/profile_one.py --config C1 --eager --calls 1 > $O/lu_small.log 2>&1; echo "cap rc=$?"
AS_LU_SMALL_PROF=1 python tools/profile_one.py --config C1 --eager --calls 3 > $O/stamps_C1.txt 2>&1
AS_LU_SMALL_PROF=2 python tools/profile_one.py --config C1 --eager --calls 3 > $O/stamps2_C1.txt 2>&1
python tools/std_vs_adaptive.py --out $O/std_vs_adaptive.json > $O/std_vs_adaptive.txt 2>&1; echo "std rc=$?"
