# r01j: after the faster one-cluster LU: full GPU suite, smoke, C1/C4 bench lines, C1 launch list,
# ncu capture of lu_small_kernel, phase stamps, default bench line
set -x
O=gpurun_out/r01j
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?"
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?"
python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench default rc=$?"
timeout 300 python bench.py --config C1 --steps 200 --warmup 10 --no-cpu-baseline > $O/bench_C1_200.json 2> $O/bench_C1_200.err
timeout 300 python bench.py --config C1 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_C1.json 2> $O/bench_C1.err
timeout 400 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_C4.json 2> $O/bench_C4.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C1_eager.csv python tools/profile_one.py --config C1 --eager --calls 1 > /dev/null 2>&1; python tools/launches.py $O/launches_C1_eager.csv > $O/launches_C1_eager.txt
timeout 600 ncu --set full --import-source on --clock-control none -k regex:lu_small_kernel --launch-count 1 \
    -o $O/lu_small_C1 python tools/profile_one.py --config C1 --eager --calls 1 > $O/lu_small.log 2>&1; echo "cap rc=$?"
AS_LU_SMALL_PROF=1 python tools/profile_one.py --config C1 --eager --calls 3 > $O/stamps_C1.txt 2>&1
AS_LU_SMALL_PROF=2 python tools/profile_one.py --config C1 --eager --calls 3 > $O/stamps2_C1.txt 2>&1
python tools/std_vs_adaptive.py --out $O/std_vs_adaptive.json > $O/std_vs_adaptive.txt 2>&1; echo "std rc=$?"
