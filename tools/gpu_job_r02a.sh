# r02a: first round-2 GPU pass: DMMA peak probe variants, full GPU suite, smoke, default bench line
# (headline C5 + every config), C5 eager launch list, ncu pipe metrics on the peak probe
set -x
O=gpurun_out/r02a
mkdir -p $O
nproc > $O/host.txt; lscpu | head -20 >> $O/host.txt
./tools/ubench_dmma > $O/ubench_dmma.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,sm__inst_executed_pipe_tensor_subpipe_dmma.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg.per_second \
    --clock-control none -c 16 --csv --log-file $O/ncu_dmma_probe.csv ./tools/ubench_dmma > /dev/null 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?"
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?"
timeout 1200 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C5_eager.csv \
    python tools/profile_one.py --config C5 --eager --calls 1 > /dev/null 2>&1
python tools/launches.py $O/launches_C5_eager.csv > $O/launches_C5_eager.txt 2>&1
