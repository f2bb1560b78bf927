# small-n one-cluster LU: parity + C1 bench + launch list
set -x
O=gpurun_out/small
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "debug_factor or lu or singular or diag_gate or force or skip_detect or chol_fail or C1 or illcond" > $O/pytest.txt 2>&1; echo "pytest rc=$?"
timeout 300 python bench.py --config C1 --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_C1.json 2> $O/bench_C1.err; echo "C1 rc=$?"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C1_eager.csv python tools/profile_one.py --config C1 --eager --calls 1 > /dev/null 2>&1; python tools/launches.py $O/launches_C1_eager.csv > $O/launches_C1_eager.txt
AS_LU_SMALL_PROF=1 python tools/profile_one.py --config C1 --eager --calls 3 > gpurun_out/small/stamps.txt 2>&1
AS_LU_SMALL_PROF=2 python tools/profile_one.py --config C1 --eager --calls 3 > gpurun_out/small/stamps2.txt 2>&1
