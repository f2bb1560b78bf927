# Re-entry check: GPU parity suite, default bench, every config's bench line, C5 LU timeline.
set -x
O=gpurun_out/r01c
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 $O/pytest_gpu.log
python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench default rc=$?"
for c in C1 C3a C3b C4 C5 C5f; do
  timeout 400 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; echo "$c rc=$?"
done
timeout 300 python tools/lu_trace.py C5 > $O/lu_trace.txt 2>&1; echo "trace rc=$?"
timeout 300 python tools/lu_check.py > $O/lu_check.txt 2>&1; echo "check rc=$?"
