# Re-entry check (r01h): GPU parity suite, smoke, and bench lines on the current tree
set -x
O=gpurun_out/r01h
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?"
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?"
python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench default rc=$?"
for c in C1 C3a C3b C4 C5 C5f; do
  timeout 400 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; echo "$c rc=$?"
done
