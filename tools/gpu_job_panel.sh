set -x
O=gpurun_out/panel
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "lu or debug_factor or chol_fail or C5 or C4 or singular or force" > $O/pytest.txt 2>&1; echo "pytest rc=$?"
for c in C5 C5f C4; do timeout 400 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; echo "$c rc=$?"; done
python tools/std_vs_adaptive.py --out $O/std_vs_adaptive.json > $O/std_vs_adaptive.txt 2>&1
