# POTF2 timing study + C3a step time (run under gpurun from the repo root)
mkdir -p gpurun_out
python tools/potf2_bench.py 4096 > gpurun_out/potf2.txt 2>&1
python bench.py --config C3a --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['stage_ms'])" >> gpurun_out/potf2.txt
cat gpurun_out/potf2.txt
