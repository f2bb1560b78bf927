# detection parity + detection-stage bandwidth on C2 / C3a / C3b (run under gpurun from the repo root)
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -k "detect or spd or sympd or band" > gpurun_out/pt_det.log 2>&1; tail -2 gpurun_out/pt_det.log
for c in C2 C3a C3b; do
  python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['ms_per_step'], d['roofline']['stage_ms'], d.get('detect_hbm'))"
done
python tools/profile_one.py --config C2 --calls 3 2>&1 | tail -2
