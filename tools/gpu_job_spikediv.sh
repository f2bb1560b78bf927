for d in 2 3 4 6 8; do
  AS_SPIKE_DIV=$d python bench.py --config C2 --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('div $d', d['ms_per_step'], d['roofline']['stage_ms'])"
done
