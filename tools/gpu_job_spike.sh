# band SPIKE parity + C2 timing and phase stamps (run under gpurun from the repo root)
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -k "band or spike or banded" > gpurun_out/pt_spike.log 2>&1; tail -2 gpurun_out/pt_spike.log
python bench.py --config C2 --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C2', d['ms_per_step'], d['roofline']['stage_ms'], d['config']['rcond'])"
python tools/profile_one.py --config C2 --calls 3 2>&1 | tail -2
