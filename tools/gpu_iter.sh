# Iteration job: GPU parity subset ($1 = pytest -k expression, "" = all), then bench configs ($2, space separated)
O=gpurun_out/iter
rm -rf $O; mkdir -p $O
if [ -n "$1" ]; then K="-k"; fi
timeout 900 python -m pytest tests -m gpu -x -q $K "$1" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
for c in $2; do
  timeout 400 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; echo "$c rc=$?"
  python -c "
import json;d=json.load(open('$O/bench_$c.json'));r=d['roofline'];print('$c',round(d['value'],2),'ms',round(d['ms_per_step'],3),r.get('stage_ms'),'frac',round(r['frac'],3),d.get('detect_hbm',{}).get('frac'),d['clocks']['sm_mhz'])"
done
shift 2
for cmd in "$@"; do echo "== $cmd"; timeout 300 bash -c "$cmd" 2>&1 | tail -40; done
