O=gpurun_out/prof
mkdir -p $O
timeout 300 python -m pytest tests -m gpu -x -q -k "spd or chol or C3a" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.log
timeout 300 python bench.py --config C3a --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_C3a.json 2>&1; echo "C3a rc=$?"
python -c "
import json;d=json.load(open('$O/bench_C3a.json'));r=d['roofline'];print('C3a',round(d['value'],2),'ms',round(d['ms_per_step'],3),r.get('stage_ms'))"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:lu_panel_leaf --launch-count 1 \
    -o $O/leaf_C1 python tools/profile_one.py --config C1 --eager --calls 1 > $O/leaf_C1.log 2>&1; echo "ncu rc=$?"
