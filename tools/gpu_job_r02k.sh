# r02k: detection modes (streaming triangle, sympd-only) parity + timing
set -x
O=gpurun_out/r02k
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_r02.py -m gpu -q -p no:cacheprovider -k "detect or triangular or spd or C3 or config or density or finite" > $O/pytest_det.txt 2>&1; echo "det rc=$?"
for c in C3a C3b C2; do timeout 600 python bench.py --config $c --only --steps 10 --no-cpu-baseline > $O/bench_$c.json 2>/dev/null; done
NF="ncu --set full --import-source on --clock-control none"
timeout 600 $NF -k regex:detect_pairs_v3 --launch-count 1 -o $O/detect_C3a python tools/profile_one.py --config C3a --eager --calls 1 > $O/ncu_det_c3a.log 2>&1
timeout 600 $NF -k regex:detect_pairs_v3 --launch-count 1 -o $O/detect_C3b python tools/profile_one.py --config C3b --eager --calls 1 > $O/ncu_det_c3b.log 2>&1
