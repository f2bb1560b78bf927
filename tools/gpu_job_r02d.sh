# r02d: leaf panel U12 fix + batched small systems
set -x
O=gpurun_out/r02d
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_batched.py -m gpu -q -p no:cacheprovider > $O/pytest_batched.txt 2>&1; echo "batched rc=$?"
timeout 1200 python -m pytest tests/test_gpu_r02.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "(lu or LU or debug_factor or c5 or C5) and not c5f" > $O/pytest_lu.txt 2>&1; echo "pytest rc=$?"
timeout 600 python bench.py --config C5 --only --steps 5 --no-cpu-baseline > $O/bench_C5.json 2> $O/bench_C5.err; echo "bench rc=$?"
