# r02h: chunked swap+U12 / GEMM on two streams, 8-CTA linv128
set -x
O=gpurun_out/r02h
mkdir -p $O
timeout 600 python bench.py --config C5 --only --steps 5 --no-cpu-baseline > $O/bench_C5.json 2> $O/bench_C5.err
for c in 1 2 8; do AS_LU_SWAP_CHUNKS=$c timeout 600 python bench.py --config C5 --only --steps 3 --no-cpu-baseline > $O/bench_C5_ch$c.json 2>/dev/null; done
timeout 600 python bench.py --config C5f --only --steps 3 --no-cpu-baseline > $O/bench_C5f.json 2>/dev/null
AS_LU_TRACE=1 AS_USE_DEBUG_LIB=1 timeout 300 python tools/lu_trace.py > $O/lu_trace_C5.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_r02.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "(lu or LU or debug_factor or c5 or C5) and not narrow" > $O/pytest_lu.txt 2>&1; echo "lu rc=$?"
