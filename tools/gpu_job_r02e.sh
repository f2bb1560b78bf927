# r02e: narrow-band chain, batched (relaxed ill-conditioned bits), swap+U12 v2 (C5)
set -x
O=gpurun_out/r02e
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_r02.py tests/test_gpu_batched.py -m gpu -q -p no:cacheprovider -k "narrow or batched" > $O/pytest_new.txt 2>&1; echo "new rc=$?"
timeout 600 python bench.py --config C5 --only --steps 5 --no-cpu-baseline > $O/bench_C5.json 2> $O/bench_C5.err
AS_LU_SWAP_V1=1 timeout 600 python bench.py --config C5 --only --steps 5 --no-cpu-baseline > $O/bench_C5_swapv1.json 2> $O/bench_C5_swapv1.err
timeout 900 python -m pytest tests/test_gpu_r02.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "(lu or LU or debug_factor or c5 or C5 or band) and not c5f" > $O/pytest_lu.txt 2>&1; echo "lu rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C5_eager.csv \
    python tools/profile_one.py --config C5 --eager --calls 1 > /dev/null 2>&1
python tools/launches.py $O/launches_C5_eager.csv > $O/launches_C5_eager.txt 2>&1
python tools/std_vs_adaptive.py --out $O/std_vs_adaptive.json > $O/std_vs_adaptive.txt 2>&1
