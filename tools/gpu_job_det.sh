set -x
O=gpurun_out/det
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "detect or triangular or C3b or tri or skip_detect or force" > $O/pytest.txt 2>&1; echo "pytest rc=$?"
timeout 400 python bench.py --config C3b --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_C3b.json 2> $O/bench_C3b.err
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv --log-file $O/launches_C3b_eager.csv python tools/profile_one.py --config C3b --eager --calls 2 > /dev/null 2>&1; python tools/launches.py $O/launches_C3b_eager.csv > $O/launches_C3b_eager.txt
timeout 600 ncu --set full --import-source on --clock-control none -k regex:detect_pairs --launch-skip 1 --launch-count 1 \
    -o $O/detect_C3b python tools/profile_one.py --config C3b --eager --calls 2 > $O/cap.log 2>&1; echo "cap rc=$?"
