set -x
O=gpurun_out/det2
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.txt 2>&1; echo "pytest rc=$?"
for c in C1 C3a C3b; do timeout 400 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; done
python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:detect_pairs --launch-skip 1 --launch-count 1 \
    -o $O/detect_C3b python tools/profile_one.py --config C3b --eager --calls 2 > $O/cap.log 2>&1; echo "cap rc=$?"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C3b_eager.csv python tools/profile_one.py --config C3b --eager --calls 1 > /dev/null 2>&1; python tools/launches.py $O/launches_C3b_eager.csv > $O/launches_C3b_eager.txt
