# r02j2: final-tree evidence (small outputs): full GPU suite, smoke, default bench line, reference
# arm, eager launch lists per config, standard-vs-adaptive
set -x
O=gpurun_out/r02j2
mkdir -p $O
nproc > $O/host.txt
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?"
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?"
timeout 1500 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err; echo "ref rc=$?"
for c in C1 C2 C3a C3b C4 C5 C5f; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_${c}_eager.csv \
      python tools/profile_one.py --config $c --eager --calls 1 > /dev/null 2>&1
  python tools/launches.py $O/launches_${c}_eager.csv > $O/launches_${c}_eager.txt 2>&1
  gzip -f $O/launches_${c}_eager.csv
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_batched.csv python tools/batched_one.py > /dev/null 2>&1
python tools/launches.py $O/launches_batched.csv > $O/launches_batched.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_band5_n1000.csv python tools/profile_kind.py banded 1000 > /dev/null 2>&1
python tools/launches.py $O/launches_band5_n1000.csv > $O/launches_band5_n1000.txt 2>&1
python tools/std_vs_adaptive.py --out $O/std_vs_adaptive.json > $O/std_vs_adaptive.txt 2>&1
du -sh $O
