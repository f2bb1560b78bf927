# ncu launch lists (eager mode: same kernels, no graph) of one solve per config
O=gpurun_out/launch
mkdir -p $O
for c in C1 C2 C3a C3b C4; do
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/$c.csv \
    python tools/profile_one.py --config $c --eager --calls 2 > $O/$c.log 2>&1; echo "$c rc=$?"
  python tools/launches.py $O/$c.csv > $O/$c.txt 2>&1
done
