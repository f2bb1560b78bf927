# ncu --set full of the detection kernel on C3a and C3b (run under gpurun from the repo root)
O=gpurun_out/det; mkdir -p $O
for c in C3a C3b; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:detect_pairs --launch-count 1 \
    -o $O/detect_$c python tools/profile_one.py --config $c --eager --calls 1 > $O/detect_$c.log 2>&1; echo "cap $c rc=$?"
done
