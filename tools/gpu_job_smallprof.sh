set -x
O=gpurun_out/smallprof
mkdir -p $O
timeout 600 ncu --set full --import-source on --clock-control none -k regex:lu_small_kernel --launch-count 1 \
    -o $O/lu_small_C1 python tools/profile_one.py --config C1 --eager --calls 1 > $O/ncu.log 2>&1; echo "cap rc=$?"
