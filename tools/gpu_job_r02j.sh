# r02j: final-tree evidence: full GPU suite, smoke, default bench line (every config + batched),
# reference arm, eager launch lists per config, ncu --set full captures of the dominant kernels
set -x
O=gpurun_out/r02j
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
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_batched.csv python tools/batched_one.py > /dev/null 2>&1
python tools/launches.py $O/launches_batched.csv > $O/launches_batched.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_band5_n1000.csv python tools/profile_kind.py banded 1000 > /dev/null 2>&1
python tools/launches.py $O/launches_band5_n1000.csv > $O/launches_band5_n1000.txt 2>&1
NF="ncu --set full --import-source on --clock-control none"
timeout 900 $NF -k regex:gemm_dmma2 --launch-skip 30 --launch-count 1 -o $O/gemm_C5 python tools/profile_one.py --config C5 --eager --calls 1 > $O/ncu_gemm.log 2>&1
timeout 900 $NF -k regex:lu_panel_lf --launch-skip 2 --launch-count 1 -o $O/panel_lf_C5 python tools/profile_one.py --config C5 --eager --calls 1 > $O/ncu_panel.log 2>&1
timeout 600 $NF -k regex:band_spike_kernel --launch-count 1 -o $O/band_spike_C2 python tools/profile_one.py --config C2 --eager --calls 1 > $O/ncu_spike.log 2>&1
timeout 600 $NF -k regex:detect_pairs_v3 --launch-count 1 -o $O/detect_C2 python tools/profile_one.py --config C2 --eager --calls 1 > $O/ncu_det.log 2>&1
timeout 600 $NF -k regex:trsm_sf_kernel --launch-count 1 -o $O/trsm_C3b python tools/profile_one.py --config C3b --eager --calls 1 > $O/ncu_trsm.log 2>&1
timeout 600 $NF -k regex:lu_small_kernel --launch-count 1 -o $O/lu_small_C1 python tools/profile_one.py --config C1 --eager --calls 1 > $O/ncu_lusmall.log 2>&1
timeout 600 $NF -k regex:small_solve_kernel --launch-count 1 -o $O/small_batched python tools/batched_one.py 1000 > $O/ncu_small.log 2>&1
timeout 600 $NF -k regex:band_chain_kernel --launch-count 1 -o $O/band_chain_n1000 python tools/profile_kind.py banded 1000 > $O/ncu_chain.log 2>&1
timeout 900 $NF -k regex:jacobi --launch-count 1 -o $O/jacobi_C4 python tools/profile_one.py --config C4 --eager --calls 1 > $O/ncu_jacobi.log 2>&1
timeout 900 $NF -k regex:potf2 --launch-skip 10 --launch-count 1 -o $O/potf2_C3a python tools/profile_one.py --config C3a --eager --calls 1 > $O/ncu_potf2.log 2>&1
timeout 900 $NF -k regex:sgemm --launch-skip 30 --launch-count 1 -o $O/sgemm_C5f python tools/profile_one.py --config C5f --eager --calls 1 > $O/ncu_sgemm.log 2>&1
python tools/std_vs_adaptive.py --out $O/std_vs_adaptive.json > $O/std_vs_adaptive.txt 2>&1
