# Round-1 final measurement job (r01g): bench lines, reference arm, launch lists, ncu captures
#   bench lines for every config, the reference arm, the eager ncu launch list of the default
#   bench command, and one ncu --set full capture per dominant kernel.
set -x
O=gpurun_out/r01g
mkdir -p $O
python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench default rc=$?"
for c in C1 C3a C3b C4 C5 C5f; do
  timeout 400 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; echo "$c rc=$?"
done
python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err; echo "ref rc=$?"
# launch list of the default bench command (eager: kernel nodes of conditional graphs are invisible to ncu)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C2_bench.csv \
  python bench.py --eager --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1; echo "launch list rc=$?"
# one full capture per dominant kernel
cap() {  # name, regex, config, skip
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$2 --launch-skip $4 --launch-count 1 \
    -o $O/$1 python tools/profile_one.py --config $3 --eager --calls 1 > $O/$1.log 2>&1; echo "cap $1 rc=$?"
}
cap band_spike_C2 band_spike_kernel C2 0
cap detect_C2 detect_pairs C2 0
cap detect_C3a detect_pairs C3a 0
cap detect_C3b detect_pairs C3b 0
cap panel_C5 lu_panel2 C5 10
cap potf2_C3a potf2_kernel C3a 10
cap trsm_C3b trsm_sf_kernel C3b 0
cap jacobi_C4 jacobi_block_sweep C4 2
python tools/gemm_bench.py > $O/gemm_bench.txt 2>&1
python tools/std_vs_adaptive.py --out $O/std_vs_adaptive.json > $O/std_vs_adaptive.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C3b_eager.csv python tools/profile_one.py --config C3b --eager --calls 1 > /dev/null 2>&1; python tools/launches.py $O/launches_C3b_eager.csv > $O/launches_C3b_eager.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C3a_eager.csv python tools/profile_one.py --config C3a --eager --calls 1 > /dev/null 2>&1; python tools/launches.py $O/launches_C3a_eager.csv > $O/launches_C3a_eager.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C1_eager.csv python tools/profile_one.py --config C1 --eager --calls 1 > /dev/null 2>&1; python tools/launches.py $O/launches_C1_eager.csv > $O/launches_C1_eager.txt
