# Evidence job (run on the GPU box through gpurun; results are copied into profiles/<round>/). Part 1: full GPU suite, smoke, default bench line (every config + batched),
# reference arm, eager launch lists per config, standard-vs-adaptive.  Part 2: ncu --set full captures
# of the dominant kernels, summarised on the box (tools/ncu_traffic.py; gpurun copies back <= 64 MiB).
set -x
O=${1:-gpurun_out/evidence}
mkdir -p $O
nproc > $O/host.txt
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,clocks.max.mem --format=csv > $O/gpu.txt 2>&1
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
python tools/launches.py $O/launches_batched.csv > $O/launches_batched.txt 2>&1; gzip -f $O/launches_batched.csv
python tools/std_vs_adaptive.py --out $O/std_vs_adaptive.json > $O/std_vs_adaptive.txt 2>&1
timeout 900 python tools/stage_time.py --config C3a --n 16384 --calls 3 > $O/chol16k.txt 2>&1
AS_USE_DEBUG_LIB=1 timeout 600 python tools/lu_trace.py C5 > $O/lu_trace_C5.txt 2>&1
timeout 600 python tools/gemm_bench.py > $O/gemm_bench.txt 2>&1
NF="ncu --set full --import-source on --clock-control none"
cap() {   # name, kernel regex, skip, command...
  local name=$1 rx=$2 skip=$3; shift 3
  timeout 900 $NF -k regex:$rx --launch-skip $skip --launch-count 1 -o $O/$name "$@" > $O/$name.log 2>&1
  python tools/ncu_traffic.py $O/$name.ncu-rep > $O/$name.json 2>> $O/$name.log
  ncu -i $O/$name.ncu-rep --page details --csv > $O/$name.details.csv 2>/dev/null
  gzip -f $O/$name.details.csv
  local sz=$(stat -c %s $O/$name.ncu-rep 2>/dev/null || echo 0)
  if [ "$sz" -gt 3000000 ]; then rm -f $O/$name.ncu-rep; fi
}
# the bulk trailing update of C5 at its dominant shape (bench.py's dominant_kernel), run alone
cap gemm_C5 gemm_dmma2 2 python -c "import paper_2007_11208_b200 as AS; print(AS.bench_gemm(12288, 12288, 128, AS.AS_F64, False, 3))"
cap swap_u12v3_C5 swap_u12v3 40 python tools/profile_one.py --config C5 --eager --calls 1
cap panel_coop_C5 lu_panel2 40 python tools/profile_one.py --config C5 --eager --calls 1
cap panel_lf_C5 lu_panel_lf 2 python tools/profile_one.py --config C5 --eager --calls 1
cap band_spike_C2 band_spike_kernel 0 python tools/profile_one.py --config C2 --eager --calls 1
cap detect_C2 detect_pairs_tma 0 python tools/profile_one.py --config C2 --eager --calls 1
cap detect_C3a detect_pairs_tma 0 python tools/profile_one.py --config C3a --eager --calls 1
cap detect_C3b detect_pairs_tma 0 python tools/profile_one.py --config C3b --eager --calls 1
cap trsm_C3b trsm_sf_kernel 0 python tools/profile_one.py --config C3b --eager --calls 1
cap lu_small_C1 lu_small_kernel 0 python tools/profile_one.py --config C1 --eager --calls 1
cap est_small_C1 est_small_kernel 0 python tools/profile_one.py --config C1 --eager --calls 1
cap small_batched small_solve_kernel 0 python tools/batched_one.py 1000
cap jacobi_C4 jacobi 0 python tools/profile_one.py --config C4 --eager --calls 1
cap potf2_C3a potf2 10 python tools/profile_one.py --config C3a --eager --calls 1
cap sgemm_C5f sgemm 2 python -c "import paper_2007_11208_b200 as AS; print(AS.bench_gemm(12288, 12288, 128, AS.AS_F32, False, 3))"
du -sh $O
cuobjdump -sass paper_2007_11208_b200/libadaptsolve.so | grep -c "UTMALDG\|UBLKCP" > $O/sass_tma_count.txt
# side measurements (same box, same build): knobs around the defaults
b() { cfg=$1; name=$2; shift 2; env "$@" timeout 600 python bench.py --config $cfg --only --steps 20 --no-cpu-baseline > $O/ab_${cfg}_$name.json 2> $O/ab_${cfg}_$name.err; }
b C3b default AS_X=0
b C3b rt16 AS_TS_RT=16
b C3b notma AS_DET_TMA=0
b C3a notma AS_DET_TMA=0
b C2 notma AS_DET_TMA=0
b C2 nohint AS_DET_TMA_HINT=0
