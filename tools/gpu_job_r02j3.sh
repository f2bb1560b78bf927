# r02j3: ncu --set full captures of the dominant kernels; summarised on the box (tools/ncu_traffic.py,
# raw-page CSV) and the reports kept only when small (gpurun copies back <= 64 MiB)
set -x
O=gpurun_out/r02j3
mkdir -p $O
NF="ncu --set full --import-source on --clock-control none"
cap() {   # name, kernel regex, skip, command...
  local name=$1 rx=$2 skip=$3; shift 3
  timeout 900 $NF -k regex:$rx --launch-skip $skip --launch-count 1 -o $O/$name "$@" > $O/$name.log 2>&1
  python tools/ncu_traffic.py $O/$name.ncu-rep > $O/$name.json 2>> $O/$name.log
  ncu -i $O/$name.ncu-rep --page details --csv > $O/$name.details.csv 2>/dev/null
  gzip -f $O/$name.details.csv
  local sz=$(stat -c %s $O/$name.ncu-rep 2>/dev/null || echo 0)
  if [ "$sz" -gt 4000000 ]; then rm -f $O/$name.ncu-rep; fi
}
cap gemm_C5 gemm_dmma 30 python tools/profile_one.py --config C5 --eager --calls 1
cap panel_lf_C5 lu_panel_lf 2 python tools/profile_one.py --config C5 --eager --calls 1
cap panel_coop_C5 lu_panel2 40 python tools/profile_one.py --config C5 --eager --calls 1
cap band_spike_C2 band_spike_kernel 0 python tools/profile_one.py --config C2 --eager --calls 1
cap detect_C2 detect_pairs_v3 0 python tools/profile_one.py --config C2 --eager --calls 1
cap detect_C3a detect_pairs_v3 0 python tools/profile_one.py --config C3a --eager --calls 1
cap detect_C3b detect_pairs_v3 0 python tools/profile_one.py --config C3b --eager --calls 1
cap trsm_C3b trsm_sf_kernel 0 python tools/profile_one.py --config C3b --eager --calls 1
cap lu_small_C1 lu_small_kernel 0 python tools/profile_one.py --config C1 --eager --calls 1
cap small_batched small_solve_kernel 0 python tools/batched_one.py 1000
cap band_chain_n1000 band_chain_kernel 0 python tools/profile_kind.py banded 1000
cap jacobi_C4 jacobi 0 python tools/profile_one.py --config C4 --eager --calls 1
cap potf2_C3a potf2 10 python tools/profile_one.py --config C3a --eager --calls 1
cap sgemm_C5f sgemm 30 python tools/profile_one.py --config C5f --eager --calls 1
du -sh $O
