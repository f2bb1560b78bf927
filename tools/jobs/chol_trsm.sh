# paired-panel Cholesky (K = 128 bulk update) A/B + parity; C3b triangular-solve timeline
set -x
O=${1:-gpurun_out/chol_trsm}
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "spd or chol or C3a or c3a or determin or config_full" > $O/pytest.txt 2>&1; echo "pytest rc=$?"
tail -4 $O/pytest.txt
b() { cfg=$1; name=$2; shift 2; env "$@" timeout 600 python bench.py --config $cfg --only --steps 20 --no-cpu-baseline > $O/bench_${cfg}_$name.json 2> $O/bench_${cfg}_$name.err; }
b C3a pairs AS_X=0
b C3a nopairs AS_CHOL_PAIRS=0
timeout 900 python tools/stage_time.py --config C3a --n 16384 --calls 3 > $O/chol16k_pairs.txt 2>&1
AS_CHOL_PAIRS=0 timeout 900 python tools/stage_time.py --config C3a --n 16384 --calls 3 > $O/chol16k_nopairs.txt 2>&1
tail -4 $O/chol16k_pairs.txt $O/chol16k_nopairs.txt
AS_USE_DEBUG_LIB=1 timeout 300 python tools/trsm_trace.py C3b 9 > $O/trsm_trace_C3b.txt 2>&1
cat $O/trsm_trace_C3b.txt
