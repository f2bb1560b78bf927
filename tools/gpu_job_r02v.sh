# r02v: two-panel (K = 256) LU schedule, opt-in AS_LU_SCHED=2
set -x
O=gpurun_out/r02v
mkdir -p $O
AS_LU_SCHED=2 timeout 1500 python -m pytest tests/test_gpu_r02.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x -k "(lu or LU or c5 or C5 or debug_factor or determin) and not narrow" > $O/pytest_sched2.txt 2>&1; echo "rc=$?"
b() { cfg=$1; name=$2; shift 2; env "$@" timeout 600 python bench.py --config $cfg --only --steps 5 --no-cpu-baseline > $O/bench_${cfg}_$name.json 2> $O/bench_${cfg}_$name.err; }
b C5 a AS_X=0
b C5 sched2 AS_LU_SCHED=2
b C5 sched2_lf99999 AS_LU_SCHED=2 AS_LU_LF_MIN_M=99999
b C5 sched2_lf10240 AS_LU_SCHED=2 AS_LU_LF_MIN_M=10240
b C5 b AS_X=0
b C5f a AS_X=0
b C5f sched2 AS_LU_SCHED=2
AS_LU_SCHED=2 AS_USE_DEBUG_LIB=1 timeout 600 python tools/lu_trace.py C5 > $O/lu_trace_C5_sched2.txt 2>&1
