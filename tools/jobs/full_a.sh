# full GPU suite + C2 detection A/B repeats + Cholesky at n = 16384
set -x
O=${1:-gpurun_out/full_a}
mkdir -p $O
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $O/pytest.txt 2>&1; echo "pytest rc=$?"
tail -5 $O/pytest.txt
b() { cfg=$1; name=$2; shift 2; env "$@" timeout 600 python bench.py --config $cfg --only --steps 30 --no-cpu-baseline > $O/bench_${cfg}_$name.json 2> $O/bench_${cfg}_$name.err; }
b C2 tma_1 AS_X=0
b C2 notma_1 AS_DET_TMA=0
b C2 tma_2 AS_X=0
b C2 notma_2 AS_DET_TMA=0
b C1 tma AS_X=0
b C5 tma AS_X=0
timeout 900 python tools/stage_time.py --config C3a --n 16384 --calls 3 > $O/chol16k.txt 2>&1
tail -5 $O/chol16k.txt
