set -x
O=${1:-gpurun_out/fuse_check}
mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $O/pytest.txt 2>&1; echo "pytest rc=$?"
tail -4 $O/pytest.txt
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?"
b() { cfg=$1; name=$2; st=$3; shift 3; env "$@" timeout 600 python bench.py --config $cfg --only --steps $st --no-cpu-baseline > $O/bench_${cfg}_$name.json 2> $O/bench_${cfg}_$name.err; }
for c in C2 C3a C3b; do
b $c fused 30 AS_X=0
b $c unfused 30 AS_DET_FUSE_DISPATCH=0
done
b C5 fused 5 AS_X=0
