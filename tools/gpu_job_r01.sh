set -x
mkdir -p gpurun_out/r01
python bench.py > gpurun_out/r01/bench_default.json 2> gpurun_out/r01/bench_default.err; echo "bench default rc=$?"
for c in C1 C3a C3b C4 C5 C5f; do timeout 400 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r01/bench_$c.json 2> gpurun_out/r01/bench_$c.err; echo "$c rc=$?"; done
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r01/bench_reference.json 2> gpurun_out/r01/bench_reference.err; echo "ref rc=$?"
python tools/gemm_bench.py > gpurun_out/r01/gemm_bench.txt 2>&1
nvidia-smi -q > gpurun_out/r01/nvidia_smi.txt 2>&1
lscpu > gpurun_out/r01/lscpu.txt 2>&1
