# r02s: compute-sanitizer (memcheck, racecheck, synccheck, initcheck) on small solves of every path
# (tools/sanitize_cases.py, eager mode: the kernels one by one)
set -x
O=gpurun_out/r02s
mkdir -p $O
python tools/sanitize_cases.py --eager > $O/plain.txt 2>&1; echo "plain rc=$?"
for t in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 50 python tools/sanitize_cases.py --eager > $O/$t.txt 2>&1
  echo "$t rc=$?"
done
