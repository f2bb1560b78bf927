import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2007_11208_b200 as AS  # noqa: E402
K = int(sys.argv[1]) if len(sys.argv) > 1 else 64
print(AS.bench_gemm(16384, 16384, K, AS.AS_F64, False, 1))
