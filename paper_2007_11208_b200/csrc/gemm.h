// gemm.h -- C -= op(A) op(B) launcher (gemm.cu).
#pragma once
#include <stdint.h>
#include <cuda_runtime.h>

namespace as {

struct GemmArgs {
    int64_t M, N, K;
    const void* A; int64_t lda; bool TA;
    const void* B; int64_t ldb; bool TB;
    void* C; int64_t ldc;
    bool lower_only;        // skip CTA tiles strictly above the diagonal (SYRK)
    const int* skip;        // device flag: kernel returns at once if *skip != 0
    bool one_per_sm;        // reserve shared memory so only one GEMM CTA fits per SM (room for a
                            // concurrently running cooperative panel kernel)
    unsigned long long* trace_min = nullptr;   // diagnostics: first CTA start / last CTA end
    unsigned long long* trace_max = nullptr;   // (%globaltimer, AS_LU_TRACE only)
};

void launch_gemm_minus(int dtype, const GemmArgs& g, cudaStream_t s);

// fp64 tensor-core (DMMA) throughput in TFLOP/s from a register-resident loop
double measure_fp64_peak(int num_sms, int iters, cudaStream_t s);

}  // namespace as
