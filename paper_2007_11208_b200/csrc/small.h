// small.h -- batched small systems: one thread block per system (small.cu).
#pragma once
#include "internal.h"

namespace as {
constexpr int kSmallN = 128;     // largest n of the one-block solver (matrix in shared memory)
constexpr int kSmallRhs = 16;    // largest nrhs of the one-block solver (fallback keeps V^T Q^T B)

struct SmallArgs {
    const void* A; int64_t lda, sA;      // system b: A + b * sA (elements), leading dimension lda
    const void* B; int64_t ldb, sB;
    void* X; int64_t ldx, sX;
    int n, nrhs;
    int64_t batch;
    uint32_t opts;
    int force;                           // forced method (AS_OPT_FORCE_METHOD)
    double thr, cut;                     // rcond threshold, least-squares cutoff
    int max_sweeps;
    as_report* rep;                      // device, one per system (nullable)
    int32_t* ret;                        // device, one per system (nullable)
    void* sigma; int64_t sS;             // device singular values (fallback), nullable
};

size_t small_smem_bytes(int dtype);
int launch_small_batched(int dtype, const SmallArgs& a, cudaStream_t s);
}  // namespace as
