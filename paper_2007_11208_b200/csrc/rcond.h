// rcond.h -- estimator launcher and band-solve hooks.
#pragma once
#include "internal.h"
#include "trsm.h"

namespace as {

enum { KIND_LU = 0, KIND_BAND = 1, KIND_TRI = 2, KIND_CHOL = 3 };

void launch_estimator(const Work& w, int kind, bool upper, SyncAlloc& sa, cudaStream_t s, const void* altres = nullptr);

// band.cu
void launch_band_norm(const Work& w, cudaStream_t s);              // anorm of the band
void launch_band_factor(const Work& w, cudaStream_t s);            // pack + gbtrf (sequential path)
void launch_band_apply(const Work& w, bool trans, int slot, cudaStream_t s);  // estimator M / M^T on xe
void launch_band_solve(const Work& w, cudaStream_t s);             // X = A^{-1} B (gbtrs)

// band_spike.cu: partitioned path for strictly diagonally dominant band matrices
void launch_band_dominance(const Work& w, cudaGraphConditionalHandle h, cudaStream_t s);  // sets band_use_spike
void launch_band_spike(const Work& w, int cls, cudaStream_t s);    // K class 2^cls: factor + estimate + X in one kernel
int64_t spike_scratch_elems(int64_t n, int num_sms);

}  // namespace as
