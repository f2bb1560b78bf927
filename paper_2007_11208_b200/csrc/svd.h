// svd.h -- fallback launchers (svd.cu).
#pragma once
#include "internal.h"

namespace as {
void launch_svd_pre(const Work& w, cudaStream_t s);                                 // W = A, QR, M = R^T, Y = Q^T B
void launch_svd_sweep(const Work& w, cudaGraphConditionalHandle h, cudaStream_t s); // one sweep + WHILE condition
void launch_svd_post(const Work& w, cudaStream_t s);                                // sigma, rank, X
}  // namespace as
