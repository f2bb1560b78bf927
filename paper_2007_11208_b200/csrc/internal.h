// internal.h -- host-side declarations shared by the libadaptsolve sources.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace as {

// Per-call pointers, written on device by set_args_kernel (first graph node).
struct DevArgs {
    const void* A;
    const void* B;
    void* X;
    void* sigma;        // optional fallback singular values (device)
    as_report* rep_dev; // optional device report
    as_report* rep_host;// optional mapped pinned host report
    int32_t* ret_dev;   // optional device return code (batched calls)
    // 2-D TMA tensor map of A (64 x 64 tiles; a CUtensorMap, encoded per call on the host) for the
    // detection pass's tile pipeline; tma_ok = 0: A or lda not 16-byte aligned, or no driver entry point
    int32_t tma_ok;
    alignas(64) unsigned long long tmapA[16];
};

// Workspace layout of a plan (all device pointers; see api.cu).
struct Work {
    int dtype;           // AS_F64 / AS_F32
    int64_t n, nrhs, lda, ldb;
    int64_t ldw;         // leading dimension of W (n rounded up to a multiple of 4)
    DevState* st;
    DevArgs* args;
    void* W;             // n x n (ld n): LU / Cholesky factors, band storage, QR/Jacobi matrix
    void* diag;          // n (detection: contiguous copy of diag(A))
    void* xe;            // n (estimator vector)
    void* Dinv0;         // n x kNB inverted diagonal blocks (first triangular factor)
    void* Dinv1;         // n x kNB (second triangular factor)
    void* vec;           // scratch n x max(nrhs,2) (QR c = Q^T b etc.)
    void* yv;            // n x nrhs (fallback V^T c)
    void* zx;            // n x (nrhs + 2): triangular path's fused solve [B | e/n | alt] (ld n)
    int64_t* ipiv;       // n
    int64_t* perm;       // n (LU row permutation)
    unsigned* flags_ts;  // sync-free triangular-solve tickets/flags: (n/kNB+1) * tiles + 64
    int64_t flags_ts_len;
    unsigned long long* ll;   // triangular-solve exchange words (epoch-tagged, zeroed once)
    int64_t ll_len;
    unsigned* bars;      // cooperative-kernel barrier counters (zeroed per solve)
    int64_t bars_len;
    void* cand;          // LU panel candidates
    void* lfbuf;         // leaf LU panel: counters, exchange slots, candidate rows, row-move staging
    void* linv;          // LU: full 128 x 128 inverse of each block's unit-lower L11 (n/128 blocks)
    void* swplan;        // LU: per block, the composed row interchanges (lu.cu SwapPlan)
    int det_tma;         // plan-level: launch the TMA instantiation of the detection pair pass as well
    int num_sms;
};

// launchers (each enqueues on `s`; used while capturing the plan's graph)
void launch_state_init(const Work& w, cudaStream_t s, uint32_t opts, int force_method, double thr, double cut,
                       int max_sweeps);
// 1: the plan also launches the TMA tile pipeline of the detection pair pass (detect.cu)
int detect_tma_plan(int dtype, int64_t n, int64_t lda);
void launch_detect(const Work& w, cudaStream_t s, bool fullscan, bool check_finite = false);
void launch_dispatch(const Work& w, cudaStream_t s, cudaGraphConditionalHandle h_method);
void launch_copy_b_to_x(const Work& w, cudaStream_t s);   // band.cu
void launch_band_chain(const Work& w, cudaStream_t s);    // band_chain.cu: kl, ku <= 3 (factor + rcond + X)

}  // namespace as
