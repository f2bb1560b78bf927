// factor.h -- LU / Cholesky launchers (factor.cu).
#pragma once
#include "internal.h"
#include "trsm.h"

namespace as {
void launch_copy_norm(const Work& w, bool with_perm, cudaStream_t s); // W = A, anorm (+ perm = id)
double lu_debug_panel_time(int dtype, int kind, void* W, int64_t ldw, int64_t n, int64_t k0, int nbp, const void* Wsrc,
                           int iters, int dbg);
double chol_debug_panel_time(int dtype, int kind, void* W, int64_t ldw, int64_t n, int64_t k0, int nbp, const void* Wsrc,
                             int iters, int dbg);
unsigned long long* debug_trace_buf(int which);   // lu.cu diagnostics (AS_LU_TRACE)
int lu_trace_copy(unsigned long long* out_min, unsigned long long* out_max, int cap);  // lu.cu diagnostics
size_t lu_cand_bytes();                        // Work::cand size (lu.cu)
size_t lu_swplan_bytes(int64_t n);             // Work::swplan size (lu.cu)
size_t lu_lfbuf_bytes(int64_t n, int dtype);   // Work::lfbuf size (lu.cu)
void launch_lu_factor(const Work& w, cudaStream_t s);                 // lu.cu: W = L\U, ipiv, perm, Dinv0/1, anorm
void launch_chol_factor(const Work& w, cudaStream_t s);               // W = L (lower), anorm, chol_failed
void launch_chol_check(const Work& w, cudaGraphConditionalHandle h, cudaStream_t s);
void launch_chol_tri_prep(const Work& w, cudaStream_t s);             // Dinv0 of L
}  // namespace as
