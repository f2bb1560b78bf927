// trsm.h -- triangular-solve launchers (trsm.cu) and sync-arena bookkeeping.
#pragma once
#include "internal.h"

namespace as {

// words of zeroed sync memory one trsm launch needs
int64_t trsm_sync_words(int64_t n, int nrhs);
// 64-bit words of epoch-tagged exchange buffer one trsm launch needs (never zeroed per solve)
int64_t trsm_ll_words(int64_t n, int nrhs);
struct SyncAlloc;

// A == nullptr -> args->A
void launch_trtri_blocks(int dtype, const void* A, int64_t lda, int64_t n, void* Dinv, bool upper, bool unit,
                         const DevState* st, bool skip_if_singular, const DevArgs* args, cudaStream_t s);

// Solve op(T) X = X in place.  A == nullptr -> args->A (with lda); X == nullptr -> args->X.
// slot >= 0: run only if st->est_next == slot (estimator gating).
void launch_trsm(int dtype, const void* A, int64_t lda, const void* Dinv, bool upper, bool trans, void* X,
                 int64_t ldx, int64_t n, int nrhs, SyncAlloc& sa, int slot, bool skip_if_singular,
                 const DevArgs* args, const DevState* st, cudaStream_t s);

// bump allocator over the plan's zeroed sync arena
// plus a bump allocator over the plan's epoch-tagged exchange arena (zeroed once at plan creation;
// the method branches of the graph are exclusive, so each branch may restart it: reset_ll)
struct SyncAlloc {
    unsigned* base = nullptr;
    int64_t cap = 0, used = 0;
    unsigned long long* llbase = nullptr;
    int64_t llcap = 0, llused = 0, llpeak = 0;
    unsigned* take(int64_t words) {
        if (used + words > cap) return nullptr;
        unsigned* p = base + used;
        used += words;
        return p;
    }
    unsigned long long* take_ll(int64_t words) {
        unsigned long long* p = llbase ? llbase + llused : nullptr;
        llused += words;
        if (llused > llpeak) llpeak = llused;
        return llused <= llcap ? p : nullptr;
    }
    void reset_ll() { llused = 0; }
};

}  // namespace as
