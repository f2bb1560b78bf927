// trsm.cu -- blocked triangular solves op(T) X = B (Eq. 3).
//
// K5 (TRTRS), the L/U solves of GETRS and POTRS, and every
// M / M^T application of the rcond estimators run through two kernels:
//
//  trtri_blocks_kernel: inverts the kNB x kNB diagonal blocks of the stored
//      triangle (all blocks in parallel, one CTA each) -> Dinv.
//  trsm_sf_kernel:      synchronization-free blocked substitution.  CTA
//      (step s, rhs-tile r) takes a ticket in launch order, accumulates
//      B_b - sum_{j before b} op(T)_{bj} X_j as soon as each X_j is flagged
//      complete by the CTA that produced it, multiplies by Dinv_b and
//      publishes X_b.  Ticket order guarantees that every CTA waits only on
//      CTAs that are already resident, so there is no deadlock and the
//      dependency chain is n/kNB hops long.
//
// The stored triangle (upper/lower), transpose and unit diagonal are template
// parameters; "forward" order = (lower && !trans) || (upper && trans).
#include "internal.h"
#include "trsm.h"

namespace as {

constexpr int kTsThreads = 256;
constexpr int kTsR = 16;          // max RHS columns per CTA tile
constexpr int kLDT = kNB + 1;     // padded smem leading dimension

// ------------------------------------------------------------------ diagonal block inverse
// Dinv block b (kNB x kNB, column-major, ld kNB) = inverse of the b-th diagonal
// block of the stored triangle; padded with identity beyond n.
template <typename T, bool UPPER, bool UNIT>
__global__ void __launch_bounds__(kTsThreads) trtri_blocks_kernel(const T* __restrict__ A_, int64_t lda, int64_t n,
                                                                   T* __restrict__ Dinv, const DevState* st,
                                                                   int skip_if_singular, const DevArgs* args) {
    if (skip_if_singular && st->info != ~0ull) return;
    const T* A = A_ ? A_ : (const T*)args->A;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* Ts = (T*)smem_raw;          // kNB x kLDT
    T* Is = Ts + kNB * kLDT;       // kNB x kLDT
    const int b = blockIdx.x;
    const int64_t o = (int64_t)b * kNB;
    const int nb = (int)min<int64_t>(kNB, n - o);
    for (int e = threadIdx.x; e < kNB * kNB; e += blockDim.x) {
        const int r = e % kNB, c = e / kNB;
        T v = T(0);
        if (r < nb && c < nb) {
            const bool in_tri = UPPER ? (r <= c) : (r >= c);
            if (in_tri) v = A[(o + r) + (o + c) * lda];
            if (r == c && UNIT) v = T(1);
        } else if (r == c) {
            v = T(1);
        }
        Ts[r + c * kLDT] = v;
    }
    __syncthreads();
    // column c of the inverse solves T x = e_c; threads split columns x 4 row-phases
    // (simple and exact enough: one thread per column, sequential substitution)
    if (threadIdx.x < kNB) {
        const int c = threadIdx.x;
        if (!UPPER) {
            for (int r = 0; r < kNB; ++r) {
                T s = (r == c) ? T(1) : T(0);
                if (r > c) {
                    for (int k = c; k < r; ++k) s -= Ts[r + k * kLDT] * Is[k + c * kLDT];
                }
                Is[r + c * kLDT] = (r < c) ? T(0) : s / Ts[r + r * kLDT];
            }
        } else {
            for (int r = kNB - 1; r >= 0; --r) {
                T s = (r == c) ? T(1) : T(0);
                if (r < c) {
                    for (int k = r + 1; k <= c; ++k) s -= Ts[r + k * kLDT] * Is[k + c * kLDT];
                }
                Is[r + c * kLDT] = (r > c) ? T(0) : s / Ts[r + r * kLDT];
            }
        }
    }
    __syncthreads();
    T* D = Dinv + (int64_t)b * kNB * kNB;
    for (int e = threadIdx.x; e < kNB * kNB; e += blockDim.x) {
        const int r = e % kNB, c = e / kNB;
        D[r + c * kNB] = Is[r + c * kLDT];
    }
}

// ------------------------------------------------------------------ sync-free blocked solve
struct TsArgs {
    const void* A; int64_t lda;      // triangle (nullptr: read args->A)
    const void* Dinv;
    void* X; int64_t ldx;            // in/out (nullptr: args->X with ldx)
    int64_t n; int nrhs;
    unsigned* sync;                  // [0] = ticket, [1..] = flags (nblk * ntiles), zeroed per solve
    int slot;                        // estimator slot gate (-1: none)
    int skip_if_singular;
};

// acc[i][c] (partial over k-quarter q) for row i = tid % 64, q = tid / 64
template <typename T, bool TRANSB>
AS_DEV void block_product(const T* __restrict__ Ms, const T* __restrict__ Xs, T (&part)[kTsR], int R) {
    const int i = threadIdx.x % kNB, q = threadIdx.x / kNB;
#pragma unroll
    for (int c = 0; c < kTsR; ++c) part[c] = T(0);
#pragma unroll 4
    for (int kk = 0; kk < kNB / 4; ++kk) {
        const int k = q * (kNB / 4) + kk;
        const T m = TRANSB ? Ms[k + i * kLDT] : Ms[i + k * kLDT];
#pragma unroll
        for (int c = 0; c < kTsR; ++c)
            if (c < R) part[c] += m * Xs[k + c * kLDT];
    }
}

template <typename T, bool UPPER, bool TRANS>
__global__ void __launch_bounds__(kTsThreads) trsm_sf_kernel(TsArgs p, const DevArgs* args, const DevState* st) {
    if (p.slot >= 0 && ld_volatile_i32(&st->est_next) != p.slot) return;
    if (p.skip_if_singular && st->info != ~0ull) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* Ms = (T*)smem_raw;                       // kNB x kLDT: T block / Dinv block
    T* Xs = Ms + kNB * kLDT;                    // kNB x kLDT (R columns used): X_j tile
    T* Red = Xs + kNB * kLDT;                   // 4 x kNB x kTsR partials
    __shared__ unsigned s_ticket;

    const T* A = (const T*)(p.A ? p.A : args->A);
    T* X = (T*)(p.X ? p.X : args->X);
    const T* Dinv = (const T*)p.Dinv;
    const int64_t n = p.n;
    const int nblk = (int)((n + kNB - 1) / kNB);
    const int ntiles = (p.nrhs + kTsR - 1) / kTsR;
    constexpr bool FWD = (!UPPER && !TRANS) || (UPPER && TRANS);

    if (threadIdx.x == 0) s_ticket = atomicAdd(&p.sync[0], 1u);
    __syncthreads();
    const unsigned t = s_ticket;
    const int s = (int)(t / ntiles), rt = (int)(t % ntiles);
    const int b = FWD ? s : nblk - 1 - s;
    const int64_t ob = (int64_t)b * kNB;
    const int nbr = (int)min<int64_t>(kNB, n - ob);
    const int c0 = rt * kTsR;
    const int R = min(kTsR, p.nrhs - c0);
    const int i = threadIdx.x % kNB, q = threadIdx.x / kNB;

    // acc = B_b (only q == 0 threads keep it)
    T acc[kTsR];
#pragma unroll
    for (int c = 0; c < kTsR; ++c) acc[c] = (q == 0 && c < R && i < nbr) ? X[(ob + i) + (c0 + c) * p.ldx] : T(0);

    T part[kTsR];
    for (int sp = 0; sp < s; ++sp) {
        const int j = FWD ? sp : nblk - 1 - sp;
        const int64_t oj = (int64_t)j * kNB;
        const int nbj = (int)min<int64_t>(kNB, n - oj);
        // stage op(T)_{bj}: no-trans: A[b rows, j cols]; trans: A[j rows, b cols] (transposed in product)
        __syncthreads();
        if (!TRANS) {
            for (int e = threadIdx.x; e < kNB * kNB; e += blockDim.x) {
                const int r = e % kNB, c = e / kNB;
                Ms[r + c * kLDT] = (r < nbr && c < nbj) ? A[(ob + r) + (oj + c) * p.lda] : T(0);
            }
        } else {
            for (int e = threadIdx.x; e < kNB * kNB; e += blockDim.x) {
                const int r = e % kNB, c = e / kNB;   // r: row within A block (j rows), c: col (b cols)
                Ms[r + c * kLDT] = (r < nbj && c < nbr) ? A[(oj + r) + (ob + c) * p.lda] : T(0);
            }
        }
        // wait for X_j (tile rt)
        if (threadIdx.x == 0) {
            const unsigned* f = &p.sync[1 + j * ntiles + rt];
            while (ld_acquire(f) == 0u) { __nanosleep(20); }
        }
        __syncthreads();
        for (int e = threadIdx.x; e < kNB * kTsR; e += blockDim.x) {
            const int r = e % kNB, c = e / kNB;
            Xs[r + c * kLDT] = (r < nbj && c < R) ? __ldcg(&X[(oj + r) + (c0 + c) * p.ldx]) : T(0);
        }
        __syncthreads();
        if (!TRANS) block_product<T, false>(Ms, Xs, part, R);
        else block_product<T, true>(Ms, Xs, part, R);
#pragma unroll
        for (int c = 0; c < kTsR; ++c) Red[(q * kTsR + c) * kNB + i] = part[c];
        __syncthreads();
        if (q == 0) {
#pragma unroll
            for (int c = 0; c < kTsR; ++c)
                acc[c] -= (Red[(0 * kTsR + c) * kNB + i] + Red[(1 * kTsR + c) * kNB + i]) +
                          (Red[(2 * kTsR + c) * kNB + i] + Red[(3 * kTsR + c) * kNB + i]);
        }
    }
    // X_b = Dinv_b * acc  (trans: Dinv_b^T)
    __syncthreads();
    {
        const T* D = Dinv + (int64_t)b * kNB * kNB;
        for (int e = threadIdx.x; e < kNB * kNB; e += blockDim.x) {
            const int r = e % kNB, c = e / kNB;
            Ms[r + c * kLDT] = D[r + c * kNB];
        }
        if (q == 0) {
#pragma unroll
            for (int c = 0; c < kTsR; ++c) Xs[i + c * kLDT] = acc[c];
        }
    }
    __syncthreads();
    if (!TRANS) block_product<T, false>(Ms, Xs, part, R);
    else block_product<T, true>(Ms, Xs, part, R);
#pragma unroll
    for (int c = 0; c < kTsR; ++c) Red[(q * kTsR + c) * kNB + i] = part[c];
    __syncthreads();
    if (q == 0 && i < nbr) {
#pragma unroll
        for (int c = 0; c < kTsR; ++c)
            if (c < R)
                X[(ob + i) + (c0 + c) * p.ldx] = (Red[(0 * kTsR + c) * kNB + i] + Red[(1 * kTsR + c) * kNB + i]) +
                                                 (Red[(2 * kTsR + c) * kNB + i] + Red[(3 * kTsR + c) * kNB + i]);
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) st_release(&p.sync[1 + b * ntiles + rt], 1u);
}

// ------------------------------------------------------------------ launchers
int64_t trsm_sync_words(int64_t n, int nrhs) {
    const int64_t nblk = (n + kNB - 1) / kNB;
    const int64_t ntiles = (nrhs + kTsR - 1) / kTsR;
    return 1 + nblk * ntiles;
}

template <typename T>
static void trtri_dispatch(const T* A, int64_t lda, int64_t n, T* Dinv, bool upper, bool unit, const DevState* st,
                           bool skip, const DevArgs* args, cudaStream_t s) {
    const int nblk = (int)((n + kNB - 1) / kNB);
    const int smem = (int)(sizeof(T) * 2 * kNB * kLDT);
    auto go = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        kern<<<nblk, kTsThreads, smem, s>>>(A, lda, n, Dinv, st, skip, args);
    };
    if (upper) {
        if (unit) go(trtri_blocks_kernel<T, true, true>);
        else go(trtri_blocks_kernel<T, true, false>);
    } else {
        if (unit) go(trtri_blocks_kernel<T, false, true>);
        else go(trtri_blocks_kernel<T, false, false>);
    }
}

void launch_trtri_blocks(int dtype, const void* A, int64_t lda, int64_t n, void* Dinv, bool upper, bool unit,
                         const DevState* st, bool skip_if_singular, const DevArgs* args, cudaStream_t s) {
    if (dtype == AS_F64) trtri_dispatch<double>((const double*)A, lda, n, (double*)Dinv, upper, unit, st, skip_if_singular, args, s);
    else trtri_dispatch<float>((const float*)A, lda, n, (float*)Dinv, upper, unit, st, skip_if_singular, args, s);
}

// A == nullptr selects args->A (the caller's matrix); X == nullptr selects args->X.
template <typename T>
static void trsm_dispatch(const TsArgs& p, bool upper, bool trans, const DevArgs* args, const DevState* st,
                          cudaStream_t s) {
    const int nblk = (int)((p.n + kNB - 1) / kNB);
    const int ntiles = (p.nrhs + kTsR - 1) / kTsR;
    const size_t smem = sizeof(T) * (2 * kNB * kLDT + 4 * kNB * kTsR);
    auto go = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<nblk * ntiles, kTsThreads, smem, s>>>(p, args, st);
    };
    if (upper) {
        if (trans) go(trsm_sf_kernel<T, true, true>);
        else go(trsm_sf_kernel<T, true, false>);
    } else {
        if (trans) go(trsm_sf_kernel<T, false, true>);
        else go(trsm_sf_kernel<T, false, false>);
    }
}

void launch_trsm(int dtype, const void* A, int64_t lda, const void* Dinv, bool upper, bool trans, void* X,
                 int64_t ldx, int64_t n, int nrhs, unsigned* sync, int slot, bool skip_if_singular,
                 const DevArgs* args, const DevState* st, cudaStream_t s) {
    TsArgs p{A, lda, Dinv, X, ldx, n, nrhs, sync, slot, skip_if_singular ? 1 : 0};
    if (n <= 0 || nrhs <= 0) return;
    if (dtype == AS_F64) trsm_dispatch<double>(p, upper, trans, args, st, s);
    else trsm_dispatch<float>(p, upper, trans, args, st, s);
}

}  // namespace as
