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
template <typename T, bool TRANSB, int RT>
AS_DEV void block_product(const T* __restrict__ Ms, const T* __restrict__ Xs, T (&part)[RT], int R) {
    const int i = threadIdx.x % kNB, q = threadIdx.x / kNB;
#pragma unroll
    for (int c = 0; c < RT; ++c) part[c] = T(0);
#pragma unroll 4
    for (int kk = 0; kk < kNB / 4; ++kk) {
        const int k = q * (kNB / 4) + kk;
        const T m = TRANSB ? Ms[k + i * kLDT] : Ms[i + k * kLDT];
#pragma unroll
        for (int c = 0; c < RT; ++c)
            if (c < R) part[c] += m * Xs[k + c * kLDT];
    }
}

template <typename T>
AS_DEV void cp_async_elem(T* smem, const T* gmem, bool ok) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    if (sizeof(T) == 8)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(sa), "l"(gmem), "r"(ok ? 8 : 0) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(sa), "l"(gmem), "r"(ok ? 4 : 0) : "memory");
}

template <typename T, bool UPPER, bool TRANS, int RT>
__global__ void __launch_bounds__(kTsThreads) trsm_sf_kernel(TsArgs p, const DevArgs* args, const DevState* st) {
    if (p.slot >= 0 && ld_volatile_i32(&st->est_next) != p.slot) return;
    if (p.skip_if_singular && st->info != ~0ull) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* Mb0 = (T*)smem_raw;                      // kNB x kLDT: T block (double buffered: Mb0, Mb1)
    T* Mb1 = Mb0 + kNB * kLDT;
    T* Xs = Mb1 + kNB * kLDT;                   // kNB x kLDT (R columns used): X_j tile
    T* Red = Xs + kNB * kLDT;                   // 4 x kNB x RT partials
    T* Ds = Red + 4 * kNB * RT;                 // kNB x kLDT: Dinv_b (prefetched off the critical path)
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
    const int R = min(RT, p.nrhs - c0);
    const int i = threadIdx.x % kNB, q = threadIdx.x / kNB;

    // async staging of op(T)_{b j} (no-trans: A[b rows, j cols]; trans: A[j rows, b cols])
    auto stage = [&](T* dst, int sp) {
        const int j = FWD ? sp : nblk - 1 - sp;
        const int64_t oj = (int64_t)j * kNB;
        const int nbj = (int)min<int64_t>(kNB, n - oj);
        for (int e = threadIdx.x; e < kNB * kNB; e += blockDim.x) {
            const int r = e % kNB, c = e / kNB;
            const bool ok = TRANS ? (r < nbj && c < nbr) : (r < nbr && c < nbj);
            const T* src = !ok ? A : TRANS ? A + (oj + r) + (ob + c) * p.lda : A + (ob + r) + (oj + c) * p.lda;
            cp_async_elem(dst + r + c * kLDT, src, ok);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    if (s > 0) stage(Mb0, 0);
    {   // Dinv_b prefetch
        const T* D = Dinv + (int64_t)b * kNB * kNB;
        for (int e = threadIdx.x; e < kNB * kNB; e += blockDim.x) Ds[(e % kNB) + (e / kNB) * kLDT] = D[e];
    }
    // acc = B_b (only q == 0 threads keep it)
    T acc[RT];
#pragma unroll
    for (int c = 0; c < RT; ++c) acc[c] = (q == 0 && c < R && i < nbr) ? X[(ob + i) + (c0 + c) * p.ldx] : T(0);

    T part[RT];
    for (int sp = 0; sp < s; ++sp) {
        const int j = FWD ? sp : nblk - 1 - sp;
        const int64_t oj = (int64_t)j * kNB;
        const int nbj = (int)min<int64_t>(kNB, n - oj);
        T* Ms = (sp & 1) ? Mb1 : Mb0;
        if (sp + 1 < s) stage((sp & 1) ? Mb0 : Mb1, sp + 1);
        else asm volatile("cp.async.commit_group;" ::: "memory");
        // wait for X_j (tile rt)
        if (threadIdx.x == 0) {
            const unsigned* f = &p.sync[1 + j * ntiles + rt];
            while (ld_acquire(f) == 0u) { __nanosleep(20); }   // (relaxed poll + fence measured slower here)
        }
        asm volatile("cp.async.wait_group 1;" ::: "memory");
        __syncthreads();
        for (int e = threadIdx.x; e < kNB * RT; e += blockDim.x) {
            const int r = e % kNB, c = e / kNB;
            Xs[r + c * kLDT] = (r < nbj && c < R) ? __ldcg(&X[(oj + r) + (c0 + c) * p.ldx]) : T(0);
        }
        __syncthreads();
        if (!TRANS) block_product<T, false, RT>(Ms, Xs, part, R);
        else block_product<T, true, RT>(Ms, Xs, part, R);
#pragma unroll
        for (int c = 0; c < RT; ++c) Red[(q * RT + c) * kNB + i] = part[c];
        __syncthreads();
        if (q == 0) {
#pragma unroll
            for (int c = 0; c < RT; ++c)
                acc[c] -= (Red[(0 * RT + c) * kNB + i] + Red[(1 * RT + c) * kNB + i]) +
                          (Red[(2 * RT + c) * kNB + i] + Red[(3 * RT + c) * kNB + i]);
        }
    }
    // X_b = Dinv_b * acc  (trans: Dinv_b^T)
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    if (q == 0) {
#pragma unroll
        for (int c = 0; c < RT; ++c) Xs[i + c * kLDT] = acc[c];
    }
    __syncthreads();
    if (!TRANS) block_product<T, false, RT>(Ds, Xs, part, R);
    else block_product<T, true, RT>(Ds, Xs, part, R);
#pragma unroll
    for (int c = 0; c < RT; ++c) Red[(q * RT + c) * kNB + i] = part[c];
    __syncthreads();
    if (q == 0 && i < nbr) {
#pragma unroll
        for (int c = 0; c < RT; ++c)
            if (c < R)
                X[(ob + i) + (c0 + c) * p.ldx] = (Red[(0 * RT + c) * kNB + i] + Red[(1 * RT + c) * kNB + i]) +
                                                 (Red[(2 * RT + c) * kNB + i] + Red[(3 * RT + c) * kNB + i]);
    }
    __syncthreads();   // release is cumulative over the CTA's X stores ordered by this barrier
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
    auto go = [&](auto kern, int rt) {
        const size_t smem = sizeof(T) * (4 * kNB * kLDT + 4 * kNB * rt);
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<nblk * ntiles, kTsThreads, smem, s>>>(p, args, st);
    };
    auto by_r = [&](auto k1, auto k4, auto k16) {
        if (p.nrhs == 1) go(k1, 1);
        else if (p.nrhs <= 4) go(k4, 4);
        else go(k16, kTsR);
    };
    if (upper) {
        if (trans) by_r(trsm_sf_kernel<T, true, true, 1>, trsm_sf_kernel<T, true, true, 4>, trsm_sf_kernel<T, true, true, kTsR>);
        else by_r(trsm_sf_kernel<T, true, false, 1>, trsm_sf_kernel<T, true, false, 4>, trsm_sf_kernel<T, true, false, kTsR>);
    } else {
        if (trans) by_r(trsm_sf_kernel<T, false, true, 1>, trsm_sf_kernel<T, false, true, 4>, trsm_sf_kernel<T, false, true, kTsR>);
        else by_r(trsm_sf_kernel<T, false, false, 1>, trsm_sf_kernel<T, false, false, 4>, trsm_sf_kernel<T, false, false, kTsR>);
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
