// factor.cu -- K7 blocked LU with partial pivoting (xGETRF / xGETRS,
// P:505-533, Eq. 4) and K6 blocked Cholesky (xPOTRF / xPOTRS).
//
// LU, right-looking, panel width kNB:
//   copy A -> W (+ column 1-norms for the estimator, + perm = identity)
//   per panel k0:
//     panel_kernel   cooperative: rows of the panel split over P CTAs and
//                    held in shared memory; per column one grid-wide exchange
//                    of (|max|, row) candidates + pivot row, first-max
//                    tie-break (Z15), swap, scale, in-panel rank-1 update
//     laswp_kernel   apply the panel's interchanges to all other columns and
//                    to the row permutation
//     u12_kernel     U12 = L11^{-1} A12
//     gemm (DMMA)    A22 -= L21 U12      (>= 99% of the flops)
//   trtri of the unit-L and U diagonal blocks for the substitutions.
// Cholesky (lower, Z12b), right-looking, panel kNB:
//   potf2_kernel (diagonal block in smem; first !(d > 0) column -> failure,
//   Z23), l21_kernel (L21 = A21 L11^{-T}), SYRK = gemm NT on lower tiles.
#include "factor.h"
#include "gemm.h"
#include "internal.h"
#include "trsm.h"

namespace as {

constexpr int kPanelThreads = 256;

// ------------------------------------------------------------------ copy + norm
// W = A (ld ldw), anorm = max_j sum_i |A_ij| (full stored A), perm = identity.
template <typename T>
__global__ void copy_norm_kernel(const DevArgs* args, int64_t lda, int64_t n, T* W, int64_t ldw, DevState* st,
                                 int64_t* perm) {
    const T* A = (const T*)args->A;
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    double best = 0.0;
    for (int64_t j = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); j < n; j += warps) {
        T s = T(0);
        const T* a = A + j * lda;
        T* w = W + j * ldw;
        for (int64_t i = lane; i < n; i += 32) {
            const T v = a[i];
            w[i] = v;
            s += v < T(0) ? -v : v;
        }
        s = warp_sum(s);
        if ((double)s > best || s != s) best = (double)s;
        if (lane == 0 && perm) perm[j] = j;
    }
    if (lane == 0 && best > 0.0) atomicMax(&st->anorm_bits, dbits(best));
}

void launch_copy_norm(const Work& w, bool with_perm, cudaStream_t s) {
    if (w.dtype == AS_F64)
        copy_norm_kernel<double><<<w.num_sms * 4, 256, 0, s>>>(w.args, w.lda, w.n, (double*)w.W, w.ldw, w.st,
                                                               with_perm ? w.perm : nullptr);
    else
        copy_norm_kernel<float><<<w.num_sms * 4, 256, 0, s>>>(w.args, w.lda, w.n, (float*)w.W, w.ldw, w.st,
                                                              with_perm ? w.perm : nullptr);
}

// X[i,:] = B[perm[i], :]  (through scratch when X aliases B)
template <typename T>
__global__ void gather_rows_kernel(const DevArgs* args, int64_t n, int64_t ldb, int64_t nrhs, const int64_t* perm,
                                   T* scratch, int phase) {
    const T* B = (const T*)args->B;
    T* X = (T*)args->X;
    const bool alias = (const void*)B == (const void*)X;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * nrhs; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e % n, c = e / n;
        if (phase == 0) {
            if (alias) scratch[i + c * n] = B[i + c * ldb];
        } else {
            X[i + c * ldb] = alias ? scratch[perm[i] + c * n] : B[perm[i] + c * ldb];
        }
    }
}

void launch_lu_solve(const Work& w, SyncAlloc& sa, cudaStream_t s) {
    const int blocks = w.num_sms * 4;
    if (w.dtype == AS_F64) {
        gather_rows_kernel<double><<<blocks, 256, 0, s>>>(w.args, w.n, w.ldb, w.nrhs, w.perm, (double*)w.vec, 0);
        gather_rows_kernel<double><<<blocks, 256, 0, s>>>(w.args, w.n, w.ldb, w.nrhs, w.perm, (double*)w.vec, 1);
    } else {
        gather_rows_kernel<float><<<blocks, 256, 0, s>>>(w.args, w.n, w.ldb, w.nrhs, w.perm, (float*)w.vec, 0);
        gather_rows_kernel<float><<<blocks, 256, 0, s>>>(w.args, w.n, w.ldb, w.nrhs, w.perm, (float*)w.vec, 1);
    }
    launch_trsm(w.dtype, w.W, w.ldw, w.Dinv0, false, false, nullptr, w.ldb, w.n, (int)w.nrhs,
                sa.take(trsm_sync_words(w.n, (int)w.nrhs)), -1, false, w.args, w.st, s);
    launch_trsm(w.dtype, w.W, w.ldw, w.Dinv1, true, false, nullptr, w.ldb, w.n, (int)w.nrhs,
                sa.take(trsm_sync_words(w.n, (int)w.nrhs)), -1, false, w.args, w.st, s);
}

// ------------------------------------------------------------------ Cholesky
template <typename T>
__global__ void __launch_bounds__(256) potf2_kernel(T* W, int64_t ldw, int64_t n, int64_t k0, int nbp, DevState* st) {
    if (st->chol_failed) return;
    constexpr int LD = kNB + 1;
    __shared__ T a[kNB * LD];
    __shared__ int s_fail;
    for (int e = threadIdx.x; e < nbp * nbp; e += blockDim.x) {
        const int r = e % nbp, c = e / nbp;
        a[r + c * LD] = (r >= c) ? W[(k0 + r) + (k0 + c) * ldw] : T(0);
    }
    if (threadIdx.x == 0) s_fail = -1;
    __syncthreads();
    for (int j = 0; j < nbp; ++j) {
        const T d = a[j + j * LD];
        if (!(d > T(0))) { if (threadIdx.x == 0) s_fail = j; break; }
        const T ljj = sqrt(d);
        __syncthreads();
        if (threadIdx.x == 0) a[j + j * LD] = ljj;
        for (int i = j + 1 + threadIdx.x; i < nbp; i += blockDim.x) a[i + j * LD] = a[i + j * LD] / ljj;
        __syncthreads();
        {   // thread = (row i, column phase); trailing lower triangle update
            const int i = threadIdx.x & (kNB - 1), ph = threadIdx.x / kNB, nph = blockDim.x / kNB;
            if (i > j && i < nbp) {
                const T lij = a[i + j * LD];
                for (int k = j + 1 + ph; k <= i; k += nph) a[i + k * LD] -= lij * a[k + j * LD];
            }
        }
        __syncthreads();
    }
    __syncthreads();
    if (s_fail >= 0) {
        if (threadIdx.x == 0) {
            st->chol_failed = 1;
            st->chol_fail_col = k0 + s_fail;
        }
        return;
    }
    for (int e = threadIdx.x; e < nbp * nbp; e += blockDim.x) {
        const int r = e % nbp, c = e / nbp;
        if (r >= c) W[(k0 + r) + (k0 + c) * ldw] = a[r + c * LD];
    }
}

// L21 = A21 L11^{-T}: each CTA solves kNB rows  x L11^T = a  (column sweep)
template <typename T>
__global__ void __launch_bounds__(256) l21_kernel(T* W, int64_t ldw, int64_t n, int64_t k0, int nbp, const DevState* st) {
    if (st->chol_failed) return;
    constexpr int LD = kNB + 1;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* L = (T*)smem_raw;         // kNB x LD
    T* X = L + kNB * LD;         // X[r + c*LD]: row r of this CTA's block, column c
    const int64_t r0 = k0 + nbp + (int64_t)blockIdx.x * kNB;
    const int nr = (int)min<int64_t>(kNB, n - r0);
    if (nr <= 0) return;
    for (int e = threadIdx.x; e < nbp * nbp; e += blockDim.x) {
        const int r = e % nbp, c = e / nbp;
        L[r + c * LD] = (r >= c) ? W[(k0 + r) + (k0 + c) * ldw] : T(0);
    }
    for (int e = threadIdx.x; e < nr * nbp; e += blockDim.x) {
        const int r = e % nr, c = e / nr;
        X[r + c * LD] = W[(r0 + r) + (k0 + c) * ldw];
    }
    __syncthreads();
    for (int c = 0; c < nbp; ++c) {
        for (int r = threadIdx.x; r < nr; r += blockDim.x) X[r + c * LD] = X[r + c * LD] / L[c + c * LD];
        __syncthreads();
        {   // thread = (row r, column phase)
            const int r = threadIdx.x & (kNB - 1), ph = threadIdx.x / kNB, nph = blockDim.x / kNB;
            if (r < nr) {
                const T xr = X[r + c * LD];
                for (int cc = c + 1 + ph; cc < nbp; cc += nph) X[r + cc * LD] -= xr * L[cc + c * LD];
            }
        }
        __syncthreads();
    }
    for (int e = threadIdx.x; e < nr * nbp; e += blockDim.x) {
        const int r = e % nr, c = e / nr;
        W[(r0 + r) + (k0 + c) * ldw] = X[r + c * LD];
    }
}

template <typename T>
static void chol_factor_t(const Work& w, cudaStream_t s) {
    const int64_t n = w.n, ldw = w.ldw;
    T* W = (T*)w.W;
    copy_norm_kernel<T><<<w.num_sms * 4, 256, 0, s>>>(w.args, w.lda, n, W, ldw, w.st, nullptr);
    for (int64_t k0 = 0; k0 < n; k0 += kNB) {
        const int nbp = (int)std::min<int64_t>(kNB, n - k0);
        potf2_kernel<T><<<1, 256, 0, s>>>(W, ldw, n, k0, nbp, w.st);
        const int64_t rest = n - k0 - nbp;
        if (rest > 0) {
            const int sm2 = (int)(sizeof(T) * 2 * kNB * (kNB + 1));
            cudaFuncSetAttribute(l21_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm2);
            l21_kernel<T><<<(unsigned)((rest + kNB - 1) / kNB), 256, sm2, s>>>(W, ldw, n, k0, nbp, w.st);
            GemmArgs g{};
            g.M = rest; g.N = rest; g.K = nbp;
            g.A = W + (k0 + nbp) + k0 * ldw; g.lda = ldw; g.TA = false;
            g.B = W + (k0 + nbp) + k0 * ldw; g.ldb = ldw; g.TB = true;
            g.C = W + (k0 + nbp) + (k0 + nbp) * ldw; g.ldc = ldw;
            g.lower_only = true;
            g.skip = &w.st->chol_failed;
            launch_gemm_minus(w.dtype, g, s);
        }
    }
}

void launch_chol_factor(const Work& w, cudaStream_t s) {
    if (w.dtype == AS_F64) chol_factor_t<double>(w, s);
    else chol_factor_t<float>(w, s);
}

// after POTRF: if it failed, switch to LU and set the IF handle
__global__ void chol_check_kernel(DevState* st, cudaGraphConditionalHandle h) {
    if (threadIdx.x != 0) return;
    const int failed = st->chol_failed;
    if (failed) {
        st->flags |= AS_FLAG_CHOL_FAILED;
        st->method = AS_METHOD_LU;
        st->primary = AS_METHOD_LU;
        st->anorm_bits = 0ull;
    }
    if (h) cudaGraphSetConditional(h, failed ? 1u : 0u);
}

void launch_chol_check(const Work& w, cudaGraphConditionalHandle h, cudaStream_t s) {
    chol_check_kernel<<<1, 32, 0, s>>>(w.st, h);
}

void launch_chol_tri_prep(const Work& w, cudaStream_t s) {
    launch_trtri_blocks(w.dtype, w.W, w.ldw, w.n, w.Dinv0, false, false, w.st, true, w.args, s);
}

void launch_chol_solve(const Work& w, SyncAlloc& sa, cudaStream_t s) {
    launch_copy_b_to_x(w, s);
    launch_trsm(w.dtype, w.W, w.ldw, w.Dinv0, false, false, nullptr, w.ldb, w.n, (int)w.nrhs,
                sa.take(trsm_sync_words(w.n, (int)w.nrhs)), -1, false, w.args, w.st, s);
    launch_trsm(w.dtype, w.W, w.ldw, w.Dinv0, false, true, nullptr, w.ldb, w.n, (int)w.nrhs,
                sa.take(trsm_sync_words(w.n, (int)w.nrhs)), -1, false, w.args, w.st, s);
}

}  // namespace as
