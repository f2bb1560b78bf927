// band.cu -- banded path: K2 band_pack into the LAPACK band layout
// ("each diagonal is stored as a vector in a separate dense matrix", P:345-346,
// Z12), K3 banded LU with partial pivoting (xGBTRF), K4 the banded
// solve (xGBTRS) and the M / M^T applications of the xGBCON estimator
// (P:350).  Band extents kl/ku are read from the device state written by the
// detection kernel, so nothing here needs the host.
//
// Row i, column c of A lives at ab[kv + i - c + c*ldab], kv = kl + ku,
// ldab = 2*kl + ku + 1 (kl fill rows on top for the pivoting fill-in).
// The band storage lives in the plan's n x n workspace W.
//
// The factor/solve are sequential chains of n pivot steps (a faithful
// GBTRF); one warp per chain keeps every step warp-synchronous.
#include "internal.h"
#include "rcond.h"

namespace as {

// ------------------------------------------------------------------ K2 pack
template <typename T>
__global__ void band_pack_kernel(const DevArgs* args, int64_t lda, int64_t n, DevState* st, T* ab) {
    const T* A = (const T*)args->A;
    const int64_t kl = st->kl, ku = st->ku, kv = kl + ku, ldab = 2 * kl + ku + 1;
    const int64_t total = ldab * n;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = e % ldab, j = e / ldab;
        const int64_t i = r + j - kv;
        T v = T(0);
        if (r >= kl && i >= 0 && i < n) v = A[i + j * lda];
        ab[e] = v;
    }
}

// anorm = max_j sum_i |A_ij| over the band (one warp per column)
template <typename T>
__global__ void band_norm_kernel(const DevArgs* args, int64_t lda, int64_t n, DevState* st) {
    const T* A = (const T*)args->A;
    const int64_t kl = st->kl, ku = st->ku;
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    double best = 0.0;
    for (int64_t j = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); j < n; j += warps) {
        const int64_t i0 = j - ku > 0 ? j - ku : 0, i1 = j + kl < n - 1 ? j + kl : n - 1;
        T s = T(0);
        for (int64_t i = i0 + lane; i <= i1; i += 32) { T a = A[i + j * lda]; s += a < T(0) ? -a : a; }
        s = warp_sum(s);
        if ((double)s > best || s != s) best = (double)s;
    }
    if (lane == 0 && best > 0.0) atomicMax(&st->anorm_bits, dbits(best));
}

// ------------------------------------------------------------------ K3 gbtrf (one warp)
template <typename T>
__global__ void __launch_bounds__(32) gbtrf_warp_kernel(T* ab, int64_t n, DevState* st, int64_t* ipiv) {
    const int lane = threadIdx.x;
    const int64_t kl = st->kl, ku = st->ku, kv = kl + ku, ldab = 2 * kl + ku + 1;
#define AB(r, c) ab[(r) + (c) * ldab]
    int64_t ju = 0;
    unsigned long long info = ~0ull;
    for (int64_t j = 0; j < n; ++j) {
        const int64_t km = kl < n - 1 - j ? kl : n - 1 - j;
        // pivot: first max |.| over r = 0..km, strict > starting from r = 0 (Z15)
        T best = T(-1);
        long long jp = 0x7fffffffffffffffll;
        for (int64_t r = lane; r <= km; r += 32) {
            T a = AB(kv + r, j);
            a = a < T(0) ? -a : a;
            if (r == 0 && a != a) { best = T(INFINITY); jp = 0; }  // NaN diagonal: serial semantics keep r = 0
            argmax_merge(best, jp, a, (long long)r);
        }
        warp_argmax(best, jp);
        if (jp == 0x7fffffffffffffffll) jp = 0;
        if (lane == 0) ipiv[j] = j + jp;
        const T piv = AB(kv + jp, j);
        if (piv != T(0)) {
            const int64_t lim = j + ku + jp < n - 1 ? j + ku + jp : n - 1;
            if (lim > ju) ju = lim;
            if (jp != 0) {
                for (int64_t c = j + lane; c <= ju; c += 32) {
                    const T t = AB(kv + j + jp - c, c);
                    AB(kv + j + jp - c, c) = AB(kv + j - c, c);
                    AB(kv + j - c, c) = t;
                }
                __syncwarp();
            }
            const T pv = AB(kv, j);
            for (int64_t r = 1 + lane; r <= km; r += 32) AB(kv + r, j) = AB(kv + r, j) / pv;
            __syncwarp();
            const int64_t wdt = ju - j;
            for (int64_t e = lane; e < km * wdt; e += 32) {
                const int64_t r = 1 + e % km, c = j + 1 + e / km;
                AB(kv + j + r - c, c) = AB(kv + j + r - c, c) - AB(kv + r, j) * AB(kv + j - c, c);
            }
            __syncwarp();
        } else if (info == ~0ull) {
            info = (unsigned long long)(j + 1);
        }
    }
    if (lane == 0 && info != ~0ull) atomicMin(&st->info, info);
#undef AB
}

// ------------------------------------------------------------------ K4 gbtrs (one warp per RHS column)
// no-trans: L (with interleaved interchanges) then U (bandwidth kv);
// trans:    U^T then L^T with the interchanges undone in reverse.
template <typename T>
AS_DEV void gb_solve_vec(const T* ab, int64_t n, int64_t kl, int64_t ku, const int64_t* ipiv, T* b, bool trans) {
    const int lane = threadIdx.x & 31;
    const int64_t kv = kl + ku, ldab = 2 * kl + ku + 1;
#define AB(r, c) ab[(r) + (c) * ldab]
    if (!trans) {
        for (int64_t j = 0; j + 1 < n; ++j) {
            const int64_t lm = kl < n - 1 - j ? kl : n - 1 - j;
            const int64_t l = ipiv[j];
            T bj;
            if (l != j) {
                const T bl = b[l];
                bj = b[j];
                __syncwarp();
                if (lane == 0) { b[l] = bj; b[j] = bl; }
                bj = bl;
            } else {
                bj = b[j];
            }
            __syncwarp();
            for (int64_t r = 1 + lane; r <= lm; r += 32) b[j + r] = b[j + r] - AB(kv + r, j) * bj;
            __syncwarp();
        }
        for (int64_t j = n - 1; j >= 0; --j) {
            const T xj = b[j] / AB(kv, j);
            __syncwarp();
            if (lane == 0) b[j] = xj;
            const int64_t i0 = j - kv > 0 ? j - kv : 0;
            for (int64_t i = i0 + lane; i < j; i += 32) b[i] = b[i] - AB(kv + i - j, j) * xj;
            __syncwarp();
        }
    } else {
        for (int64_t j = 0; j < n; ++j) {
            const int64_t i0 = j - kv > 0 ? j - kv : 0;
            T s = T(0);
            for (int64_t i = i0 + lane; i < j; i += 32) s += AB(kv + i - j, j) * b[i];
            s = warp_sum(s);
            const T v = (b[j] - s) / AB(kv, j);
            __syncwarp();
            if (lane == 0) b[j] = v;
            __syncwarp();
        }
        for (int64_t j = n - 2; j >= 0; --j) {
            const int64_t lm = kl < n - 1 - j ? kl : n - 1 - j;
            T s = T(0);
            for (int64_t r = 1 + lane; r <= lm; r += 32) s += AB(kv + r, j) * b[j + r];
            s = warp_sum(s);
            const T v = b[j] - s;
            const int64_t l = ipiv[j];
            __syncwarp();
            if (lane == 0) {
                if (l != j) { b[j] = b[l]; b[l] = v; }
                else b[j] = v;
            }
            __syncwarp();
        }
    }
#undef AB
}

template <typename T>
__global__ void __launch_bounds__(32) gbtrs_kernel(const T* ab, int64_t n, const DevState* st, const int64_t* ipiv,
                                                    const DevArgs* args, int64_t ldb, T* xvec, int trans, int slot) {
    if (slot >= 0 && ld_volatile_i32(&st->est_next) != slot) return;
    if (st->info != ~0ull) return;
    if (st->band_fast) return;    // the partitioned solver already produced X
    T* b = xvec ? xvec : (T*)args->X + (int64_t)blockIdx.x * ldb;
    gb_solve_vec<T>(ab, n, st->kl, st->ku, ipiv, b, trans != 0);
}

// X = B (column by column; skipped when X aliases B)
template <typename T>
__global__ void copy_b_to_x_kernel(const DevArgs* args, int64_t n, int64_t ldb, int64_t nrhs, const DevState* st) {
    const T* B = (const T*)args->B;
    T* X = (T*)args->X;
    if ((const void*)B == (const void*)X) return;
    if (st && st->band_fast) return;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * nrhs; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e % n, c = e / n;
        X[i + c * ldb] = B[i + c * ldb];
    }
}

// ------------------------------------------------------------------ launchers
void launch_band_norm(const Work& w, cudaStream_t s) {
    const int blocks = w.num_sms * 4;
    if (w.dtype == AS_F64) band_norm_kernel<double><<<blocks, 256, 0, s>>>(w.args, w.lda, w.n, w.st);
    else band_norm_kernel<float><<<blocks, 256, 0, s>>>(w.args, w.lda, w.n, w.st);
}

// sequential (faithful xGBTF2) path: pack + factor
void launch_band_factor(const Work& w, cudaStream_t s) {
    const int blocks = w.num_sms * 4;
    if (w.dtype == AS_F64) {
        band_pack_kernel<double><<<blocks, 256, 0, s>>>(w.args, w.lda, w.n, w.st, (double*)w.W);
        gbtrf_warp_kernel<double><<<1, 32, 0, s>>>((double*)w.W, w.n, w.st, w.ipiv);
    } else {
        band_pack_kernel<float><<<blocks, 256, 0, s>>>(w.args, w.lda, w.n, w.st, (float*)w.W);
        gbtrf_warp_kernel<float><<<1, 32, 0, s>>>((float*)w.W, w.n, w.st, w.ipiv);
    }
}

void launch_band_apply(const Work& w, bool trans, int slot, cudaStream_t s) {
    if (w.dtype == AS_F64)
        gbtrs_kernel<double><<<1, 32, 0, s>>>((const double*)w.W, w.n, w.st, w.ipiv, w.args, w.n, (double*)w.xe, trans, slot);
    else
        gbtrs_kernel<float><<<1, 32, 0, s>>>((const float*)w.W, w.n, w.st, w.ipiv, w.args, w.n, (float*)w.xe, trans, slot);
}

void launch_copy_b_to_x(const Work& w, cudaStream_t s) {
    const int blocks = w.num_sms * 4;
    if (w.dtype == AS_F64) copy_b_to_x_kernel<double><<<blocks, 256, 0, s>>>(w.args, w.n, w.ldb, w.nrhs, w.st);
    else copy_b_to_x_kernel<float><<<blocks, 256, 0, s>>>(w.args, w.n, w.ldb, w.nrhs, w.st);
}

void launch_band_solve(const Work& w, cudaStream_t s) {
    launch_copy_b_to_x(w, s);
    if (w.dtype == AS_F64)
        gbtrs_kernel<double><<<(unsigned)w.nrhs, 32, 0, s>>>((const double*)w.W, w.n, w.st, w.ipiv, w.args, w.ldb, nullptr, 0, -1);
    else
        gbtrs_kernel<float><<<(unsigned)w.nrhs, 32, 0, s>>>((const float*)w.W, w.n, w.st, w.ipiv, w.args, w.ldb, nullptr, 0, -1);
}

}  // namespace as
