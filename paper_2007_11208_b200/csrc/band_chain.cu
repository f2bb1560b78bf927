// band_chain.cu -- narrow non-dominant bands (kl, ku <= 3: the tridiagonal fast path of SURVEY
// 8(f) row 4, and the paper's own 5-diagonal Table 1 class) in ONE launch of one warp:
//
//   xGBTRF with partial pivoting as a register-window chain: the active
//   (kl+1) x (kl+ku+1) window of the factorization lives in registers of lane 0 (compile-time
//   shape), the next rows of A are prefetched 8 steps ahead (they do not depend on the chain), the
//   factor columns go to the LAPACK band layout (Z12) as they complete;
//   xGBCON: the xLACN2 steps of the oracle on lane 0 with xGBTRS / xGBTRS^T chains, the
//   sums / argmax reductions by the warp;
//   xGBTRS: one right-hand side per lane, all lanes' chains in parallel.
//
// For kl = ku = 1 this is xGTTRF / xGTTRS (LAPACK's tridiagonal LU with partial pivoting): the same
// pivot rule (|d_j| vs |dl_j|, ties keep the diagonal) and the same operations as the band LU, so it
// is graded against the oracle's band path.  Every step is a short dependent chain (~50-100 cycles)
// instead of the warp-synchronous window of the general sequential kernel (~1.2 us per column).
// X is written before the gate (like the partitioned path), so the path is not used for X == B.
#include "internal.h"
#include "rcond.h"

namespace as {
namespace {

template <typename T>
AS_DEV T cabs(T x) { return x < T(0) ? -x : x; }

// ------------------------------------------------------------------ xGBTRF, lane 0
template <typename T, int KL, int KU>
AS_DEV int64_t chain_gbtrf(const T* __restrict__ A, int64_t lda, int64_t n, T* ab, int64_t* ipiv) {
    constexpr int KV = KL + KU;
    constexpr int LDAB = 2 * KL + KU + 1;
    constexpr int kPF = KV >= 4 ? 4 : 8;   // prefetch depth (rows); shallower for wide windows (registers)
    T w[KL + 1][KV + 1];
    // window at j = 0: rows 0..KL, columns 0..KV (in-band entries of A)
#pragma unroll
    for (int r = 0; r <= KL; ++r)
#pragma unroll
        for (int c = 0; c <= KV; ++c) {
            const bool inb = (r - c <= KL) && (c - r <= KU) && r < n && c < n;
            w[r][c] = inb ? A[r + (int64_t)c * lda] : T(0);
        }
    // prefetch queue: row j + KL + 1 (entering at the end of step j), columns j + 1 .. j + 1 + KV
    T q[kPF][KV + 1];
    auto load_row = [&](int64_t j, T (&dst)[KV + 1]) {
        const int64_t i = j + KL + 1;
#pragma unroll
        for (int c = 0; c <= KV; ++c) {
            const int64_t k = j + 1 + c;
            dst[c] = (i < n && k < n) ? __ldg(&A[i + k * lda]) : T(0);
        }
    };
#pragma unroll
    for (int d = 0; d < kPF; ++d) load_row(d, q[d]);
    int64_t info = 0;
    for (int64_t j0 = 0; j0 < n; j0 += kPF) {
        T nq[kPF][KV + 1];
#pragma unroll
        for (int d = 0; d < kPF; ++d) load_row(j0 + kPF + d, nq[d]);
#pragma unroll
        for (int d = 0; d < kPF; ++d) {
            const int64_t j = j0 + d;
            if (j >= n) break;
            const int km = (int)min<int64_t>(KL, n - 1 - j);
            // first max |w[r][0]|, r = 0..km (Z15: strict >, NaN never wins)
            int p = 0;
            T best = cabs(w[0][0]);
#pragma unroll
            for (int r = 1; r <= KL; ++r)
                if (r <= km && cabs(w[r][0]) > best) { best = cabs(w[r][0]); p = r; }
            ipiv[j] = j + p;
            T pv = w[0][0];
#pragma unroll
            for (int r = 1; r <= KL; ++r) if (r == p) pv = w[r][0];
            T l[KL + 1];
#pragma unroll
            for (int r = 0; r <= KL; ++r) l[r] = T(0);
            if (pv != T(0)) {
                // interchange rows 0 and p of the window
#pragma unroll
                for (int r = 1; r <= KL; ++r)
                    if (r == p)
#pragma unroll
                        for (int c = 0; c <= KV; ++c) { const T t = w[0][c]; w[0][c] = w[r][c]; w[r][c] = t; }
#pragma unroll
                for (int r = 1; r <= KL; ++r)
                    if (r <= km) l[r] = w[r][0] / w[0][0];       // multipliers by division (Z15)
#pragma unroll
                for (int r = 1; r <= KL; ++r)
#pragma unroll
                    for (int c = 1; c <= KV; ++c) w[r][c] = w[r][c] - l[r] * w[0][c];
            } else if (info == 0) {
                info = j + 1;
            }
            // factor column j: U(j, j + c) at AB(KV - c, j + c), L(j + r, j) at AB(KV + r, j)
#pragma unroll
            for (int c = 0; c <= KV; ++c)
                if (j + c < n) ab[(KV - c) + (j + c) * (int64_t)LDAB] = w[0][c];
#pragma unroll
            for (int r = 1; r <= KL; ++r) ab[(KV + r) + j * (int64_t)LDAB] = l[r];
            // shift the window: rows j+1.., columns j+1..; the new last row from the queue
#pragma unroll
            for (int r = 0; r < KL; ++r)
#pragma unroll
                for (int c = 0; c < KV; ++c) w[r][c] = w[r + 1][c + 1];
#pragma unroll
            for (int r = 0; r < KL; ++r) w[r][KV] = T(0);
            if (KL > 0) {
#pragma unroll
                for (int c = 0; c <= KV; ++c) w[KL][c] = q[d][c];
            } else {
                // KL = 0: the window is row j+1 only, columns j+1 .. j+1+KU
#pragma unroll
                for (int c = 0; c <= KV; ++c) w[0][c] = q[d][c];
            }
        }
#pragma unroll
        for (int d = 0; d < kPF; ++d)
#pragma unroll
            for (int c = 0; c <= KV; ++c) q[d][c] = nq[d][c];
    }
    return info;
}

// ------------------------------------------------------------------ xGBTRS ('N' and 'T'), one lane
// b (global, stride 1) overwritten.  'N': interchanges + L forward, U backward.  'T': U^T forward,
// L^T backward with the interchanges undone in reverse (the oracle's gbtrs_vec / gbtrs_vec_t).
template <typename T, int KL, int KU>
AS_DEV void chain_gbtrs(const T* ab, const int64_t* ipiv, int64_t n, T* b, bool trans) {
    constexpr int KV = KL + KU;
    constexpr int LDAB = 2 * KL + KU + 1;
    if (!trans) {
        // forward: window b[j .. j+KL]
        T v[KL + 1];
#pragma unroll
        for (int r = 0; r <= KL; ++r) v[r] = r < n ? b[r] : T(0);
        for (int64_t j = 0; j < n; ++j) {
            const T nxt = (j + KL + 1 < n) ? b[j + KL + 1] : T(0);
            if (j + 1 < n) {
                const int lm = (int)min<int64_t>(KL, n - 1 - j);
                const int p = (int)(ipiv[j] - j);
#pragma unroll
                for (int r = 1; r <= KL; ++r)
                    if (r == p) { const T t = v[0]; v[0] = v[r]; v[r] = t; }
#pragma unroll
                for (int r = 1; r <= KL; ++r)
                    if (r <= lm) v[r] = v[r] - (ab[(KV + r) + j * (int64_t)LDAB]) * v[0];
            }
            b[j] = v[0];
#pragma unroll
            for (int r = 0; r < KL; ++r) v[r] = v[r + 1];
            if (KL > 0) v[KL] = nxt;
            else v[0] = nxt;
        }
        // backward: x_j = b_j / U(j,j); b_i -= U(i, j) x_j for i = j - KV .. j - 1 (window b[j-KV .. j])
        T u[KV + 1];
#pragma unroll
        for (int c = 0; c <= KV; ++c) u[c] = (n - 1 - KV + c >= 0) ? b[n - 1 - KV + c] : T(0);   // u[KV] = b[j]
        for (int64_t j = n - 1; j >= 0; --j) {
            const T prev = (j - KV - 1 >= 0) ? b[j - KV - 1] : T(0);
            const T x = u[KV] / (ab[KV + j * (int64_t)LDAB]);
            b[j] = x;
#pragma unroll
            for (int c = 0; c < KV; ++c) {
                const int64_t i = j - KV + c;
                if (i >= 0) u[c] = u[c] - (ab[(KV + i - j) + j * (int64_t)LDAB]) * x;
            }
#pragma unroll
            for (int c = KV; c > 0; --c) u[c] = u[c - 1];
            u[0] = prev;
        }
    } else {
        // U^T forward: b_j = (b_j - sum_{i=j-KV}^{j-1} U(i, j) x_i) / U(j, j); window of the last KV x
        T xs[KV + 1];
#pragma unroll
        for (int c = 0; c <= KV; ++c) xs[c] = T(0);      // xs[c] = x_{j - KV + c}, c < KV
        for (int64_t j = 0; j < n; ++j) {
            T s = b[j];
#pragma unroll
            for (int c = 0; c < KV; ++c) {
                const int64_t i = j - KV + c;
                if (i >= 0) s = s - (ab[(KV + i - j) + j * (int64_t)LDAB]) * xs[c];
            }
            const T x = s / (ab[KV + j * (int64_t)LDAB]);
            b[j] = x;
#pragma unroll
            for (int c = 0; c + 1 < KV; ++c) xs[c] = xs[c + 1];
            if (KV > 0) xs[KV - 1] = x;
        }
        // L^T backward: b_j = b_j - sum_{r=1..lm} L(j + r, j) b_{j+r}; then swap b_j, b_ipiv(j)
        if (KL > 0 && n >= 2) {
            T v[KL + 1];                                   // v[r] = b[j + r]
#pragma unroll
            for (int r = 0; r <= KL; ++r) v[r] = (n - 2 + r < n) ? b[n - 2 + r] : T(0);
            for (int64_t j = n - 2; j >= 0; --j) {
                const T prev = j >= 1 ? b[j - 1] : T(0);
                const int lm = (int)min<int64_t>(KL, n - 1 - j);
                T s = v[0];
#pragma unroll
                for (int r = 1; r <= KL; ++r)
                    if (r <= lm) s = s - (ab[(KV + r) + j * (int64_t)LDAB]) * v[r];
                v[0] = s;
                const int p = (int)(ipiv[j] - j);
#pragma unroll
                for (int r = 1; r <= KL; ++r)
                    if (r == p) { const T t = v[0]; v[0] = v[r]; v[r] = t; b[j + r] = v[r]; }
                b[j] = v[0];
#pragma unroll
                for (int r = KL; r > 0; --r) v[r] = v[r - 1];
                v[0] = prev;
            }
        }
    }
}

// ------------------------------------------------------------------ the kernel (one warp)
template <typename T, int KL, int KU>
AS_DEV void band_chain_body(const DevArgs* args, int64_t lda, int64_t n, int64_t ldb, int64_t nrhs, T* ab,
                            int64_t* ipiv, T* xv, signed char* isgn, DevState* st) {
    const int lane = threadIdx.x;
    const T* A = (const T*)args->A;
    __shared__ long long s_info;
    if (lane == 0) s_info = chain_gbtrf<T, KL, KU>(A, lda, n, ab, ipiv);
    __syncwarp();
    __threadfence_block();
    const long long info = s_info;
    if (info) {
        if (lane == 0) atomicMin(&st->info, (unsigned long long)info);
        return;
    }
    // ---- xGBCON: the oracle's xLACN2 steps (Z13b), chains on lane 0, reductions by the warp
    auto sync = [&]() { __syncwarp(); __threadfence_block(); };
    auto asum = [&]() { T s = T(0); for (int64_t i = lane; i < n; i += 32) s += cabs(xv[i]); return warp_sum(s); };
    auto iamax = [&]() {
        T bk = T(-1);
        long long bi = 0x7fffffffffffffffll;
        for (int64_t i = lane; i < n; i += 32) { const T a = cabs(xv[i]); if (a > bk) { bk = a; bi = i; } }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const T k2 = __shfl_xor_sync(0xffffffffu, bk, o);
            const long long i2 = __shfl_xor_sync(0xffffffffu, bi, o);
            if (k2 > bk || (k2 == bk && i2 < bi)) { bk = k2; bi = i2; }
        }
        return bi == 0x7fffffffffffffffll ? 0ll : bi;
    };
    auto apply = [&](bool tr) { if (lane == 0) chain_gbtrs<T, KL, KU>(ab, ipiv, n, xv, tr); sync(); };
    for (int64_t i = lane; i < n; i += 32) xv[i] = T(1) / (T)n;
    sync();
    apply(false);
    T est;
    if (n == 1) {
        est = cabs(xv[0]);
    } else {
        est = asum();
        for (int64_t i = lane; i < n; i += 32) { const T s = xv[i] >= T(0) ? T(1) : T(-1); xv[i] = s; isgn[i] = s > T(0) ? 1 : -1; }
        sync();
        apply(true);
        long long j = iamax();
        int iter = 2;
        for (;;) {
            for (int64_t i = lane; i < n; i += 32) xv[i] = i == j ? T(1) : T(0);
            sync();
            apply(false);
            const T estold = est;
            est = asum();
            bool same = true;
            for (int64_t i = lane; i < n; i += 32) same &= (xv[i] >= T(0) ? 1 : -1) == isgn[i];
            same = __all_sync(0xffffffffu, same);
            if (same || est <= estold) break;
            for (int64_t i = lane; i < n; i += 32) { const T s = xv[i] >= T(0) ? T(1) : T(-1); xv[i] = s; isgn[i] = s > T(0) ? 1 : -1; }
            sync();
            apply(true);
            const long long jlast = j;
            j = iamax();
            if (xv[jlast] != cabs(xv[j]) && iter < 5) { ++iter; continue; }
            break;
        }
        for (int64_t i = lane; i < n; i += 32) xv[i] = ((i & 1) ? T(-1) : T(1)) * (T(1) + (T)i / (T)(n - 1));
        sync();
        apply(false);
        const T temp = T(2) * (asum() / (T)(3 * n));
        if (temp > est) est = temp;
    }
    if (lane == 0) {
        const T anorm = (T)dfrom(st->anorm_bits);
        T rc = T(0);
        if (anorm > T(0) && est != T(0)) rc = (T(1) / est) / anorm;
        st->rcond = (double)rc;
    }
    // ---- the primary solve, one right-hand side per lane (X written before the gate, like the
    // partitioned path; the fallback overwrites it)
    T* X = (T*)args->X;
    const T* B = (const T*)args->B;
    for (int64_t c = lane; c < nrhs; c += 32) {
        T* x = X + c * ldb;
        for (int64_t i = 0; i < n; ++i) x[i] = B[i + c * ldb];
        chain_gbtrs<T, KL, KU>(ab, ipiv, n, x, false);
    }
    if (lane == 0) st->band_fast = 1;
}

// one kernel, the (kl, ku) instance picked on device (kl / ku are only known after detection)
template <typename T>
__global__ void __launch_bounds__(32, 1) band_chain_kernel(const DevArgs* args, int64_t lda, int64_t n, int64_t ldb,
                                                           int64_t nrhs, T* ab, int64_t* ipiv, T* xv,
                                                           signed char* isgn, DevState* st) {
    switch (st->band_chain) {
#define AS_CHAIN_CASE(KL, KU) \
    case 1 + 4 * KL + KU: band_chain_body<T, KL, KU>(args, lda, n, ldb, nrhs, ab, ipiv, xv, isgn, st); break;
    AS_CHAIN_CASE(0, 0) AS_CHAIN_CASE(0, 1) AS_CHAIN_CASE(0, 2) AS_CHAIN_CASE(0, 3)
    AS_CHAIN_CASE(1, 0) AS_CHAIN_CASE(1, 1) AS_CHAIN_CASE(1, 2) AS_CHAIN_CASE(1, 3)
    AS_CHAIN_CASE(2, 0) AS_CHAIN_CASE(2, 1) AS_CHAIN_CASE(2, 2) AS_CHAIN_CASE(2, 3)
    AS_CHAIN_CASE(3, 0) AS_CHAIN_CASE(3, 1) AS_CHAIN_CASE(3, 2) AS_CHAIN_CASE(3, 3)
#undef AS_CHAIN_CASE
    default: break;
    }
}

}  // namespace

void launch_band_chain(const Work& w, cudaStream_t s) {
    if (w.dtype == AS_F64)
        band_chain_kernel<double><<<1, 32, 0, s>>>(w.args, w.lda, w.n, w.ldb, w.nrhs, (double*)w.W, w.ipiv,
                                                    (double*)w.xe, (signed char*)w.zx, w.st);
    else
        band_chain_kernel<float><<<1, 32, 0, s>>>(w.args, w.lda, w.n, w.ldb, w.nrhs, (float*)w.W, w.ipiv,
                                                   (float*)w.xe, (signed char*)w.zx, w.st);
}

}  // namespace as
