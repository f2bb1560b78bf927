// small.cu -- batched small systems: many independent A_b X_b = B_b with
// n <= kSmallN, ONE thread block per system, the paper's whole flowchart inside the block with the
// matrix in shared memory:
//
//   detection (kl/ku, triangularity, Fig. 4 likely_sympd; every element is read once anyway, so the
//   verdicts and kl/ku are always exact) -> first-match dispatch -> factor -> xLACN2 rcond estimate
//   -> gate -> solve, or the QR + one-sided Jacobi minimum-norm fallback.
//
// The paper's workload is "1000 unique random systems" per size: the per-system path
// of the large solver is latency bound for such sizes (one graph launch, grid-wide exchanges per
// column), here a launch carries the whole batch.  Method by method the arithmetic is the
// unblocked algorithm the oracle states:
//   BAND      partial-pivoting LU of the (dense-stored) band matrix: the pivot search over rows
//             j..n-1 meets only zeros below j+kl, so the pivots and the non-zero arithmetic are
//             xGBTRF's; GBCON applies the interchanges (as xGBCON), anorm = band 1-norm;
//   TRI       exact-zero diagonal check, Eq. (3) substitution, xTRCON;
//   CHOL      right-looking xPOTF2 on the lower triangle, failure -> LU on the original A
//             (P:449-457), xPOCON;
//   LU        xGETF2 (first max |.|, Z15), xGECON (inv(U) inv(L), no interchanges), xGETRS
//             (P:505-533);
//   fallback  Householder QR, one-sided Jacobi on R^T (round-robin pairs, rotate iff
//             |gamma| > n eps sqrt(alpha) sqrt(beta), Z16), min-norm with cut n eps sigma_max (Z14).
// Triangular solves run on one warp (lane l owns rows l, l+32, ...): no block barrier per column.
#include <cstdio>

#include "internal.h"
#include "rcond.h"
#include "small.h"

namespace as {
namespace {   // internal linkage: these helpers must not merge with other translation units' templates

template <typename T> AS_DEV T tabs(T x);
template <> AS_DEV double tabs<double>(double x) { return fabs(x); }
template <> AS_DEV float tabs<float>(float x) { return fabsf(x); }

constexpr int KIND_LDLT = 4;      // one-block solver only: Bunch-Kaufman L D L^T (Z30)
constexpr int kSmallT = 256;
constexpr int kSmallWarps = kSmallT / 32;
constexpr int kRows = kSmallN / 32;      // rows per lane in the warp substitutions

template <typename T>
struct SmallSmem {
    T W[kSmallN * (kSmallN + 1)];          // factor (ld n + 1)
    T x[kSmallN], y[kSmallN], z[kSmallN];  // estimator / solve vectors
    T Y[kSmallRhs * kSmallN];              // fallback: V^T Q^T B
    T sig[kSmallN];
    T red[32];
    int ipiv[kSmallN];
    int isgn[kSmallN];
    int ired[32];
    int kl, ku, flags, nonfinite, spd_dead, rot, asym;
    T max_diag;
};

// ------------------------------------------------------------------ block reductions
template <typename T>
AS_DEV T block_sum(T v, T* red) {
    v = warp_sum(v);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    T s = T(0);
#pragma unroll
    for (int w = 0; w < kSmallWarps; ++w) s += red[w];
    return s;
}
// first index of the maximum of key (keys are >= 0 or -1 = none; never NaN)
template <typename T>
AS_DEV int block_argmax(T key, int idx, T* red, int* ired) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const T k2 = __shfl_xor_sync(0xffffffffu, key, o);
        const int i2 = __shfl_xor_sync(0xffffffffu, idx, o);
        if (k2 > key || (k2 == key && i2 < idx)) { key = k2; idx = i2; }
    }
    __syncthreads();
    if ((threadIdx.x & 31) == 0) { red[threadIdx.x >> 5] = key; ired[threadIdx.x >> 5] = idx; }
    __syncthreads();
    T bk = red[0];
    int bi = ired[0];
#pragma unroll
    for (int w = 1; w < kSmallWarps; ++w) {
        const T k2 = red[w];
        const int i2 = ired[w];
        if (k2 > bk || (k2 == bk && i2 < bi)) { bk = k2; bi = i2; }
    }
    return bi;
}

// ------------------------------------------------------------------ one-warp substitution
// op(T) x = x for the n x n triangle stored in W (ld): upper selects the stored triangle, trans
// solves with its transpose, unit ignores the stored diagonal.  Column-oriented (x_j final ->
// broadcast -> the rows still pending subtract T(i, j) x_j).
template <typename T>
AS_DEV void warp_trsv(const T* W, int ld, int n, bool upper, bool trans, bool unit, T* x) {
    const int lane = threadIdx.x & 31;
    T r[kRows];
#pragma unroll
    for (int k = 0; k < kRows; ++k) r[k] = lane + 32 * k < n ? x[lane + 32 * k] : T(0);
    const bool fwd = upper == trans;       // effective lower triangle
    for (int s = 0; s < n; ++s) {
        const int j = fwd ? s : n - 1 - s;
        T xj = T(0);
#pragma unroll
        for (int k = 0; k < kRows; ++k)
            if (lane + 32 * k == j) xj = unit ? r[k] : r[k] / W[j + j * ld];
        xj = __shfl_sync(0xffffffffu, xj, j & 31);
#pragma unroll
        for (int k = 0; k < kRows; ++k) {
            const int i = lane + 32 * k;
            if (i == j) r[k] = xj;
            else if (i < n && (fwd ? i > j : i < j)) r[k] -= (trans ? W[j + i * ld] : W[i + j * ld]) * xj;
        }
    }
#pragma unroll
    for (int k = 0; k < kRows; ++k)
        if (lane + 32 * k < n) x[lane + 32 * k] = r[k];
    __syncwarp();
}

// xSYTRS (lower) on one warp: v <- A^{-1} v from the Bunch-Kaufman factors in W (the oracle's
// sytrs_vec: L D forward with the interleaved interchanges, then L^T backward)
template <typename T>
AS_DEV void warp_sytrs(const T* W, int ld, int n, const int* ipiv, T* v) {
    const int lane = threadIdx.x & 31;
    int k = 0;
    while (k < n) {
        if (ipiv[k] >= 0) {
            const int kp = ipiv[k];
            if (lane == 0 && kp != k) { const T t = v[k]; v[k] = v[kp]; v[kp] = t; }
            __syncwarp();
            const T bk = v[k];
            for (int i = k + 1 + lane; i < n; i += 32) v[i] = v[i] - W[i + k * ld] * bk;
            __syncwarp();
            if (lane == 0) v[k] = bk / W[k + k * ld];
            __syncwarp();
            k += 1;
        } else {
            const int kp = -ipiv[k] - 1;
            if (lane == 0 && kp != k + 1) { const T t = v[k + 1]; v[k + 1] = v[kp]; v[kp] = t; }
            __syncwarp();
            const T b0 = v[k], b1 = v[k + 1];
            for (int i = k + 2 + lane; i < n; i += 32) v[i] = v[i] - W[i + k * ld] * b0 - W[i + (k + 1) * ld] * b1;
            __syncwarp();
            if (lane == 0) {
                const T akm1k = W[(k + 1) + k * ld];
                const T akm1 = W[k + k * ld] / akm1k;
                const T ak = W[(k + 1) + (k + 1) * ld] / akm1k;
                const T denom = akm1 * ak - T(1);
                const T bkm1 = b0 / akm1k;
                const T bk = b1 / akm1k;
                v[k] = (ak * bkm1 - bk) / denom;
                v[k + 1] = (akm1 * bk - bkm1) / denom;
            }
            __syncwarp();
            k += 2;
        }
    }
    k = n - 1;
    while (k >= 0) {
        const bool one = ipiv[k] >= 0;
        T s = T(0), s1 = T(0);
        for (int i = k + 1 + lane; i < n; i += 32) {
            s += W[i + k * ld] * v[i];
            if (!one) s1 += W[i + (k - 1) * ld] * v[i];
        }
        s = warp_sum(s);
        s1 = warp_sum(s1);
        if (lane == 0) {
            v[k] = v[k] - s;
            if (!one) v[k - 1] = v[k - 1] - s1;
            const int kp = one ? ipiv[k] : -ipiv[k] - 1;
            if (kp != k) { const T t = v[k]; v[k] = v[kp]; v[kp] = t; }
        }
        __syncwarp();
        k -= one ? 1 : 2;
    }
}

// y <- M y or M^T y, M = A^{-1} through the path's factors (the oracle's applyM); warp 0 only.
template <typename T>
AS_DEV void small_apply(SmallSmem<T>& sm, int n, int kind, bool upper, bool trans, T* v) {
    const int lane = threadIdx.x & 31;
    const int ld = n + 1;
    auto swaps_fwd = [&]() {               // v <- P v (interchanges in order)
        if (lane == 0)
            for (int j = 0; j < n; ++j) { const int p = sm.ipiv[j]; if (p != j) { const T t = v[j]; v[j] = v[p]; v[p] = t; } }
        __syncwarp();
    };
    auto swaps_bwd = [&]() {               // v <- P^T v
        if (lane == 0)
            for (int j = n - 1; j >= 0; --j) { const int p = sm.ipiv[j]; if (p != j) { const T t = v[j]; v[j] = v[p]; v[p] = t; } }
        __syncwarp();
    };
    switch (kind) {
    case KIND_LU:                           // xGECON: inv(U) inv(L) / inv(L^T) inv(U^T), no interchanges
        if (!trans) { warp_trsv(sm.W, ld, n, false, false, true, v); warp_trsv(sm.W, ld, n, true, false, false, v); }
        else { warp_trsv(sm.W, ld, n, true, true, false, v); warp_trsv(sm.W, ld, n, false, true, true, v); }
        break;
    case KIND_BAND:                         // xGBCON: with the interchanges (A^{-1} = U^{-1} L^{-1} P)
        if (!trans) { swaps_fwd(); warp_trsv(sm.W, ld, n, false, false, true, v); warp_trsv(sm.W, ld, n, true, false, false, v); }
        else { warp_trsv(sm.W, ld, n, true, true, false, v); warp_trsv(sm.W, ld, n, false, true, true, v); swaps_bwd(); }
        break;
    case KIND_TRI:
        warp_trsv(sm.W, ld, n, upper, trans, false, v);
        break;
    case KIND_LDLT:                         // xSYCON: symmetric, both kases through xSYTRS
        warp_sytrs(sm.W, ld, n, sm.ipiv, v);
        break;
    default:                                // KIND_CHOL: inv(L^T) inv(L)
        warp_trsv(sm.W, ld, n, false, false, false, v);
        warp_trsv(sm.W, ld, n, false, true, false, v);
        break;
    }
}

// xLACN2 (the oracle's lacn2, Z13b) on warp 0; returns est (valid on warp 0)
template <typename T>
AS_DEV T small_lacn2(SmallSmem<T>& sm, int n, int kind, bool upper) {
    const int lane = threadIdx.x & 31;
    T* x = sm.x;
    auto asum = [&]() { T s = T(0); for (int i = lane; i < n; i += 32) s += tabs(x[i]); s = warp_sum(s); return s; };
    auto iamax = [&]() {
        T bk = T(-1);
        int bi = 0x7fffffff;
        for (int i = lane; i < n; i += 32) { const T a = tabs(x[i]); if (a > bk) { bk = a; bi = i; } }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const T k2 = __shfl_xor_sync(0xffffffffu, bk, o);
            const int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
            if (k2 > bk || (k2 == bk && i2 < bi)) { bk = k2; bi = i2; }
        }
        return bi == 0x7fffffff ? 0 : bi;
    };
    for (int i = lane; i < n; i += 32) x[i] = T(1) / (T)n;
    __syncwarp();
    small_apply(sm, n, kind, upper, false, x);
    T est;
    if (n == 1) return tabs(x[0]);
    est = asum();
    for (int i = lane; i < n; i += 32) { x[i] = x[i] >= T(0) ? T(1) : T(-1); sm.isgn[i] = x[i] > T(0) ? 1 : -1; }
    __syncwarp();
    small_apply(sm, n, kind, upper, true, x);
    int j = iamax();
    int iter = 2;
    for (;;) {
        for (int i = lane; i < n; i += 32) x[i] = i == j ? T(1) : T(0);
        __syncwarp();
        small_apply(sm, n, kind, upper, false, x);
        const T estold = est;
        est = asum();
        bool same = true;
        for (int i = lane; i < n; i += 32) same &= (x[i] >= T(0) ? 1 : -1) == sm.isgn[i];
        same = __all_sync(0xffffffffu, same);
        if (same || est <= estold) break;
        for (int i = lane; i < n; i += 32) { x[i] = x[i] >= T(0) ? T(1) : T(-1); sm.isgn[i] = x[i] > T(0) ? 1 : -1; }
        __syncwarp();
        small_apply(sm, n, kind, upper, true, x);
        const int jlast = j;
        j = iamax();
        if (x[jlast] != tabs(x[j]) && iter < 5) { ++iter; continue; }
        break;
    }
    T alt = T(1);
    for (int i = 0; i < n; ++i) {          // (-1)^i (1 + i/(n-1)), every lane the same sign sequence
        if (i % 32 == lane) x[i] = alt * (T(1) + (T)i / (T)(n - 1));
        alt = -alt;
    }
    __syncwarp();
    small_apply(sm, n, kind, upper, false, x);
    const T temp = T(2) * (asum() / (T)(3 * n));
    return temp > est ? temp : est;
}

template <typename T>
AS_DEV T rcond_from(T anorm, T est) {
    if (!(anorm > T(0))) return T(0);
    if (est == T(0)) return T(0);
    return (T(1) / est) / anorm;
}

// copy A (global, original) into W
template <typename T>
AS_DEV void load_w(SmallSmem<T>& sm, const T* A, int64_t lda, int n) {
    for (int e = threadIdx.x; e < n * n; e += kSmallT) { const int i = e % n, j = e / n; sm.W[i + j * (n + 1)] = A[i + j * lda]; }
    __syncthreads();
}

// xGETF2 on W; returns info (1 + first zero pivot, 0 otherwise)
template <typename T>
AS_DEV int small_getrf(SmallSmem<T>& sm, int n) {
    const int ld = n + 1;
    int info = 0;
    for (int j = 0; j < n; ++j) {
        // the serial sweep (oracle getrf): start from |a_jj|, move only on a strictly larger |a_ij|:
        // the first maximum; a NaN never wins, a NaN at j keeps j
        T key = T(-1);
        int idx = 0x7fffffff;
        for (int i = j + threadIdx.x; i < n; i += kSmallT) {
            const T v = tabs(sm.W[i + j * ld]);
            if (v == v && v > key) { key = v; idx = i; }
        }
        int p = block_argmax(key, idx, sm.red, sm.ired);
        {
            const T d = sm.W[j + j * ld];
            if (d != d || p == 0x7fffffff) p = j;
        }
        if (threadIdx.x == 0) sm.ipiv[j] = p;
        const T pv = sm.W[p + j * ld];
        if (pv == T(0)) { if (info == 0) info = j + 1; __syncthreads(); continue; }
        if (p != j)
            for (int c = threadIdx.x; c < n; c += kSmallT) { const T t = sm.W[j + c * ld]; sm.W[j + c * ld] = sm.W[p + c * ld]; sm.W[p + c * ld] = t; }
        __syncthreads();
        const T piv = sm.W[j + j * ld];
        for (int i = j + 1 + threadIdx.x; i < n; i += kSmallT) sm.W[i + j * ld] = sm.W[i + j * ld] / piv;
        __syncthreads();
        const int m = n - j - 1;
        for (int e = threadIdx.x; e < m * m; e += kSmallT) {
            const int i = j + 1 + e % m, c = j + 1 + e / m;
            sm.W[i + c * ld] -= sm.W[i + j * ld] * sm.W[j + c * ld];
        }
        __syncthreads();
    }
    return info;
}

// Bunch-Kaufman xSYTF2 (lower) on W, the oracle's sytrf step by step; returns info (1 + first zero
// pivot column); ipiv as the oracle (1x1: kp; 2x2 at k, k+1: -(kp + 1) twice)
template <typename T>
AS_DEV int small_sytrf(SmallSmem<T>& sm, int n) {
    const int ld = n + 1;
    const T alpha = (T(1) + sqrt(T(17))) / T(8);
    int info = 0, k = 0;
    while (k < n) {
        int kstep = 1, kp = k;
        const T absakk = tabs(sm.W[k + k * ld]);
        T colmax = T(0);
        int imax = k;
        if (k < n - 1) {
            T key = T(-1);
            int idx = 0x7fffffff;
            for (int i = k + 1 + threadIdx.x; i < n; i += kSmallT) {
                const T v = tabs(sm.W[i + k * ld]);
                if (v == v && v > key) { key = v; idx = i; }
            }
            imax = block_argmax(key, idx, sm.red, sm.ired);
            if (imax == 0x7fffffff) imax = k + 1;
            colmax = tabs(sm.W[imax + k * ld]);
        }
        if ((absakk > colmax ? absakk : colmax) == T(0) || absakk != absakk) {
            if (info == 0) info = k + 1;
            kp = k;
        } else {
            if (absakk >= alpha * colmax) {
                kp = k;
            } else {
                T rm = T(0);
                for (int j = k + threadIdx.x; j < imax; j += kSmallT) rm = fmax(rm, tabs(sm.W[imax + j * ld]));
                for (int i = imax + 1 + threadIdx.x; i < n; i += kSmallT) rm = fmax(rm, tabs(sm.W[i + imax * ld]));
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) rm = fmax(rm, __shfl_xor_sync(0xffffffffu, rm, o));
                __syncthreads();
                if ((threadIdx.x & 31) == 0) sm.red[threadIdx.x >> 5] = rm;
                __syncthreads();
                T rowmax = T(0);
                for (int w = 0; w < kSmallWarps; ++w) rowmax = fmax(rowmax, sm.red[w]);
                if (absakk >= alpha * colmax * (colmax / rowmax)) kp = k;
                else if (tabs(sm.W[imax + imax * ld]) >= alpha * rowmax) kp = imax;
                else { kp = imax; kstep = 2; }
            }
            const int kk = k + kstep - 1;
            __syncthreads();
            if (kp != kk) {                 // interchange rows and columns kk and kp of A(k:n, k:n)
                for (int i = kp + 1 + threadIdx.x; i < n; i += kSmallT) {
                    const T t = sm.W[i + kk * ld]; sm.W[i + kk * ld] = sm.W[i + kp * ld]; sm.W[i + kp * ld] = t;
                }
                for (int j = kk + 1 + threadIdx.x; j < kp; j += kSmallT) {
                    const T t = sm.W[j + kk * ld]; sm.W[j + kk * ld] = sm.W[kp + j * ld]; sm.W[kp + j * ld] = t;
                }
                if (threadIdx.x == 0) {
                    T t = sm.W[kk + kk * ld]; sm.W[kk + kk * ld] = sm.W[kp + kp * ld]; sm.W[kp + kp * ld] = t;
                    if (kstep == 2) { t = sm.W[(k + 1) + k * ld]; sm.W[(k + 1) + k * ld] = sm.W[kp + k * ld]; sm.W[kp + k * ld] = t; }
                }
            }
            __syncthreads();
            if (kstep == 1) {
                if (k < n - 1) {            // A := A - d11 x x^T (lower), x *= d11
                    const T d11 = T(1) / sm.W[k + k * ld];
                    const int m = n - k - 1;
                    for (int e = threadIdx.x; e < m * m; e += kSmallT) {
                        const int i = k + 1 + e % m, j = k + 1 + e / m;
                        if (i >= j) sm.W[i + j * ld] = sm.W[i + j * ld] + sm.W[i + k * ld] * (-d11 * sm.W[j + k * ld]);
                    }
                    __syncthreads();
                    for (int i = k + 1 + threadIdx.x; i < n; i += kSmallT) sm.W[i + k * ld] = d11 * sm.W[i + k * ld];
                }
            } else if (k < n - 2) {
                T d21 = sm.W[(k + 1) + k * ld];
                const T d11 = sm.W[(k + 1) + (k + 1) * ld] / d21;
                const T d22 = sm.W[k + k * ld] / d21;
                const T t = T(1) / (d11 * d22 - T(1));
                d21 = t / d21;
                for (int j = k + 2 + threadIdx.x; j < n; j += kSmallT) {
                    sm.x[j] = d21 * (d11 * sm.W[j + k * ld] - sm.W[j + (k + 1) * ld]);
                    sm.y[j] = d21 * (d22 * sm.W[j + (k + 1) * ld] - sm.W[j + k * ld]);
                }
                __syncthreads();
                const int m = n - k - 2;
                for (int e = threadIdx.x; e < m * m; e += kSmallT) {
                    const int i = k + 2 + e % m, j = k + 2 + e / m;
                    if (i >= j) sm.W[i + j * ld] = sm.W[i + j * ld] - sm.W[i + k * ld] * sm.x[j] - sm.W[i + (k + 1) * ld] * sm.y[j];
                }
                __syncthreads();
                for (int j = k + 2 + threadIdx.x; j < n; j += kSmallT) { sm.W[j + k * ld] = sm.x[j]; sm.W[j + (k + 1) * ld] = sm.y[j]; }
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            if (kstep == 1) sm.ipiv[k] = kp;
            else { sm.ipiv[k] = -(kp + 1); sm.ipiv[k + 1] = -(kp + 1); }
        }
        __syncthreads();
        k += kstep;
    }
    return info;
}

// xPOTF2 (lower, right-looking) on W; returns 1 + failing column, 0 on success
template <typename T>
AS_DEV int small_potrf(SmallSmem<T>& sm, int n) {
    const int ld = n + 1;
    for (int j = 0; j < n; ++j) {
        const T d = sm.W[j + j * ld];
        if (!(d > T(0))) return j + 1;
        const T ljj = sqrt(d);
        __syncthreads();
        if (threadIdx.x == 0) sm.W[j + j * ld] = ljj;
        for (int i = j + 1 + threadIdx.x; i < n; i += kSmallT) sm.W[i + j * ld] = sm.W[i + j * ld] / ljj;
        __syncthreads();
        const int m = n - j - 1;
        for (int e = threadIdx.x; e < m * m; e += kSmallT) {
            const int i = j + 1 + e % m, k = j + 1 + e / m;
            if (i >= k) sm.W[i + k * ld] -= sm.W[i + j * ld] * sm.W[k + j * ld];
        }
        __syncthreads();
    }
    return 0;
}

// ------------------------------------------------------------------ the kernel
template <typename T>
__global__ void __launch_bounds__(kSmallT, 1) small_solve_kernel(SmallArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SmallSmem<T>& sm = *(SmallSmem<T>*)smem_raw;
    const int64_t b = blockIdx.x;
    const int n = a.n, nrhs = a.nrhs, ld = n + 1;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const T* A = (const T*)a.A + b * a.sA;
    const T* B = (const T*)a.B + b * a.sB;
    T* X = (T*)a.X + b * a.sX;
    const T eps = Eps<T>::v;

    // ---- detection: every element is read here anyway -> exact kl / ku
    if (tid == 0) { sm.kl = 0; sm.ku = 0; sm.flags = 0; sm.nonfinite = 0; sm.spd_dead = 0; sm.rot = 0; sm.asym = 0; }
    __syncthreads();
    {
        int kl = 0, ku = 0, f = 0;
        bool bad = false;
        for (int e = tid; e < n * n; e += kSmallT) {
            const int i = e % n, j = e / n;
            const T v = A[i + j * a.lda];
            sm.W[i + j * ld] = v;
            bad |= !is_finite_val(v);
            if (v != T(0)) {                                   // Z1: IEEE non-zero
                if (i > j) { kl = max(kl, i - j); f |= 1; }   // something below the diagonal
                else if (i < j) { ku = max(ku, j - i); f |= 2; }
            }
        }
        if (a.opts & AS_OPT_CHECK_FINITE)
            for (int e = tid; e < n * nrhs; e += kSmallT) bad |= !is_finite_val(B[e % n + (e / n) * a.ldb]);
        kl = __reduce_max_sync(0xffffffffu, kl);
        ku = __reduce_max_sync(0xffffffffu, ku);
        f = __reduce_or_sync(0xffffffffu, f);
        bad = __any_sync(0xffffffffu, bad);
        if (lane == 0) { atomicMax(&sm.kl, kl); atomicMax(&sm.ku, ku); atomicOr(&sm.flags, f); if (bad) sm.nonfinite = 1; }
    }
    __syncthreads();
    // Fig. 4 with its printed operators (Z7): pass 1 on the diagonal, pass 2 on pairs
    {
        T md = T(0);
        bool dead = false;
        for (int j = tid; j < n; j += kSmallT) {
            const T d = sm.W[j + j * ld];
            if (d <= T(0)) dead = true;                                   // line 8
            if (d > md) md = d;                                           // line 9
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) { const T o2 = __shfl_xor_sync(0xffffffffu, md, o); if (o2 > md) md = o2; }
        dead = __any_sync(0xffffffffu, dead);
        if (lane == 0) sm.red[warp] = md;
        if (lane == 0 && dead) sm.spd_dead = 1;
        __syncthreads();
        if (tid == 0) {
            T m = T(0);
            for (int w = 0; w < kSmallWarps; ++w) if (sm.red[w] > m) m = sm.red[w];
            sm.max_diag = m;
        }
        __syncthreads();
        const T max_diag = sm.max_diag;
        const T tol = T(100) * eps;                                       // line 5
        dead = false;
        if (!sm.spd_dead)
            for (int e = tid; e < n * n; e += kSmallT) {
                const int i = e % n, j = e / n;
                if (i <= j) continue;
                const T aij = sm.W[i + j * ld], aji = sm.W[j + i * ld];
                const T aa = aij < T(0) ? -aij : aij, ab = aji < T(0) ? -aji : aji;
                const T df = aij - aji;
                const T delta = df < T(0) ? -df : df;                     // line 12
                const T m = aa > ab ? aa : ab;
                if (delta > tol && delta > tol * m) dead = true;           // lines 13-14
                if (aa >= max_diag) dead = true;                          // line 15
                if (aa + ab >= sm.W[i + i * ld] + sm.W[j + j * ld]) dead = true;   // line 16
            }
        dead = __any_sync(0xffffffffu, dead);
        if (lane == 0 && dead) sm.spd_dead = 1;
        if (a.opts & AS_OPT_SYM_INDEF) {                                  // exact symmetry (Z30)
            bool asym = false;
            for (int e = tid; e < n * n; e += kSmallT) {
                const int i = e % n, j = e / n;
                if (i > j && !(sm.W[i + j * ld] == sm.W[j + i * ld])) asym = true;
            }
            asym = __any_sync(0xffffffffu, asym);
            if (lane == 0 && asym) sm.asym = 1;
        }
    }
    __syncthreads();
    const int kl = sm.kl, ku = sm.ku;
    const bool sym = (a.opts & AS_OPT_SYM_INDEF) && !sm.asym;
    unsigned det = 0;
    if (band_density_ok(n, kl, ku)) det |= AS_FLAG_BANDED;                // P:339, Z2/Z3
    if (!(sm.flags & 2)) det |= AS_FLAG_LOWER;
    if (!(sm.flags & 1)) det |= AS_FLAG_UPPER;
    if (!sm.spd_dead) det |= AS_FLAG_SPD_CANDIDATE;
    int method;
    if (a.opts & AS_OPT_FORCE_METHOD) method = a.force;
    else if (det & AS_FLAG_BANDED) method = AS_METHOD_BAND;
    else if (det & AS_FLAG_LOWER) method = AS_METHOD_TRI_LOWER;
    else if (det & AS_FLAG_UPPER) method = AS_METHOD_TRI_UPPER;
    else if (det & AS_FLAG_SPD_CANDIDATE) method = AS_METHOD_CHOL;
    else if (sym) method = AS_METHOD_LDLT;
    else method = AS_METHOD_LU;
    const bool fullscan = (a.opts & (AS_OPT_FULLSCAN | AS_OPT_FORCE_METHOD)) != 0;

    uint32_t flags = det | (sym ? AS_FLAG_SYMMETRIC : 0u);
    int32_t ret = AS_OK;
    int primary = method;
    double rcond = 0.0, anorm_out = 0.0;
    int64_t info = 0, chol_col = 0, rank = -1;
    int sweeps = 0;
    bool run_fallback = false, write_primary = false;

    if ((a.opts & AS_OPT_CHECK_FINITE) && sm.nonfinite) {                // Z28
        flags |= AS_FLAG_NONFINITE;
        ret = AS_ERR_NONFINITE;
        method = primary = AS_METHOD_NONE;
    } else {
        // ---- anorm (of the original A: triangle for TRI, everything else the full 1-norm)
        T anorm = T(0);
        {
            const bool tri = method == AS_METHOD_TRI_LOWER || method == AS_METHOD_TRI_UPPER;
            const bool up = method == AS_METHOD_TRI_UPPER;
            T best = T(0);
            for (int j = warp; j < n; j += kSmallWarps) {
                T s = T(0);
                for (int i = lane; i < n; i += 32)
                    if (!tri || (up ? i <= j : i >= j)) s += tabs(sm.W[i + j * ld]);
                s = warp_sum(s);
                if (s > best || s != s) best = s;
            }
            if (lane == 0) sm.red[warp] = best;
            __syncthreads();
            for (int w = 0; w < kSmallWarps; ++w) { const T v = sm.red[w]; if (v > anorm || v != v) anorm = v; }
            __syncthreads();
        }
        int kind = KIND_LU;
        bool upper = false, singular = false;
        if (method == AS_METHOD_TRI_LOWER || method == AS_METHOD_TRI_UPPER) {
            kind = KIND_TRI;
            upper = method == AS_METHOD_TRI_UPPER;
            for (int j = 0; j < n; ++j) if (sm.W[j + j * ld] == T(0)) { info = j + 1; break; }
            singular = info != 0;
        } else if (method == AS_METHOD_CHOL) {
            const int f = small_potrf(sm, n);
            if (f) {                                                      // general LU
                flags |= AS_FLAG_CHOL_FAILED;                             // (Z30: LDL^T if exactly symmetric)
                chol_col = f - 1;
                method = primary = sym ? AS_METHOD_LDLT : AS_METHOD_LU;
                __syncthreads();
                load_w(sm, A, a.lda, n);
            } else {
                kind = KIND_CHOL;
            }
        }
        if (method == AS_METHOD_LDLT) {
            kind = KIND_LDLT;
            info = small_sytrf(sm, n);
            singular = info != 0;
        }
        if (method == AS_METHOD_LU || method == AS_METHOD_BAND) {
            kind = method == AS_METHOD_BAND ? KIND_BAND : KIND_LU;
            info = small_getrf(sm, n);
            singular = info != 0;
        }
        __syncthreads();
        T rc = T(0);
        if (!singular) {
            T est = T(0);
            if (warp == 0) est = small_lacn2(sm, n, kind, upper);
            if (tid == 0) sm.red[0] = est;
            __syncthreads();
            est = sm.red[0];
            rc = rcond_from(anorm, est);
        }
        __syncthreads();
        anorm_out = (double)anorm;
        rcond = singular ? 0.0 : (double)rc;
        if (singular) flags |= AS_FLAG_SINGULAR;
        const T thr = (T)a.thr;
        const bool gate = singular || !(rc >= thr);                       // Z11
        if (gate) {
            flags |= AS_FLAG_RCOND_LOW;
            if (a.opts & AS_OPT_NO_FALLBACK) {
                if (singular) ret = AS_ERR_SINGULAR_NO_FALLBACK;
                else { flags |= AS_FLAG_POORLY_COND; write_primary = true; }
            } else {
                run_fallback = true;
            }
        } else {
            write_primary = true;
        }
        // ---- primary solve, one right-hand side per warp (X = M B)
        if (write_primary) {
            for (int c = warp; c < nrhs; c += kSmallWarps) {
                T* v = warp == 0 ? sm.x : (warp == 1 ? sm.y : (warp == 2 ? sm.z : nullptr));
                // warps 3.. use the fallback's Y area as vectors (not needed on this path)
                if (!v) v = sm.Y + (warp - 3) * kSmallN;
                for (int i = lane; i < n; i += 32) v[i] = B[i + (int64_t)c * a.ldb];
                __syncwarp();
                if (kind == KIND_LU) {             // xGETRS: P b, then L, then U
                    if (lane == 0)
                        for (int j = 0; j < n; ++j) { const int p = sm.ipiv[j]; if (p != j) { const T t = v[j]; v[j] = v[p]; v[p] = t; } }
                    __syncwarp();
                    warp_trsv(sm.W, ld, n, false, false, true, v);
                    warp_trsv(sm.W, ld, n, true, false, false, v);
                } else {
                    small_apply(sm, n, kind, upper, false, v);
                }
                for (int i = lane; i < n; i += 32) X[i + (int64_t)c * a.ldx] = v[i];
                __syncwarp();
            }
        }
        __syncthreads();
        if (run_fallback) {
            // ---- SVD minimum-norm fallback on the original A
            flags |= AS_FLAG_FALLBACK;
            method = AS_METHOD_SVD;
            load_w(sm, A, a.lda, n);
            for (int e = tid; e < n * nrhs; e += kSmallT) sm.Y[e] = B[e % n + (int64_t)(e / n) * a.ldb];
            __syncthreads();
            // (1) Householder QR, C = Q^T B (xGEQR2 / xLARFG as the oracle)
            for (int j = 0; j < n; ++j) {
                T ss = T(0);
                for (int i = j + 1 + tid; i < n; i += kSmallT) ss += sm.W[i + j * ld] * sm.W[i + j * ld];
                ss = block_sum(ss, sm.red);
                const T xnorm = sqrt(ss);
                const T alpha = sm.W[j + j * ld];
                __syncthreads();
                if (xnorm == T(0)) continue;
                const T aa = tabs(alpha), wv = aa > xnorm ? aa : xnorm, zv = aa > xnorm ? xnorm : aa;
                const T hyp = wv * sqrt(T(1) + (zv / wv) * (zv / wv));
                const T beta = alpha >= T(0) ? -hyp : hyp;
                const T tau = (beta - alpha) / beta;
                const T scal = T(1) / (alpha - beta);
                for (int i = j + 1 + tid; i < n; i += kSmallT) sm.x[i] = sm.W[i + j * ld] * scal;
                if (tid == 0) { sm.x[j] = T(1); sm.W[j + j * ld] = beta; }
                __syncthreads();
                for (int i = j + 1 + tid; i < n; i += kSmallT) sm.W[i + j * ld] = T(0);
                for (int k = j + 1 + warp; k < n + nrhs; k += kSmallWarps) {
                    T* col = k < n ? sm.W + k * ld : sm.Y + (k - n) * n;
                    T s = T(0);
                    for (int i = j + lane; i < n; i += 32) s += sm.x[i] * col[i];
                    s = warp_sum(s) * tau;
                    for (int i = j + lane; i < n; i += 32) col[i] = col[i] - s * sm.x[i];
                }
                __syncthreads();
            }
            // (2) M = R^T (in place) and one-sided Jacobi, round-robin pairs
            for (int e = tid; e < n * n; e += kSmallT) {
                const int i = e % n, j = e / n;
                if (i > j) { sm.W[i + j * ld] = sm.W[j + i * ld]; sm.W[j + i * ld] = T(0); }
            }
            __syncthreads();
            const T tol = (T)n * eps;
            const int n2 = n + (n & 1), npairs = n2 / 2, rounds = n2 - 1;
            bool conv = false;
            while (sweeps < a.max_sweeps) {
                ++sweeps;
                if (tid == 0) sm.rot = 0;
                __syncthreads();
                int myrot = 0;
                for (int r = 0; r < rounds; ++r) {
                    for (int k = warp; k < npairs; k += kSmallWarps) {
                        const int s1 = k, s2 = n2 - 1 - k;
                        const int pa = s1 == 0 ? 0 : 1 + (s1 - 1 + r) % (n2 - 1);
                        const int pb = s2 == 0 ? 0 : 1 + (s2 - 1 + r) % (n2 - 1);
                        if (pa >= n || pb >= n) continue;
                        const int p = pa < pb ? pa : pb, q = pa < pb ? pb : pa;
                        T* mp = sm.W + p * ld;
                        T* mq = sm.W + q * ld;
                        T al = T(0), be = T(0), ga = T(0);
                        for (int i = lane; i < n; i += 32) { const T u = mp[i], v = mq[i]; al += u * u; be += v * v; ga += u * v; }
                        al = warp_sum(al); be = warp_sum(be); ga = warp_sum(ga);
                        if (ga == T(0) || !(tabs(ga) > tol * sqrt(al) * sqrt(be))) continue;
                        ++myrot;
                        const T zeta = (be - al) / (T(2) * ga);
                        const T t = (zeta >= T(0) ? T(1) : T(-1)) / (tabs(zeta) + sqrt(T(1) + zeta * zeta));
                        const T c = T(1) / sqrt(T(1) + t * t);
                        const T s = c * t;
                        for (int i = lane; i < n; i += 32) { const T u = mp[i], v = mq[i]; mp[i] = c * u - s * v; mq[i] = s * u + c * v; }
                        for (int rr = lane; rr < nrhs; rr += 32) {
                            const T u = sm.Y[p + rr * n], v = sm.Y[q + rr * n];
                            sm.Y[p + rr * n] = c * u - s * v;
                            sm.Y[q + rr * n] = s * u + c * v;
                        }
                        __syncwarp();
                    }
                    __syncthreads();
                }
                if (lane == 0 && myrot) atomicAdd(&sm.rot, myrot);
                __syncthreads();
                if (sm.rot == 0) { conv = true; break; }
                __syncthreads();
            }
            // (3) sigma_k = ||m_k||, rank, sigma_max
            for (int k = warp; k < n; k += kSmallWarps) {
                T s = T(0);
                for (int i = lane; i < n; i += 32) s += sm.W[i + k * ld] * sm.W[i + k * ld];
                s = warp_sum(s);
                if (lane == 0) sm.sig[k] = sqrt(s);
            }
            __syncthreads();
            T smax = T(0);
            bool bad = false;
            for (int k = 0; k < n; ++k) { const T v = sm.sig[k]; if (v > smax) smax = v; bad |= !is_finite_val(v); }
            const T cut = (T)a.cut;
            if (bad) {                                                    // Z29
                flags |= AS_FLAG_NONFINITE;
                ret = AS_ERR_NONFINITE;
                rank = -1;
            } else {
                int64_t kept = 0;
                for (int k = 0; k < n; ++k) kept += sm.sig[k] > cut * smax;
                rank = kept;
                if (rank < n) flags |= AS_FLAG_RANK_DEF;
                if (!conv) { flags |= AS_FLAG_SVD_NOCONV; ret = AS_ERR_SVD_NOT_CONVERGED; }
                // (4) x = sum_kept m_k y_k / sigma_k^2
                for (int e = tid; e < n * nrhs; e += kSmallT) {
                    const int i = e % n, r = e / n;
                    T acc = T(0);
                    for (int k = 0; k < n; ++k) {
                        const T sk = sm.sig[k];
                        if (!(sk > cut * smax)) continue;
                        acc += sm.W[i + k * ld] * (sm.Y[k + r * n] / (sk * sk));
                    }
                    X[i + (int64_t)r * a.ldx] = acc;
                }
                if (a.sigma) {                                            // descending, stable
                    T* so = (T*)a.sigma + b * a.sS;
                    for (int k = tid; k < n; k += kSmallT) {
                        const T sk = sm.sig[k];
                        int pos = 0;
                        for (int j = 0; j < n; ++j) { const T sj = sm.sig[j]; pos += (sj > sk || (sj == sk && j < k)); }
                        so[pos] = sk;
                    }
                }
            }
        }
    }
    if (tid == 0) {
        if (a.rep) {
            as_report r;
            r.flags = flags | ((unsigned)method << AS_FLAG_METHOD_SHIFT);
            r.method = method;
            r.primary_method = primary;
            r.sweeps = sweeps;
            const bool banded = (det & AS_FLAG_BANDED) || primary == AS_METHOD_BAND;
            r.kl = (banded || fullscan) ? kl : -1;
            r.ku = (banded || fullscan) ? ku : -1;
            r.rcond = rcond;
            r.anorm = anorm_out;
            r.rank = (flags & AS_FLAG_FALLBACK) ? rank : -1;
            r.info = info;
            r.chol_fail_col = chol_col;
            a.rep[b] = r;
        }
        if (a.ret) a.ret[b] = ret;
    }
}

}  // namespace

size_t small_smem_bytes(int dtype) { return dtype == AS_F64 ? sizeof(SmallSmem<double>) : sizeof(SmallSmem<float>); }

int launch_small_batched(int dtype, const SmallArgs& a, cudaStream_t s) {
    if (a.batch <= 0) return 0;
    const size_t smem = small_smem_bytes(dtype);
    void* kern = dtype == AS_F64 ? (void*)small_solve_kernel<double> : (void*)small_solve_kernel<float>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int64_t b0 = 0; b0 < a.batch; b0 += 0x7fffffff) {
        SmallArgs c = a;
        const int64_t nb = std::min<int64_t>(a.batch - b0, 0x7fffffff);
        const size_t es = dtype == AS_F64 ? 8 : 4;
        c.A = (const char*)a.A + b0 * a.sA * es;
        c.B = (const char*)a.B + b0 * a.sB * es;
        c.X = (char*)a.X + b0 * a.sX * es;
        if (c.rep) c.rep += b0;
        if (c.ret) c.ret += b0;
        if (c.sigma) c.sigma = (char*)a.sigma + b0 * a.sS * es;
        c.batch = nb;
        void* args[] = {&c};
        const cudaError_t e = cudaLaunchKernel(kern, dim3((unsigned)nb), dim3(kSmallT), args, smem, s);
        if (e != cudaSuccess) return AS_ERR_CUDA_BASE + (int)e;
    }
    return 0;
}

}  // namespace as
