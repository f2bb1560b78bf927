/*
 * oracle_impl.h -- TEST INFRASTRUCTURE ONLY.  Plain, slow, unblocked CPU
 * implementation of the adaptive solve of A X = B from
 *   C. Sanderson, R. Curtin, "An Adaptive Solver for Systems of Linear
 *   Equations" (arXiv 2007.11208), /root/reference/PAPER.md (cited as P:<line>).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * use this code.  It shares nothing with the CUDA path
 * (paper_2007_11208_b200/csrc); neither includes the other.
 *
 * This file is included twice by oracle.c, once with T=double and once with
 * T=float (a poor man's template).  Every operation is done in T.
 * Column-major storage: element (i,j) of A is A[i + j*lda], zero-based
 * (Fig. 4 caption).  Readings of the paper where it is silent are
 * tagged Z<k> and listed in DESIGN.md ("Readings of the paper").
 *
 * Parallelism: OpenMP only over independent columns of a rank-1 update or
 * a reflector application, where each output element's operation order is
 * independent of the thread count -> results are bitwise identical for any
 * number of threads (tested).
 */

/* ------------------------------------------------------------------ */
/* constants (P:441-443 footnote: eps = gap between 1 and next value)  */
/* ------------------------------------------------------------------ */
static T FN(eps)(void) { return NEXTAFTER((T)1, (T)2) - (T)1; }

/* ------------------------------------------------------------------ */
/* Detection                                                           */
/* ------------------------------------------------------------------ */

/* Band extent by the paper's per-column scan, P:328-337 (Sec. II-A):
 *  ku: traverse column j from the top to the diagonal, note the distance of
 *      the first non-zero above-or-on the diagonal; max over columns.
 *  kl: traverse from the diagonal to the bottom, note the distance of the
 *      last non-zero; max over columns.
 * "non-zero" is IEEE a != 0 (Z1).  The paper's early stop only
 * saves work, never changes the verdict (kl, ku only grow), so the oracle
 * scans everything and applies the 25% rule afterwards (Z2, Z3). */
static void FN(band_extent)(const T* A, int64_t lda, int64_t n, int64_t* kl_out, int64_t* ku_out)
{
    int64_t kl = 0, ku = 0;
    for (int64_t j = 0; j < n; ++j) {
        const T* col = A + j * lda;
        for (int64_t i = 0; i <= j; ++i) {          /* top -> diagonal */
            if (col[i] != (T)0) { if (j - i > ku) ku = j - i; break; }
        }
        for (int64_t i = n - 1; i >= j; --i) {      /* bottom -> diagonal: last non-zero */
            if (col[i] != (T)0) { if (i - j > kl) kl = i - j; break; }
        }
    }
    *kl_out = kl; *ku_out = ku;
}

/* Fig. 4, likely_sympd, literally: lines 5-17 with the printed
 * operators (Z7); loop order j outer, i inner as printed. */
static int FN(likely_sympd)(const T* A, int64_t lda, int64_t n, T* max_diag_out)
{
    const T tol = (T)100 * FN(eps)();                      /* line 5 */
    T max_diag = (T)0;                                     /* line 6 */
    for (int64_t j = 0; j < n; ++j) {                      /* line 7 */
        const T ajj = A[j + j * lda];
        if (ajj <= (T)0) { *max_diag_out = max_diag; return 0; }   /* line 8 */
        if (ajj > max_diag) max_diag = ajj;                /* line 9 */
    }
    *max_diag_out = max_diag;
    for (int64_t j = 0; j + 1 < n; ++j) {                  /* line 10 */
        for (int64_t i = j + 1; i < n; ++i) {              /* line 11 */
            const T aij = A[i + j * lda], aji = A[j + i * lda];
            const T delta = ABS(aij - aji);                /* line 12 */
            const T m = ABS(aij) > ABS(aji) ? ABS(aij) : ABS(aji);
            if (delta > tol && delta > tol * m) return 0;  /* lines 13-14 */
            if (ABS(aij) >= max_diag) return 0;            /* line 15 */
            if ((ABS(aij) + ABS(aji)) >= (A[i + i * lda] + A[j + j * lda])) return 0;  /* line 16 */
        }
    }
    return 1;                                              /* line 17 */
}

/* Triangular detection: "If all elements above the main diagonal
 * are zero, a lower triangular matrix is present.  Conversely, if all
 * elements below the main diagonal are zero, an upper triangular matrix".
 * Exact zero, no tolerance (Z6). */
static int FN(is_lower)(const T* A, int64_t lda, int64_t n)
{
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i < j; ++i)
            if (A[i + j * lda] != (T)0) return 0;
    return 1;
}
static int FN(is_upper)(const T* A, int64_t lda, int64_t n)
{
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = j + 1; i < n; ++i)
            if (A[i + j * lda] != (T)0) return 0;
    return 1;
}

/* Exact symmetry, A_ij == A_ji for every pair (IEEE compare: a NaN breaks it).  Evaluated only
 * for the symmetric-indefinite specialisation the paper names as future work, which
 * is an option (OR_OPT_SYM_INDEF, Z30). */
static int FN(is_symmetric)(const T* A, int64_t lda, int64_t n)
{
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = j + 1; i < n; ++i)
            if (!(A[i + j * lda] == A[j + i * lda])) return 0;
    return 1;
}

/* Band capacity count(n,kl,ku) = n(kl+ku+1) - kl(kl+1)/2 - ku(ku+1)/2 and
 * the 25% rule of P:339 ("more than 25% ... non-zero" -> non-banded):
 * banded <=> 4*count <= n^2, exact integer arithmetic (Z2, Z3). */
static int FN(band_density_ok)(int64_t n, int64_t kl, int64_t ku)
{
    uint64_t un = (uint64_t)n;
    uint64_t cnt = un * (uint64_t)(kl + ku + 1) - (uint64_t)(kl * (kl + 1) / 2) - (uint64_t)(ku * (ku + 1) / 2);
    return 4u * cnt <= un * un;
}

/* Every element of the m x n column-major array finite?  Z28:
 * SPEC S:91 / S:409 reject NaN/Inf input at solve entry; the paper asks for
 * robustness to floating-point limits.  isfinite() of C99. */
static int FN(all_finite)(const T* A, int64_t lda, int64_t m, int64_t n)
{
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i < m; ++i)
            if (!isfinite(A[i + j * lda])) return 0;
    return 1;
}

/* ------------------------------------------------------------------ */
/* Norms                                                               */
/* ------------------------------------------------------------------ */
/* 1-norm (max column sum) of the full stored matrix (Z13b). */
static T FN(norm1_full)(const T* A, int64_t lda, int64_t n)
{
    T best = (T)0;
    for (int64_t j = 0; j < n; ++j) {
        T s = (T)0;
        for (int64_t i = 0; i < n; ++i) s += ABS(A[i + j * lda]);
        if (s > best || s != s) best = s;
    }
    return best;
}
/* 1-norm of the lower (uplo=0) or upper (uplo=1) triangle incl. diagonal. */
static T FN(norm1_tri)(const T* A, int64_t lda, int64_t n, int upper)
{
    T best = (T)0;
    for (int64_t j = 0; j < n; ++j) {
        T s = (T)0;
        int64_t i0 = upper ? 0 : j, i1 = upper ? j : n - 1;
        for (int64_t i = i0; i <= i1; ++i) s += ABS(A[i + j * lda]);
        if (s > best || s != s) best = s;
    }
    return best;
}

/* ------------------------------------------------------------------ */
/* Banded LU: compact band storage, xGBTRF / xGBTRS*/
/* ------------------------------------------------------------------ */
/* LAPACK band layout with kl fill rows (Z12): ldab = 2kl+ku+1,
 * ab[kl+ku+i-j, j] = A[i,j] for max(0,j-ku) <= i <= min(n-1,j+kl).
 * Returns the band 1-norm. */
static T FN(band_pack)(const T* A, int64_t lda, int64_t n, int64_t kl, int64_t ku, T* ab, int64_t ldab)
{
    T anorm = (T)0;
    for (int64_t j = 0; j < n; ++j) {
        for (int64_t r = 0; r < ldab; ++r) ab[r + j * ldab] = (T)0;
        int64_t i0 = j - ku > 0 ? j - ku : 0;
        int64_t i1 = j + kl < n - 1 ? j + kl : n - 1;
        T s = (T)0;
        for (int64_t i = i0; i <= i1; ++i) {
            ab[kl + ku + i - j + j * ldab] = A[i + j * lda];
            s += ABS(A[i + j * lda]);
        }
        if (s > anorm || s != s) anorm = s;
    }
    return anorm;
}

#define AB(r, c) ab[(r) + (c) * ldab]

/* Unblocked banded LU with partial pivoting (the xGBTF2 algorithm behind
 * xGBTRF).  Row i, column c of A lives at AB(kv+i-c, c).
 * Pivot = first max |.| among rows j..j+km (Z15); multipliers by division.
 * Returns 0, or 1+j for the first exactly-zero pivot (singular). */
static int64_t FN(gbtrf)(int64_t n, int64_t kl, int64_t ku, T* ab, int64_t ldab, int64_t* ipiv)
{
    const int64_t kv = kl + ku;
    int64_t info = 0, ju = 0;
    for (int64_t j = 0; j < n; ++j) {
        int64_t km = kl < n - 1 - j ? kl : n - 1 - j;
        int64_t jp = 0;
        T best = ABS(AB(kv, j));
        for (int64_t r = 1; r <= km; ++r)
            if (ABS(AB(kv + r, j)) > best) { best = ABS(AB(kv + r, j)); jp = r; }
        ipiv[j] = j + jp;
        if (AB(kv + jp, j) != (T)0) {
            int64_t lim = j + ku + jp < n - 1 ? j + ku + jp : n - 1;
            if (lim > ju) ju = lim;
            if (jp != 0)                                     /* swap rows j and j+jp, columns j..ju */
                for (int64_t c = j; c <= ju; ++c) {
                    T t = AB(kv + j + jp - c, c);
                    AB(kv + j + jp - c, c) = AB(kv + j - c, c);
                    AB(kv + j - c, c) = t;
                }
            const T piv = AB(kv, j);
            for (int64_t r = 1; r <= km; ++r) AB(kv + r, j) = AB(kv + r, j) / piv;
            for (int64_t c = j + 1; c <= ju; ++c) {           /* rank-1 update of the km x (ju-j) block */
                const T u = AB(kv + j - c, c);
                for (int64_t r = 1; r <= km; ++r)
                    AB(kv + j + r - c, c) = AB(kv + j + r - c, c) - AB(kv + r, j) * u;
            }
        } else if (info == 0) {
            info = j + 1;
        }
    }
    return info;
}

/* xGBTRS 'N': apply L with the interleaved interchanges, then
 * back-substitute with U (upper bandwidth kl+ku).  b is overwritten. */
static void FN(gbtrs_vec)(int64_t n, int64_t kl, int64_t ku, const T* ab, int64_t ldab, const int64_t* ipiv, T* b)
{
    const int64_t kv = kl + ku;
    for (int64_t j = 0; j + 1 < n; ++j) {
        int64_t lm = kl < n - 1 - j ? kl : n - 1 - j;
        int64_t l = ipiv[j];
        if (l != j) { T t = b[l]; b[l] = b[j]; b[j] = t; }
        for (int64_t r = 1; r <= lm; ++r) b[j + r] = b[j + r] - AB(kv + r, j) * b[j];
    }
    for (int64_t j = n - 1; j >= 0; --j) {
        b[j] = b[j] / AB(kv, j);
        int64_t i0 = j - kv > 0 ? j - kv : 0;
        for (int64_t i = i0; i < j; ++i) b[i] = b[i] - AB(kv + i - j, j) * b[j];
    }
}
/* A^T x = b with the band LU (used by the xGBCON estimator): U^T forward,
 * then L^T backward with the interchanges undone in reverse order. */
static void FN(gbtrs_vec_t)(int64_t n, int64_t kl, int64_t ku, const T* ab, int64_t ldab, const int64_t* ipiv, T* b)
{
    const int64_t kv = kl + ku;
    for (int64_t j = 0; j < n; ++j) {
        int64_t i0 = j - kv > 0 ? j - kv : 0;
        T s = b[j];
        for (int64_t i = i0; i < j; ++i) s = s - AB(kv + i - j, j) * b[i];
        b[j] = s / AB(kv, j);
    }
    for (int64_t j = n - 2; j >= 0; --j) {
        int64_t lm = kl < n - 1 - j ? kl : n - 1 - j;
        T s = b[j];
        for (int64_t r = 1; r <= lm; ++r) s = s - AB(kv + r, j) * b[j + r];
        b[j] = s;
        int64_t l = ipiv[j];
        if (l != j) { T t = b[l]; b[l] = b[j]; b[j] = t; }
    }
}
#undef AB

/* ------------------------------------------------------------------ */
/* Triangular solve, Eq. (3), back-substitution */
/* ------------------------------------------------------------------ */
/* Solves op(T) x = b in place; upper selects the stored triangle; trans
 * solves with the transpose (for xTRCON's estimator); unit ignores
 * the stored diagonal (the unit-lower L of the LU). */
static void FN(trsv)(const T* A, int64_t lda, int64_t n, int upper, int trans, int unit, T* b)
{
    /* effective lower <=> (lower && !trans) || (upper && trans) */
    int eff_lower = (!upper && !trans) || (upper && trans);
#define OP(i, j) (trans ? A[(j) + (i) * lda] : A[(i) + (j) * lda])
    if (eff_lower) {                   /* Eq. (3): x_i = (b_i - sum_{j<i} a_ij x_j) / a_ii */
        for (int64_t i = 0; i < n; ++i) {
            T s = b[i];
            for (int64_t j = 0; j < i; ++j) s = s - OP(i, j) * b[j];
            b[i] = unit ? s : s / OP(i, i);
        }
    } else {                           /* back-substitution: x_n first */
        for (int64_t i = n - 1; i >= 0; --i) {
            T s = b[i];
            for (int64_t j = i + 1; j < n; ++j) s = s - OP(i, j) * b[j];
            b[i] = unit ? s : s / OP(i, i);
        }
    }
#undef OP
}

/* ------------------------------------------------------------------ */
/* Cholesky xPOTRF / xPOTRS, lower triangle (Z12b)         */
/* ------------------------------------------------------------------ */
/* Unblocked right-looking (outer product) Cholesky on the lower triangle of
 * a copy L (the strict upper part is ignored).  Fails (returns 1+j) at the
 * first column whose pivot is not > 0 (Z23). */
static int64_t FN(potrf)(T* L, int64_t ld, int64_t n)
{
    for (int64_t j = 0; j < n; ++j) {
        T d = L[j + j * ld];
        if (!(d > (T)0)) return j + 1;
        T ljj = SQRT(d);
        L[j + j * ld] = ljj;
        for (int64_t i = j + 1; i < n; ++i) L[i + j * ld] = L[i + j * ld] / ljj;
        #pragma omp parallel for schedule(static)
        for (int64_t k = j + 1; k < n; ++k) {
            const T lkj = L[k + j * ld];
            for (int64_t i = k; i < n; ++i) L[i + k * ld] = L[i + k * ld] - L[i + j * ld] * lkj;
        }
    }
    return 0;
}

/* ------------------------------------------------------------------ */
/* General LU xGETRF / xGETRS (Eq. 4)                       */
/* ------------------------------------------------------------------ */
/* Unblocked right-looking LU with partial pivoting, PA = LU.  Pivot: first
 * max |a_ij| over i >= j (Z15); whole rows are swapped; multipliers by
 * division.  Returns 0, or 1+j for the first exactly-zero pivot. */
static int64_t FN(getrf)(T* W, int64_t ld, int64_t n, int64_t* ipiv)
{
    int64_t info = 0;
    for (int64_t j = 0; j < n; ++j) {
        int64_t p = j;
        T best = ABS(W[j + j * ld]);
        for (int64_t i = j + 1; i < n; ++i)
            if (ABS(W[i + j * ld]) > best) { best = ABS(W[i + j * ld]); p = i; }
        ipiv[j] = p;
        if (W[p + j * ld] == (T)0) { if (info == 0) info = j + 1; continue; }
        if (p != j)
            for (int64_t c = 0; c < n; ++c) { T t = W[j + c * ld]; W[j + c * ld] = W[p + c * ld]; W[p + c * ld] = t; }
        const T piv = W[j + j * ld];
        for (int64_t i = j + 1; i < n; ++i) W[i + j * ld] = W[i + j * ld] / piv;
        #pragma omp parallel for schedule(static)
        for (int64_t k = j + 1; k < n; ++k) {
            const T u = W[j + k * ld];
            for (int64_t i = j + 1; i < n; ++i) W[i + k * ld] = W[i + k * ld] - W[i + j * ld] * u;
        }
    }
    return info;
}
/* xGETRS: b <- P b, then L y = b (forward, unit), U x = y (back). */
static void FN(getrs_vec)(const T* W, int64_t ld, int64_t n, const int64_t* ipiv, T* b)
{
    for (int64_t j = 0; j < n; ++j) { int64_t p = ipiv[j]; if (p != j) { T t = b[j]; b[j] = b[p]; b[p] = t; } }
    FN(trsv)(W, ld, n, 0, 0, 1, b);
    FN(trsv)(W, ld, n, 1, 0, 0, b);
}

/* ------------------------------------------------------------------ */
/* Symmetric indefinite LDL^T with Bunch-Kaufman pivoting (P:741-743,   */
/* "plain symmetric matrices" as future work; the xSYTF2 algorithm,    */
/* lower triangle, Z30)                                      */
/* ------------------------------------------------------------------ */
/* P A P^T = L D L^T with 1x1 and 2x2 diagonal blocks; only the lower
 * triangle of W is read and overwritten (D on the block diagonal, the
 * multipliers below).  ipiv (0-based): 1x1 block at k: ipiv[k] = kp (rows
 * and columns k and kp interchanged); 2x2 block at k, k+1: ipiv[k] =
 * ipiv[k+1] = -(kp + 1) (k+1 and kp interchanged).  alpha = (1+sqrt(17))/8.
 * Returns 0, or 1+k for the first exactly zero (or NaN) pivot column. */
static int64_t FN(sytrf)(T* W, int64_t ld, int64_t n, int64_t* ipiv)
{
#define WL(i, j) W[(i) + (j) * ld]
    const T alpha = ((T)1 + SQRT((T)17)) / (T)8;
    int64_t info = 0, k = 0;
    while (k < n) {
        int kstep = 1;
        int64_t kp = k, imax = k;
        const T absakk = ABS(WL(k, k));
        T colmax = (T)0;
        if (k < n - 1) {
            imax = k + 1;
            colmax = ABS(WL(k + 1, k));
            for (int64_t i = k + 2; i < n; ++i) if (ABS(WL(i, k)) > colmax) { colmax = ABS(WL(i, k)); imax = i; }
        }
        if ((absakk > colmax ? absakk : colmax) == (T)0 || absakk != absakk) {
            if (info == 0) info = k + 1;
            kp = k;
        } else {
            if (absakk >= alpha * colmax) {
                kp = k;
            } else {
                /* largest off-diagonal |.| in row imax: A(imax, k..imax-1), then column imax below */
                int64_t jmax = k;
                T rowmax = ABS(WL(imax, k));
                for (int64_t j = k + 1; j < imax; ++j) if (ABS(WL(imax, j)) > rowmax) { rowmax = ABS(WL(imax, j)); jmax = j; }
                if (imax < n - 1) {
                    int64_t j2 = imax + 1;
                    T m2 = ABS(WL(imax + 1, imax));
                    for (int64_t i = imax + 2; i < n; ++i) if (ABS(WL(i, imax)) > m2) { m2 = ABS(WL(i, imax)); j2 = i; }
                    if (m2 > rowmax) rowmax = m2;
                    (void)j2;
                }
                (void)jmax;
                if (absakk >= alpha * colmax * (colmax / rowmax)) kp = k;
                else if (ABS(WL(imax, imax)) >= alpha * rowmax) kp = imax;
                else { kp = imax; kstep = 2; }
            }
            const int64_t kk = k + kstep - 1;
            if (kp != kk) {        /* interchange rows and columns kk and kp of A(k:n, k:n) */
                for (int64_t i = kp + 1; i < n; ++i) { T t = WL(i, kk); WL(i, kk) = WL(i, kp); WL(i, kp) = t; }
                for (int64_t j = kk + 1; j < kp; ++j) { T t = WL(j, kk); WL(j, kk) = WL(kp, j); WL(kp, j) = t; }
                { T t = WL(kk, kk); WL(kk, kk) = WL(kp, kp); WL(kp, kp) = t; }
                if (kstep == 2) { T t = WL(k + 1, k); WL(k + 1, k) = WL(kp, k); WL(kp, k) = t; }
            }
            if (kstep == 1) {
                if (k < n - 1) {   /* A := A - d11 x x^T (xSYR), x = A(k+1:n, k); then x *= d11 */
                    const T d11 = (T)1 / WL(k, k);
                    #pragma omp parallel for schedule(static)
                    for (int64_t j = k + 1; j < n; ++j) {
                        const T temp = -d11 * WL(j, k);
                        for (int64_t i = j; i < n; ++i) WL(i, j) = WL(i, j) + WL(i, k) * temp;
                    }
                    for (int64_t i = k + 1; i < n; ++i) WL(i, k) = d11 * WL(i, k);
                }
            } else if (k < n - 2) {
                T d21 = WL(k + 1, k);
                const T d11 = WL(k + 1, k + 1) / d21;
                const T d22 = WL(k, k) / d21;
                const T t = (T)1 / (d11 * d22 - (T)1);
                d21 = t / d21;
                for (int64_t j = k + 2; j < n; ++j) {
                    const T wk = d21 * (d11 * WL(j, k) - WL(j, k + 1));
                    const T wkp1 = d21 * (d22 * WL(j, k + 1) - WL(j, k));
                    for (int64_t i = j; i < n; ++i) WL(i, j) = WL(i, j) - WL(i, k) * wk - WL(i, k + 1) * wkp1;
                    WL(j, k) = wk;
                    WL(j, k + 1) = wkp1;
                }
            }
        }
        if (kstep == 1) ipiv[k] = kp;
        else { ipiv[k] = -(kp + 1); ipiv[k + 1] = -(kp + 1); }
        k += kstep;
    }
    return info;
#undef WL
}

/* xSYTRS (lower): b <- A^{-1} b from sytrf's factors (L D L^T with the interchanges). */
static void FN(sytrs_vec)(const T* W, int64_t ld, int64_t n, const int64_t* ipiv, T* b)
{
#define WL(i, j) W[(i) + (j) * ld]
    int64_t k = 0;
    while (k < n) {                       /* solve L D y = P b */
        if (ipiv[k] >= 0) {
            const int64_t kp = ipiv[k];
            if (kp != k) { T t = b[k]; b[k] = b[kp]; b[kp] = t; }
            for (int64_t i = k + 1; i < n; ++i) b[i] = b[i] - WL(i, k) * b[k];
            b[k] = b[k] / WL(k, k);
            k += 1;
        } else {
            const int64_t kp = -ipiv[k] - 1;
            if (kp != k + 1) { T t = b[k + 1]; b[k + 1] = b[kp]; b[kp] = t; }
            for (int64_t i = k + 2; i < n; ++i) b[i] = b[i] - WL(i, k) * b[k] - WL(i, k + 1) * b[k + 1];
            const T akm1k = WL(k + 1, k);
            const T akm1 = WL(k, k) / akm1k;
            const T ak = WL(k + 1, k + 1) / akm1k;
            const T denom = akm1 * ak - (T)1;
            const T bkm1 = b[k] / akm1k;
            const T bk = b[k + 1] / akm1k;
            b[k] = (ak * bkm1 - bk) / denom;
            b[k + 1] = (akm1 * bk - bkm1) / denom;
            k += 2;
        }
    }
    k = n - 1;
    while (k >= 0) {                      /* solve L^T P x = y */
        if (ipiv[k] >= 0) {
            T s = b[k];
            for (int64_t i = k + 1; i < n; ++i) s = s - WL(i, k) * b[i];
            b[k] = s;
            const int64_t kp = ipiv[k];
            if (kp != k) { T t = b[k]; b[k] = b[kp]; b[kp] = t; }
            k -= 1;
        } else {
            T s = b[k], s1 = b[k - 1];
            for (int64_t i = k + 1; i < n; ++i) { s = s - WL(i, k) * b[i]; s1 = s1 - WL(i, k - 1) * b[i]; }
            b[k] = s;
            b[k - 1] = s1;
            const int64_t kp = -ipiv[k] - 1;
            if (kp != k) { T t = b[k]; b[k] = b[kp]; b[kp] = t; }
            k -= 2;
        }
    }
#undef WL
}

/* ------------------------------------------------------------------ */
/* Reciprocal condition estimate (the xxCON family P:350,     */
/* P:386): 1-norm estimate of ||A^-1||_1 by the Hager-Higham */
/* procedure in the form LAPACK's xLACN2 uses (Z13b), with M = A^-1 and    */
/* M^T applied through the path's factors.                               */
/* ------------------------------------------------------------------ */
typedef struct {
    int kind;               /* 0 LU, 1 band LU, 2 triangular, 3 Cholesky, 4 LDL^T (ipiv = sytrf's) */
    const T* F; int64_t ldf; int64_t n;
    int64_t kl, ku; const int64_t* ipiv;
    int upper;
} FN(opM);

/* y <- M y (trans=0) or M^T y (trans=1). */
static void FN(applyM)(const FN(opM)* op, int trans, T* y)
{
    const int64_t n = op->n;
    switch (op->kind) {
    case 0:   /* xGECON: inv(U)*inv(L) resp. inv(L^T)*inv(U^T), no interchanges (1-norm invariant) */
        if (!trans) { FN(trsv)(op->F, op->ldf, n, 0, 0, 1, y); FN(trsv)(op->F, op->ldf, n, 1, 0, 0, y); }
        else        { FN(trsv)(op->F, op->ldf, n, 1, 1, 0, y); FN(trsv)(op->F, op->ldf, n, 0, 1, 1, y); }
        break;
    case 1:   /* xGBCON: band L with interchanges, then band U */
        if (!trans) FN(gbtrs_vec)(n, op->kl, op->ku, op->F, op->ldf, op->ipiv, y);
        else        FN(gbtrs_vec_t)(n, op->kl, op->ku, op->F, op->ldf, op->ipiv, y);
        break;
    case 2:   /* xTRCON */
        FN(trsv)(op->F, op->ldf, n, op->upper, trans, 0, y);
        break;
    case 3:   /* xPOCON: inv(L^T) * inv(L), symmetric */
        FN(trsv)(op->F, op->ldf, n, 0, 0, 0, y);
        FN(trsv)(op->F, op->ldf, n, 0, 1, 0, y);
        break;
    case 4:   /* xSYCON: A^{-1} through xSYTRS, symmetric (both kases the same) */
        FN(sytrs_vec)(op->F, op->ldf, n, op->ipiv, y);
        break;
    }
}

static T FN(asum)(const T* x, int64_t n) { T s = (T)0; for (int64_t i = 0; i < n; ++i) s += ABS(x[i]); return s; }
/* IxAMAX: first index of the maximum |x_i| (strict >). */
static int64_t FN(iamax)(const T* x, int64_t n)
{
    int64_t k = 0; T m = ABS(x[0]);
    for (int64_t i = 1; i < n; ++i) if (ABS(x[i]) > m) { m = ABS(x[i]); k = i; }
    return k;
}

/* Returns the estimate of ||M||_1; *nsolves counts applications of M/M^T. */
static T FN(lacn2)(const FN(opM)* op, int* nsolves)
{
    const int64_t n = op->n;
    const int itmax = 5;
    T* x = (T*)malloc(sizeof(T) * (size_t)n);
    signed char* isgn = (signed char*)malloc((size_t)n);
    int ns = 0;
    T est;
    /* step 1: x = e/n, x <- M x */
    for (int64_t i = 0; i < n; ++i) x[i] = (T)1 / (T)n;
    FN(applyM)(op, 0, x); ++ns;
    if (n == 1) { est = ABS(x[0]); goto done; }
    est = FN(asum)(x, n);
    for (int64_t i = 0; i < n; ++i) { x[i] = x[i] >= (T)0 ? (T)1 : (T)-1; isgn[i] = x[i] > 0 ? 1 : -1; }
    FN(applyM)(op, 1, x); ++ns;
    int64_t j = FN(iamax)(x, n);
    int iter = 2;
    for (;;) {
        /* step 2: x = e_j, x <- M x */
        for (int64_t i = 0; i < n; ++i) x[i] = (T)0;
        x[j] = (T)1;
        FN(applyM)(op, 0, x); ++ns;
        T estold = est;
        est = FN(asum)(x, n);
        int same = 1;
        for (int64_t i = 0; i < n; ++i) { int s = x[i] >= (T)0 ? 1 : -1; if (s != isgn[i]) { same = 0; break; } }
        if (same) break;                 /* repeated sign vector: converged */
        if (est <= estold) break;
        for (int64_t i = 0; i < n; ++i) { x[i] = x[i] >= (T)0 ? (T)1 : (T)-1; isgn[i] = x[i] > 0 ? 1 : -1; }
        FN(applyM)(op, 1, x); ++ns;
        int64_t jlast = j;
        j = FN(iamax)(x, n);
        if (x[jlast] != ABS(x[j]) && iter < itmax) { ++iter; continue; }
        break;
    }
    /* step 3: alternating-sign probe x_i = (-1)^i (1 + i/(n-1)) */
    {
        T altsgn = (T)1;
        for (int64_t i = 0; i < n; ++i) { x[i] = altsgn * ((T)1 + (T)i / (T)(n - 1)); altsgn = -altsgn; }
        FN(applyM)(op, 0, x); ++ns;
        T temp = (T)2 * (FN(asum)(x, n) / (T)(3 * n));
        if (temp > est) est = temp;
    }
done:
    free(x); free(isgn);
    if (nsolves) *nsolves = ns;
    return est;
}

/* rcond = (1/est)/anorm (xGECON convention); 0 if anorm or est is 0. */
static T FN(rcond_from)(T anorm, T est)
{
    if (!(anorm > (T)0)) return (T)0;
    if (est == (T)0) return (T)0;
    return ((T)1 / est) / anorm;
}

/* ------------------------------------------------------------------ */
/* SVD-based minimum-norm fallback (xGELSD role; Z14, Z16, Z17) */
/* ------------------------------------------------------------------ */
/* Householder QR, A = QR (the xGEQR2 algorithm with xLARFG reflectors):
 * R overwrites the upper triangle of W; each reflector is applied to the
 * remaining columns and to the nrhs columns of C (C <- Q^T C). */
static void FN(geqr_apply)(T* W, int64_t ld, int64_t n, T* C, int64_t ldc, int64_t nrhs)
{
    T* v = (T*)malloc(sizeof(T) * (size_t)n);
    for (int64_t j = 0; j < n; ++j) {
        T alpha = W[j + j * ld];
        T ss = (T)0;
        for (int64_t i = j + 1; i < n; ++i) ss += W[i + j * ld] * W[i + j * ld];
        T xnorm = SQRT(ss);
        if (xnorm == (T)0) continue;     /* H = I (tau = 0) */
        /* beta = -sign(alpha) * hypot(alpha, xnorm) */
        T aa = ABS(alpha), w = aa > xnorm ? aa : xnorm, z = aa > xnorm ? xnorm : aa;
        T hyp = w * SQRT((T)1 + (z / w) * (z / w));
        T beta = alpha >= (T)0 ? -hyp : hyp;
        T tau = (beta - alpha) / beta;
        T scal = (T)1 / (alpha - beta);
        v[j] = (T)1;
        for (int64_t i = j + 1; i < n; ++i) { v[i] = W[i + j * ld] * scal; W[i + j * ld] = (T)0; }
        W[j + j * ld] = beta;
        /* apply H = I - tau v v^T to W[j:n, j+1:n] and C[j:n, :] */
        #pragma omp parallel for schedule(static)
        for (int64_t k = j + 1; k < n + nrhs; ++k) {
            T* col = k < n ? W + k * ld : C + (k - n) * ldc;
            T s = (T)0;
            for (int64_t i = j; i < n; ++i) s += v[i] * col[i];
            s = tau * s;
            for (int64_t i = j; i < n; ++i) col[i] = col[i] - s * v[i];
        }
    }
    free(v);
}

/* One-sided (Hestenes) Jacobi on M (n x n, column-major), cyclic-by-rows
 * pair order p<q; V accumulates the rotations (V starts as I).  Rotation of
 * (p,q) iff gamma != 0 and |gamma| > tol*sqrt(alpha)*sqrt(beta),
 * tol = n*eps (Z16).  Returns the number of sweeps executed; *conv = 1 if
 * the last sweep made no rotation, 0 if the cap was hit. */
static int FN(jacobi)(T* M, int64_t ld, int64_t n, T* V, int max_sweeps, int* conv)
{
    const T tol = (T)n * FN(eps)();
    int sweeps = 0;
    *conv = 0;
    for (int64_t j = 0; j < n; ++j) for (int64_t i = 0; i < n; ++i) V[i + j * n] = i == j ? (T)1 : (T)0;
    while (sweeps < max_sweeps) {
        int64_t rotations = 0;
        ++sweeps;
        for (int64_t p = 0; p + 1 < n; ++p) {
            for (int64_t q = p + 1; q < n; ++q) {
                T* mp = M + p * ld; T* mq = M + q * ld;
                T alpha = (T)0, beta = (T)0, gamma = (T)0;
                for (int64_t i = 0; i < n; ++i) { alpha += mp[i] * mp[i]; beta += mq[i] * mq[i]; gamma += mp[i] * mq[i]; }
                if (gamma == (T)0 || !(ABS(gamma) > tol * SQRT(alpha) * SQRT(beta))) continue;
                ++rotations;
                T zeta = (beta - alpha) / ((T)2 * gamma);
                T t = (zeta >= (T)0 ? (T)1 : (T)-1) / (ABS(zeta) + SQRT((T)1 + zeta * zeta));
                T c = (T)1 / SQRT((T)1 + t * t);
                T s = c * t;
                for (int64_t i = 0; i < n; ++i) {
                    T a = mp[i], b = mq[i];
                    mp[i] = c * a - s * b; mq[i] = s * a + c * b;
                }
                T* vp = V + p * n; T* vq = V + q * n;
                for (int64_t i = 0; i < n; ++i) {
                    T a = vp[i], b = vq[i];
                    vp[i] = c * a - s * b; vq[i] = s * a + c * b;
                }
            }
        }
        if (rotations == 0) { *conv = 1; break; }
    }
    return sweeps;
}

/* Minimum-norm solution x = V_A Sigma^+ U_A^T b via the SVD (Z17), with
 * A = QR, R^T V_J = M (orthogonal columns), so A = (Q V_J) Sigma (M/Sigma)^T:
 * x = sum_{kept k} m_k (V_J^T Q^T b)_k / sigma_k^2.  Kept: sigma_k > cut*sigma_max
 * (cut = n*eps by default, Z14).  sigma_out (optional) gets sigma sorted
 * descending (stable).  Returns the rank (number kept); *sweeps_out and
 * *conv_out report the Jacobi iteration. */
static int64_t FN(lsq_svd)(const T* A, int64_t lda, int64_t n, const T* B, int64_t ldb, int64_t nrhs,
                           T* X, int64_t ldx, T cut, int max_sweeps, T* sigma_out, int* sweeps_out, int* conv_out,
                           int* nonfinite_out)
{
    T* W = (T*)malloc(sizeof(T) * (size_t)(n * n));
    T* C = (T*)malloc(sizeof(T) * (size_t)(n * (nrhs > 0 ? nrhs : 1)));
    T* M = (T*)malloc(sizeof(T) * (size_t)(n * n));
    T* V = (T*)malloc(sizeof(T) * (size_t)(n * n));
    T* sig = (T*)malloc(sizeof(T) * (size_t)n);
    int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
    for (int64_t j = 0; j < n; ++j) for (int64_t i = 0; i < n; ++i) W[i + j * n] = A[i + j * lda];
    for (int64_t j = 0; j < nrhs; ++j) for (int64_t i = 0; i < n; ++i) C[i + j * n] = B[i + j * ldb];
    /* (1) A = QR, C = Q^T B */
    FN(geqr_apply)(W, n, n, C, n, nrhs);
    /* (2) M = R^T */
    for (int64_t j = 0; j < n; ++j) for (int64_t i = 0; i < n; ++i) M[i + j * n] = i >= j ? W[j + i * n] : (T)0;
    int conv = 0;
    int sweeps = FN(jacobi)(M, n, n, V, max_sweeps, &conv);
    /* (3) sigma_k = ||m_k||_2, sorted descending (stable insertion sort) */
    int nonfinite = 0;
    for (int64_t k = 0; k < n; ++k) {
        T s = (T)0;
        for (int64_t i = 0; i < n; ++i) s += M[i + k * n] * M[i + k * n];
        sig[k] = SQRT(s);
        order[k] = k;
        if (!isfinite(sig[k])) nonfinite = 1;   /* Z29: non-finite input reached the SVD */
    }
    if (nonfinite_out) *nonfinite_out = nonfinite;
    for (int64_t a = 1; a < n; ++a) {
        int64_t key = order[a]; int64_t b = a - 1;
        while (b >= 0 && sig[order[b]] < sig[key]) { order[b + 1] = order[b]; --b; }
        order[b + 1] = key;
    }
    if (sigma_out) for (int64_t k = 0; k < n; ++k) sigma_out[k] = sig[order[k]];
    T smax = n > 0 ? sig[order[0]] : (T)0;
    /* (4) x = sum_kept m_k (V^T c)_k / sigma_k^2 */
    int64_t rank = 0;
    for (int64_t k = 0; k < n; ++k) if (sig[k] > cut * smax) ++rank;
    for (int64_t r = 0; r < nrhs; ++r) {
        T* x = X + r * ldx;
        const T* c = C + r * n;
        for (int64_t i = 0; i < n; ++i) x[i] = (T)0;
        for (int64_t k = 0; k < n; ++k) {
            if (!(sig[k] > cut * smax)) continue;
            T y = (T)0;
            for (int64_t i = 0; i < n; ++i) y += V[i + k * n] * c[i];
            T coef = y / (sig[k] * sig[k]);
            for (int64_t i = 0; i < n; ++i) x[i] += coef * M[i + k * n];
        }
    }
    free(W); free(C); free(M); free(V); free(sig); free(order);
    if (sweeps_out) *sweeps_out = sweeps;
    if (conv_out) *conv_out = conv;
    return rank;
}

/* ------------------------------------------------------------------ */
/* Public oracle entry points (C ABI, host buffers)                     */
/* ------------------------------------------------------------------ */

/* Detection verdict: literal flags + kl/ku exact + max_diag. */
int FN(or_detect)(const T* A, int64_t lda, int64_t n, or_structure* out)
{
    memset(out, 0, sizeof(*out));
    if (n <= 0) return 0;
    int64_t kl, ku;
    FN(band_extent)(A, lda, n, &kl, &ku);
    out->kl = kl; out->ku = ku;
    uint32_t f = 0;
    if (FN(band_density_ok)(n, kl, ku)) f |= OR_BANDED;
    if (FN(is_lower)(A, lda, n)) f |= OR_LOWER;
    if (FN(is_upper)(A, lda, n)) f |= OR_UPPER;
    T md = 0;
    if (FN(likely_sympd)(A, lda, n, &md)) f |= OR_SPD;
    out->max_diag = (double)md;
    out->flags = f;
    return 0;
}

/* Pieces exported for the oracle's own pin tests. */
int64_t FN(or_getrf)(T* W, int64_t ld, int64_t n, int64_t* ipiv) { return FN(getrf)(W, ld, n, ipiv); }
void FN(or_getrs)(const T* W, int64_t ld, int64_t n, const int64_t* ipiv, T* B, int64_t ldb, int64_t nrhs)
{ for (int64_t r = 0; r < nrhs; ++r) FN(getrs_vec)(W, ld, n, ipiv, B + r * ldb); }
int64_t FN(or_potrf)(T* L, int64_t ld, int64_t n) { return FN(potrf)(L, ld, n); }
int64_t FN(or_sytrf)(T* W, int64_t ld, int64_t n, int64_t* ipiv) { return FN(sytrf)(W, ld, n, ipiv); }
void FN(or_sytrs)(const T* W, int64_t ld, int64_t n, const int64_t* ipiv, T* B, int64_t ldb, int64_t nrhs)
{ for (int64_t r = 0; r < nrhs; ++r) FN(sytrs_vec)(W, ld, n, ipiv, B + r * ldb); }
void FN(or_trsv)(const T* A, int64_t lda, int64_t n, int upper, int trans, int unit, T* b) { FN(trsv)(A, lda, n, upper, trans, unit, b); }
double FN(or_band_pack)(const T* A, int64_t lda, int64_t n, int64_t kl, int64_t ku, T* ab, int64_t ldab)
{ return (double)FN(band_pack)(A, lda, n, kl, ku, ab, ldab); }
int64_t FN(or_gbtrf)(int64_t n, int64_t kl, int64_t ku, T* ab, int64_t ldab, int64_t* ipiv) { return FN(gbtrf)(n, kl, ku, ab, ldab, ipiv); }
void FN(or_gbtrs)(int64_t n, int64_t kl, int64_t ku, const T* ab, int64_t ldab, const int64_t* ipiv, T* B, int64_t ldb, int64_t nrhs, int trans)
{ for (int64_t r = 0; r < nrhs; ++r) { if (trans) FN(gbtrs_vec_t)(n, kl, ku, ab, ldab, ipiv, B + r * ldb); else FN(gbtrs_vec)(n, kl, ku, ab, ldab, ipiv, B + r * ldb); } }
double FN(or_norm1)(const T* A, int64_t lda, int64_t n) { return (double)FN(norm1_full)(A, lda, n); }
/* rcond estimators from factors: kind 0 LU (F=W), 1 band (F=ab), 2 tri (F=A), 3 Cholesky (F=L),
 * 4 LDL^T (F=W, ipiv = sytrf's). */
double FN(or_rcond)(int kind, const T* F, int64_t ldf, int64_t n, int64_t kl, int64_t ku, const int64_t* ipiv, int upper, double anorm, int* nsolves)
{
    FN(opM) op = { kind, F, ldf, n, kl, ku, ipiv, upper };
    if (n == 0) return 1.0;
    T est = FN(lacn2)(&op, nsolves);
    return (double)FN(rcond_from)((T)anorm, est);
}
void FN(or_geqr)(T* W, int64_t ld, int64_t n, T* C, int64_t ldc, int64_t nrhs) { FN(geqr_apply)(W, ld, n, C, ldc, nrhs); }
int FN(or_jacobi)(T* M, int64_t ld, int64_t n, T* V, int max_sweeps, int* conv) { return FN(jacobi)(M, ld, n, V, max_sweeps, conv); }
int64_t FN(or_lsq_svd)(const T* A, int64_t lda, int64_t n, const T* B, int64_t ldb, int64_t nrhs, T* X, int64_t ldx,
                       double cut, int max_sweeps, T* sigma_out, int* sweeps_out, int* conv_out)
{ return FN(lsq_svd)(A, lda, n, B, ldb, nrhs, X, ldx, (T)cut, max_sweeps, sigma_out, sweeps_out, conv_out, NULL); }

/* The adaptive solve, the paper's flowchart (Fig. 2
 * caption P:237-243) as read in Z9-Z11, Z24, Z25:
 *   banded -> GBTRF/GBCON/GBTRS; lower/upper -> TRTRS/TRCON;
 *   likely-sympd -> POTRF/POCON/POTRS, POTRF failure -> general LU;
 *   general -> GETRF/GECON/GETRS;
 *   factor failure or !(rcond >= 0.5 eps) -> SVD min-norm (unless NO_FALLBACK).
 * Returns 0 or an OR_ERR_* code; X (ldx) gets the solution. */
int FN(or_solve)(const T* A, int64_t lda, int64_t n, const T* B, int64_t ldb, int64_t nrhs,
                 T* X, int64_t ldx, const or_options* opt, or_report* rep, T* sigma_out)
{
    or_options o;
    if (opt) o = *opt; else { memset(&o, 0, sizeof(o)); o.rcond_threshold = -1; o.lsq_cutoff = -1; o.max_sweeps = 30; }
    memset(rep, 0, sizeof(*rep));
    rep->kl = -1; rep->ku = -1; rep->rcond = 1.0; rep->rank = -1;
    if (n == 0 || nrhs == 0) return 0;
    const T eps = FN(eps)();
    const T thr = o.rcond_threshold >= 0 ? (T)o.rcond_threshold : (T)0.5 * eps;
    const T cut = o.lsq_cutoff >= 0 ? (T)o.lsq_cutoff : (T)n * eps;
    const int max_sweeps = o.max_sweeps > 0 ? o.max_sweeps : 30;

    or_structure st;
    FN(or_detect)(A, lda, n, &st);
    uint32_t flags = st.flags;
    /* Z30: with SYM_INDEF the exact symmetry is evaluated; a symmetric matrix that is not likely
     * sympd (or whose Cholesky fails) takes LDL^T instead of the general LU */
    const int symind = (o.flags & OR_OPT_SYM_INDEF) != 0 && n <= 128;   /* Z30: larger systems ignore it */
    const int sym = symind && FN(is_symmetric)(A, lda, n);
    if (sym) flags |= OR_F_SYMMETRIC;
    int method;
    if (o.flags & OR_OPT_FORCE_METHOD) method = o.force_method;
    else if (st.flags & OR_BANDED) method = OR_M_BAND;
    else if (st.flags & OR_LOWER) method = OR_M_TRI_LOWER;
    else if (st.flags & OR_UPPER) method = OR_M_TRI_UPPER;
    else if (st.flags & OR_SPD) method = OR_M_CHOL;
    else if (sym) method = OR_M_LDLT;
    else method = OR_M_LU;
    if (method == OR_M_BAND || (o.flags & OR_OPT_FULLSCAN)) { rep->kl = st.kl; rep->ku = st.ku; }
    /* Z28: with CHECK_FINITE a NaN/Inf anywhere in A or B is rejected before
     * any factorization (the detection verdicts are still reported). */
    if ((o.flags & OR_OPT_CHECK_FINITE) &&
        !(FN(all_finite)(A, lda, n, n) && FN(all_finite)(B, ldb, n, nrhs))) {
        rep->rcond = 0.0;
        rep->flags = flags | OR_F_NONFINITE;
        return OR_ERR_NONFINITE;
    }

    int singular = 0, factored = 0;
    T rcond = 0, anorm = 0;
    int64_t info = 0;
    /* X <- B (every primary path solves in place in X) */
    for (int64_t r = 0; r < nrhs; ++r) for (int64_t i = 0; i < n; ++i) X[i + r * ldx] = B[i + r * ldb];

    if (method == OR_M_BAND) {
        const int64_t kl = st.kl, ku = st.ku, ldab = 2 * kl + ku + 1;
        T* ab = (T*)malloc(sizeof(T) * (size_t)(ldab * n));
        int64_t* ipiv = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
        anorm = FN(band_pack)(A, lda, n, kl, ku, ab, ldab);
        info = FN(gbtrf)(n, kl, ku, ab, ldab, ipiv);
        if (info) singular = 1;
        else {
            FN(opM) op = { 1, ab, ldab, n, kl, ku, ipiv, 0 };
            rcond = FN(rcond_from)(anorm, FN(lacn2)(&op, NULL));
            factored = 1;
            for (int64_t r = 0; r < nrhs; ++r) FN(gbtrs_vec)(n, kl, ku, ab, ldab, ipiv, X + r * ldx);
        }
        free(ab); free(ipiv);
    } else if (method == OR_M_TRI_LOWER || method == OR_M_TRI_UPPER) {
        const int upper = method == OR_M_TRI_UPPER;
        for (int64_t j = 0; j < n; ++j) if (A[j + j * lda] == (T)0) { info = j + 1; break; }
        if (info) singular = 1;
        else {
            anorm = FN(norm1_tri)(A, lda, n, upper);
            FN(opM) op = { 2, A, lda, n, 0, 0, NULL, upper };
            rcond = FN(rcond_from)(anorm, FN(lacn2)(&op, NULL));
            factored = 1;
            for (int64_t r = 0; r < nrhs; ++r) FN(trsv)(A, lda, n, upper, 0, 0, X + r * ldx);
        }
    } else {
        T* W = (T*)malloc(sizeof(T) * (size_t)(n * n));
        for (int64_t j = 0; j < n; ++j) for (int64_t i = 0; i < n; ++i) W[i + j * n] = A[i + j * lda];
        if (method == OR_M_CHOL) {
            info = FN(potrf)(W, n, n);
            if (info) {              /* not actually sympd -> generic solver (Z30: LDL^T if symmetric) */
                flags |= OR_F_CHOL_FAILED;
                rep->chol_fail_col = info - 1;
                info = 0;
                method = sym ? OR_M_LDLT : OR_M_LU;
                for (int64_t j = 0; j < n; ++j) for (int64_t i = 0; i < n; ++i) W[i + j * n] = A[i + j * lda];
            } else {
                anorm = FN(norm1_full)(A, lda, n);
                FN(opM) op = { 3, W, n, n, 0, 0, NULL, 0 };
                rcond = FN(rcond_from)(anorm, FN(lacn2)(&op, NULL));
                factored = 1;
                for (int64_t r = 0; r < nrhs; ++r) { FN(trsv)(W, n, n, 0, 0, 0, X + r * ldx); FN(trsv)(W, n, n, 0, 1, 0, X + r * ldx); }
            }
        }
        if (method == OR_M_LDLT) {   /* xSYTRF / xSYCON / xSYTRS, lower (Z30) */
            int64_t* ipiv = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
            anorm = FN(norm1_full)(A, lda, n);
            info = FN(sytrf)(W, n, n, ipiv);
            if (info) singular = 1;
            else {
                FN(opM) op = { 4, W, n, n, 0, 0, ipiv, 0 };
                rcond = FN(rcond_from)(anorm, FN(lacn2)(&op, NULL));
                factored = 1;
                for (int64_t r = 0; r < nrhs; ++r) FN(sytrs_vec)(W, n, n, ipiv, X + r * ldx);
            }
            free(ipiv);
        }
        if (method == OR_M_LU) {
            int64_t* ipiv = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
            anorm = FN(norm1_full)(A, lda, n);
            info = FN(getrf)(W, n, n, ipiv);
            if (info) singular = 1;
            else {
                FN(opM) op = { 0, W, n, n, 0, 0, ipiv, 0 };
                rcond = FN(rcond_from)(anorm, FN(lacn2)(&op, NULL));
                factored = 1;
                for (int64_t r = 0; r < nrhs; ++r) FN(getrs_vec)(W, n, n, ipiv, X + r * ldx);
            }
            free(ipiv);
        }
        free(W);
    }
    rep->primary_method = method;
    rep->anorm = (double)anorm;
    rep->rcond = singular ? 0.0 : (double)rcond;
    rep->info = info;
    if (singular) flags |= OR_F_SINGULAR;
    int gate = singular || !(rcond >= thr);        /* Z11: NaN rcond -> gate */
    (void)factored;
    if (gate) flags |= OR_F_RCOND_LOW;
    int ret = 0;
    if (gate) {
        if (o.flags & OR_OPT_NO_FALLBACK) {
            if (singular) ret = OR_ERR_SINGULAR_NO_FALLBACK;
            else flags |= OR_F_POORLY_COND;
        } else {
            int sweeps = 0, conv = 0, nonfinite = 0;
            int64_t rank = FN(lsq_svd)(A, lda, n, B, ldb, nrhs, X, ldx, cut, max_sweeps, sigma_out, &sweeps, &conv,
                                       &nonfinite);
            rep->rank = rank; rep->sweeps = sweeps;
            flags |= OR_F_FALLBACK;
            method = OR_M_SVD;
            if (nonfinite) {          /* Z29: min-norm solution undefined, X unspecified */
                flags |= OR_F_NONFINITE;
                rep->rank = -1;
                ret = OR_ERR_NONFINITE;
            } else {
                if (rank < n) flags |= OR_F_RANK_DEF;
                if (!conv) { flags |= OR_F_SVD_NOCONV; ret = OR_ERR_SVD_NOT_CONVERGED; }
            }
        }
    }
    rep->method = method;
    rep->flags = flags | ((uint32_t)method << 4);
    return ret;
}
