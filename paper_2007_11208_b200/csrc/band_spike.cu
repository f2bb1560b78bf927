// band_spike.cu -- partitioned (SPIKE-style) banded solve for the band path
// (P:345-350), used when A is strictly diagonally dominant by rows or by
// columns (checked on device).  Then Gaussian elimination needs no row
// interchanges for stability, every diagonal partition block is nonsingular,
// and the paper's GBTRF / GBTRS / GBCON steps can be reorganised without the
// serial chain of n pivot steps:
//
//   A = D S,  D = diag(A_0 .. A_{p-1})  (partition blocks, no-pivot band LU in smem)
//   S = I + spikes V_i = A_i^{-1}[0; B_i], W_i = A_i^{-1}[C_i; 0]
//   reduced block-tridiagonal system on the interface unknowns
//   z_i = [x_i(bottom K) ; x_{i+1}(top K)], factored by block Thomas
//   (explicit inverses of the 2K x 2K pivots) and kept in the shared memory
//   of a dedicated "reduced" CTA for the whole call.
//
// Solves with A^T use the same partition LU (A_i^T = U_i^T L_i^T) and their
// own spikes / reduced system (second reduced CTA).  The whole band path --
// factor, the xLACN2 estimate of ||A^{-1}||_1 (state machine with distributed
// reductions), and the primary solve X = A^{-1} B -- runs in ONE cooperative
// kernel of p + 2 CTAs; phases are separated by grid barriers.  Bandwidths are
// padded to a K class (1, 2, 4, 8) >= max(kl, ku); a SWITCH node (value set by
// band_mode_kernel) launches the matching variant only.
#include "internal.h"
#include "rcond.h"

namespace as {

constexpr int kSpThreads = 256;
constexpr int kSpR = 8;    // RHS columns per partition-solve chunk (one thread per column)
constexpr int kRedR = 8;   // RHS columns per reduced-solve chunk (the serial chains: 32/K columns per warp)

struct SpikeArgs {
    const DevArgs* args;
    int64_t lda, ldb, n, nrhs;
    DevState* st;
    int p, m;            // partitions, rows per partition (last one: n - (p-1) m)
    void* scratch;       // global scratch (plan W workspace)
    void* xe;            // estimator vector (n)
    void* xs;            // estimator sign vector (n)
    unsigned* bar;       // grid barrier counter (zeroed per solve)
};

// global scratch layout (elements of T)
template <int K>
struct SpLayout {
    static constexpr int S = 2 * K;
    int64_t tips, gt, zz, part;
    __host__ __device__ explicit SpLayout(int p) {
        tips = 0;                                        // [dir][i][4][K*K]
        gt = tips + (int64_t)2 * p * 4 * K * K;          // [i][2K][kSpR]
        zz = gt + (int64_t)p * 2 * K * kSpR;             // [i][S][kSpR]
        part = zz + (int64_t)p * S * kSpR;               // [cta][8] partial reductions
    }
    static int64_t total(int p) { return SpLayout(p).part + (int64_t)(p + 2) * 8; }
};

// ------------------------------------------------------------------ partition-level chains
// LU rows: LU[r*LDR + k], k = col - row + K; the diagonal slot holds 1/u_jj (reciprocal pivot).
// Solve A_i y = r (trans=0) or A_i^T y = r (trans=1) in place on v[0..m) (stride vs), one thread.
// LU rows (pitch LDR = 2K+2), zero pad rows -K..-1 and m..m+K-1; LU[j][K] = 1/u_jj.
// LC rows hold the factor's columns: LC[j][q] = L(j+1+q, j), LC[j][K+1+q] = U(j-1-q, j).
//
// One substitution sweep, column-oriented: once s_j is known it is folded into the pending
// right-hand sides of the next K rows of the sweep (acc[0..K-1]), so the dependency chain per
// row is one FMA (+ one multiply by 1/u) and the K updates are independent.  CASE: 0 unit L
// (forward, LC), 1 U (backward, LC), 2 U^T (forward, LU rows), 3 unit L^T (backward, LU rows).
// The right-hand sides entering the window are read kChunk rows ahead.
constexpr int kChunk = 8;
template <typename T, int K, int CASE>
AS_DEV void sweep_row(const T* __restrict__ LU, const T* __restrict__ LC, int j, T (&acc)[K], T enter,
                      T* __restrict__ v, int vs) {
    constexpr int LDR = 2 * K + 2;
    T c[K];
#pragma unroll
    for (int q = 0; q < K; ++q) {
        if (CASE == 0) c[q] = LC[j * LDR + q];               // L(j+1+q, j)
        if (CASE == 1) c[q] = LC[j * LDR + K + 1 + q];       // U(j-1-q, j)
        if (CASE == 2) c[q] = LU[j * LDR + K + 1 + q];       // U(j, j+1+q)
        if (CASE == 3) c[q] = LU[j * LDR + K - 1 - q];       // L(j, j-1-q)
    }
    T s = acc[0];
    if (CASE == 1 || CASE == 2) s *= LU[j * LDR + K];
    v[j * vs] = s;
#pragma unroll
    for (int q = 0; q + 1 < K; ++q) acc[q] = acc[q + 1] - c[q] * s;
    acc[K - 1] = enter - c[K - 1] * s;
}
template <typename T, int K, int CASE>
AS_DEV void sweep(const T* __restrict__ LU, const T* __restrict__ LC, int jb, int je, T* __restrict__ v, int vs) {
    constexpr bool FWD = (CASE == 0 || CASE == 2);
    const int cnt = je - jb;
    T acc[K];
#pragma unroll
    for (int q = 0; q < K; ++q) acc[q] = q < cnt ? v[(FWD ? jb + q : je - 1 - q) * vs] : T(0);
    int t = 0;
    for (; t + kChunk <= cnt; t += kChunk) {
        T vv[kChunk];
#pragma unroll
        for (int u = 0; u < kChunk; ++u) {
            const int te = t + u + K;
            vv[u] = te < cnt ? v[(FWD ? jb + te : je - 1 - te) * vs] : T(0);
        }
#pragma unroll
        for (int u = 0; u < kChunk; ++u) sweep_row<T, K, CASE>(LU, LC, FWD ? jb + t + u : je - 1 - t - u, acc, vv[u], v, vs);
    }
    for (; t < cnt; ++t) {
        const int te = t + K;
        const T ent = te < cnt ? v[(FWD ? jb + te : je - 1 - te) * vs] : T(0);
        sweep_row<T, K, CASE>(LU, LC, FWD ? jb + t : je - 1 - t, acc, ent, v, vs);
    }
}
template <typename T, int K>
AS_DEV void part_solve(const T* __restrict__ LU, const T* __restrict__ LC, int m, T* __restrict__ v, int vs, bool trans,
                       int first_nz) {
    if (!trans) {
        sweep<T, K, 0>(LU, LC, first_nz, m, v, vs);    // L y = r (rows before first_nz are zero)
        sweep<T, K, 1>(LU, LC, 0, m, v, vs);           // U x = y
    } else {
        sweep<T, K, 2>(LU, LC, first_nz, m, v, vs);    // U^T y = r
        sweep<T, K, 3>(LU, LC, 0, m, v, vs);           // L^T x = y
    }
}

// Reciprocal on the factor's dependency chain: MUFU approximation + two Newton steps
// (~55 cycles against ~127 for the IEEE division; within 1 ulp, not correctly rounded).
AS_DEV double recip(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    double e = fma(-x, r, 1.0);
    r = fma(r, e, r);
    e = fma(-x, r, 1.0);
    return fma(r, e, r);
}
AS_DEV float recip(float x) { return 1.0f / x; }

// Warp-level in-place Gauss-Jordan inverse of an S x S row-major matrix (S <= 32, no
// pivoting: the reduced pivots of a strictly dominant band matrix are dominant).
// Lane c owns column c of [M | I] (two register columns when S == 32... S <= 16 here:
// lanes 0..S-1 own M's columns, lanes S..2S-1 own the identity's).
template <typename T, int S>
AS_DEV void warp_gj_inverse(T* M) {
    static_assert(2 * S <= 32, "warp Gauss-Jordan handles S <= 16");
    const int lane = threadIdx.x & 31;
    T col[S];
#pragma unroll
    for (int r = 0; r < S; ++r) col[r] = lane < S ? M[r * S + lane] : (lane - S == r ? T(1) : T(0));
#pragma unroll
    for (int k = 0; k < S; ++k) {
        const T piv = __shfl_sync(0xffffffffu, col[k], k);
        const T inv = recip(piv);
        const T pk = col[k] * inv;          // normalized pivot-row entry of my column
        T f[S];
#pragma unroll
        for (int r = 0; r < S; ++r) f[r] = __shfl_sync(0xffffffffu, col[r], k);   // column k (multipliers)
#pragma unroll
        for (int r = 0; r < S; ++r) col[r] = (r == k) ? pk : col[r] - f[r] * pk;
    }
    if (lane >= S && lane < 2 * S)
#pragma unroll
        for (int r = 0; r < S; ++r) M[r * S + (lane - S)] = col[r];
    __syncwarp();
}

// ------------------------------------------------------------------ the kernel
template <typename T, int K>
__global__ void __launch_bounds__(kSpThreads, 1) band_spike_kernel(SpikeArgs a) {
    constexpr int kCPW = (32 / K < kRedR) ? 32 / K : kRedR;   // reduced-chain columns per warp
    constexpr int BW = 2 * K + 2, S = 2 * K;     // BW: LU row pitch (odd lane stride 2K+1 in the factor loop)
    {   // exactly one K-class variant runs (uniform exit for all CTAs of the others)
        const int km = max(a.st->kl, a.st->ku);
        const int cls = km <= 1 ? 1 : km <= 2 ? 2 : km <= 4 ? 4 : km <= 8 ? 8 : 16;
        if (!a.st->band_use_spike || cls != K) return;
    }
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int P = a.p, cta = blockIdx.x;
    const bool is_part = cta < P;
    const int rdir = cta - P;                  // reduced CTA direction (0: A, 1: A^T)
    const int64_t n = a.n;
    const int m = !is_part ? 0 : (cta == P - 1) ? (int)(n - (int64_t)(P - 1) * a.m) : a.m;
    const int64_t o = (int64_t)cta * a.m;
    DevState* st = a.st;
    const T* A = (const T*)a.args->A;
    const int64_t lda = a.lda;
    const int kl = st->kl, ku = st->ku;
    T* scr = (T*)a.scratch;
    const SpLayout<K> L(P);
    __shared__ T red_s[32];
    __shared__ long long redi_s[32];
    __shared__ T zsh[2 * K * kSpR];            // interface values a partition needs (solve correction)
    unsigned gen = 0;
    auto gbar = [&]() { grid_barrier(a.bar, ++gen, (unsigned)gridDim.x); };

    // smem carve-up: partition CTAs
    T* LU = (T*)smem_raw + (int64_t)K * BW;     // rows -K .. a.m+K-1, pitch BW
    T* SP = LU + (int64_t)(a.m + K) * BW;       // [4][K][a.m]: V, W (A), V', W' (A^T)
    T* G = SP + (int64_t)4 * K * a.m;           // a.m x kSpR
    T* LC = G + (int64_t)a.m * kSpR;            // a.m rows, pitch BW: the factor's columns (sweeps)
    // smem carve-up: reduced CTAs  [i][Lr(K x S) | Dinv(S x S) | Fv(K x K)] then h, y
    constexpr int RSZ = 7 * K * K;
    T* RM = (T*)smem_raw;
    T* RH = RM + (int64_t)(P - 1) * RSZ;        // [i][2K][kRedR] tips of g
    T* RY = RH + (int64_t)P * 2 * K * kRedR;    // 3 x [i][K][kRedR]  (c/a, u, d/b)
    T* RT = RY + (int64_t)3 * (P - 1) * K * kRedR;  // per-warp temps: 9 x K*max(K,kRedR)

#define STAMP(k) do { if (cta == 0 && threadIdx.x == 0) st->dbg_t[k] = gtimer(); } while (0)
    STAMP(0);
    // ---------------- F1: load the partition band and factor it (no pivoting)
    if (is_part) {
        {   // zero rows -K..a.m+K-1 (pads, out-of-band slots), then the band column by column:
            // e = (column c, slot k) with k fastest reads a contiguous run of rows of column c
            T* LU0 = LU - (int64_t)K * BW;
            for (int e = threadIdx.x; e < (a.m + 2 * K) * BW; e += blockDim.x) LU0[e] = T(0);
            __syncthreads();
            batched<8, T>(
                m * BW,
                [&](int e) -> T {
                    const int c = e / BW, k = e - c * BW, r = c + K - k;
                    const bool ok = k <= 2 * K && r >= 0 && r < m && k - K <= ku && K - k <= kl;
                    return ok ? A[(o + r) + (o + c) * lda] : T(0);
                },
                [&](int e, T v) {
                    const int c = e / BW, k = e - c * BW, r = c + K - k;
                    if (k <= 2 * K && r >= 0 && r < m) LU[r * BW + k] = v;
                });
        }
        __syncthreads();
        if (threadIdx.x < 32) {
            // lane r (1..K) owns row j+r of the active window: multiplier + its K updates.  Entries
            // outside the band / partition are zero in LU, so padding kl, ku to K adds zero work.
            // (A register-resident window with shuffle broadcasts measured 2.5x slower per step:
            // the step is instruction-issue bound for a single warp.)
            const int lane = threadIdx.x;
            for (int j = 0; j < m; ++j) {
                const T* prow = LU + j * BW + K;               // prow[c] = U(j, j+c)
                const T inv = recip(prow[0]);
                if (lane >= 1 && lane <= K && j + lane < m) {
                    T* row = LU + (j + lane) * BW + K - lane;  // row[c] = A(j+lane, j+c)
                    T rv[K + 1], pv[K + 1];
#pragma unroll
                    for (int c = 0; c <= K; ++c) { rv[c] = row[c]; pv[c] = prow[c]; }
                    const T l = rv[0] * inv;
                    row[0] = l;
#pragma unroll
                    for (int c = 1; c <= K; ++c) row[c] = rv[c] - l * pv[c];
                }
                __syncwarp();
                if (lane == 0) LU[j * BW + K] = inv;   // keep the reciprocal pivot
            }
            __syncwarp();
        }
        __syncthreads();

        // column copies of L and U for the column-oriented sweeps
        for (int e = threadIdx.x; e < m * 2 * K; e += blockDim.x) {
            const int j = e / (2 * K), qq = e - j * 2 * K;
            if (qq < K) LC[j * BW + qq] = LU[(j + 1 + qq) * BW + K - 1 - qq];
            else { const int q = qq - K; LC[j * BW + K + 1 + q] = LU[(j - 1 - q) * BW + K + 1 + q]; }
        }
        __syncthreads();
        STAMP(1);
        // ---------------- F2: spikes (kind 0 V, 1 W for A; 2 V', 3 W' for A^T), column q
        for (int e = threadIdx.x; e < 4 * K * a.m; e += blockDim.x) SP[e] = T(0);
        __syncthreads();
        if (threadIdx.x < 4 * K) {
            const int kind = threadIdx.x / K, q = threadIdx.x % K;
            T* v = SP + (int64_t)(kind * K + q) * a.m;
            int first = 0;
            const int64_t on = o + m;
            bool nz = false;
            if (kind == 0 && cta < P - 1) {          // B_i(aa, q) = A(o+m-K+aa, on+q)
                for (int aa = 0; aa < K; ++aa) {
                    const int64_t gr = o + m - K + aa, gc = on + q;
                    if (gc < n && gc - gr <= ku && gr - gc <= kl) v[m - K + aa] = A[gr + gc * lda];
                }
                first = m - K; nz = true;
            } else if (kind == 1 && cta > 0) {       // C_i(aa, q) = A(o+aa, o-K+q)
                for (int aa = 0; aa < K; ++aa) {
                    const int64_t gr = o + aa, gc = o - K + q;
                    if (gr - gc <= kl && gc - gr <= ku) v[aa] = A[gr + gc * lda];
                }
                nz = true;
            } else if (kind == 2 && cta < P - 1) {   // (A^T)(o+m-K+aa, on+q) = A(on+q, o+m-K+aa)
                for (int aa = 0; aa < K; ++aa) {
                    const int64_t gc = o + m - K + aa, gr = on + q;
                    if (gr < n && gr - gc <= kl && gc - gr <= ku) v[m - K + aa] = A[gr + gc * lda];
                }
                first = m - K; nz = true;
            } else if (kind == 3 && cta > 0) {       // (A^T)(o+aa, o-K+q) = A(o-K+q, o+aa)
                for (int aa = 0; aa < K; ++aa) {
                    const int64_t gr = o - K + q, gc = o + aa;
                    if (gc - gr <= ku && gr - gc <= kl) v[aa] = A[gr + gc * lda];
                }
                nz = true;
            }
            if (nz) part_solve<T, K>(LU, LC, m, v, 1, kind >= 2, first);
        }
        __syncthreads();
        // tips: [dir][i][w][rr][q], w: 0 Vtop, 1 Vbot, 2 Wtop, 3 Wbot
        for (int e = threadIdx.x; e < 2 * 4 * K * K; e += blockDim.x) {
            const int dir = e / (4 * K * K), w = (e / (K * K)) % 4, rr = (e / K) % K, q = e % K;
            const T* spk = SP + (int64_t)((dir * 2 + (w >= 2 ? 1 : 0)) * K + q) * a.m;
            const int row = (w == 0 || w == 2) ? rr : m - K + rr;
            scr[L.tips + (((int64_t)dir * P + cta) * 4 + w) * K * K + rr * K + q] = spk[row];
        }
    }
    STAMP(2);
    gbar();
    STAMP(3);

    // ---------------- F3 (reduced CTAs): block-Thomas factorization kept in smem
    //   z_i = [x_i(bottom K); x_{i+1}(top K)], i = 0..P-2:
    //   D_i = [[I, Vbot_i], [Wtop_{i+1}, I]],  E_i = [[Wbot_i, 0],[0,0]],  F_i = [[0,0],[0, Vtop_{i+1}]]
    //   Every pivot Dh_i = D_i - E_i Dh_{i-1}^{-1} F_{i-1} has the form [[I, X_i], [Y_i, I]], so with
    //   Si_i = (I - Y_i X_i)^{-1}, Q_i = X_i Si_i:
    //     Dh_i^{-1} [u; v] = [u - X_i b; b],  b = Si_i (v - Y_i u)
    //     X_0 = Vbot_0,  X_{i+1} = Vbot_{i+1} + Wbot_{i+1} Q_i Vtop_{i+1},  Y_i = Wtop_{i+1}
    //   and the solve reduces to two 1-matvec chains (see solve()):
    //     a_i = c_i - M_i a_{i-1},  M_i = Wbot_i + Q_i Y_i Wbot_i     (forward)
    //     b_i = d_i - N_i b_{i+1},  N_i = Si_i Vtop_{i+1}             (backward)
    //   Slots per interface: [0] X [1] Y [2] Si [3] Wb [4] Vt->N [5] Q [6] M  (K x K, row-major).
    if (!is_part && P > 1) {
        const T* tp = scr + L.tips + (int64_t)rdir * P * 4 * K * K;
        // e = (interface i, part w4, entry q): slot 0 X <- Vbot_i, 1 Y <- Wtop_{i+1}, 3 Wb <- Wbot_i,
        // 4 Vt <- Vtop_{i+1}
        batched<16, T>(
            (P - 1) * 4 * K * K,
            [&](int e) -> T {
                const int i = e / (4 * K * K), w4 = (e / (K * K)) & 3, q = e % (K * K);
                const int blk = (w4 == 1 || w4 == 3) ? i + 1 : i;
                const int tw = w4 == 0 ? 1 : w4 == 1 ? 2 : w4 == 2 ? 3 : 0;
                return __ldcg(&tp[((int64_t)blk * 4 + tw) * K * K + q]);
            },
            [&](int e, T v) {
                const int i = e / (4 * K * K), w4 = (e / (K * K)) & 3, q = e % (K * K);
                const int slot = w4 == 0 ? 0 : w4 == 1 ? 1 : w4 == 2 ? 3 : 4;
                RM[(int64_t)i * RSZ + slot * K * K + q] = v;
            });
        __syncthreads();
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        // C = A B (+ C if acc), K x K, one warp
        auto wmm = [&](T* C, const T* Am, const T* Bm, bool acc) {
            for (int e = lane; e < K * K; e += 32) {
                const int r = e / K, c = e % K;
                T s = T(0);
#pragma unroll
                for (int k = 0; k < K; ++k) s += Am[r * K + k] * Bm[k * K + c];
                C[e] = acc ? C[e] + s : s;
            }
            __syncwarp();
        };
        if (warp == 0) {
            T* t1 = RT;
            for (int i = 0; i <= P - 2; ++i) {
                T* X = RM + (int64_t)i * RSZ;
                T* Y = X + K * K;
                T* Si = Y + K * K;
                T* Q = X + 5 * K * K;
                if (i > 0) {
                    const T* Xp = RM + (int64_t)(i - 1) * RSZ;
                    wmm(t1, Xp + 5 * K * K, Xp + 4 * K * K, false);   // Q_{i-1} Vtop_i
                    wmm(X, X + 3 * K * K, t1, true);                 // X_i = Vbot_i + Wbot_i (...)
                }
                for (int e = lane; e < K * K; e += 32) {             // I - Y X
                    const int r = e / K, c = e % K;
                    T s = T(0);
#pragma unroll
                    for (int k = 0; k < K; ++k) s += Y[r * K + k] * X[k * K + c];
                    Si[e] = (r == c ? T(1) : T(0)) - s;
                }
                __syncwarp();
                warp_gj_inverse<T, K>(Si);
                wmm(Q, X, Si, false);
            }
        }
        __syncthreads();
        // independent per interface: N_i = Si_i Vt_i, M_i = Wb_i + Q_i (Y_i Wb_i)
        for (int i = warp; i <= P - 2; i += (int)(blockDim.x >> 5)) {
            T* R7 = RM + (int64_t)i * RSZ;
            T* tw = RT + (int64_t)(1 + warp) * K * K;
            wmm(tw, R7 + 2 * K * K, R7 + 4 * K * K, false);          // Si Vt
            for (int e = lane; e < K * K; e += 32) R7[4 * K * K + e] = tw[e];
            __syncwarp();
            wmm(tw, R7 + 1 * K * K, R7 + 3 * K * K, false);          // Y Wb
            for (int e = lane; e < K * K; e += 32) R7[6 * K * K + e] = R7[3 * K * K + e];
            __syncwarp();
            wmm(R7 + 6 * K * K, R7 + 5 * K * K, tw, true);           // M = Wb + Q (Y Wb)
        }
        __syncthreads();
    }
    // ---------------- the solve primitive: X(part) = A^{-1} F (dir 0) or A^{-T} F (dir 1)
    // input: G[r*kSpR + c] holds F rows of this partition (R <= kSpR columns); output overwrites G.
    if (!is_part && rdir == 0 && threadIdx.x == 0) st->dbg_t[4] = gtimer();
    int nsolve = 0;
#define STAMP1(k) do { if (nsolve == 0 && cta == 0 && threadIdx.x == 0) st->dbg_t[k] = gtimer(); } while (0)
    auto solve = [&](int dir, int R) {
        if (is_part) {
            if (threadIdx.x < R) part_solve<T, K>(LU, LC, m, G + threadIdx.x, kSpR, dir == 1, 0);
            __syncthreads();
            for (int e = threadIdx.x; e < 2 * K * R; e += blockDim.x) {
                const int rr = e / R, c = e % R;
                const int row = rr < K ? rr : m - 2 * K + rr;
                scr[L.gt + ((int64_t)cta * 2 * K + rr) * kSpR + c] = G[row * kSpR + c];
            }
        }
        STAMP1(8);
        gbar();
        STAMP1(9);
        if (!is_part && rdir == dir && P > 1) {
            const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (int)(blockDim.x >> 5);
            for (int c0 = 0; c0 < R; c0 += kRedR) {
                const int Rr = min(kRedR, R - c0);
                batched<16, T>(
                    P * 2 * K * Rr,
                    [&](int e) -> T {
                        const int c = e % Rr, ir = e / Rr;      // ir = i * 2K + rr
                        return __ldcg(&scr[L.gt + (int64_t)ir * kSpR + c0 + c]);
                    },
                    [&](int e, T v) { const int c = e % Rr, ir = e / Rr; RH[(int64_t)ir * kRedR + c] = v; });
                __syncthreads();
                // vectors [k][c], stride kRedR; gb_i = RH[i][K..2K), gt_{i+1} = RH[i+1][0..K)
                auto GB = [&](int i) { return RH + ((int64_t)i * 2 * K + K) * kRedR; };
                auto GT = [&](int i) { return RH + ((int64_t)(i + 1) * 2 * K) * kRedR; };
                T* CA = RY;                                             // (P-1) x K x kRedR
                T* UU = RY + (int64_t)(P - 1) * K * kRedR;
                T* DB = RY + (int64_t)2 * (P - 1) * K * kRedR;
                // Parallel phases: every (interface i, row r, column c) entry is one thread's K-term
                // dot product; a phase is a few block-wide passes separated by barriers.
                // pass(out, x, M, y): out_i = x_i - M_i y_i for i in [i0, P-2]   (K x Rr each)
                const int ne = K * Rr;
                auto pass = [&](int i0, auto&& fn) {
                    for (int e = threadIdx.x; e < (P - 1 - i0) * ne; e += blockDim.x) {
                        const int i = i0 + e / ne, f = e % ne, r = f / Rr, c = f - (f / Rr) * Rr;
                        fn(i, r, c);
                    }
                };
                auto dotM = [&](const T* M, const T* y, int r, int c) -> T {   // (M y)(r, c), tree sum
                    T pr[K];
#pragma unroll
                    for (int k = 0; k < K; ++k) pr[k] = M[r * K + k] * y[k * kRedR + c];
#pragma unroll
                    for (int h = 1; h < K; h *= 2)
#pragma unroll
                        for (int k = 0; k + h < K; k += 2 * h) pr[k] += pr[k + h];
                    return pr[0];
                };
#define RSTAMP(k) do { if (nsolve == 2 && rdir == 0 && threadIdx.x == 0) st->dbg_t[k] = gtimer(); } while (0)
                RSTAMP(11);
                RSTAMP(13);
                // A: c_i = gb_i - Q_i (gt_{i+1} - Y_i gb_i)      (UU: temporary)
                pass(0, [&](int i, int r, int c) {
                    const T* R7 = RM + (int64_t)i * RSZ;
                    UU[(int64_t)i * K * kRedR + r * kRedR + c] = GT(i)[r * kRedR + c] - dotM(R7 + 1 * K * K, GB(i), r, c);
                });
                __syncthreads();
                pass(0, [&](int i, int r, int c) {
                    const T* R7 = RM + (int64_t)i * RSZ;
                    CA[(int64_t)i * K * kRedR + r * kRedR + c] =
                        GB(i)[r * kRedR + c] - dotM(R7 + 5 * K * K, UU + (int64_t)i * K * kRedR, r, c);
                });
                __syncthreads();
                // serial chain  v_i = w_i - C_i v_{i -/+ 1}  (registers + shuffles; the next step's
                // coefficients and right-hand side are loaded while the current step waits)
                // one right-hand side: warp 0, lane = (row r = lane / 4, quarter q = lane % 4) holds
                // columns 2q, 2q+1 of C_i's row r; a step is 2 products, a 2-level xor reduction and
                // two shuffles that hand v_i to the lanes of the next step
                auto chain1 = [&](T* V, int slot, bool fwd) {
                    static_assert(K == 8 || K < 8, "");
                    if (warp != 0) return;
                    constexpr int KP = (K + 3) / 4;                    // columns per lane (K = 8: 2)
                    const int r = lane >> 2, q = lane & 3;
                    const bool act = r < K;
                    const int i_first = fwd ? 0 : P - 2, i_last = fwd ? P - 2 : 0, step = fwd ? 1 : -1;
                    T vpr[KP];
                    const T v0 = (act && q == 0) ? V[(int64_t)i_first * K * kRedR + r * kRedR] : T(0);
#pragma unroll
                    for (int u = 0; u < KP; ++u) {
                        const int k = q * KP + u;
                        vpr[u] = __shfl_sync(0xffffffffu, v0, (k < K ? k : 0) * 4);
                        if (k >= K) vpr[u] = T(0);
                    }
                    if (i_first == i_last) return;
                    int i = i_first + step;
                    auto ldc = [&](int ii, T (&mc)[KP], T& wc) {
#pragma unroll
                        for (int u = 0; u < KP; ++u) {
                            const int k = q * KP + u;
                            mc[u] = (act && k < K) ? RM[(int64_t)ii * RSZ + slot * K * K + r * K + k] : T(0);
                        }
                        wc = act ? V[(int64_t)ii * K * kRedR + r * kRedR] : T(0);
                    };
                    T mc[KP], wc;
                    ldc(i, mc, wc);
                    for (;;) {
                        const bool more = i != i_last;
                        const int inx = more ? i + step : i;
                        T mn[KP], wn;
                        ldc(inx, mn, wn);
                        T pr = T(0);
#pragma unroll
                        for (int u = 0; u < KP; ++u) pr += mc[u] * vpr[u];
                        pr += __shfl_xor_sync(0xffffffffu, pr, 1);
                        pr += __shfl_xor_sync(0xffffffffu, pr, 2);
                        const T v = wc - pr;
                        if (act && q == 0) V[(int64_t)i * K * kRedR + r * kRedR] = v;
#pragma unroll
                        for (int u = 0; u < KP; ++u) {
                            const int k = q * KP + u;
                            const T t = __shfl_sync(0xffffffffu, v, (k < K ? k : 0) * 4);
                            vpr[u] = k < K ? t : T(0);
                        }
                        if (!more) break;
                        i = inx;
#pragma unroll
                        for (int u = 0; u < KP; ++u) mc[u] = mn[u];
                        wc = wn;
                    }
                };
                auto chain = [&](T* V, int slot, bool fwd) {
                    if (Rr == 1) { chain1(V, slot, fwd); return; }
                    if (warp * kCPW >= Rr) return;                       // column group of this warp
                    const int cb = warp * kCPW, Rw = min(kCPW, Rr - cb);
                    const bool act = lane < K * Rw;
                    const int r = act ? lane / Rw : 0, cl = act ? lane % Rw : 0, c = cb + cl;
                    const int i_first = fwd ? 0 : P - 2, i_last = fwd ? P - 2 : 0, step = fwd ? 1 : -1;
                    T vp = act ? V[(int64_t)i_first * K * kRedR + r * kRedR + c] : T(0);
                    if (i_first == i_last) return;
                    int i = i_first + step;
                    T mc[K], wc;
#pragma unroll
                    for (int k = 0; k < K; ++k) mc[k] = act ? RM[(int64_t)i * RSZ + slot * K * K + r * K + k] : T(0);
                    wc = act ? V[(int64_t)i * K * kRedR + r * kRedR + c] : T(0);
                    for (;;) {
                        const bool more = i != i_last;
                        const int inx = more ? i + step : i;
                        T mn[K], wn;
#pragma unroll
                        for (int k = 0; k < K; ++k) mn[k] = act ? RM[(int64_t)inx * RSZ + slot * K * K + r * K + k] : T(0);
                        wn = act ? V[(int64_t)inx * K * kRedR + r * kRedR + c] : T(0);
                        T pr[K];
#pragma unroll
                        for (int k = 0; k < K; ++k) pr[k] = mc[k] * __shfl_sync(0xffffffffu, vp, k * Rw + cl);
#pragma unroll
                        for (int h = 1; h < K; h *= 2)
#pragma unroll
                            for (int k = 0; k + h < K; k += 2 * h) pr[k] += pr[k + h];
                        vp = wc - pr[0];
                        if (act) V[(int64_t)i * K * kRedR + r * kRedR + c] = vp;
                        if (!more) break;
                        i = inx;
#pragma unroll
                        for (int k = 0; k < K; ++k) mc[k] = mn[k];
                        wc = wn;
                    }
                };
                // B: a_i = c_i - M_i a_{i-1}
                chain(CA, 6, true);
                __syncthreads();
                RSTAMP(14);
                // C: u_i = gb_i - Wb_i a_{i-1};  d_i = Si_i (gt_{i+1} - Y_i u_i)   (CA reused as temporary
                //    after the first pass)
                pass(0, [&](int i, int r, int c) {
                    const T* R7 = RM + (int64_t)i * RSZ;
                    const T g = GB(i)[r * kRedR + c];
                    UU[(int64_t)i * K * kRedR + r * kRedR + c] =
                        i > 0 ? g - dotM(R7 + 3 * K * K, CA + (int64_t)(i - 1) * K * kRedR, r, c) : g;
                });
                __syncthreads();
                pass(0, [&](int i, int r, int c) {
                    const T* R7 = RM + (int64_t)i * RSZ;
                    CA[(int64_t)i * K * kRedR + r * kRedR + c] =
                        GT(i)[r * kRedR + c] - dotM(R7 + 1 * K * K, UU + (int64_t)i * K * kRedR, r, c);
                });
                __syncthreads();
                pass(0, [&](int i, int r, int c) {
                    const T* R7 = RM + (int64_t)i * RSZ;
                    DB[(int64_t)i * K * kRedR + r * kRedR + c] = dotM(R7 + 2 * K * K, CA + (int64_t)i * K * kRedR, r, c);
                });
                __syncthreads();
                // D: b_i = d_i - N_i b_{i+1}
                chain(DB, 4, false);
                __syncthreads();
                RSTAMP(15);
                // E: a_i = u_i - X_i b_i;  z_i = [a_i; b_i]
                pass(0, [&](int i, int r, int c) {
                    const T* R7 = RM + (int64_t)i * RSZ;
                    const T* bi = DB + (int64_t)i * K * kRedR;
                    scr[L.zz + ((int64_t)i * S + r) * kSpR + c0 + c] =
                        UU[(int64_t)i * K * kRedR + r * kRedR + c] - dotM(R7, bi, r, c);
                    scr[L.zz + ((int64_t)i * S + K + r) * kSpR + c0 + c] = bi[r * kRedR + c];
                });
                __syncthreads();
                RSTAMP(12);
            }
            if (nsolve == 0 && threadIdx.x == 0) st->dbg_t[10] = gtimer();
        }
        gbar();
        if (is_part) {
            // x_i = g_i - V_i t_{i+1} - W_i b_{i-1};  t_{i+1} = z_i[K:S], b_{i-1} = z_{i-1}[0:K]
            const T* V = SP + (int64_t)(dir * 2 + 0) * K * a.m;
            const T* Wsp = SP + (int64_t)(dir * 2 + 1) * K * a.m;
            // zsh[q][c]: q < K: t_{i+1}[q] = z_i[K+q];  q >= K: b_{i-1}[q-K] = z_{i-1}[q-K]
            batched<4, T>(
                2 * K * R,
                [&](int e) -> T {
                    const int q = e / R, c = e - q * R;
                    if (q < K) return cta < P - 1 ? __ldcg(&scr[L.zz + ((int64_t)cta * S + K + q) * kSpR + c]) : T(0);
                    return cta > 0 ? __ldcg(&scr[L.zz + ((int64_t)(cta - 1) * S + q - K) * kSpR + c]) : T(0);
                },
                [&](int e, T v) { zsh[e] = v; });
            __syncthreads();
            for (int e = threadIdx.x; e < m * R; e += blockDim.x) {
                const int r = e / R, c = e - r * R;
                T v = G[r * kSpR + c];
#pragma unroll
                for (int q = 0; q < K; ++q) v -= V[(int64_t)q * a.m + r] * zsh[q * R + c];
#pragma unroll
                for (int q = 0; q < K; ++q) v -= Wsp[(int64_t)q * a.m + r] * zsh[(K + q) * R + c];
                G[r * kSpR + c] = v;
            }
            __syncthreads();
        }
        ++nsolve;
    };

    // ---------------- rcond estimate (xLACN2 state machine, distributed reductions)
    T* xe = (T*)a.xe;
    T* xsg = (T*)a.xs;
    T* part = scr + L.part;
    const int64_t nn = n;
    auto block_sum = [&](T v) -> T {   // result valid on thread 0
        v = warp_sum(v);
        __syncthreads();               // red_s may still be read by a previous reduction
        if ((threadIdx.x & 31) == 0) red_s[threadIdx.x >> 5] = v;
        __syncthreads();
        T r = T(0);
        if (threadIdx.x == 0) for (int w = 0; w < (int)(blockDim.x >> 5); ++w) r += red_s[w];
        __syncthreads();
        return r;
    };
    // sum of the P partition partials, the same fixed tree in every CTA (so every thread of the
    // grid takes the same estimator branch): one L2 round trip, then a block reduction
    auto all_sum = [&](int slot) -> T {
        T v = (int)threadIdx.x < P ? __ldcg(&part[threadIdx.x * 8 + slot]) : T(0);
        v = warp_sum(v);
        __syncthreads();
        if ((threadIdx.x & 31) == 0) red_s[threadIdx.x >> 5] = v;
        __syncthreads();
        T r = T(0);
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) r += red_s[w];
        return r;
    };
    auto asum_local = [&](int col) -> T {
        T s = T(0);
        for (int r = threadIdx.x; r < m; r += blockDim.x) { const T v = G[r * kSpR + col]; s += v < T(0) ? -v : v; }
        return block_sum(s);
    };
    auto set_G_col0 = [&](auto f) {
        for (int r = threadIdx.x; r < m; r += blockDim.x) G[r * kSpR] = f(o + r);
        __syncthreads();
    };
    auto iamax_global = [&]() -> long long {
        if (is_part) {
            T v = T(-1);
            long long idx = 0x7fffffffffffffffll;
            for (int r = threadIdx.x; r < m; r += blockDim.x) {
                T x = G[r * kSpR];
                x = x < T(0) ? -x : x;
                argmax_merge(v, idx, x, (long long)(o + r));
                xe[o + r] = G[r * kSpR];      // publish z for the x[jlast] comparison
            }
            warp_argmax(v, idx);
            __syncthreads();
            if ((threadIdx.x & 31) == 0) { red_s[threadIdx.x >> 5] = v; redi_s[threadIdx.x >> 5] = idx; }
            __syncthreads();
            if (threadIdx.x == 0) {
                T bv = T(-1);
                long long bi = 0x7fffffffffffffffll;
                for (int w = 0; w < (int)(blockDim.x >> 5); ++w) argmax_merge(bv, bi, red_s[w], redi_s[w]);
                part[cta * 8 + 2] = bv;
                part[cta * 8 + 3] = (T)(double)bi;
            }
        }
        gbar();
        T bv = T(-1);
        long long bi = 0x7fffffffffffffffll;
        if ((int)threadIdx.x < P) { bv = __ldcg(&part[threadIdx.x * 8 + 2]); bi = (long long)(double)__ldcg(&part[threadIdx.x * 8 + 3]); }
        warp_argmax(bv, bi);
        __syncthreads();
        if ((threadIdx.x & 31) == 0) { red_s[threadIdx.x >> 5] = bv; redi_s[threadIdx.x >> 5] = bi; }
        __syncthreads();
        bv = T(-1);
        bi = 0x7fffffffffffffffll;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) argmax_merge(bv, bi, red_s[w], redi_s[w]);
        return bi == 0x7fffffffffffffffll ? 0 : bi;
    };

    STAMP(5);
    double est = 0.0;
    const T* Bm = (const T*)a.args->B;
    T* X = (T*)a.args->X;
    // The first solve carries every application of M = A^{-1} that does not depend on the
    // estimator's iteration: the start vector e/n (col 0), xLACN2's closing alternating-sign
    // probe (col 1), and the primary solve X = A^{-1} B (cols 2.., speculative: the gate may
    // still replace it; the spike path is not selected for X == B).
    const int R0 = (int)min<int64_t>(a.nrhs, kSpR - 2);
    {
        if (is_part) {
            for (int r = threadIdx.x; r < m; r += blockDim.x) {
                const int64_t i = o + r;
                const T sg = (i & 1) ? T(-1) : T(1);
                G[r * kSpR + 0] = T(1) / (T)nn;
                G[r * kSpR + 1] = sg * (T(1) + (T)i / (T)(nn - 1));
            }
            batched<8, T>(
                m * R0, [&](int e) -> T { const int c = e / m, r = e - c * m; return Bm[(o + r) + c * a.ldb]; },
                [&](int e, T v) { const int c = e / m, r = e - c * m; G[r * kSpR + 2 + c] = v; });
            __syncthreads();
        }
        solve(0, 2 + R0);                                    // y = M (e/n), alt probe, X = M B
        T s = T(0), s3 = T(0);
        if (is_part) {
            for (int c = 0; c < R0; ++c)
                for (int r = threadIdx.x; r < m; r += blockDim.x) X[(o + r) + c * a.ldb] = G[r * kSpR + 2 + c];
            s = asum_local(0);
            s3 = asum_local(1);
            if (threadIdx.x == 0) { part[cta * 8 + 0] = s; part[cta * 8 + 4] = s3; }
        }
        gbar();
        est = (double)all_sum(0);
        if (is_part)
            set_G_col0([&](int64_t i) { const T v = G[(i - o) * kSpR]; const T sg = v >= T(0) ? T(1) : T(-1); xsg[i] = sg; return sg; });
        solve(1, 1);                                         // z = M^T s
        long long j = iamax_global();
        int iter = 2;
        for (;;) {
            if (is_part) set_G_col0([&](int64_t i) { return i == j ? T(1) : T(0); });
            solve(0, 1);                                     // y = M e_j
            int diff = 0;
            T s2 = T(0);
            if (is_part) {
                s2 = asum_local(0);
                for (int r = threadIdx.x; r < m; r += blockDim.x) {
                    const T v = G[r * kSpR];
                    const T sg = v >= T(0) ? T(1) : T(-1);
                    if (sg != xsg[o + r]) diff = 1;
                }
                diff = __syncthreads_or(diff);
                if (threadIdx.x == 0) { part[cta * 8 + 0] = s2; part[cta * 8 + 1] = diff ? T(1) : T(0); }
            }
            gbar();
            const double estold = est;
            est = (double)all_sum(0);
            const bool anydiff = all_sum(1) > T(0);
            if (!anydiff || (T)est <= (T)estold) break;       // converged / no increase -> alternating probe
            if (is_part)
                set_G_col0([&](int64_t i) { const T v = G[(i - o) * kSpR]; const T sg = v >= T(0) ? T(1) : T(-1); xsg[i] = sg; return sg; });
            solve(1, 1);                                     // z = M^T s
            const long long jlast = j;
            j = iamax_global();
            const T zjl = __ldcg(&xe[jlast]);
            const T zj = __ldcg(&xe[j]);
            const T azj = zj < T(0) ? -zj : zj;
            if (zjl != azj && iter < 5) { ++iter; continue; }
            break;
        }
        // alternating-sign probe (applied in the first solve, column 1)
        const T tot = all_sum(4);
        const T temp = T(2) * (tot / (T)(3 * nn));
        if (temp > (T)est) est = (double)temp;
    }
    if (cta == 0 && threadIdx.x == 0) {
        const T anorm = (T)dfrom(st->anorm_bits);
        const T e = (T)est;
        T r;
        if (!(anorm > T(0)) || e == T(0)) r = T(0);
        else r = (T(1) / e) / anorm;
        st->rcond = (double)r;
        st->est = est;
    }

    STAMP(6);
    // ---------------- primary solve X = A^{-1} B (speculative: the gate may still replace it)
    // remaining right-hand sides (each CTA reads and writes only its own rows of B and X)
    for (int64_t c0 = R0; c0 < a.nrhs; c0 += kSpR) {
        const int R = (int)min<int64_t>(kSpR, a.nrhs - c0);
        if (is_part) {
            batched<8, T>(
                m * R, [&](int e) -> T { const int c = e / m, r = e - c * m; return Bm[(o + r) + (c0 + c) * a.ldb]; },
                [&](int e, T v) { const int c = e / m, r = e - c * m; G[r * kSpR + c] = v; });
            __syncthreads();
        }
        solve(0, R);
        if (is_part)
            for (int e = threadIdx.x; e < m * R; e += blockDim.x) {
                const int r = e % m, c = e / m;
                X[(o + r) + (c0 + c) * a.ldb] = G[r * kSpR + c];
            }
    }
    STAMP(7);
    if (cta == 0 && threadIdx.x == 0) st->band_fast = 1;
}

// ------------------------------------------------------------------ mode selection
// (strict diagonal dominance by rows or by columns: st->band_dom, set by band_norm_kernel in band.cu)
// feasible_mask bit c: the K = 2^c variant was captured (fits in shared memory, enough SMs)
__global__ void band_mode_kernel(const DevArgs* args, DevState* st, cudaGraphConditionalHandle h, int feasible_mask) {
    if (threadIdx.x != 0) return;
    // the spike kernel writes X speculatively before the gate: not for an in-place solve (X == B),
    // whose fallback still needs B
    const int km = max(st->kl, st->ku);
    const int cbit = km <= 1 ? 0 : km <= 2 ? 1 : km <= 4 ? 2 : km <= 8 ? 3 : 4;
    const int use = (st->band_dom != 0) && st->kl + st->ku > 0 && km <= 16 && ((feasible_mask >> cbit) & 1) &&
                    st->primary == AS_METHOD_BAND &&
                    (const void*)args->X != args->B;
    st->band_fast = 0;
    st->band_use_spike = use ? 1 + cbit : 0;      // 1 + K class index (SWITCH value; 0 = sequential)
    // not partitioned, kl, ku <= 3 (tridiagonal, the paper's 5-diagonal class): the register chain
    // (band_chain.cu, SWITCH value 5); it writes X before the gate, so not for X == B either
    const int chain = !use && st->kl <= 3 && st->ku <= 3 && st->primary == AS_METHOD_BAND &&
                      (const void*)args->X != args->B ? 1 + 4 * st->kl + st->ku : 0;
    st->band_chain = chain;
    if (h) cudaGraphSetConditional(h, use ? (unsigned)(1 + cbit) : chain ? 5u : 0u);
}

// ------------------------------------------------------------------ host side
template <typename T, int K>
static size_t part_smem(int M) {
    constexpr int BW = 2 * K + 2;
    return sizeof(T) * ((size_t)(M + 2 * K) * BW + (size_t)4 * K * M + (size_t)M * kSpR + (size_t)M * BW) + 64;
}
template <typename T, int K>
static size_t red_smem(int P) {
    constexpr int RSZ = 7 * K * K;
    return sizeof(T) * ((size_t)(P - 1) * RSZ + (size_t)P * 2 * K * kRedR + (size_t)3 * std::max(P - 1, 1) * K * kRedR +
                        (size_t)9 * K * std::max(K, kRedR)) + 64;
}

static size_t smem_optin() {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    return (size_t)v;
}

// Partition count balancing the partition chain (2m steps) against the reduced chain (2(p-1)
// block steps), limited by the reduced CTA's shared memory and the SM count.
template <typename T, int K>
static bool spike_geometry(int64_t n, int num_sms, int* P, int* M) {
    if (n < 256) return false;
    const size_t lim = smem_optin();
    double div = 4.0;
    if (const char* e = getenv("AS_SPIKE_DIV")) div = atof(e);   // tuning knob: p ~ sqrt(n / div)
    int p = (int)std::max<double>(2.0, std::floor(std::sqrt((double)n / div)));
    p = std::min(p, num_sms - 2);
    while (p > 2 && red_smem<T, K>(p) > lim) --p;
    int64_t m = (n + p - 1) / p;
    while (p > 2 && (m < 4 * K || n - (int64_t)(p - 1) * m < 2 * K)) { --p; m = (n + p - 1) / p; }
    if (p < 2 || red_smem<T, K>(p) > lim || part_smem<T, K>((int)m) > lim || m < 4 * K) return false;
    if (n - (int64_t)(p - 1) * m < 2 * K) return false;
    *P = p;
    *M = (int)m;
    return true;
}

template <typename T, int K>
static bool launch_spike_k(const Work& w, cudaStream_t s) {
    int P, M;
    if (!spike_geometry<T, K>(w.n, w.num_sms, &P, &M)) return false;
    SpikeArgs a;
    a.args = w.args; a.lda = w.lda; a.ldb = w.ldb; a.n = w.n; a.nrhs = w.nrhs; a.st = w.st;
    a.p = P; a.m = M; a.scratch = w.W; a.xe = w.xe; a.xs = w.vec; a.bar = w.bars + 2;
    const size_t smem = std::max(part_smem<T, K>(M), red_smem<T, K>(P));
    auto kern = band_spike_kernel<T, K>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(P + 2);
    cfg.blockDim = dim3(kSpThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, a);
    return true;
}

template <typename T>
static int feasible_mask_t(int64_t n, int num_sms) {
    int P, M, mask = 0;
    if (spike_geometry<T, 1>(n, num_sms, &P, &M)) mask |= 1;
    if (spike_geometry<T, 2>(n, num_sms, &P, &M)) mask |= 2;
    if (spike_geometry<T, 4>(n, num_sms, &P, &M)) mask |= 4;
    if (spike_geometry<T, 8>(n, num_sms, &P, &M)) mask |= 8;
    // K = 16 (2K = 32 pivots) is left to the sequential path: the warp Gauss-Jordan handles 2K <= 16
    return mask;
}

void launch_band_spike(const Work& w, int cls, cudaStream_t s) {
    if (w.dtype == AS_F64) {
        switch (cls) {
        case 0: launch_spike_k<double, 1>(w, s); break;
        case 1: launch_spike_k<double, 2>(w, s); break;
        case 2: launch_spike_k<double, 4>(w, s); break;
        case 3: launch_spike_k<double, 8>(w, s); break;
        default: break;
        }
    } else {
        switch (cls) {
        case 0: launch_spike_k<float, 1>(w, s); break;
        case 1: launch_spike_k<float, 2>(w, s); break;
        case 2: launch_spike_k<float, 4>(w, s); break;
        case 3: launch_spike_k<float, 8>(w, s); break;
        default: break;
        }
    }
}

void launch_band_dominance(const Work& w, cudaGraphConditionalHandle h, cudaStream_t s) {
    const int mask = w.dtype == AS_F64 ? feasible_mask_t<double>(w.n, w.num_sms) : feasible_mask_t<float>(w.n, w.num_sms);
    band_mode_kernel<<<1, 32, 0, s>>>(w.args, w.st, h, mask);
}

int64_t spike_scratch_elems(int64_t n, int num_sms) {
    (void)n;
    return SpLayout<16>::total(std::max(num_sms, 2));
}

}  // namespace as
