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

// Every chain reads its operands from shared memory: the warp stages the NEXT chunk of kCH steps
// (factor columns, pivots, entering right-hand-side values) into registers before lane 0 (or every
// lane, one vector each) runs the current chunk, and stores them after it -- the global-memory
// latency of the next chunk hides behind the ~kCH dependent steps of the current one.
constexpr int kCH = 64;
constexpr int kMaxKV = 6, kMaxLdab = 10;   // kl, ku <= 3

template <typename T>
struct ChainSm {
    T ab[kCH * kMaxLdab];          // factor columns of the chunk (or A's entering rows for xGBTRF)
    long long ip[kCH];
    T rd[kCH];                     // 1 / u_jj of the chunk
    T b[32 * (kCH + 1)];           // entering right-hand-side values, one row of kCH + 1 per lane
};

// asynchronous element copy global -> shared (zero-filled when !ok)
template <typename U>
AS_DEV void cpa(U* dst, const U* src, bool ok) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    const void* g = ok ? (const void*)src : (const void*)dst;
    if (sizeof(U) == 8)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(g), "r"(ok ? 8 : 0) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(d), "l"(g), "r"(ok ? 4 : 0) : "memory");
}
AS_DEV void cpa_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
AS_DEV void cpa_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// ------------------------------------------------------------------ xGBTRF (chain on lane 0)
template <typename T, int KL, int KU>
AS_DEV int64_t chain_gbtrf(ChainSm<T> (&sm)[2], const T* __restrict__ A, int64_t lda, int64_t n, T* ab,
                           int64_t* ipiv, T* rdiag) {
    constexpr int KV = KL + KU;
    constexpr int LDAB = 2 * KL + KU + 1;
    constexpr int NE = kCH * (KV + 1);
    const int lane = threadIdx.x;
    // entering row of step j: A(j + KL + 1, j + 1 + c), c = 0..KV (all in the band)
    auto issue = [&](int64_t c0, int buf) {
        for (int e = lane; e < NE; e += 32) {
            const int d = e / (KV + 1), c = e - d * (KV + 1);
            const int64_t i = c0 + d + KL + 1, k = c0 + d + 1 + c;
            const bool ok = i < n && k < n;
            cpa(&sm[buf].ab[e], ok ? &A[i + k * lda] : (const T*)nullptr, ok);
        }
        cpa_commit();
    };
    issue(0, 0);
    cpa_wait_all();
    __syncwarp();
    T w[KL + 1][KV + 1];
    int64_t info = 0;
    if (lane == 0) {
#pragma unroll
        for (int r = 0; r <= KL; ++r)
#pragma unroll
            for (int c = 0; c <= KV; ++c) {
                const bool inb = (r - c <= KL) && (c - r <= KU) && r < n && c < n;
                w[r][c] = inb ? A[r + (int64_t)c * lda] : T(0);
            }
    }
    for (int64_t c0 = 0, q = 0; c0 < n; c0 += kCH, ++q) {
        const int cur = (int)(q & 1);
        if (c0 + kCH < n) issue(c0 + kCH, cur ^ 1);                  // next chunk in flight
        if (lane == 0) {
            const int cnt = (int)min<int64_t>(kCH, n - c0);
            for (int d = 0; d < cnt; ++d) {
                const int64_t j = c0 + d;
                const int km = (int)min<int64_t>(KL, n - 1 - j);
                int p = 0;
                T best = cabs(w[0][0]);                              // first max (Z15)
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
                rdiag[j] = T(1) / w[0][0];                              // the solves multiply by 1/u_jj
                // factor column j: U(j, j + c) at AB(KV - c, j + c), L(j + r, j) at AB(KV + r, j)
#pragma unroll
                for (int c = 0; c <= KV; ++c)
                    if (j + c < n) ab[(KV - c) + (j + c) * (int64_t)LDAB] = w[0][c];
#pragma unroll
                for (int r = 1; r <= KL; ++r) ab[(KV + r) + j * (int64_t)LDAB] = l[r];
#pragma unroll
                for (int r = 0; r < KL; ++r)
#pragma unroll
                    for (int c = 0; c < KV; ++c) w[r][c] = w[r + 1][c + 1];
#pragma unroll
                for (int r = 0; r < KL; ++r) w[r][KV] = T(0);
#pragma unroll
                for (int c = 0; c <= KV; ++c) w[KL][c] = sm[cur].ab[d * (KV + 1) + c];
            }
        }
        cpa_wait_all();
        __syncwarp();
    }
    return __shfl_sync(0xffffffffu, (long long)info, 0);
}

// ------------------------------------------------------------------ xGBTRS ('N' / 'T') on nv vectors
// Lane l < nv solves vector l (b + l * ldv) in place; the factor chunk and the pivots are shared.
// 'N': interchanges + L forward, U backward.  'T': U^T forward, L^T backward with the interchanges
// undone in reverse (the oracle's gbtrs_vec / gbtrs_vec_t).
template <typename T, int KL, int KU>
AS_DEV void chain_gbtrs(ChainSm<T> (&sm)[2], const T* ab, const int64_t* ipiv, const T* rdiag, int64_t n, T* b,
                        int64_t ldv, int nv, bool trans) {
    constexpr int KV = KL + KU;
    constexpr int LDAB = 2 * KL + KU + 1;
    constexpr int NAB = kCH * LDAB;
    const int lane = threadIdx.x;
    const bool act = lane < nv;
    T* bl = b + (int64_t)(act ? lane : 0) * ldv;
    int cur = 0;
    // one sweep: chunks of kCH steps in direction fwd; per step j: factor column j, pivot j, and the
    // entering value b[j + boff] of every vector, staged by cp.async one chunk ahead
    auto sweep = [&](bool fwd, int64_t first, int64_t last, int boff, auto&& step) {
        const int64_t cnt_all = fwd ? last - first + 1 : first - last + 1;
        if (cnt_all <= 0) return;
        auto jof = [&](int64_t q, int d) { return fwd ? first + q * kCH + d : first - q * kCH - d; };
        auto issue = [&](int64_t q, int buf) {
            for (int e = lane; e < NAB; e += 32) {
                const int d = e / LDAB, r = e - d * LDAB;
                const int64_t j = jof(q, d);
                const bool ok = j >= 0 && j < n;
                cpa(&sm[buf].ab[e], ok ? &ab[r + j * (int64_t)LDAB] : (const T*)nullptr, ok);
            }
            for (int d = lane; d < kCH; d += 32) {
                const int64_t j = jof(q, d);
                const bool ok = j >= 0 && j < n;
                cpa(&sm[buf].ip[d], ok ? (const long long*)&ipiv[j] : (const long long*)nullptr, ok);
                cpa(&sm[buf].rd[d], ok ? &rdiag[j] : (const T*)nullptr, ok);
            }
            for (int e = lane; e < nv * kCH; e += 32) {
                const int v = e / kCH, d = e - v * kCH;
                const int64_t i = jof(q, d) + boff;
                const bool ok = i >= 0 && i < n;
                cpa(&sm[buf].b[v * (kCH + 1) + d], ok ? &b[i + v * ldv] : (const T*)nullptr, ok);
            }
            cpa_commit();
        };
        issue(0, cur);
        cpa_wait_all();
        __syncwarp();
        const int64_t nq = (cnt_all + kCH - 1) / kCH;
        for (int64_t q = 0; q < nq; ++q) {
            if (q + 1 < nq) issue(q + 1, cur ^ 1);
            const int cnt = (int)min<int64_t>(kCH, cnt_all - q * kCH);
            if (act)
                for (int d = 0; d < cnt; ++d) step(jof(q, d), d);
            cpa_wait_all();
            __syncwarp();
            cur ^= 1;
        }
    };
    auto col = [&](int d, int r) -> T { return sm[cur].ab[d * LDAB + r]; };
    auto ent = [&](int d) -> T { return sm[cur].b[lane * (kCH + 1) + d]; };
    if (!trans) {
        // forward: window v[r] = b[j + r]
        T v[KL + 1];
#pragma unroll
        for (int r = 0; r <= KL; ++r) v[r] = (act && r < n) ? bl[r] : T(0);
        sweep(true, 0, n - 1, KL + 1, [&](int64_t j, int d) {
            const T nxt = ent(d);
            if (j + 1 < n) {
                const int lm = (int)min<int64_t>(KL, n - 1 - j);
                const int p = (int)(sm[cur].ip[d] - j);
#pragma unroll
                for (int r = 1; r <= KL; ++r)
                    if (r == p) { const T t = v[0]; v[0] = v[r]; v[r] = t; }
#pragma unroll
                for (int r = 1; r <= KL; ++r)
                    if (r <= lm) v[r] = v[r] - col(d, KV + r) * v[0];
            }
            bl[j] = v[0];
#pragma unroll
            for (int r = 0; r < KL; ++r) v[r] = v[r + 1];
            if (KL > 0) v[KL] = nxt;
            else v[0] = nxt;
        });
        __syncwarp();
        // backward: window u[c] = b[j - KV + c], u[KV] = b[j]
        T u[KV + 1];
#pragma unroll
        for (int c = 0; c <= KV; ++c) u[c] = (act && n - 1 - KV + c >= 0) ? bl[n - 1 - KV + c] : T(0);
        sweep(false, n - 1, 0, -KV - 1, [&](int64_t j, int d) {
            const T prev = ent(d);
            const T x = u[KV] * sm[cur].rd[d];
            bl[j] = x;
#pragma unroll
            for (int c = 0; c < KV; ++c)
                if (j - KV + c >= 0) u[c] = u[c] - col(d, c) * x;       // U(j - KV + c, j) at AB(c, j)
#pragma unroll
            for (int c = KV; c > 0; --c) u[c] = u[c - 1];
            u[0] = prev;
        });
    } else {
        // U^T forward: x_j = (b_j - sum_{i=j-KV}^{j-1} U(i, j) x_i) / U(j, j); xs = last KV x
        T xs[KV + 1];
#pragma unroll
        for (int c = 0; c <= KV; ++c) xs[c] = T(0);
        sweep(true, 0, n - 1, 0, [&](int64_t j, int d) {
            T s = ent(d);
#pragma unroll
            for (int c = 0; c < KV; ++c)
                if (j - KV + c >= 0) s = s - col(d, c) * xs[c];
            const T x = s * sm[cur].rd[d];
            bl[j] = x;
#pragma unroll
            for (int c = 0; c + 1 < KV; ++c) xs[c] = xs[c + 1];
            if (KV > 0) xs[KV - 1] = x;
        });
        __syncwarp();
        // L^T backward with the interchanges in reverse: window v[r] = b[j + r]
        if (KL > 0 && n >= 2) {
            T v[KL + 1];
#pragma unroll
            for (int r = 0; r <= KL; ++r) v[r] = (act && n - 2 + r < n) ? bl[n - 2 + r] : T(0);
            sweep(false, n - 2, 0, -1, [&](int64_t j, int d) {
                const T prev = ent(d);
                const int lm = (int)min<int64_t>(KL, n - 1 - j);
                T s = v[0];
#pragma unroll
                for (int r = 1; r <= KL; ++r)
                    if (r <= lm) s = s - col(d, KV + r) * v[r];
                v[0] = s;
                const int p = (int)(sm[cur].ip[d] - j);
#pragma unroll
                for (int r = 1; r <= KL; ++r)
                    if (r == p) { const T t = v[0]; v[0] = v[r]; v[r] = t; bl[j + r] = v[r]; }
                bl[j] = v[0];
#pragma unroll
                for (int r = KL; r > 0; --r) v[r] = v[r - 1];
                v[0] = prev;
            });
        }
    }
    __syncwarp();
}

// ------------------------------------------------------------------ the kernel (one warp)
template <typename T, int KL, int KU>
AS_DEV void band_chain_body(ChainSm<T> (&sm)[2], const DevArgs* args, int64_t lda, int64_t n, int64_t ldb,
                            int64_t nrhs, T* ab, int64_t* ipiv, T* xv, signed char* isgn, T* rdiag, DevState* st) {
    const int lane = threadIdx.x;
    const T* A = (const T*)args->A;
    const long long info = chain_gbtrf<T, KL, KU>(sm, A, lda, n, ab, ipiv, rdiag);
    __syncwarp();
    __threadfence_block();
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
    auto apply = [&](bool tr) { chain_gbtrs<T, KL, KU>(sm, ab, ipiv, rdiag, n, xv, n, 1, tr); sync(); };
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
    for (int64_t c0 = 0; c0 < nrhs; c0 += 32) {
        const int nv = (int)min<int64_t>(32, nrhs - c0);
        for (int64_t e = lane; e < n * nv; e += 32) {
            const int64_t i = e % n, c = c0 + e / n;
            X[i + c * ldb] = B[i + c * ldb];
        }
        sync();
        chain_gbtrs<T, KL, KU>(sm, ab, ipiv, rdiag, n, X + c0 * ldb, ldb, nv, false);
    }
    if (lane == 0) st->band_fast = 1;
}

// one kernel, the (kl, ku) instance picked on device (kl / ku are only known after detection)
template <typename T>
__global__ void __launch_bounds__(32, 1) band_chain_kernel(const DevArgs* args, int64_t lda, int64_t n, int64_t ldb,
                                                           int64_t nrhs, T* ab, int64_t* ipiv, T* xv,
                                                           signed char* isgn, T* rdiag, DevState* st) {
    __shared__ ChainSm<T> sm[2];
    switch (st->band_chain) {
#define AS_CHAIN_CASE(KL, KU) \
    case 1 + 4 * KL + KU: band_chain_body<T, KL, KU>(sm, args, lda, n, ldb, nrhs, ab, ipiv, xv, isgn, rdiag, st); break;
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
                                                    (double*)w.xe, (signed char*)w.zx, (double*)w.vec, w.st);
    else
        band_chain_kernel<float><<<1, 32, 0, s>>>(w.args, w.lda, w.n, w.ldb, w.nrhs, (float*)w.W, w.ipiv,
                                                   (float*)w.xe, (signed char*)w.zx, (float*)w.vec, w.st);
}

}  // namespace as
