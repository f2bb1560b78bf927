// rcond.cu -- K10: reciprocal condition estimate (the xxCON family
// P:350).  1-norm estimate of ||A^{-1}||_1 by the
// Hager-Higham procedure in the form of LAPACK's xLACN2 (Z13b), run as a
// device-resident state machine: 11 fixed "apply" slots (M or M^T through the
// path's factors, see launch_estimator) interleaved with single-CTA step
// kernels; a slot whose turn never comes exits at once, so the host never
// synchronizes.  rcond = (1/est)/anorm.
#include <cstdlib>

#include "internal.h"
#include "rcond.h"
#include "trsm.h"

namespace as {

constexpr int kEstThreads = 1024;
constexpr int kEstSlots = 11;

// block-wide helpers (1024 threads)
template <typename T>
AS_DEV T block_sum(T v, T* sh) {
    v = warp_sum(v);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) sh[w] = v;
    __syncthreads();
    T r = (threadIdx.x < (blockDim.x >> 5)) ? sh[threadIdx.x] : T(0);
    if (w == 0) r = warp_sum(r);
    if (threadIdx.x == 0) sh[0] = r;
    __syncthreads();
    r = sh[0];
    __syncthreads();
    return r;
}

template <typename T>
AS_DEV long long block_iamax(const T* x, int64_t n, T* shv, long long* shi) {
    T v = T(-1);
    long long idx = 0x7fffffffffffffffll;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        T a = x[i] < T(0) ? -x[i] : x[i];
        argmax_merge(v, idx, a, (long long)i);
    }
    warp_argmax(v, idx);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) { shv[w] = v; shi[w] = idx; }
    __syncthreads();
    if (w == 0) {
        v = (l < (int)(blockDim.x >> 5)) ? shv[l] : T(-1);
        idx = (l < (int)(blockDim.x >> 5)) ? shi[l] : 0x7fffffffffffffffll;
        warp_argmax(v, idx);
        if (l == 0) shi[0] = idx;
    }
    __syncthreads();
    long long r = shi[0];
    __syncthreads();
    return r == 0x7fffffffffffffffll ? 0 : r;
}

template <typename T>
AS_DEV void set_alt(T* x, int64_t n) {
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        const T sgn = (i & 1) ? T(-1) : T(1);
        x[i] = sgn * (T(1) + (T)i / (T)(n - 1));
    }
}

// x = e/n, est_next = 0 (or done if the factor was singular / n == 0)
template <typename T>
__global__ void est_begin_kernel(DevState* st, T* x, int64_t n, int init_x) {
    const bool singular = st->info != ~0ull;
    if (init_x)
        for (int64_t i = threadIdx.x; i < n; i += blockDim.x) x[i] = T(1) / (T)n;
    if (threadIdx.x == 0) {
        st->est_next = singular ? -1 : 0;
        st->est = 0.0;
        st->est_iter = 0;
        st->est_j = 0;
        st->est_jlast = 0;
    }
}

// After apply slot `slot` ran on x (only if est_next == slot).
// xs holds the stored sign vector (isgn) as +-1.
// altres != nullptr: M applied to the closing alternating-sign probe was computed up front (fused
// into the primary solve): the probe's estimate temp = 2 ||M alt||_1 / (3n) is taken at once
// instead of requesting one more application.
template <typename T>
__global__ void __launch_bounds__(kEstThreads) est_step_kernel(DevState* st, T* x, T* xs, int64_t n, int slot,
                                                               const T* altres) {
    if (ld_volatile_i32(&st->est_next) != slot) return;
    __shared__ T sh[32];
    __shared__ T shv[32];
    __shared__ long long shi[32];
    __shared__ int s_flag;
    // the closing probe from the precomputed M alt (block-uniform call): est = max(est_now, temp)
    auto alt_now = [&](T est_now) {
        T sa = T(0);
        for (int64_t i = threadIdx.x; i < n; i += blockDim.x) sa += altres[i] < T(0) ? -altres[i] : altres[i];
        sa = block_sum(sa, sh);
        if (threadIdx.x == 0) {
            const T temp = T(2) * (sa / (T)(3 * n));
            st->est = (double)(temp > est_now ? temp : est_now);
            st->est_iter = -1;
            st->est_next = -1;
        }
    };
    if (slot == 0) {
        if (n == 1) {
            if (threadIdx.x == 0) {
                T a = x[0] < T(0) ? -x[0] : x[0];
                st->est = (double)a;
                st->est_next = -1;
            }
            return;
        }
        T s = T(0);
        for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += x[i] < T(0) ? -x[i] : x[i];
        s = block_sum(s, sh);
        for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
            const T sg = x[i] >= T(0) ? T(1) : T(-1);
            x[i] = sg;
            xs[i] = sg;
        }
        if (threadIdx.x == 0) { st->est = (double)s; st->est_next = 1; }
        return;
    }
    if (slot == 1) {  // after z = M^T s
        long long j = block_iamax(x, n, shv, shi);
        for (int64_t i = threadIdx.x; i < n; i += blockDim.x) x[i] = (i == j) ? T(1) : T(0);
        if (threadIdx.x == 0) { st->est_j = (int)j; st->est_iter = 2; st->est_next = 2; }
        return;
    }
    if ((slot & 1) == 0) {  // after y = M x (either M e_j, or the alternating probe)
        if (st->est_iter < 0) {  // alternating probe result: temp = 2*asum/(3n)
            T s = T(0);
            for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += x[i] < T(0) ? -x[i] : x[i];
            s = block_sum(s, sh);
            if (threadIdx.x == 0) {
                const T temp = T(2) * (s / (T)(3 * n));
                const T est = (T)st->est;
                if (temp > est) st->est = (double)temp;
                st->est_next = -1;
            }
            return;
        }
        T s = T(0);
        for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += x[i] < T(0) ? -x[i] : x[i];
        s = block_sum(s, sh);
        if (threadIdx.x == 0) s_flag = 0;
        __syncthreads();
        for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
            const T sg = x[i] >= T(0) ? T(1) : T(-1);
            if (sg != xs[i]) s_flag = 1;   // benign race: any writer sets 1
        }
        __syncthreads();
        const T estold = (T)st->est;
        const bool differ = s_flag != 0;
        __syncthreads();
        const bool go_alt = !differ || (s <= estold);
        if (go_alt && altres) {
            if (threadIdx.x == 0) st->est_old = (double)estold;
            alt_now(s);
        } else if (go_alt) {
            set_alt(x, n);
            if (threadIdx.x == 0) { st->est = (double)s; st->est_old = (double)estold; st->est_iter = -1; st->est_next = slot + 2; }
        } else {
            for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
                const T sg = x[i] >= T(0) ? T(1) : T(-1);
                x[i] = sg;
                xs[i] = sg;
            }
            if (threadIdx.x == 0) { st->est = (double)s; st->est_old = (double)estold; st->est_next = slot + 1; }
        }
        return;
    }
    // odd slot >= 3: after z = M^T s
    {
        const int jlast = st->est_j;
        const T xjl = __ldcg(&x[jlast]);
        long long j = block_iamax(x, n, shv, shi);
        const T xj = x[j] < T(0) ? -x[j] : x[j];
        const int iter = st->est_iter;
        __syncthreads();
        if (xjl != xj && iter < 5) {
            for (int64_t i = threadIdx.x; i < n; i += blockDim.x) x[i] = (i == j) ? T(1) : T(0);
            if (threadIdx.x == 0) { st->est_jlast = jlast; st->est_j = (int)j; st->est_iter = iter + 1; st->est_next = slot + 1; }
        } else if (altres) {
            if (threadIdx.x == 0) { st->est_jlast = jlast; st->est_j = (int)j; }
            alt_now((T)st->est);
        } else {
            set_alt(x, n);
            if (threadIdx.x == 0) { st->est_jlast = jlast; st->est_j = (int)j; st->est_iter = -1; st->est_next = slot + 1; }
        }
    }
}

template <typename T>
__global__ void est_finish_kernel(DevState* st) {
    if (threadIdx.x != 0) return;
    if (st->info != ~0ull) { st->rcond = 0.0; return; }
    const T anorm = (T)dfrom(st->anorm_bits);
    const T est = (T)st->est;
    T r;
    if (!(anorm > T(0)) || est == T(0)) r = T(0);
    else r = (T(1) / est) / anorm;
    st->rcond = (double)r;
}

// ------------------------------------------------------------------ small n: the whole estimator in one CTA
// For n <= kEstFusedN the 11-slot state machine above (1 + 11 x (1-2 triangular-solve launches + 1
// step launch) + 1 kernels, most of them exiting at once) costs more in launches than in work: C1's
// estimate was ~190 us of a 545 us solve.  Here one 1024-thread CTA runs xLACN2 (Z13b) start to
// finish with the vectors in shared memory and the triangular factors read from L2.
// cta_trsv: blocked substitution op(T) x = x with the inverted 64 x 64 diagonal blocks (Dinv, the
// same blocks the multi-CTA solves use): x_b <- op(Dinv_b) x_b, then the block's contribution is
// removed from the remaining right-hand sides (no-trans: a thread per row, coalesced columns; trans:
// a warp per unknown, the 64 contiguous elements of its column).
constexpr int kEstFusedN = 512;
template <typename T, bool UPPER, bool TRANS>
AS_DEV void cta_trsv(const T* __restrict__ A, int64_t lda, const T* __restrict__ Dinv, T* x, int n, T* red) {
    constexpr bool FWD = (!UPPER && !TRANS) || (UPPER && TRANS);
    const int nblk = (n + kNB - 1) / kNB;
    const int t = threadIdx.x;
    for (int s = 0; s < nblk; ++s) {
        const int b = FWD ? s : nblk - 1 - s, ob = b * kNB;
        {
            const int i = t & 63, q = t >> 6;                 // 16 k-slices of 4
            const T* D = Dinv + (int64_t)b * kNB * kNB;
            T p = T(0);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int k = 4 * q + u;
                const T xv = ob + k < n ? x[ob + k] : T(0);
                p += (TRANS ? D[k + i * kNB] : D[i + k * kNB]) * xv;
            }
            red[q * 64 + i] = p;
            __syncthreads();
            if (t < 64 && ob + t < n) {
                T sum = T(0);
#pragma unroll
                for (int q2 = 0; q2 < 16; ++q2) sum += red[q2 * 64 + t];
                x[ob + t] = sum;
            }
            __syncthreads();
        }
        const int r0 = FWD ? ob + kNB : 0, r1 = FWD ? n : ob;   // unknowns still to come
        if (r1 <= r0) continue;
        const int nb = min(kNB, n - ob);
        if (!TRANS) {
            const int rl = t & 255, kq = t >> 8;              // 4 k-slices of 16
            for (int rb = r0; rb < r1; rb += 512) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int r = rb + rl + 256 * h;
                    T p = T(0);
                    if (r < r1) {
#pragma unroll
                        for (int u = 0; u < 16; ++u) {
                            const int k = 16 * kq + u;
                            if (k < nb) p += A[r + (int64_t)(ob + k) * lda] * x[ob + k];
                        }
                    }
                    red[kq * 512 + rl + 256 * h] = p;
                }
                __syncthreads();
                if (kq == 0) {
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int r = rb + rl + 256 * h, e = rl + 256 * h;
                        if (r < r1) x[r] -= (red[e] + red[512 + e]) + (red[1024 + e] + red[1536 + e]);
                    }
                }
                __syncthreads();
            }
        } else {
            const int lane = t & 31, wp = t >> 5;
            for (int c = r0 + wp; c < r1; c += 32) {
                const T* col = A + ob + (int64_t)c * lda;
                T p = (lane < nb ? col[lane] * x[ob + lane] : T(0)) + (lane + 32 < nb ? col[lane + 32] * x[ob + lane + 32] : T(0));
                p = warp_sum(p);
                if (lane == 0) x[c] -= p;
            }
            __syncthreads();
        }
    }
}

template <typename T>
__global__ void __launch_bounds__(kEstThreads) est_small_kernel(DevState* st, const DevArgs* args, const T* W, int64_t ldw,
                                                                int64_t lda, const T* Dinv0, const T* Dinv1, int n, int kind,
                                                                int upper, const T* xe, const T* altres) {
    __shared__ T x[kEstFusedN];
    __shared__ T xs[kEstFusedN];
    __shared__ T red[2048];
    __shared__ T sh[32];
    __shared__ T shv[32];
    __shared__ long long shi[32];
    __shared__ int s_flag;
    const int t = threadIdx.x;
    if (st->info != ~0ull) {                     // singular factor: rcond = 0 (est_begin / est_finish)
        if (t == 0) { st->est_next = -1; st->est = 0.0; st->rcond = 0.0; }
        return;
    }
    const T* A = kind == KIND_TRI ? (const T*)args->A : W;
    const int64_t ld = kind == KIND_TRI ? lda : ldw;
    auto apply = [&](bool trans) {               // x <- M x or M^T x, M = A^{-1} through the path's factors
        if (kind == KIND_LU) {
            if (!trans) { cta_trsv<T, false, false>(A, ld, Dinv0, x, n, red); cta_trsv<T, true, false>(A, ld, Dinv1, x, n, red); }
            else { cta_trsv<T, true, true>(A, ld, Dinv1, x, n, red); cta_trsv<T, false, true>(A, ld, Dinv0, x, n, red); }
        } else if (kind == KIND_CHOL) {
            cta_trsv<T, false, false>(A, ld, Dinv0, x, n, red);
            cta_trsv<T, false, true>(A, ld, Dinv0, x, n, red);
        } else if (upper) {
            if (!trans) cta_trsv<T, true, false>(A, ld, Dinv0, x, n, red);
            else cta_trsv<T, true, true>(A, ld, Dinv0, x, n, red);
        } else {
            if (!trans) cta_trsv<T, false, false>(A, ld, Dinv0, x, n, red);
            else cta_trsv<T, false, true>(A, ld, Dinv0, x, n, red);
        }
    };
    auto asum = [&]() {
        T sv = T(0);
        for (int i = t; i < n; i += blockDim.x) sv += x[i] < T(0) ? -x[i] : x[i];
        return block_sum(sv, sh);
    };
    // x = M (e/n): computed with the primary solve (altres given) or here
    if (altres) { for (int i = t; i < n; i += blockDim.x) x[i] = xe[i]; __syncthreads(); }
    else { for (int i = t; i < n; i += blockDim.x) x[i] = T(1) / (T)n; __syncthreads(); apply(false); }
    T est;
    if (n == 1) {
        est = x[0] < T(0) ? -x[0] : x[0];
    } else {
        est = asum();
        for (int i = t; i < n; i += blockDim.x) { const T sg = x[i] >= T(0) ? T(1) : T(-1); x[i] = sg; xs[i] = sg; }
        __syncthreads();
        apply(true);
        int j = (int)block_iamax(x, (int64_t)n, shv, shi);
        int iter = 2;
        bool alt = false;                          // the closing alternating-sign probe is due
        for (;;) {
            for (int i = t; i < n; i += blockDim.x) x[i] = (i == j) ? T(1) : T(0);
            __syncthreads();
            apply(false);                           // y = M e_j
            const T sv = asum();
            if (t == 0) s_flag = 0;
            __syncthreads();
            for (int i = t; i < n; i += blockDim.x) {
                const T sg = x[i] >= T(0) ? T(1) : T(-1);
                if (sg != xs[i]) s_flag = 1;        // benign race: any writer sets 1
            }
            __syncthreads();
            const bool differ = s_flag != 0;
            const T estold = est;
            __syncthreads();
            if (!differ || sv <= estold) { est = sv; alt = true; break; }   // (est_step: est = s before the probe)
            est = sv;
            for (int i = t; i < n; i += blockDim.x) { const T sg = x[i] >= T(0) ? T(1) : T(-1); x[i] = sg; xs[i] = sg; }
            __syncthreads();
            apply(true);                            // z = M^T s
            const int jlast = j;
            const T xjl = x[jlast];
            __syncthreads();
            j = (int)block_iamax(x, (int64_t)n, shv, shi);
            const T xj = x[j] < T(0) ? -x[j] : x[j];
            __syncthreads();
            if (xjl != xj && iter < 5) { ++iter; continue; }
            alt = true;
            break;
        }
        if (alt) {
            T sa;
            if (altres) {
                T v = T(0);
                for (int i = t; i < n; i += blockDim.x) v += altres[i] < T(0) ? -altres[i] : altres[i];
                sa = block_sum(v, sh);
            } else {
                for (int i = t; i < n; i += blockDim.x) {
                    const T sgn = (i & 1) ? T(-1) : T(1);
                    x[i] = sgn * (T(1) + (T)i / (T)(n - 1));
                }
                __syncthreads();
                apply(false);
                sa = asum();
            }
            const T temp = T(2) * (sa / (T)(3 * n));
            if (temp > est) est = temp;
        }
    }
    if (t == 0) {
        const T anorm = (T)dfrom(st->anorm_bits);
        T r;
        if (!(anorm > T(0)) || est == T(0)) r = T(0);
        else r = (T(1) / est) / anorm;
        st->est = (double)est;
        st->est_next = -1;
        st->rcond = (double)r;
    }
}

// ------------------------------------------------------------------ launcher
// kind: KIND_LU (W = L\U, Dinv0 = inv blocks of unit L, Dinv1 = of U),
//       KIND_TRI (args->A triangle, Dinv0), KIND_CHOL (W = L, Dinv0),
//       KIND_BAND (band solves, see band.cu).
void launch_estimator(const Work& w, int kind, bool upper, SyncAlloc& sa, cudaStream_t s, const void* altres) {
    const int dt = w.dtype;
    const int64_t n = w.n;
    const int64_t ldw = w.ldw;  // W leading dimension
    // altres != nullptr: xe already holds M (e/n) and altres M alt (fused into the primary solve)
    const int init_x = altres ? 0 : 1;
    static const bool fused_off = getenv("AS_EST_FUSED_OFF") != nullptr;
    if (n <= kEstFusedN && kind != KIND_BAND && !fused_off) {      // one CTA, one launch (est_small_kernel)
        if (dt == AS_F64)
            est_small_kernel<double><<<1, kEstThreads, 0, s>>>(w.st, w.args, (const double*)w.W, ldw, w.lda, (const double*)w.Dinv0,
                                                              (const double*)w.Dinv1, (int)n, kind, upper ? 1 : 0,
                                                              (const double*)w.xe, (const double*)altres);
        else
            est_small_kernel<float><<<1, kEstThreads, 0, s>>>(w.st, w.args, (const float*)w.W, ldw, w.lda, (const float*)w.Dinv0,
                                                             (const float*)w.Dinv1, (int)n, kind, upper ? 1 : 0,
                                                             (const float*)w.xe, (const float*)altres);
        return;
    }
    if (dt == AS_F64) est_begin_kernel<double><<<1, kEstThreads, 0, s>>>(w.st, (double*)w.xe, n, init_x);
    else est_begin_kernel<float><<<1, kEstThreads, 0, s>>>(w.st, (float*)w.xe, n, init_x);
    void* xs = (char*)w.vec;  // sign vector scratch (n elements)
    for (int slot = 0; slot < kEstSlots; ++slot) {
        const bool trans = (slot & 1) != 0;
        if (altres && slot == 0) {                 // first application already done
            if (dt == AS_F64) est_step_kernel<double><<<1, kEstThreads, 0, s>>>(w.st, (double*)w.xe, (double*)xs, n, 0, (const double*)altres);
            else est_step_kernel<float><<<1, kEstThreads, 0, s>>>(w.st, (float*)w.xe, (float*)xs, n, 0, (const float*)altres);
            continue;
        }
        auto tr = [&](const void* A, int64_t lda, const void* Dinv, bool up, bool t) {
            launch_trsm(dt, A, lda, Dinv, up, t, w.xe, n, n, 1, sa, slot, true, w.args,
                        w.st, s);
        };
        switch (kind) {
        case KIND_LU:
            if (!trans) { tr(w.W, ldw, w.Dinv0, false, false); tr(w.W, ldw, w.Dinv1, true, false); }
            else { tr(w.W, ldw, w.Dinv1, true, true); tr(w.W, ldw, w.Dinv0, false, true); }
            break;
        case KIND_TRI:
            tr(nullptr, w.lda, w.Dinv0, upper, trans);
            break;
        case KIND_CHOL:
            tr(w.W, ldw, w.Dinv0, false, false);
            tr(w.W, ldw, w.Dinv0, false, true);
            break;
        case KIND_BAND:
            launch_band_apply(w, trans, slot, s);
            break;
        }
        if (dt == AS_F64) est_step_kernel<double><<<1, kEstThreads, 0, s>>>(w.st, (double*)w.xe, (double*)xs, n, slot, (const double*)altres);
        else est_step_kernel<float><<<1, kEstThreads, 0, s>>>(w.st, (float*)w.xe, (float*)xs, n, slot, (const float*)altres);
    }
    if (dt == AS_F64) est_finish_kernel<double><<<1, 32, 0, s>>>(w.st);
    else est_finish_kernel<float><<<1, 32, 0, s>>>(w.st);
}

}  // namespace as
