// rcond.cu -- K10: reciprocal condition estimate (the xxCON family
// P:350).  1-norm estimate of ||A^{-1}||_1 by the
// Hager-Higham procedure in the form of LAPACK's xLACN2 (Z13b), run as a
// device-resident state machine: 11 fixed "apply" slots (M or M^T through the
// path's factors, see launch_estimator) interleaved with single-CTA step
// kernels; a slot whose turn never comes exits at once, so the host never
// synchronizes.  rcond = (1/est)/anorm.
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
