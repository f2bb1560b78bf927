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
#include <cstdlib>
#include <type_traits>

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

// anorm = max_j sum_i |A_ij| over the band (one warp per column), and in the same pass over the band the
// strict diagonal dominance by rows / by columns that selects the partitioned solver (st->band_dom, preset
// to 3): the column sums without their diagonal term come from the same loads, the row sums from a thread
// per row (coalesced across rows).  (Was two kernels; the column sums of the dominance test were one thread
// per column, 13.7 us on C2.)
template <typename T>
__global__ void band_norm_kernel(const DevArgs* args, int64_t lda, int64_t n, DevState* st) {
    const T* A = (const T*)args->A;
    const int64_t kl = st->kl, ku = st->ku;
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    double best = 0.0;
    int row_ok = 1, col_ok = 1;
    for (int64_t j = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); j < n; j += warps) {
        const int64_t i0 = j - ku > 0 ? j - ku : 0, i1 = j + kl < n - 1 ? j + kl : n - 1;
        T s = T(0), cs = T(0), ad = T(0);
        for (int64_t i = i0 + lane; i <= i1; i += 32) {
            T a = A[i + j * lda];
            a = a < T(0) ? -a : a;
            s += a;
            if (i != j) cs += a;
            else ad = a;
        }
        s = warp_sum(s);
        cs = warp_sum(cs);
        ad = warp_sum(ad);                      // one lane holds |a_jj|, the others 0
        if ((double)s > best || s != s) best = (double)s;
        if (!(ad > cs)) col_ok = 0;
    }
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        T rs = T(0);
        const int64_t j0 = i - kl > 0 ? i - kl : 0, j1 = i + ku < n - 1 ? i + ku : n - 1;
        for (int64_t j = j0; j <= j1; ++j) if (j != i) { const T v = A[i + j * lda]; rs += v < T(0) ? -v : v; }
        const T d = A[i + i * lda];
        const T ad = d < T(0) ? -d : d;
        if (!(ad > rs)) row_ok = 0;
    }
    if (lane == 0 && best > 0.0) atomicMax(&st->anorm_bits, dbits(best));
    row_ok = __syncthreads_and(row_ok);
    col_ok = __syncthreads_and(col_ok);
    if (threadIdx.x == 0) {
        if (!row_ok) atomicAnd(&st->band_dom, ~1u);
        if (!col_ok) atomicAnd(&st->band_dom, ~2u);
    }
}

// ------------------------------------------------------------------ K3 gbtrf (one warp)
template <typename T>
AS_DEV void gbtrf_global(T* ab, int64_t n, DevState* st, int64_t* ipiv) {
    const int lane = threadIdx.x & 31;
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
template <typename T>
__global__ void __launch_bounds__(32) gbtrf_warp_kernel(T* ab, int64_t n, DevState* st, int64_t* ipiv) {
    gbtrf_global<T>(ab, n, st, ipiv);
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

// ------------------------------------------------------------------ shared-memory windows
// The sequential chains touch a window of <= kl + kv + 1 band columns at a time: the warp keeps a
// ring of kRing columns in shared memory, prefetched kDist columns ahead with cp.async (one group
// per step, so "all but the last 8 groups done" covers every column the step reads) and, for the
// factor, writes each column back once it is final.  b (and ipiv) live in shared memory for the
// whole sweep.  Every chain step then costs shared-memory latencies instead of L2 round trips.
constexpr int kRing = 128;           // power of two
constexpr int kRingWait = 32;        // prefetch groups in flight (~32 chain steps of memory latency)
constexpr int64_t kRingLdab = 85;     // 2 kl + ku + 1: keeps the factor's prefetch distance < kRing - 1

template <typename T>
AS_DEV void ring_fetch(T* ring, const T* ab, int64_t ldab, int64_t n, int64_t c) {
    if (c >= n) { asm volatile("cp.async.commit_group;" ::: "memory"); return; }
    const int lane = threadIdx.x & 31;
    T* dst = ring + (int64_t)((unsigned)c & (kRing - 1)) * ldab;
    const T* src = ab + c * ldab;
    for (int64_t r = lane; r < ldab; r += 32) {
        const unsigned sa = (unsigned)__cvta_generic_to_shared(dst + r);
        if (sizeof(T) == 8) asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(src + r) : "memory");
        else asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa), "l"(src + r) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
}
AS_DEV void ring_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(kRingWait) : "memory"); __syncwarp(); }

// windowed band LU (xGBTF2 semantics identical to gbtrf_warp_kernel), one warp
template <typename T>
__global__ void __launch_bounds__(32) gbtrf_ring_kernel(T* ab, int64_t n, DevState* st, int64_t* ipiv) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* ring = (T*)smem_raw;
    const int lane = threadIdx.x;
    const int64_t kl = st->kl, ku = st->ku, kv = kl + ku, ldab = 2 * kl + ku + 1;
    const int64_t dist = kl + kv + kRingWait + 2;            // prefetch distance (< kRing - 1)
    if (ldab > kRingLdab || dist >= kRing - 1) { gbtrf_global<T>(ab, n, st, ipiv); return; }   // wide band
#define RB(r, c) ring[(r) + (int64_t)((unsigned)(c) & (kRing - 1)) * ldab]
    for (int64_t c = 0; c < dist; ++c) ring_fetch(ring, ab, ldab, n, c);
    int64_t ju = 0;
    unsigned long long info = ~0ull;
    for (int64_t j = 0; j < n; ++j) {
        ring_fetch(ring, ab, ldab, n, j + dist);
        ring_wait();
        const int64_t km = kl < n - 1 - j ? kl : n - 1 - j;
        T best = T(-1);
        long long jp = 0x7fffffffffffffffll;
        for (int64_t r = lane; r <= km; r += 32) {
            T a = RB(kv + r, j);
            a = a < T(0) ? -a : a;
            if (r == 0 && a != a) { best = T(INFINITY); jp = 0; }
            argmax_merge(best, jp, a, (long long)r);
        }
        warp_argmax(best, jp);
        if (jp == 0x7fffffffffffffffll) jp = 0;
        if (lane == 0) ipiv[j] = j + jp;
        const T piv = RB(kv + jp, j);
        if (piv != T(0)) {
            const int64_t lim = j + ku + jp < n - 1 ? j + ku + jp : n - 1;
            if (lim > ju) ju = lim;
            if (jp != 0) {
                for (int64_t c = j + lane; c <= ju; c += 32) {
                    const T t = RB(kv + j + jp - c, c);
                    RB(kv + j + jp - c, c) = RB(kv + j - c, c);
                    RB(kv + j - c, c) = t;
                }
                __syncwarp();
            }
            const T pv = RB(kv, j);
            // multipliers and the rank-1 update with lanes over the km <= kl rows (no 64-bit
            // division on the chain: column loop outside, rows across lanes)
            const int ikm = (int)km, iwdt = (int)(ju - j);
            for (int r0 = 1; r0 <= ikm; r0 += 32) {
                const int r = r0 + lane;
                const T lr = r <= ikm ? RB(kv + r, j) / pv : T(0);
                if (r <= ikm) RB(kv + r, j) = lr;
                for (int cc = 1; cc <= iwdt; ++cc) {
                    const int64_t c = j + cc;
                    const T u = RB(kv - cc, c);                 // pivot row j at column c
                    if (r <= ikm) RB(kv + r - cc, c) -= lr * u;
                }
            }
            __syncwarp();
        } else if (info == ~0ull) {
            info = (unsigned long long)(j + 1);
        }
        // column j is final: write it back (its ring slot is reused dist steps later)
        for (int64_t r = lane; r < ldab; r += 32) ab[r + j * ldab] = RB(r, j);
    }
    if (lane == 0 && info != ~0ull) atomicMin(&st->info, info);
#undef RB
}

// windowed GBTRS sweep (gb_solve_vec semantics) on a vector b held in shared memory
template <typename T>
AS_DEV void gb_solve_ring(const T* ab, T* ring, int64_t n, int64_t kl, int64_t ku, const int* piv, T* b, bool trans) {
    const int lane = threadIdx.x & 31;
    const int64_t kv = kl + ku, ldab = 2 * kl + ku + 1;
    const int64_t dist = kv + kRingWait + 2;
#define RB(r, c) ring[(r) + (int64_t)((unsigned)(c) & (kRing - 1)) * ldab]
    // forward sweeps read columns j .. ; backward sweeps read columns j .. downwards: the ring is
    // filled in sweep order (column index mapped through `order`)
    auto sweep_fwd = [&](auto&& body) {
        for (int64_t c = 0; c < dist; ++c) ring_fetch(ring, ab, ldab, n, c);
        for (int64_t j = 0; j < n; ++j) {
            ring_fetch(ring, ab, ldab, n, j + dist);
            ring_wait();
            body(j);
        }
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncwarp();
    };
    auto fetch_rev = [&](int64_t c) {   // column c (may be < 0: no-op group)
        if (c < 0) { asm volatile("cp.async.commit_group;" ::: "memory"); return; }
        ring_fetch(ring, ab, ldab, n, c);
    };
    auto sweep_bwd = [&](auto&& body) {
        for (int64_t c = 0; c < dist; ++c) fetch_rev(n - 1 - c);
        for (int64_t j = n - 1; j >= 0; --j) {
            fetch_rev(j - dist);
            ring_wait();
            body(j);
        }
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncwarp();
    };
    if (!trans) {
        sweep_fwd([&](int64_t j) {
            if (j + 1 >= n) return;
            const int64_t lm = kl < n - 1 - j ? kl : n - 1 - j;
            const int64_t l = piv[j];
            T bj = b[j];
            if (l != j) {
                const T bl = b[l];
                __syncwarp();
                if (lane == 0) { b[l] = bj; b[j] = bl; }
                bj = bl;
            }
            __syncwarp();
            for (int64_t r = 1 + lane; r <= lm; r += 32) b[j + r] = b[j + r] - RB(kv + r, j) * bj;
            __syncwarp();
        });
        sweep_bwd([&](int64_t j) {
            const T xj = b[j] / RB(kv, j);
            __syncwarp();
            if (lane == 0) b[j] = xj;
            const int64_t i0 = j - kv > 0 ? j - kv : 0;
            for (int64_t i = i0 + lane; i < j; i += 32) b[i] = b[i] - RB(kv + i - j, j) * xj;
            __syncwarp();
        });
    } else {
        sweep_fwd([&](int64_t j) {
            const int64_t i0 = j - kv > 0 ? j - kv : 0;
            T sacc = T(0);
            for (int64_t i = i0 + lane; i < j; i += 32) sacc += RB(kv + i - j, j) * b[i];
            sacc = warp_sum(sacc);
            const T v = (b[j] - sacc) / RB(kv, j);
            __syncwarp();
            if (lane == 0) b[j] = v;
            __syncwarp();
        });
        sweep_bwd([&](int64_t j) {
            if (j > n - 2) return;
            const int64_t lm = kl < n - 1 - j ? kl : n - 1 - j;
            T sacc = T(0);
            for (int64_t r = 1 + lane; r <= lm; r += 32) sacc += RB(kv + r, j) * b[j + r];
            sacc = warp_sum(sacc);
            const T v = b[j] - sacc;
            const int64_t l = piv[j];
            __syncwarp();
            if (lane == 0) {
                if (l != j) { b[j] = b[l]; b[l] = v; }
                else b[j] = v;
            }
            __syncwarp();
        });
    }
#undef RB
}

// one warp per right-hand side; b and ipiv staged in shared memory
template <typename T>
__global__ void __launch_bounds__(32) gbtrs_ring_kernel(const T* ab, int64_t n, const DevState* st, const int64_t* ipiv,
                                                         const DevArgs* args, int64_t ldb, T* xvec, int trans, int slot) {
    if (slot >= 0 && ld_volatile_i32(&st->est_next) != slot) return;
    if (st->info != ~0ull) return;
    if (st->band_fast) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int64_t kl = st->kl, ku = st->ku, ldab = 2 * kl + ku + 1;
    if (ldab > kRingLdab || kl + ku + kRingWait + 2 >= kRing - 1) {     // wide band: global sweep
        T* bg = xvec ? xvec : (T*)args->X + (int64_t)blockIdx.x * ldb;
        gb_solve_vec<T>(ab, n, kl, ku, ipiv, bg, trans != 0);
        return;
    }
    T* ring = (T*)smem_raw;
    T* b = ring + kRing * ldab;
    int* piv = (int*)(b + n + (n & 1));
    T* bg = xvec ? xvec : (T*)args->X + (int64_t)blockIdx.x * ldb;
    for (int64_t i = threadIdx.x; i < n; i += 32) { b[i] = bg[i]; piv[i] = (int)ipiv[i]; }
    __syncwarp();
    gb_solve_ring<T>(ab, ring, n, kl, ku, piv, b, trans != 0);
    __syncwarp();
    for (int64_t i = threadIdx.x; i < n; i += 32) bg[i] = b[i];
}

template <typename T>
static size_t ring_solve_smem(int64_t n, int64_t ldab_max) {
    return sizeof(T) * (kRing * ldab_max + n + 1) + sizeof(int) * n + 16;
}

// ------------------------------------------------------------------ launchers
void launch_band_norm(const Work& w, cudaStream_t s) {
    const int blocks = w.num_sms * 4;
    if (w.dtype == AS_F64) band_norm_kernel<double><<<blocks, 256, 0, s>>>(w.args, w.lda, w.n, w.st);
    else band_norm_kernel<float><<<blocks, 256, 0, s>>>(w.args, w.lda, w.n, w.st);
}

// The windowed kernels need ldab = 2 kl + ku + 1 <= kRingLdab (the ring's shared memory is sized
// for it at capture time, before kl / ku are known) and, for the solves, b + ipiv in shared memory.
// Wider bands (or huge n) run the global-memory warp kernels -- checked on device.
static bool ring_ok_host(const Work& w) {
    const size_t es = w.dtype == AS_F64 ? 8 : 4;
    return es * (kRing * kRingLdab + w.n + 1) + 4 * w.n + 16 <= 200 * 1024 && getenv("AS_BAND_NO_RING") == nullptr;
}

// sequential (faithful xGBTF2) path: pack + factor
void launch_band_factor(const Work& w, cudaStream_t s) {
    const int blocks = w.num_sms * 4;
    const bool ring = ring_ok_host(w);
    auto go = [&](auto* W) {
        using T = std::remove_pointer_t<decltype(W)>;
        band_pack_kernel<T><<<blocks, 256, 0, s>>>(w.args, w.lda, w.n, w.st, W);
        if (ring) {
            const int smem = (int)(sizeof(T) * kRing * kRingLdab);
            cudaFuncSetAttribute(gbtrf_ring_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            gbtrf_ring_kernel<T><<<1, 32, smem, s>>>(W, w.n, w.st, w.ipiv);
        } else {
            gbtrf_warp_kernel<T><<<1, 32, 0, s>>>(W, w.n, w.st, w.ipiv);
        }
    };
    if (w.dtype == AS_F64) go((double*)w.W);
    else go((float*)w.W);
}

template <typename T>
static void gbtrs_launch(const Work& w, unsigned grid, T* xvec, int64_t ldb, int trans, int slot, cudaStream_t s) {
    if (ring_ok_host(w)) {
        const int smem = (int)ring_solve_smem<T>(w.n, kRingLdab);
        cudaFuncSetAttribute(gbtrs_ring_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        gbtrs_ring_kernel<T><<<grid, 32, smem, s>>>((const T*)w.W, w.n, w.st, w.ipiv, w.args, ldb, xvec, trans, slot);
    } else {
        gbtrs_kernel<T><<<grid, 32, 0, s>>>((const T*)w.W, w.n, w.st, w.ipiv, w.args, ldb, xvec, trans, slot);
    }
}

void launch_band_apply(const Work& w, bool trans, int slot, cudaStream_t s) {
    if (w.dtype == AS_F64) gbtrs_launch<double>(w, 1, (double*)w.xe, w.n, trans, slot, s);
    else gbtrs_launch<float>(w, 1, (float*)w.xe, w.n, trans, slot, s);
}

void launch_copy_b_to_x(const Work& w, cudaStream_t s) {
    const int blocks = w.num_sms * 4;
    if (w.dtype == AS_F64) copy_b_to_x_kernel<double><<<blocks, 256, 0, s>>>(w.args, w.n, w.ldb, w.nrhs, w.st);
    else copy_b_to_x_kernel<float><<<blocks, 256, 0, s>>>(w.args, w.n, w.ldb, w.nrhs, w.st);
}

void launch_band_solve(const Work& w, cudaStream_t s) {
    launch_copy_b_to_x(w, s);
    if (w.dtype == AS_F64) gbtrs_launch<double>(w, (unsigned)w.nrhs, (double*)nullptr, w.ldb, 0, -1, s);
    else gbtrs_launch<float>(w, (unsigned)w.nrhs, (float*)nullptr, w.ldb, 0, -1, s);
}

}  // namespace as
