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

// ------------------------------------------------------------------ LU panel (cooperative)
template <typename T>
struct PanelCand { T v; long long idx; };

template <typename T>
__global__ void __launch_bounds__(kPanelThreads, 1) lu_panel_kernel(T* W, int64_t ldw, int64_t n, int64_t k0, int nbp,
                                                                    int64_t* ipiv, DevState* st, unsigned* bar,
                                                                    PanelCand<T>* cand, T* rowbuf, T* diagbuf,
                                                                    int use_smem) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int P = gridDim.x, cta = blockIdx.x;
    const int64_t m = n - k0;
    const int64_t chunk = (m + P - 1) / P;
    const int64_t rbeg = k0 + (int64_t)cta * chunk;
    const int64_t rend = min(n, rbeg + chunk);
    const int nr = (int)max<int64_t>(0, rend - rbeg);
    const int64_t cp = use_smem ? chunk : ldw;                  // leading dimension of my row block
    T* Ps = use_smem ? (T*)smem_raw : W + rbeg + k0 * ldw;     // Ps[r + c*cp], r local row, c panel col
    T* ubuf = use_smem ? (T*)smem_raw + chunk * nbp : (T*)smem_raw;
    __shared__ T sv[32];
    __shared__ long long si[32];
    __shared__ long long s_p;
    __shared__ int s_owner;
    __shared__ T s_piv;
    __shared__ int s_diag_nan;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;

    if (use_smem) {
        for (int64_t e = threadIdx.x; e < (int64_t)nr * nbp; e += blockDim.x) {
            const int64_t r = e % nr, c = e / nr;
            Ps[r + c * cp] = W[(rbeg + r) + (k0 + c) * ldw];
        }
        __syncthreads();
    }
    unsigned long long info = ~0ull;
    for (int j = 0; j < nbp; ++j) {
        const int64_t g = k0 + j;                  // diagonal row / column
        const int par = j & 1;
        // local first-max over my rows >= g (NaN never wins, Z15)
        T v = T(-1);
        long long idx = 0x7fffffffffffffffll;
        int dnan = 0;
        for (int r = threadIdx.x; r < nr; r += blockDim.x) {
            const int64_t gr = rbeg + r;
            if (gr < g) continue;
            T a = Ps[r + j * cp];
            a = a < T(0) ? -a : a;
            if (gr == g && a != a) dnan = 1;
            argmax_merge(v, idx, a, (long long)gr);
        }
        warp_argmax(v, idx);
        dnan = __any_sync(0xffffffffu, dnan);
        if (lane == 0) { sv[warp] = v; si[warp] = idx; }
        if (threadIdx.x == 0) s_diag_nan = 0;
        __syncthreads();
        if (lane == 0 && dnan) s_diag_nan = 1;
        if (warp == 0) {
            v = lane < nw ? sv[lane] : T(-1);
            idx = lane < nw ? si[lane] : 0x7fffffffffffffffll;
            warp_argmax(v, idx);
            if (lane == 0) { sv[0] = v; si[0] = idx; }
        }
        __syncthreads();
        v = sv[0];
        idx = si[0];
        // publish candidate + its row; the owner of row g publishes old row g
        if (threadIdx.x == 0) {
            PanelCand<T> c;
            c.v = s_diag_nan ? T(INFINITY) : v;     // NaN diagonal: serial semantics keep row g
            c.idx = s_diag_nan ? (long long)g : idx;
            cand[par * P + cta] = c;
        }
        const long long pub = s_diag_nan ? (long long)g : idx;
        if (pub != 0x7fffffffffffffffll && pub >= rbeg && pub < rend) {
            const int r = (int)(pub - rbeg);
            for (int c = threadIdx.x; c < nbp; c += blockDim.x) rowbuf[((int64_t)par * P + cta) * nbp + c] = Ps[r + c * cp];
        }
        if (g >= rbeg && g < rend) {
            const int r = (int)(g - rbeg);
            for (int c = threadIdx.x; c < nbp; c += blockDim.x) diagbuf[par * nbp + c] = Ps[r + c * cp];
        }
        if (P > 1) grid_barrier(bar, (unsigned)(j + 1), (unsigned)P);
        else { __threadfence_block(); __syncthreads(); }
        // global winner
        if (warp == 0) {
            T bv = T(-1);
            long long bi = 0x7fffffffffffffffll;
            int bo = 0;
            for (int t = lane; t < P; t += 32) {
                PanelCand<T> c;
                c.v = __ldcg(&cand[par * P + t].v);
                c.idx = __ldcg(&cand[par * P + t].idx);
                if (c.v > bv || (c.v == bv && c.idx < bi)) { bv = c.v; bi = c.idx; bo = t; }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                T v2 = __shfl_xor_sync(0xffffffffu, bv, o);
                long long i2 = __shfl_xor_sync(0xffffffffu, bi, o);
                int o2 = __shfl_xor_sync(0xffffffffu, bo, o);
                if (v2 > bv || (v2 == bv && i2 < bi)) { bv = v2; bi = i2; bo = o2; }
            }
            if (lane == 0) { s_p = bi; s_owner = bo; }
        }
        __syncthreads();
        const long long p = s_p;
        const int owner = s_owner;
        for (int c = threadIdx.x; c < nbp; c += blockDim.x) ubuf[c] = __ldcg(&rowbuf[((int64_t)owner * 1 + (int64_t)par * P) * nbp + c]);
        __syncthreads();
        const T piv = ubuf[j];
        if (cta == 0 && threadIdx.x == 0) ipiv[g] = (p == 0x7fffffffffffffffll) ? g : p;
        if (piv == T(0)) {                       // exact zero pivot: singular column (no elimination)
            if (info == ~0ull) info = (unsigned long long)(g + 1);
            __syncthreads();
            continue;
        }
        // swap: row p <- old row g, row g <- pivot row
        if (p != g && p >= rbeg && p < rend) {
            const int r = (int)(p - rbeg);
            for (int c = threadIdx.x; c < nbp; c += blockDim.x) Ps[r + c * cp] = __ldcg(&diagbuf[par * nbp + c]);
        }
        if (g >= rbeg && g < rend) {
            const int r = (int)(g - rbeg);
            for (int c = threadIdx.x; c < nbp; c += blockDim.x) Ps[r + c * cp] = ubuf[c];
        }
        __syncthreads();
        // eliminate my rows > g
        const int64_t r0 = max<int64_t>(0, g + 1 - rbeg);
        for (int64_t r = r0 + threadIdx.x; r < nr; r += blockDim.x) {
            const T l = Ps[r + j * cp] / piv;
            Ps[r + j * cp] = l;
            for (int c = j + 1; c < nbp; ++c) Ps[r + c * cp] -= l * ubuf[c];
        }
        __syncthreads();
    }
    if (use_smem) {
        for (int64_t e = threadIdx.x; e < (int64_t)nr * nbp; e += blockDim.x) {
            const int64_t r = e % nr, c = e / nr;
            W[(rbeg + r) + (k0 + c) * ldw] = Ps[r + c * cp];
        }
    }
    if (threadIdx.x == 0 && cta == 0 && info != ~0ull) atomicMin(&st->info, info);
}

// ------------------------------------------------------------------ laswp
// Apply ipiv[k0..k0+nbp) (in order) to every column outside the panel and to perm.
template <typename T>
__global__ void laswp_kernel(T* W, int64_t ldw, int64_t n, int64_t k0, int nbp, const int64_t* ipiv, int64_t* perm) {
    const int64_t ncols = n - nbp + 1;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ncols; t += (int64_t)gridDim.x * blockDim.x) {
        if (t == ncols - 1) {
            for (int j = 0; j < nbp; ++j) {
                const int64_t a = k0 + j, b = ipiv[a];
                if (b != a) { const int64_t x = perm[a]; perm[a] = perm[b]; perm[b] = x; }
            }
            continue;
        }
        const int64_t col = t < k0 ? t : t + nbp;
        T* c = W + col * ldw;
        for (int j = 0; j < nbp; ++j) {
            const int64_t a = k0 + j, b = ipiv[a];
            if (b != a) { const T x = c[a]; c[a] = c[b]; c[b] = x; }
        }
    }
}

// ------------------------------------------------------------------ U12 = L11^{-1} A12
template <typename T>
__global__ void __launch_bounds__(256) u12_kernel(T* W, int64_t ldw, int64_t n, int64_t k0, int nbp) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* L = (T*)smem_raw;                 // kNB x (kNB+1)
    T* Bt = L + kNB * (kNB + 1);         // kNB x (kNB+1)
    const int64_t c0 = k0 + nbp + (int64_t)blockIdx.x * kNB;
    const int nc = (int)min<int64_t>(kNB, n - c0);
    if (nc <= 0) return;
    constexpr int LD = kNB + 1;
    for (int e = threadIdx.x; e < nbp * nbp; e += blockDim.x) {
        const int r = e % nbp, c = e / nbp;
        L[r + c * LD] = W[(k0 + r) + (k0 + c) * ldw];
    }
    for (int e = threadIdx.x; e < nbp * nc; e += blockDim.x) {
        const int r = e % nbp, c = e / nbp;
        Bt[r + c * LD] = W[(k0 + r) + (c0 + c) * ldw];
    }
    __syncthreads();
    for (int i = 0; i < nbp - 1; ++i) {
        const int rows = nbp - 1 - i;
        for (int e = threadIdx.x; e < rows * nc; e += blockDim.x) {
            const int r = i + 1 + e % rows, c = e / rows;
            Bt[r + c * LD] -= L[r + i * LD] * Bt[i + c * LD];
        }
        __syncthreads();
    }
    for (int e = threadIdx.x; e < nbp * nc; e += blockDim.x) {
        const int r = e % nbp, c = e / nbp;
        W[(k0 + r) + (c0 + c) * ldw] = Bt[r + c * LD];
    }
}

// ------------------------------------------------------------------ LU driver
template <typename T>
static void lu_factor_t(const Work& w, cudaStream_t s) {
    const int64_t n = w.n, ldw = w.ldw;
    T* W = (T*)w.W;
    copy_norm_kernel<T><<<w.num_sms * 4, 256, 0, s>>>(w.args, w.lda, n, W, ldw, w.st, w.perm);
    int panel_idx = 0;
    for (int64_t k0 = 0; k0 < n; k0 += kNB, ++panel_idx) {
        const int nbp = (int)std::min<int64_t>(kNB, n - k0);
        const int64_t m = n - k0;
        int P = (int)std::min<int64_t>(w.num_sms, (m + 127) / 128);
        P = std::max(P, 1);
        int64_t chunk = (m + P - 1) / P;
        size_t smem = sizeof(T) * (chunk * nbp + nbp);
        int use_smem = 1;
        if (smem > 200 * 1024) { use_smem = 0; smem = sizeof(T) * nbp; }
        unsigned* bar = w.bars + 8 + (panel_idx % (int)(w.bars_len - 8));
        PanelCand<T>* cand = (PanelCand<T>*)w.cand;
        T* rowbuf = (T*)((char*)w.cand + sizeof(PanelCand<T>) * 2 * 1024);
        T* diagbuf = rowbuf + (int64_t)2 * 1024 * kNB;
        auto kern = lu_panel_kernel<T>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)std::max<size_t>(smem, 1024));
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(P);
        cfg.blockDim = dim3(kPanelThreads);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeCooperative;
        attr[0].val.cooperative = 1;
        cfg.attrs = attr;
        cfg.numAttrs = P > 1 ? 1 : 0;
        cudaLaunchKernelEx(&cfg, kern, W, ldw, n, k0, nbp, w.ipiv, w.st, bar, cand, rowbuf, diagbuf, use_smem);
        const int64_t ncols = n - nbp + 1;
        laswp_kernel<T><<<(unsigned)std::min<int64_t>((ncols + 127) / 128, 4096), 128, 0, s>>>(W, ldw, n, k0, nbp,
                                                                                                 w.ipiv, w.perm);
        const int64_t rest = n - k0 - nbp;
        if (rest > 0) {
            const int sm2 = (int)(sizeof(T) * 2 * kNB * (kNB + 1));
            cudaFuncSetAttribute(u12_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm2);
            u12_kernel<T><<<(unsigned)((rest + kNB - 1) / kNB), 256, sm2, s>>>(W, ldw, n, k0, nbp);
            GemmArgs g{};
            g.M = rest; g.N = rest; g.K = nbp;
            g.A = W + (k0 + nbp) + k0 * ldw; g.lda = ldw; g.TA = false;
            g.B = W + k0 + (k0 + nbp) * ldw; g.ldb = ldw; g.TB = false;
            g.C = W + (k0 + nbp) + (k0 + nbp) * ldw; g.ldc = ldw;
            launch_gemm_minus(w.dtype, g, s);
        }
    }
    launch_trtri_blocks(w.dtype, W, ldw, n, w.Dinv0, false, true, w.st, true, w.args, s);
    launch_trtri_blocks(w.dtype, W, ldw, n, w.Dinv1, true, false, w.st, true, w.args, s);
}

void launch_lu_factor(const Work& w, cudaStream_t s) {
    if (w.dtype == AS_F64) lu_factor_t<double>(w, s);
    else lu_factor_t<float>(w, s);
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
        const int rem = nbp - j - 1;
        for (int e = threadIdx.x; e < rem * rem; e += blockDim.x) {
            const int i = j + 1 + e % rem, k = j + 1 + e / rem;
            if (i >= k) a[i + k * LD] -= a[i + j * LD] * a[k + j * LD];
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
        const int rem = nbp - c - 1;
        for (int e = threadIdx.x; e < nr * rem; e += blockDim.x) {
            const int r = e % nr, cc = c + 1 + e / nr;
            X[r + cc * LD] -= X[r + c * LD] * L[cc + c * LD];
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
