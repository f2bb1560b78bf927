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
#include <cstdlib>
#include <cstring>

#include "factor.h"
#include "gemm.h"
#include "internal.h"
#include "trsm.h"
#include "blk64.cuh"
#include <cooperative_groups.h>
#include <type_traits>

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

void launch_copy_norm(const Work& w, bool with_perm, cudaStream_t s) {
    if (w.dtype == AS_F64)
        copy_norm_kernel<double><<<w.num_sms * 4, 256, 0, s>>>(w.args, w.lda, w.n, (double*)w.W, w.ldw, w.st,
                                                               with_perm ? w.perm : nullptr);
    else
        copy_norm_kernel<float><<<w.num_sms * 4, 256, 0, s>>>(w.args, w.lda, w.n, (float*)w.W, w.ldw, w.st,
                                                              with_perm ? w.perm : nullptr);
}

// ------------------------------------------------------------------ Cholesky
// POTF2 of one kNB x kNB diagonal block in shared memory, plus its inverse.
// Factor: right-looking with the scaling deferred (a_ik -= a_ij a_kj / d_j, then column j is
// divided by sqrt(d_j) at the end) so every column step needs a single barrier; the first
// !(d_j > 0) stops it (Z23).  The inverse L11^{-1} (lower, column-major ld kNB) goes to the
// block's Dinv slot: the substitutions of POTRS / POCON use it, and L21 = A21 L11^{-T}
// becomes a small product instead of a second column sweep.
constexpr int kChLD = kNB + 1;
template <typename T>
__global__ void __launch_bounds__(256) potf2_kernel(T* W, int64_t ldw, int64_t n, int64_t k0, int nbp, DevState* st,
                                                    T* Dinv) {
    if (st->chol_failed) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* a = (T*)smem_raw;           // kNB x kChLD, lower triangle
    T* x = a + kNB * kChLD;        // kNB x kChLD, L^{-1}
    __shared__ int s_fail;
    batched<8, T>(
        nbp * nbp,
        [&](int e) -> T { const int r = e % nbp, c = e / nbp; return r >= c ? W[(k0 + r) + (k0 + c) * ldw] : T(0); },
        [&](int e, T v) { const int r = e % nbp, c = e / nbp; a[r + c * kChLD] = v; });
    for (int e = threadIdx.x; e < kNB * kNB; e += blockDim.x) {
        const int r = e % kNB, c = e / kNB;
        x[r + c * kChLD] = (r == c) ? T(1) : T(0);
    }
    if (threadIdx.x == 0) s_fail = -1;
    __syncthreads();
    const int i = threadIdx.x & (kNB - 1), ph = threadIdx.x / kNB;  // 256 threads: 4 phases
    // thread (row i, phase ph) owns columns k = ph + 4 m of its row: loads first, then stores,
    // so a step is one smem round trip instead of one per column
    for (int j = 0; j < nbp; ++j) {
        const T d = a[j + j * kChLD];
        if (!(d > T(0))) { if (threadIdx.x == 0) s_fail = j; break; }   // uniform
        if (i > j && i < nbp) {
            const T aij = a[i + j * kChLD] / d;
            T va[kNB / 4], vb[kNB / 4];
#pragma unroll
            for (int m = 0; m < kNB / 4; ++m) {
                const int k = j + 1 + ph + 4 * m;
                if (k <= i) { va[m] = a[i + k * kChLD]; vb[m] = a[k + j * kChLD]; }
            }
#pragma unroll
            for (int m = 0; m < kNB / 4; ++m) {
                const int k = j + 1 + ph + 4 * m;
                if (k <= i) a[i + k * kChLD] = va[m] - aij * vb[m];
            }
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
    __shared__ T sq[kNB];
    if (threadIdx.x < nbp) sq[threadIdx.x] = sqrt(a[threadIdx.x + threadIdx.x * kChLD]);
    __syncthreads();
    for (int e = threadIdx.x; e < kNB * kNB; e += blockDim.x) {
        const int r = e % kNB, c = e / kNB;
        if (r >= nbp || c >= nbp) a[r + c * kChLD] = (r == c) ? T(1) : T(0);   // identity pad
        else if (r > c) a[r + c * kChLD] /= sq[c];
        else if (r == c) a[r + c * kChLD] = sq[c];
    }
    __syncthreads();
    // X = L^{-1} (lower, non-unit): diagonal 16 x 16 blocks by substitution, the rest by
    // block diagonals (blk64.cuh)
    block_trinv64<T, false>(a, x, x + kNB * kChLD);
    T* D = Dinv + (k0 / kNB) * (int64_t)kNB * kNB;
    for (int e = threadIdx.x; e < kNB * kNB; e += blockDim.x) {
        const int r = e % kNB, c = e / kNB;
        T v;
        if (r < nbp && c < nbp) v = x[r + c * kChLD];
        else v = (r == c) ? T(1) : T(0);
        D[r + c * kNB] = v;
    }
    for (int e = threadIdx.x; e < nbp * nbp; e += blockDim.x) {
        const int r = e % nbp, c = e / nbp;
        if (r >= c) W[(k0 + r) + (k0 + c) * ldw] = a[r + c * kChLD];
    }
}

// L21 = A21 L11^{-T} = A21 (Dinv block)^T: each CTA multiplies one kNB-row block in place.
// 256 threads, 4 x 4 register tile each; As[k][r], Ls[k][c] = Linv(c, k).
constexpr int kL21LD = kNB + 4;
template <typename T>
__global__ void __launch_bounds__(256) l21_kernel(T* W, int64_t ldw, int64_t n, int64_t k0, int nbp, const DevState* st,
                                                  const T* Dinv) {
    if (st->chol_failed) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* As = (T*)smem_raw;             // kNB x kL21LD
    T* Ls = As + kNB * kL21LD;        // kNB x kL21LD
    const int64_t r0 = k0 + nbp + (int64_t)blockIdx.x * kNB;
    const int nr = (int)min<int64_t>(kNB, n - r0);
    if (nr <= 0) return;
    const T* Li = Dinv + (k0 / kNB) * (int64_t)kNB * kNB;
    batched<16, T>(
        2 * kNB * kNB,
        [&](int e) -> T {
            if (e < kNB * kNB) {
                const int r = e % kNB, k = e / kNB;
                return (r < nr && k < nbp) ? W[(r0 + r) + (k0 + k) * ldw] : T(0);
            }
            const int f = e - kNB * kNB;
            return Li[f];                     // Linv(c, k) at c + k * kNB
        },
        [&](int e, T v) {
            if (e < kNB * kNB) { const int r = e % kNB, k = e / kNB; As[k * kL21LD + r] = v; }
            else { const int f = e - kNB * kNB, c = f % kNB, k = f / kNB; Ls[k * kL21LD + c] = v; }
        });
    __syncthreads();
    const int tr = threadIdx.x & 15, tc = threadIdx.x >> 4;
    T acc[4][4] = {};
    for (int k = 0; k < nbp; ++k) {
        T av[4], bv[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) { av[q] = As[k * kL21LD + 4 * tr + q]; bv[q] = Ls[k * kL21LD + 4 * tc + q]; }
#pragma unroll
        for (int p = 0; p < 4; ++p)
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[p][q] += av[p] * bv[q];
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int c = 4 * tc + q;
        if (c >= nbp) continue;
#pragma unroll
        for (int p = 0; p < 4; ++p) {
            const int r = 4 * tr + p;
            if (r < nr) W[(r0 + r) + (k0 + c) * ldw] = acc[p][q];
        }
    }
}

// Right-looking with look-ahead: after block k's panel, the next block column is updated first
// (M = rest, N = 64, K = 64) and the next panel (POTF2 + inverse, L21) starts on a
// high-priority stream while the bulk SYRK of block k runs on the main stream.
struct CholStreams {
    cudaStream_t hi = nullptr;
    cudaEvent_t ev[8];
};
static CholStreams& chol_streams() {
    static thread_local CholStreams C;
    if (!C.hi) {
        int lo = 0, hi = 0;
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        cudaStreamCreateWithPriority(&C.hi, cudaStreamNonBlocking, hi);
        for (auto& e : C.ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    }
    return C;
}

template <typename T>
static void chol_factor_t(const Work& w, cudaStream_t s) {
    const int64_t n = w.n, ldw = w.ldw;
    T* W = (T*)w.W;
    T* Dinv = (T*)w.Dinv0;
    copy_norm_kernel<T><<<w.num_sms * 4, 256, 0, s>>>(w.args, w.lda, n, W, ldw, w.st, nullptr);
    const int sm1 = (int)(sizeof(T) * (2 * kNB * kChLD + 3 * 256));
    const int sm2 = (int)(sizeof(T) * 2 * kNB * kL21LD);
    cudaFuncSetAttribute(potf2_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm1);
    cudaFuncSetAttribute(l21_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm2);
    auto panel = [&](int64_t k0, cudaStream_t st) {
        const int nbp = (int)std::min<int64_t>(kNB, n - k0);
        potf2_kernel<T><<<1, 256, sm1, st>>>(W, ldw, n, k0, nbp, w.st, Dinv);
        const int64_t rest = n - k0 - nbp;
        if (rest > 0) l21_kernel<T><<<(unsigned)((rest + kNB - 1) / kNB), 256, sm2, st>>>(W, ldw, n, k0, nbp, w.st, Dinv);
    };
    // C[r0.., c0..c0+N) -= L21[r0..] L21[c0..]^T with L21 the panel columns of block k0
    auto syrk = [&](int64_t k0, int nbp, int64_t r0, int64_t c0, int64_t M, int64_t N, cudaStream_t st) {
        if (M <= 0 || N <= 0) return;
        GemmArgs g{};
        g.M = M; g.N = N; g.K = nbp;
        g.A = W + r0 + k0 * ldw; g.lda = ldw; g.TA = false;
        g.B = W + c0 + k0 * ldw; g.ldb = ldw; g.TB = true;
        g.C = W + r0 + c0 * ldw; g.ldc = ldw;
        g.lower_only = true;
        g.skip = &w.st->chol_failed;
        launch_gemm_minus(w.dtype, g, st);
    };
    const bool lookahead = n > 2 * kNB && getenv("AS_CHOL_NO_LOOKAHEAD") == nullptr;
    CholStreams& CS = chol_streams();
    int evi = 0;
    // Two 64-column panels per step: the second panel's columns take the first panel's K = 64 update, then
    // everything to the right takes ONE K = 128 update (half the passes over the trailing matrix, and the
    // DMMA GEMM's per-tile fixed cost -- C in and out of the accumulators -- is spread over twice the
    // k-steps).  Look-ahead: the next pair's 128 columns are updated first and
    // both of its panels are factored on the high-priority stream beside the bulk update.
    static const bool pairs_off = getenv("AS_CHOL_PAIRS") != nullptr && atoi(getenv("AS_CHOL_PAIRS")) == 0;
    // measured: n = 16384 86.2 -> 77.5 ms, n = 4096 6.03 -> 6.16 ms (chain-bound there: nothing to gain from K = 128)
    static const int64_t pairs_min_n = getenv("AS_CHOL_PAIRS_MIN_N") ? atoll(getenv("AS_CHOL_PAIRS_MIN_N")) : 6144;
    if (!pairs_off && n >= pairs_min_n) {
        constexpr int kPair = 2 * kNB;
        // both panels of the pair starting at column c (the columns already carry every earlier update)
        auto pair_panels = [&](int64_t c, cudaStream_t st) {
            panel(c, st);
            const int64_t cb = c + kNB;
            if (cb >= n) return;
            syrk(c, kNB, cb, cb, n - cb, std::min<int64_t>(kNB, n - cb), st);
            panel(cb, st);
        };
        pair_panels(0, s);
        for (int64_t c = 0; c < n; c += kPair) {
            const int kw = (int)std::min<int64_t>(kPair, n - c);
            const int64_t r1 = c + kw, rest = n - r1;
            if (rest <= 0) break;
            const int64_t nb2 = std::min<int64_t>(kPair, rest);
            if (lookahead && rest > nb2) {
                cudaEvent_t e0 = CS.ev[(evi++) % 8];
                cudaEventRecord(e0, s);
                cudaStreamWaitEvent(CS.hi, e0, 0);
                syrk(c, kw, r1, r1, rest, nb2, CS.hi);                          // next pair's columns
                pair_panels(r1, CS.hi);
                syrk(c, kw, r1 + nb2, r1 + nb2, rest - nb2, rest - nb2, s);     // bulk, K = 128
                cudaEvent_t e1 = CS.ev[(evi++) % 8];
                cudaEventRecord(e1, CS.hi);
                cudaStreamWaitEvent(s, e1, 0);
            } else {
                syrk(c, kw, r1, r1, rest, rest, s);
                pair_panels(r1, s);
            }
        }
        return;
    }
    panel(0, s);
    for (int64_t k0 = 0; k0 < n; k0 += kNB) {
        const int nbp = (int)std::min<int64_t>(kNB, n - k0);
        const int64_t r1 = k0 + nbp, rest = n - r1;
        if (rest <= 0) break;
        const int64_t nb2 = std::min<int64_t>(kNB, rest);
        if (lookahead && rest > nb2) {
            cudaEvent_t e0 = CS.ev[(evi++) % 8];
            cudaEventRecord(e0, s);
            cudaStreamWaitEvent(CS.hi, e0, 0);
            syrk(k0, nbp, r1, r1, rest, nb2, CS.hi);                      // next block column
            panel(r1, CS.hi);                                              // next panel
            syrk(k0, nbp, r1 + nb2, r1 + nb2, rest - nb2, rest - nb2, s);  // bulk
            cudaEvent_t e1 = CS.ev[(evi++) % 8];
            cudaEventRecord(e1, CS.hi);
            cudaStreamWaitEvent(s, e1, 0);
        } else {
            syrk(k0, nbp, r1, r1, rest, rest, s);
            panel(r1, s);
        }
    }
    // the register panels do not form L11^{-1}: all diagonal-block inverses (POTRS / POCON) at once
}

// Diagnostics: average time (us) of one Cholesky panel of W (restored from Wsrc before each
// launch).  kind 0: the cluster panel; kind 1: POTF2 + L21 (the fallback kernels).
double chol_debug_panel_time(int dtype, int kind, void* W, int64_t ldw, int64_t n, int64_t k0, int nbp, const void* Wsrc,
                             int iters, int dbg) {
    Work w{};
    w.dtype = dtype; w.n = n; w.ldw = ldw; w.W = W;
    cudaDeviceGetAttribute(&w.num_sms, cudaDevAttrMultiProcessorCount, 0);
    cudaMalloc(&w.st, sizeof(DevState));
    cudaMalloc(&w.Dinv0, 8 * (n + kNB) * kNB);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const size_t es = dtype == AS_F64 ? 8 : 4;
    double tot = 0.0;
    for (int it = 0; it < iters; ++it) {
        // dbg 4: restore only the panel's columns (no L2 flush between launches)
        if (dbg & 4) cudaMemcpy((char*)W + es * ldw * k0, (const char*)Wsrc + es * ldw * k0, es * ldw * nbp, cudaMemcpyDeviceToDevice);
        else cudaMemcpy(W, Wsrc, es * ldw * n, cudaMemcpyDeviceToDevice);
        cudaMemset(w.st, 0, sizeof(DevState));
        cudaEventRecord(e0, 0);
        auto run = [&](auto tag) {
            using T = decltype(tag);
            const int sm1 = (int)(sizeof(T) * (2 * kNB * kChLD + 3 * 256));
            const int sm2 = (int)(sizeof(T) * 2 * kNB * kL21LD);
            cudaFuncSetAttribute(potf2_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm1);
            cudaFuncSetAttribute(l21_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm2);
            potf2_kernel<T><<<1, 256, sm1, 0>>>((T*)W, ldw, n, k0, nbp, w.st, (T*)w.Dinv0);
            const int64_t rest = n - k0 - nbp;
            if (rest > 0 && !(dbg & 2)) l21_kernel<T><<<(unsigned)((rest + kNB - 1) / kNB), 256, sm2, 0>>>((T*)W, ldw, n, k0, nbp, w.st, (T*)w.Dinv0);
        };
        if (dtype == AS_F64) run(double{});
        else run(float{});
        cudaEventRecord(e1, 0);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (it > 0 || iters == 1) tot += ms;
    }
    const cudaError_t err = cudaGetLastError();
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(w.st);
    cudaFree(w.Dinv0);
    if (err != cudaSuccess) return -(double)err;
    return 1000.0 * tot / (iters > 1 ? iters - 1 : 1);
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
    (void)w; (void)s;   // potf2_kernel already wrote the inverse diagonal blocks of L to Dinv0
}

}  // namespace as
