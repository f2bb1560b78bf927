// svd.cu -- K8/K9: the SVD-based minimum-norm fallback (the xGELSD
// role).  x = V_A Sigma^+ U_A^T b (Z17) computed as
//   (1) Householder QR of the original A (cooperative kernel, 2 grid barriers
//       per column), c = Q^T b applied to the right-hand sides;
//   (2) one-sided (Hestenes) Jacobi on M = R^T (Z16: QR preconditioning),
//       parallel round-robin ("circle method") pair ordering, one
//       cooperative kernel per sweep, sweeps driven by a CUDA-graph WHILE
//       node until a sweep makes no rotation (cap max_sweeps);
//       the rotations are applied to y = V_J^T c instead of accumulating V_J;
//   (3) sigma_k = ||m_k||, rank = #{sigma_k > cut * sigma_max} (Z14);
//   (4) x = sum_{kept k} m_k y_k / sigma_k^2.
#include "internal.h"
#include "svd.h"

namespace as {

constexpr int kSvdThreads = 256;

template <typename T>
AS_DEV T block_sum256(T v, T* sh) {
    v = warp_sum(v);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) sh[w] = v;
    __syncthreads();
    if (w == 0) {
        v = l < (int)(blockDim.x >> 5) ? sh[l] : T(0);
        v = warp_sum(v);
        if (l == 0) sh[0] = v;
    }
    __syncthreads();
    v = sh[0];
    __syncthreads();
    return v;
}

// 1/sqrt(x): hardware approximation + two Newton steps (within ~1 ulp; x >= 1 here)
AS_DEV double rsqrt_nr(double x) {
    double y = rsqrt(x);
    y = y * (1.5 - 0.5 * x * y * y);
    return y * (1.5 - 0.5 * x * y * y);
}
AS_DEV float rsqrt_nr(float x) { return 1.0f / sqrtf(x); }

// ------------------------------------------------------------------ setup
// W = A, Y = B (n x nrhs, ld n)
template <typename T>
__global__ void svd_setup_kernel(const DevArgs* args, int64_t lda, int64_t ldb, int64_t n, int64_t nrhs, T* W,
                                 int64_t ldw, T* Y, DevState* st) {
    const T* A = (const T*)args->A;
    const T* B = (const T*)args->B;
    const int64_t tot = n * n + n * nrhs;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
        if (e < n * n) { const int64_t i = e % n, j = e / n; W[i + j * ldw] = A[i + j * lda]; }
        else { const int64_t f = e - n * n, i = f % n, j = f / n; Y[i + j * n] = B[i + j * ldb]; }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) { st->sweeps = 0; st->rotated = 0; st->svd_conv = 0; }
}

// ------------------------------------------------------------------ (1) Householder QR
template <typename T>
__global__ void __launch_bounds__(kSvdThreads, 1) qr_kernel(T* W, int64_t ldw, int64_t n, T* Y, int64_t nrhs,
                                                            T* tau, unsigned* bar) {
    __shared__ T sh[32];
    const int P = gridDim.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp, nwarps = (int64_t)P * (blockDim.x >> 5);
    unsigned gen = 0;
    for (int64_t j = 0; j < n; ++j) {
        if (blockIdx.x == 0) {
            T* col = W + j * ldw;
            T ss = T(0);
            for (int64_t i = j + 1 + threadIdx.x; i < n; i += blockDim.x) { const T x = __ldcg(&col[i]); ss += x * x; }
            ss = block_sum256(ss, sh);
            const T alpha = __ldcg(&col[j]);
            const T xnorm = sqrt(ss);
            T t = T(0);
            if (xnorm != T(0)) {
                const T aa = alpha < T(0) ? -alpha : alpha;
                const T wv = aa > xnorm ? aa : xnorm, z = aa > xnorm ? xnorm : aa;
                const T hyp = wv * sqrt(T(1) + (z / wv) * (z / wv));
                const T beta = alpha >= T(0) ? -hyp : hyp;
                t = (beta - alpha) / beta;
                const T scal = T(1) / (alpha - beta);
                for (int64_t i = j + 1 + threadIdx.x; i < n; i += blockDim.x) col[i] = __ldcg(&col[i]) * scal;
                __syncthreads();
                if (threadIdx.x == 0) col[j] = beta;
            }
            if (threadIdx.x == 0) tau[j] = t;
        }
        grid_barrier(bar, ++gen, (unsigned)P);
        const T tj = __ldcg(&tau[j]);
        if (tj != T(0)) {
            const T* v = W + j * ldw;
            for (int64_t k = j + 1 + gw; k < n + nrhs; k += nwarps) {
                T* col = k < n ? W + k * ldw : Y + (k - n) * n;
                // 8 loads in flight per iteration (a lane-serial loop was bound by one L2 latency per
                // 32 rows); the lane's sum keeps the serial order i = j+lane, j+lane+32, ... (the C4
                // least-squares residual is sensitive to the rounding of the reflector products)
                T s = T(0);
                for (int64_t i0 = j + lane; i0 < n; i0 += 128) {
                    T vv[4], cv[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int64_t i = i0 + 32 * u;
                        vv[u] = i < n ? (i == j ? T(1) : __ldcg(&v[i])) : T(0);
                        cv[u] = i < n ? __ldcg(&col[i]) : T(0);
                    }
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        if (i0 + 32 * u < n) s += vv[u] * cv[u];
                }
                s = warp_sum(s) * tj;
                for (int64_t i0 = j + lane; i0 < n; i0 += 128) {
                    T vv[4], cv[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int64_t i = i0 + 32 * u;
                        vv[u] = i < n ? (i == j ? T(1) : __ldcg(&v[i])) : T(0);
                        cv[u] = i < n ? __ldcg(&col[i]) : T(0);
                    }
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int64_t i = i0 + 32 * u;
                        if (i < n) col[i] = cv[u] - s * vv[u];
                    }
                }
            }
        }
        grid_barrier(bar, ++gen, (unsigned)P);
    }
}

// M = R^T in place: M_ij = R_ji (i >= j), 0 above the diagonal
template <typename T>
__global__ void transpose_r_kernel(T* W, int64_t ldw, int64_t n) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * n; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e % n, j = e / n;
        if (i > j) { W[i + j * ldw] = W[j + i * ldw]; W[j + i * ldw] = T(0); }
    }
}

// ------------------------------------------------------------------ (2) one Jacobi sweep
template <typename T>
__global__ void __launch_bounds__(kSvdThreads, 1) jacobi_sweep_kernel(T* M, int64_t ldw, int64_t n, T* Y, int64_t nrhs,
                                                                      DevState* st, unsigned* bar) {
    const int P = gridDim.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp, nwarps = (int64_t)P * (blockDim.x >> 5);
    const T tol = (T)n * Eps<T>::v;
    const int64_t n2 = n + (n & 1), npairs = n2 / 2, rounds = n2 - 1;
    int my_rot = 0;
    for (int64_t r = 0; r < rounds; ++r) {
        for (int64_t k = gw; k < npairs; k += nwarps) {
            const int64_t s1 = k, s2 = n2 - 1 - k;
            const int64_t a = s1 == 0 ? 0 : 1 + (s1 - 1 + r) % (n2 - 1);
            const int64_t b = s2 == 0 ? 0 : 1 + (s2 - 1 + r) % (n2 - 1);
            if (a >= n || b >= n) continue;
            const int64_t p = a < b ? a : b, q = a < b ? b : a;
            T* mp = M + p * ldw;
            T* mq = M + q * ldw;
            T al = T(0), be = T(0), ga = T(0);
            for (int64_t i = lane; i < n; i += 32) {
                const T x = __ldcg(&mp[i]), y = __ldcg(&mq[i]);
                al += x * x; be += y * y; ga += x * y;
            }
            al = warp_sum(al); be = warp_sum(be); ga = warp_sum(ga);
            if (ga == T(0) || !((ga < T(0) ? -ga : ga) > tol * sqrt(al) * sqrt(be))) continue;
            ++my_rot;
            const T zeta = (be - al) / (T(2) * ga);
            const T t = (zeta >= T(0) ? T(1) : T(-1)) / ((zeta < T(0) ? -zeta : zeta) + sqrt(T(1) + zeta * zeta));
            const T c = T(1) / sqrt(T(1) + t * t);
            const T s = c * t;
            for (int64_t i = lane; i < n; i += 32) {
                const T x = __ldcg(&mp[i]), y = __ldcg(&mq[i]);
                mp[i] = c * x - s * y;
                mq[i] = s * x + c * y;
            }
            for (int64_t rr = lane; rr < nrhs; rr += 32) {
                const T x = __ldcg(&Y[p + rr * n]), y = __ldcg(&Y[q + rr * n]);
                Y[p + rr * n] = c * x - s * y;
                Y[q + rr * n] = s * x + c * y;
            }
        }
        grid_barrier(bar, (unsigned)(r + 1), (unsigned)P);
    }
    if (lane == 0 && my_rot) atomicAdd(&st->rotated, my_rot);
}

// ------------------------------------------------------------------ (2') one block-Jacobi sweep
// Columns are grouped in blocks of BS; a round-robin tournament over the NB blocks pairs them,
// each CTA stages its two blocks (2*BS columns of M and the matching rows of Y) in shared
// memory and rotates every pair among its 2*BS columns (a local round-robin), then writes
// them back.  One sweep = NB-1 block rounds, each ending in one grid barrier (instead of
// n-1 rounds of single pairs); every pair (p, q) meets at least once per sweep.
template <typename T, int BS>
__global__ void __launch_bounds__(kSvdThreads, 1) jacobi_block_sweep_kernel(T* M, int64_t ldw, int64_t n, T* Y,
                                                                            int64_t nrhs, DevState* st, unsigned* bar) {
    constexpr int C2 = 2 * BS;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* Ms = (T*)smem_raw;                  // C2 columns x n
    T* Ys = Ms + (int64_t)C2 * n;          // C2 rows x nrhs
    __shared__ int s_gc[C2];
    const int P = gridDim.x, k = blockIdx.x;
    const int NB = 2 * P;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const T tol = (T)n * Eps<T>::v;
    int my_rot = 0;
    const bool stamp = (k == 0 && threadIdx.x == 0 && st->sweeps == 0);
#define JSTAMP(q) do { if (stamp && r == 5) st->dbg_t[q] = gtimer(); } while (0)
    for (int r = 0; r < NB - 1; ++r) {
        JSTAMP(0);
        const int s1 = k, s2 = NB - 1 - k;
        const int ba = s1 == 0 ? 0 : 1 + (s1 - 1 + r) % (NB - 1);
        const int bb = s2 == 0 ? 0 : 1 + (s2 - 1 + r) % (NB - 1);
        if (threadIdx.x < C2) {
            const int blk = threadIdx.x < BS ? ba : bb;
            const int64_t gc = (int64_t)blk * BS + (threadIdx.x % BS);
            s_gc[threadIdx.x] = gc < n ? (int)gc : -1;
        }
        __syncthreads();
        {   // stage the C2 columns: per thread C2 x 4 independent loads in flight (no index division)
            const int nn = (int)n;
            for (int i0 = 0; i0 < nn; i0 += 4 * (int)blockDim.x) {
                T v[C2][4];
#pragma unroll
                for (int c = 0; c < C2; ++c) {
                    const int gc = s_gc[c];
                    const T* col = M + (int64_t)(gc >= 0 ? gc : 0) * ldw;
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const int i = i0 + (int)threadIdx.x + k * (int)blockDim.x;
                        v[c][k] = (gc >= 0 && i < nn) ? __ldcg(col + i) : T(0);
                    }
                }
#pragma unroll
                for (int c = 0; c < C2; ++c)
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const int i = i0 + (int)threadIdx.x + k * (int)blockDim.x;
                        if (i < nn) Ms[(int64_t)c * n + i] = v[c][k];
                    }
            }
        }
        {   // the C2 rows of Y: element-parallel (a column-outer loop with one active thread for one
            // right-hand side serialised C2 global latencies per round)
            const int nr = (int)nrhs;
            batched<8, T>(
                C2 * nr,
                [&](int e) -> T {
                    const int rr = e / C2, c = e - rr * C2;
                    const int gc = s_gc[c];
                    return gc >= 0 ? __ldcg(&Y[gc + (int64_t)rr * n]) : T(0);
                },
                [&](int e, T v) { Ys[e] = v; });          // Ys[c + rr * C2] = Ys[e]
        }
        __syncthreads();
        JSTAMP(1);
        // local round-robin over C2 columns: C2-1 sub-rounds of BS disjoint pairs; each pair is
        // handled by G = 8 / BS warps, each covering a contiguous slice of the n rows: slice partial
        // sums meet in shared memory (one barrier), every warp of the pair forms the same rotation
        // and applies it to its own slice
        constexpr int G = (kSvdThreads / 32) / BS > 0 ? (kSvdThreads / 32) / BS : 1;
        __shared__ T s_part[BS][G][3];
        const int nn = (int)n;
        const int u_pair = warp % BS, gsl = warp / BS;                   // pair, slice of this warp
        const int slice = (nn + G - 1) / G;
        const int i_lo = gsl * slice, i_hi = min(nn, i_lo + slice);
        // round 0 (every block takes part once per round): all C2(C2-1)/2 pairs of the two blocks
        // (a local round-robin); later rounds: only the BS^2 cross pairs (A_u, B_(u+sr) mod BS) --
        // every pair of columns still meets once per sweep, without re-rotating the intra-block
        // pairs in every round
        const int nsub = (r == 0) ? C2 - 1 : BS;
        for (int sr = 0; sr < nsub; ++sr) {
            int la, lb;
            if (r == 0) {
                const int t1 = u_pair, t2 = C2 - 1 - u_pair;
                la = t1 == 0 ? 0 : 1 + (t1 - 1 + sr) % (C2 - 1);
                lb = t2 == 0 ? 0 : 1 + (t2 - 1 + sr) % (C2 - 1);
            } else {
                la = u_pair;
                lb = BS + (u_pair + sr) % BS;
            }
            int lp = la, lq = lb;
            const bool live = gsl < G && s_gc[lp] >= 0 && s_gc[lq] >= 0;
            if (live && s_gc[lp] > s_gc[lq]) { lp = lb; lq = la; }   // p < q by global column index
            T* mp = Ms + (int64_t)lp * n;
            T* mq = Ms + (int64_t)lq * n;
            if (live) {
                // alpha, beta, gamma over this warp's slice, 4 independent partial sums per lane
                T al4[4] = {}, be4[4] = {}, ga4[4] = {};
                for (int i0 = i_lo + lane; i0 < i_hi; i0 += 128) {
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int i = i0 + 32 * u;
                        if (i < i_hi) { const T x = mp[i], y = mq[i]; al4[u] += x * x; be4[u] += y * y; ga4[u] += x * y; }
                    }
                }
                T al = (al4[0] + al4[1]) + (al4[2] + al4[3]);
                T be = (be4[0] + be4[1]) + (be4[2] + be4[3]);
                T ga = (ga4[0] + ga4[1]) + (ga4[2] + ga4[3]);
                al = warp_sum(al); be = warp_sum(be); ga = warp_sum(ga);
                if (lane == 0) { s_part[u_pair][gsl][0] = al; s_part[u_pair][gsl][1] = be; s_part[u_pair][gsl][2] = ga; }
            }
            __syncthreads();
            if (live) {
                T al = T(0), be = T(0), ga = T(0);
#pragma unroll
                for (int gg = 0; gg < G; ++gg) { al += s_part[u_pair][gg][0]; be += s_part[u_pair][gg][1]; ga += s_part[u_pair][gg][2]; }
                // rotation skipped when |gamma| <= tol sqrt(alpha beta) (Z14 reading)
                const T sa = sqrt(al), sb = sqrt(be);
                const bool rot = !(ga == T(0) || !((ga < T(0) ? -ga : ga) > tol * sa * sb));
                if (rot) {
                    if (gsl == 0) ++my_rot;
                    const T zeta = (be - al) / (T(2) * ga);
                    const T az = zeta < T(0) ? -zeta : zeta;
                    const T t = (zeta >= T(0) ? T(1) : T(-1)) / (az + sqrt(T(1) + zeta * zeta));
                    const T c = rsqrt_nr(T(1) + t * t);
                    const T sn = c * t;
                    for (int i0 = i_lo + lane; i0 < i_hi; i0 += 128) {
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const int i = i0 + 32 * u;
                            if (i < i_hi) {
                                const T x = mp[i], y = mq[i];
                                mp[i] = c * x - sn * y;
                                mq[i] = sn * x + c * y;
                            }
                        }
                    }
                    if (gsl == 0)
                        for (int64_t rr = lane; rr < nrhs; rr += 32) {
                            const T x = Ys[lp + rr * C2], y = Ys[lq + rr * C2];
                            Ys[lp + rr * C2] = c * x - sn * y;
                            Ys[lq + rr * C2] = sn * x + c * y;
                        }
                }
            }
            __syncthreads();
        }
        JSTAMP(2);
        for (int c = 0; c < C2; ++c) {
            const int gc = s_gc[c];
            if (gc < 0) continue;
            const T* src = Ms + (int64_t)c * n;
            T* dst = M + (int64_t)gc * ldw;
            for (int64_t i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
        }
        for (int e = threadIdx.x; e < C2 * (int)nrhs; e += blockDim.x) {
            const int rr = e / C2, c = e - rr * C2;
            const int gc = s_gc[c];
            if (gc >= 0) Y[gc + (int64_t)rr * n] = Ys[e];
        }
        JSTAMP(3);
        grid_barrier(bar, (unsigned)(r + 1), (unsigned)P);
        JSTAMP(4);
    }
#undef JSTAMP
    if (lane == 0 && my_rot) atomicAdd(&st->rotated, my_rot);
}

// WHILE-node condition: another sweep iff this one rotated and the cap is not hit
__global__ void sweep_check_kernel(DevState* st, unsigned* bar, cudaGraphConditionalHandle h) {
    if (threadIdx.x != 0) return;
    st->sweeps += 1;
    const int rot = st->rotated;
    st->rotated = 0;
    *bar = 0u;  // fresh barrier counter for the next sweep
    __threadfence();
    unsigned cont = 0;
    if (rot == 0) st->svd_conv = 1;
    else if (st->sweeps < st->max_sweeps) cont = 1;
    if (h) cudaGraphSetConditional(h, cont);
}

// ------------------------------------------------------------------ (3) sigma, rank
template <typename T>
__global__ void sigma_kernel(const T* M, int64_t ldw, int64_t n, T* sig, DevState* st) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    double best = 0.0;
    bool bad = false;
    for (int64_t k = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); k < n; k += warps) {
        T s = T(0);
        for (int64_t i = lane; i < n; i += 32) { const T x = M[i + k * ldw]; s += x * x; }
        s = warp_sum(s);
        const T sg = sqrt(s);
        if (lane == 0) sig[k] = sg;
        if ((double)sg > best) best = (double)sg;
        bad |= !is_finite_val(sg);
    }
    if (lane == 0 && best > 0.0) atomicMax(&st->smax_bits, dbits(best));
    // non-finite input reached the SVD: the minimum-norm solution is undefined (Z29)
    if (lane == 0 && bad) atomicOr(&st->flags, AS_FLAG_NONFINITE);
}

// rank and the optional descending copy of sigma (rank-based placement, stable)
template <typename T>
__global__ void rank_sort_kernel(const T* sig, int64_t n, DevState* st, const DevArgs* args) {
    T* out = (T*)args->sigma;
    const T smax = (T)dfrom(st->smax_bits);
    const T cut = (T)st->lsq_cut;
    long long kept = 0;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
        const T sk = sig[k];
        if (sk > cut * smax) ++kept;
        if (out) {
            int64_t pos = 0;
            for (int64_t j = 0; j < n; ++j) {
                const T sj = sig[j];
                if (sj > sk || (sj == sk && j < k)) ++pos;
            }
            out[pos] = sk;
        }
    }
    if (kept) atomicAdd((unsigned long long*)&st->rank, (unsigned long long)kept);
}

// ------------------------------------------------------------------ (4) x = sum m_k y_k / sigma_k^2
template <typename T>
__global__ void minnorm_kernel(const T* M, int64_t ldw, int64_t n, const T* Y, int64_t nrhs, const T* sig,
                               const DevState* st, const DevArgs* args, int64_t ldb) {
    T* X = (T*)args->X;
    const T smax = (T)dfrom(st->smax_bits);
    const T cut = (T)st->lsq_cut;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * nrhs; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e % n, r = e / n;
        T acc = T(0);
        for (int64_t k = 0; k < n; ++k) {
            const T sk = sig[k];
            if (!(sk > cut * smax)) continue;
            acc += M[i + k * ldw] * (Y[k + r * n] / (sk * sk));
        }
        X[i + r * ldb] = acc;
    }
}

__global__ void svd_done_kernel(DevState* st) {
    if (threadIdx.x != 0) return;
    st->flags |= AS_FLAG_FALLBACK;
    st->method = AS_METHOD_SVD;
    if (st->flags & AS_FLAG_NONFINITE) { st->rank = -1; st->ret = AS_ERR_NONFINITE; return; }   // Z29
    if (st->rank < 0) st->rank = 0;
    if (st->rank < st->n) st->flags |= AS_FLAG_RANK_DEF;
    if (!st->svd_conv) { st->flags |= AS_FLAG_SVD_NOCONV; st->ret = AS_ERR_SVD_NOT_CONVERGED; }
}

__global__ void svd_rank_reset_kernel(DevState* st) {
    if (threadIdx.x == 0) { st->rank = 0; st->smax_bits = 0ull; }
}

// ------------------------------------------------------------------ launchers
template <typename K, typename... Args>
static void coop_launch(K kern, int P, cudaStream_t s, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(P);
    cfg.blockDim = dim3(kSvdThreads);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, args...);
}

template <typename T>
static void svd_pre_t(const Work& w, cudaStream_t s) {
    T* W = (T*)w.W;
    T* Y = (T*)w.yv;
    svd_setup_kernel<T><<<w.num_sms * 4, 256, 0, s>>>(w.args, w.lda, w.ldb, w.n, w.nrhs, W, w.ldw, Y, w.st);
    coop_launch(qr_kernel<T>, w.num_sms, s, W, w.ldw, w.n, Y, w.nrhs, (T*)w.xe, w.bars + 0);
    transpose_r_kernel<T><<<w.num_sms * 4, 256, 0, s>>>(W, w.ldw, w.n);
}

template <typename T, int BS>
static bool launch_block_sweep(const Work& w, cudaStream_t s) {
    const int64_t nb = (w.n + BS - 1) / BS;
    const int P = (int)((nb + 1) / 2);                     // NB = 2P blocks (one may be a dummy)
    const size_t smem = sizeof(T) * ((size_t)2 * BS * w.n + (size_t)2 * BS * std::max<int64_t>(w.nrhs, 1));
    int optin = 0, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (P >= 2 && P <= w.num_sms && smem <= (size_t)optin) {
        auto kern = jacobi_block_sweep_kernel<T, BS>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(P);
        cfg.blockDim = dim3(kSvdThreads);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeCooperative;
        attr[0].val.cooperative = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, kern, (T*)w.W, w.ldw, w.n, (T*)w.yv, w.nrhs, w.st, w.bars + 1);
        return true;
    }
    return false;
}

// one sweep: column blocks of 4 (8 columns per CTA) when they fit in shared memory and on the
// SMs, else the per-pair kernel
template <typename T>
static void svd_sweep_t(const Work& w, cudaGraphConditionalHandle h, cudaStream_t s) {
    // (blocks of 8 measured slower: the pair updates are shared-memory bandwidth bound and only
    //  half as many CTAs take part)
    if (!launch_block_sweep<T, 4>(w, s))
        coop_launch(jacobi_sweep_kernel<T>, w.num_sms, s, (T*)w.W, w.ldw, w.n, (T*)w.yv, w.nrhs, w.st, w.bars + 1);
    sweep_check_kernel<<<1, 32, 0, s>>>(w.st, w.bars + 1, h);
}

template <typename T>
static void svd_post_t(const Work& w, cudaStream_t s) {
    T* sig = (T*)w.xe;
    svd_rank_reset_kernel<<<1, 32, 0, s>>>(w.st);
    sigma_kernel<T><<<w.num_sms * 2, 256, 0, s>>>((const T*)w.W, w.ldw, w.n, sig, w.st);
    rank_sort_kernel<T><<<(unsigned)std::min<int64_t>((w.n + 255) / 256, 1024), 256, 0, s>>>(sig, w.n, w.st, w.args);
    minnorm_kernel<T><<<w.num_sms * 4, 256, 0, s>>>((const T*)w.W, w.ldw, w.n, (const T*)w.yv, w.nrhs, sig, w.st,
                                                     w.args, w.ldb);
    svd_done_kernel<<<1, 32, 0, s>>>(w.st);
}

void launch_svd_pre(const Work& w, cudaStream_t s) {
    if (w.dtype == AS_F64) svd_pre_t<double>(w, s); else svd_pre_t<float>(w, s);
}
void launch_svd_sweep(const Work& w, cudaGraphConditionalHandle h, cudaStream_t s) {
    if (w.dtype == AS_F64) svd_sweep_t<double>(w, h, s); else svd_sweep_t<float>(w, h, s);
}
void launch_svd_post(const Work& w, cudaStream_t s) {
    if (w.dtype == AS_F64) svd_post_t<double>(w, s); else svd_post_t<float>(w, s);
}

}  // namespace as
