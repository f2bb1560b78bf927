// detect.cu -- K1: single-pass structure detection.
//
//   banded:     kl/ku = max distance of a non-zero below/above the diagonal,
//               the per-column scan of P:328-337, and the 25% capacity rule of
//               P:339 (banded <=> 4*count(n,kl,ku) <= n^2, Z2/Z3);
//   triangular: all elements above (lower) / below (upper) the diagonal are
//               exactly zero (Z6);
//   sympd:      Fig. 4 likely_sympd with its literal operators (Z7).
//
// Every verdict is an AND/OR/max of per-element predicates, so the order in
// which tiles are visited cannot change it (Z8): the kernel visits mirror tile
// pairs (I,J)/(J,I) from a device work queue, far-from-diagonal pairs first, so
// a dense asymmetric matrix kills all four candidates within the first pair
// and the kernel exits early (the paper's "all further processing is stopped",
// P:339-340), while a banded matrix is read exactly once (HBM-bound).
#include "internal.h"

namespace as {

// ------------------------------------------------------------------ per-call args
__global__ void set_args_kernel(DevArgs a, DevArgs* dst) { *dst = a; }

// ------------------------------------------------------------------ state init
__global__ void state_init_kernel(DevState* st, int64_t n, uint32_t opts, int force_method, double thr, double cut,
                                  int max_sweeps) {
    if (threadIdx.x != 0) return;
    DevState s = {};
    s.alive = AS_FLAG_BANDED | AS_FLAG_LOWER | AS_FLAG_UPPER | AS_FLAG_SPD_CANDIDATE;
    s.kl = 0; s.ku = 0;
    s.max_diag = 0ull;
    s.opts = opts;
    s.force_method = force_method;
    s.n = n;
    s.info = ~0ull;
    s.rcond = 0.0;
    s.thr = thr;
    s.lsq_cut = cut;
    s.max_sweeps = max_sweeps;
    s.est_next = 0;
    s.rank = -1;
    *st = s;
}

// ------------------------------------------------------------------ pass 1: diagonal
// Fig. 4 lines 7-9: any A_jj <= 0 kills SPD; max_diag = max A_jj over A_jj > 0.
// Also gathers diag(A) contiguously for the pair pass (line 16).
template <typename T>
__global__ void detect_diag_kernel(const DevArgs* args, int64_t lda, int64_t n, DevState* st, T* diag) {
    const T* A = (const T*)args->A;
    double local = 0.0;
    bool kill = false;
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        T a = A[j + j * lda];
        diag[j] = a;
        if (a <= T(0)) kill = true;                 // line 8 (NaN: false -> no kill)
        if (a > T(0) && (double)a > local) local = (double)a;   // line 9
    }
    // block reduce
    __shared__ double smax[32];
    __shared__ int skill;
    if (threadIdx.x == 0) skill = 0;
    __syncthreads();
    for (int o = 16; o > 0; o >>= 1) local = fmax(local, __shfl_xor_sync(0xffffffffu, local, o));
    if ((threadIdx.x & 31) == 0) smax[threadIdx.x >> 5] = local;
    if (kill) skill = 1;
    __syncthreads();
    if (threadIdx.x == 0) {
        double m = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) m = fmax(m, smax[w]);
        if (m > 0.0) atomicMax(&st->max_diag, dbits(m));
        if (skill) atomicAnd(&st->alive, ~AS_FLAG_SPD_CANDIDATE);
    }
}

AS_DEV bool band_density_ok(long long n, long long kl, long long ku) {
    unsigned long long un = (unsigned long long)n;
    unsigned long long cnt = un * (unsigned long long)(kl + ku + 1) - (unsigned long long)(kl * (kl + 1) / 2) -
                             (unsigned long long)(ku * (ku + 1) / 2);
    return 4ull * cnt <= un * un;
}

// ------------------------------------------------------------------ pass 2: tile pairs
// CTA = 256 threads = 8 warps.  Tile 64x64.  Lane l of warp w holds rows l and
// l+32 of columns w, w+8, ..., w+56 of the lower tile (I,J) in registers; the
// mirror tile (J,I) is staged in shared memory (padded, conflict-free
// transposed reads).  Diagonal tiles (I==J) pair with themselves.
constexpr int kDetThreads = 256;
constexpr int kLD = kTile + 1;

template <typename T>
__global__ void __launch_bounds__(kDetThreads) detect_pairs_kernel(const DevArgs* args, int64_t lda, int64_t n,
                                                                    DevState* st, const T* diag, int fullscan) {
    __shared__ T up[kTile * kLD];
    __shared__ unsigned s_pair;
    __shared__ unsigned s_alive;
    __shared__ int s_kl, s_ku;
    __shared__ unsigned s_kill;
    const T* A = (const T*)args->A;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long long nt = (n + kTile - 1) / kTile;
    const unsigned long long total = (unsigned long long)(nt * (nt + 1) / 2);
    const T tol = T(100) * Eps<T>::v;                       // Fig. 4 line 5
    const double maxd = dfrom(st->max_diag);                 // final after pass 1
    const T max_diag = (T)maxd;                              // exact (it was a T value)
    int my_kl = 0, my_ku = 0;                                // CTA-cached global maxima

    for (;;) {
        if (threadIdx.x == 0) {
            unsigned al = *(volatile unsigned*)&st->alive;
            s_alive = al;
            s_pair = (fullscan || al) ? atomicAdd(&st->pair_ticket, 1u) : 0xffffffffu;
            s_kl = 0; s_ku = 0; s_kill = 0;
        }
        __syncthreads();
        const unsigned p = s_pair;
        const unsigned alive = fullscan ? 0xFu : s_alive;
        if (p >= total) break;
        // pair index -> (I, J): distance-major, far pairs first
        long long q = (long long)((sqrt(8.0 * (double)p + 1.0) - 1.0) * 0.5) + 1;
        while (q * (q - 1) / 2 > (long long)p) --q;
        while (q * (q + 1) / 2 <= (long long)p) ++q;
        const long long D = nt - q;
        const long long J = (long long)p - q * (q - 1) / 2;
        const long long I = J + D;
        const bool diag_tile = (D == 0);
        const bool need_lower = fullscan || (alive & (AS_FLAG_BANDED | AS_FLAG_UPPER | AS_FLAG_SPD_CANDIDATE));
        const bool need_upper = fullscan || diag_tile || (alive & (AS_FLAG_BANDED | AS_FLAG_LOWER | AS_FLAG_SPD_CANDIDATE));
        const long long r0 = I * kTile, c0 = J * kTile;     // lower tile origin (rows I, cols J)
        const int rows_lo = (int)min<long long>(kTile, n - r0), cols_lo = (int)min<long long>(kTile, n - c0);

        // ---- stage the mirror tile (rows J, cols I) into smem: up[c' * kLD + r']
        if (need_upper) {
            const int rows_up = cols_lo, cols_up = rows_lo;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int c = warp + 8 * k;
                if (c < cols_up) {
                    const T* col = A + (c0) + (r0 + c) * lda;     // column (I*64 + c), rows J*64..
                    up[c * kLD + lane] = lane < rows_up ? col[lane] : T(0);
                    up[c * kLD + lane + 32] = lane + 32 < rows_up ? col[lane + 32] : T(0);
                }
            }
        }
        // ---- lower tile into registers
        T lo0[8], lo1[8];
        if (need_lower || diag_tile) {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int c = warp + 8 * k;
                const T* col = A + r0 + (c0 + c) * lda;
                const bool cv = c < cols_lo;
                lo0[k] = (cv && lane < rows_lo) ? col[lane] : T(0);
                lo1[k] = (cv && lane + 32 < rows_lo) ? col[lane + 32] : T(0);
            }
        }
        __syncthreads();

        int kl_loc = 0, ku_loc = 0;
        bool lower_nz = false, upper_nz = false, spd_dead = false;
        const bool chk_spd = (alive & AS_FLAG_SPD_CANDIDATE) != 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int c = warp + 8 * k;
            if (c >= cols_lo) continue;
            const long long gj = c0 + c;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int r = lane + 32 * h;
                if (r >= rows_lo) continue;
                const long long gi = r0 + r;
                const T a = h ? lo1[k] : lo0[k];   // A(gi, gj)
                if (gi > gj) {
                    // mirror b = A(gj, gi) = up tile element (row r' = c, col c' = r)
                    const T b = need_upper ? up[r * kLD + c] : T(0);
                    const int dist = (int)(gi - gj);
                    if (a != T(0)) { lower_nz = true; kl_loc = max(kl_loc, dist); }
                    if (b != T(0)) { upper_nz = true; ku_loc = max(ku_loc, dist); }
                    if (chk_spd) {
                        const T aa = a < T(0) ? -a : a, ab = b < T(0) ? -b : b;
                        const T delta = (a - b) < T(0) ? -(a - b) : (a - b);          // line 12
                        const T m = aa > ab ? aa : ab;
                        if (delta > tol && delta > tol * m) spd_dead = true;           // lines 13-14
                        if (aa >= max_diag) spd_dead = true;                            // line 15
                        const T lhs = aa + ab;
                        const T rhs = diag[gi] + diag[gj];
                        if (lhs >= rhs) spd_dead = true;                                // line 16
                    }
                } else if (gi < gj && diag_tile) {
                    // strictly-upper element of a diagonal tile (its pair is handled from the lower side)
                    if (a != T(0)) { upper_nz = true; ku_loc = max(ku_loc, (int)(gj - gi)); }
                }
            }
        }
        // ---- reduce within the CTA
        kl_loc = __reduce_max_sync(0xffffffffu, kl_loc);
        ku_loc = __reduce_max_sync(0xffffffffu, ku_loc);
        const unsigned kill = (__any_sync(0xffffffffu, lower_nz) ? AS_FLAG_UPPER : 0u) |
                              (__any_sync(0xffffffffu, upper_nz) ? AS_FLAG_LOWER : 0u) |
                              (__any_sync(0xffffffffu, spd_dead) ? AS_FLAG_SPD_CANDIDATE : 0u);
        if (lane == 0) {
            if (kl_loc) atomicMax(&s_kl, kl_loc);
            if (ku_loc) atomicMax(&s_ku, ku_loc);
            if (kill) atomicOr(&s_kill, kill);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            int gkl = my_kl, gku = my_ku;
            if (s_kl > my_kl) gkl = max(s_kl, atomicMax(&st->kl, s_kl));
            if (s_ku > my_ku) gku = max(s_ku, atomicMax(&st->ku, s_ku));
            my_kl = gkl; my_ku = gku;
            unsigned k2 = s_kill;
            if (!band_density_ok(n, gkl, gku)) k2 |= AS_FLAG_BANDED;
            if (k2 & alive) atomicAnd(&st->alive, ~k2);
        }
        // (thread 0 is the only reader of my_kl/my_ku)
        __syncthreads();
    }
}

// ------------------------------------------------------------------ dispatch
// First match in the paper's order: banded, lower, upper, sympd,
// else general LU; or the forced method.  Sets the SWITCH handle.
__global__ void dispatch_kernel(DevState* st, cudaGraphConditionalHandle h_method, int use_handle) {
    if (threadIdx.x != 0) return;
    const unsigned f = st->alive;
    st->det_flags = f;
    int m;
    if (st->opts & AS_OPT_FORCE_METHOD) m = st->force_method;
    else if (f & AS_FLAG_BANDED) m = AS_METHOD_BAND;
    else if (f & AS_FLAG_LOWER) m = AS_METHOD_TRI_LOWER;
    else if (f & AS_FLAG_UPPER) m = AS_METHOD_TRI_UPPER;
    else if (f & AS_FLAG_SPD_CANDIDATE) m = AS_METHOD_CHOL;
    else m = AS_METHOD_LU;
    st->method = m;
    st->primary = m;
    if (use_handle) cudaGraphSetConditional(h_method, (unsigned)m);
}

// ------------------------------------------------------------------ launchers
void launch_state_init(const Work& w, cudaStream_t s, uint32_t opts, int force_method, double thr, double cut,
                       int max_sweeps) {
    state_init_kernel<<<1, 32, 0, s>>>(w.st, w.n, opts, force_method, thr, cut, max_sweeps);
    cudaMemsetAsync(w.bars, 0, sizeof(unsigned) * w.bars_len, s);
}

void launch_detect(const Work& w, cudaStream_t s, bool fullscan) {
    const int dthreads = 256;
    const int dblocks = (int)std::min<int64_t>((w.n + dthreads - 1) / dthreads, 4 * w.num_sms);
    const long long nt = (w.n + kTile - 1) / kTile;
    const long long pairs = nt * (nt + 1) / 2;
    const int pblocks = (int)std::min<long long>(pairs, (long long)w.num_sms * 6);
    if (w.dtype == AS_F64) {
        detect_diag_kernel<double><<<std::max(dblocks, 1), dthreads, 0, s>>>(w.args, w.lda, w.n, w.st, (double*)w.diag);
        detect_pairs_kernel<double><<<std::max(pblocks, 1), kDetThreads, 0, s>>>(w.args, w.lda, w.n, w.st,
                                                                                 (const double*)w.diag, fullscan);
    } else {
        detect_diag_kernel<float><<<std::max(dblocks, 1), dthreads, 0, s>>>(w.args, w.lda, w.n, w.st, (float*)w.diag);
        detect_pairs_kernel<float><<<std::max(pblocks, 1), kDetThreads, 0, s>>>(w.args, w.lda, w.n, w.st,
                                                                               (const float*)w.diag, fullscan);
    }
}

void launch_dispatch(const Work& w, cudaStream_t s, cudaGraphConditionalHandle h_method) {
    dispatch_kernel<<<1, 32, 0, s>>>(w.st, h_method, h_method != 0);
}

}  // namespace as
