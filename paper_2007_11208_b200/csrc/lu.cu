// lu.cu -- K7: blocked LU with partial pivoting (xGETRF).
//
// Right-looking, 128-column blocks, each block factored as two 64-column
// panels (a two-level recursive panel: the second half is updated by a
// rank-64 DMMA GEMM before it is factored), so that the trailing update is a
// K = 128 DMMA GEMM (86% of the measured fp64 tensor peak at n = 16384).
//
//   per block b (columns k0 .. k0+127):
//     panel(k0, 64)          cooperative kernel: rows split over P CTAs, held in
//                            shared memory; per column one grid-wide exchange of
//                            (|max|, row) candidates -- published with a sequence
//                            number and polled, so barrier and data arrive
//                            together -- first-max tie-break (Z15), swap, scale,
//                            in-panel rank-1 update
//     laswp + u12 + gemm      bring columns k0+64..k0+127 up to date
//     panel(k0+64, 64)
//     laswp                  all other columns (and the row permutation)
//     u12                    U12 = L11^{-1} A12 (128 x (n - k0 - 128))
//     gemm (DMMA, K = 128)   A22 -= L21 U12
//   look-ahead: the GEMM is split; the columns of the next block are updated
//   first on a high-priority stream and the next block's panels start there
//   while the bulk of the GEMM is still running.
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <mutex>

#include "factor.h"
#include "gemm.h"
#include "internal.h"
#include <cooperative_groups.h>
#include "blk64.cuh"
#include "trsm.h"

namespace as {

constexpr int kPT = 256;     // panel threads
constexpr int kPW = 128;     // panel width (= block width: one cooperative panel per block, so the
                             // look-ahead chain is panel + L11 inverse only)
constexpr int kBW = 128;     // block width
constexpr int kHalf = 64;    // U12 and Dinv work in 64-row halves of a block

// ---- diagnostics: per-block timeline of the factorization (AS_LU_TRACE=1; %globaltimer)
// slots per 128-column block k: 0 main-stream trailing GEMM, 1 panel 1, 2 panel 2, 3 look-ahead GEMM
constexpr int kTraceBlocks = 512;
struct LuTrace {
    unsigned long long* tmin = nullptr;   // [4 * kTraceBlocks] first start
    unsigned long long* tmax = nullptr;   // [4 * kTraceBlocks] last end
};
static LuTrace& lu_trace() {
    static LuTrace t;
    static bool init = false;
    if (!init) {
        init = true;
        if (getenv("AS_LU_TRACE")) {
            cudaMalloc(&t.tmin, sizeof(unsigned long long) * 4 * kTraceBlocks);
            cudaMalloc(&t.tmax, sizeof(unsigned long long) * 4 * kTraceBlocks);
        }
    }
    return t;
}

struct __align__(32) PSlot {
    double v;
    long long idx;
    unsigned long long seq;
    long long pad;
};

// Order-preserving integer key of a candidate |a| >= +0 (0 is reserved for "no candidate"): the
// first-max argmax becomes three integer warp reductions (max high word, max low word among the
// high maxima, min row among the full maxima).
template <typename T> AS_DEV void cand_key(T x, unsigned& hi, unsigned& lo);
template <> AS_DEV void cand_key<double>(double x, unsigned& hi, unsigned& lo) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(x);   // x >= +0: bits are monotone
    hi = (unsigned)(b >> 32) + 1u;
    lo = (unsigned)b;
}
template <> AS_DEV void cand_key<float>(float x, unsigned& hi, unsigned& lo) {
    hi = __float_as_uint(x) + 1u;
    lo = 0u;
}

// ------------------------------------------------------------------ panel (cooperative)
// Rows of the panel are split over the P CTAs (shared memory when they fit).  Per column j:
// every CTA publishes its local first-max candidate row (and the owner of row g the old row g)
// and a sequence-numbered slot; all CTAs poll the P slots (barrier and data in one), read the
// winning row, swap, form the multipliers and update column j+1 first, so that column j+1's
// candidate can be published before the bulk of the rank-1 update -- the other CTAs' exchange
// latency then overlaps this CTA's update.
template <typename T>
AS_DEV void panel_local_argmax(const T* Ps, int64_t cp, int nr, int64_t rbeg, int64_t g, int col, T& v, long long& idx,
                               T* sv, long long* si, int* sdn) {
    // first max |a(r, col)| over local rows at positions >= g; NaN never wins, a NaN at row g keeps
    // g (the serial sweep's semantics).  Warp level: fmax shuffles + ballot + integer min of the
    // row; CTA level: every warp merges the 8 warp results the same way (one barrier).
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    T bv = T(-1);
    unsigned br = 0xffffffffu;
    int dnan = 0;
    for (int r = threadIdx.x; r < nr; r += blockDim.x) {
        const int64_t gr = rbeg + r;
        if (gr < g) continue;
        T a = Ps[r + col * cp];
        a = a < T(0) ? -a : a;
        if (gr == g && a != a) dnan = 1;
        if (a > bv) { bv = a; br = (unsigned)r; }     // rows increase: strict > keeps the first
    }
    unsigned kh = 0u, kl = 0u;
    if (br != 0xffffffffu) cand_key<T>(bv == T(0) ? T(0) : bv, kh, kl);   // (-0 -> +0)
    unsigned mh = __reduce_max_sync(0xffffffffu, kh);
    unsigned ml = __reduce_max_sync(0xffffffffu, kh == mh ? kl : 0u);
    const unsigned wr = __reduce_min_sync(0xffffffffu, (mh != 0u && kh == mh && kl == ml) ? br : 0xffffffffu);
    const T wm = __shfl_sync(0xffffffffu, bv, (int)(__ffs(__ballot_sync(0xffffffffu, br == wr && wr != 0xffffffffu)) - 1) & 31);
    dnan = __any_sync(0xffffffffu, dnan);
    if (lane == 0) { sv[warp] = (wr == 0xffffffffu) ? T(-1) : wm; si[warp] = (long long)wr; sdn[warp] = dnan; }
    __syncthreads();
    const int nw = (int)(blockDim.x >> 5);
    const T v8 = (lane & 7) < nw ? sv[lane & 7] : T(-1);
    const unsigned r8 = (lane & 7) < nw ? (unsigned)si[lane & 7] : 0xffffffffu;
    const int d8 = (lane & 7) < nw ? sdn[lane & 7] : 0;
    kh = 0u; kl = 0u;
    if (r8 != 0xffffffffu) cand_key<T>(v8, kh, kl);
    mh = __reduce_max_sync(0xffffffffu, kh);
    ml = __reduce_max_sync(0xffffffffu, kh == mh ? kl : 0u);
    const unsigned rmin = __reduce_min_sync(0xffffffffu, (mh != 0u && kh == mh && kl == ml) ? r8 : 0xffffffffu);
    const T m8 = __shfl_sync(0xffffffffu, v8, (int)(__ffs(__ballot_sync(0xffffffffu, r8 == rmin && rmin != 0xffffffffu)) - 1) & 31);
    const int dn = __any_sync(0xffffffffu, d8);
    v = (rmin == 0xffffffffu) ? T(-1) : m8;
    idx = (rmin == 0xffffffffu) ? 0x7fffffffffffffffll : (long long)(rbeg + rmin);
    if (dn) { v = T(INFINITY); idx = g; }
}

// Bulk rank-1 update of the panel rows r0 .. nr-1 (local), columns j+2 .. nbp-1:
// a(r, c) -= a(r, j) * u(c), rows skip0 / skip1 excluded.  Thread tile: 4 rows (lane + 32 i) x
// columns cg + 8 q (warp = column group), 4 columns per batch with every load before the stores
// (one u load feeds 4 rows; Ps and u are both shared memory: unbatched code would serialise).
template <typename T>
AS_DEV void panel_bulk_update(T* __restrict__ Ps, int64_t cp, const T* __restrict__ u, int r0, int nr, int j, int nbp,
                              int skip0, int skip1) {
    const int lane = threadIdx.x & 31, cgp = threadIdx.x >> 5, ncg = (int)(blockDim.x >> 5);
    for (int rb = r0; rb < nr; rb += 128) {
        int rr[4];
        T l[4];
        bool ok[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            rr[i] = rb + lane + 32 * i;
            ok[i] = rr[i] < nr && rr[i] != skip0 && rr[i] != skip1;
            l[i] = ok[i] ? Ps[rr[i] + j * cp] : T(0);
        }
        for (int c0 = j + 2 + cgp; c0 < nbp; c0 += 4 * ncg) {
            T uv[4], av[4][4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int c = c0 + q * ncg;
                uv[q] = c < nbp ? u[c] : T(0);
#pragma unroll
                for (int i = 0; i < 4; ++i) av[q][i] = (ok[i] && c < nbp) ? Ps[rr[i] + c * cp] : T(0);
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int c = c0 + q * ncg;
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    if (ok[i] && c < nbp) Ps[rr[i] + c * cp] = av[q][i] - l[i] * uv[q];
            }
        }
    }
}

template <typename T>
__global__ void __launch_bounds__(kPT, 1) lu_panel2_kernel(T* W, int64_t ldw, int64_t n, int64_t k0, int nbp,
                                                            int64_t* ipiv, DevState* st, PSlot* slots, T* rowbuf,
                                                            T* diagbuf, unsigned long long seq_base, int use_smem,
                                                            unsigned long long* tr_min, unsigned long long* tr_max) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    if (tr_min && threadIdx.x == 0) atomicMin(tr_min, gtimer());
    const int P = gridDim.x, cta = blockIdx.x;
    const int64_t m = n - k0;
    const int64_t chunk = (m + P - 1) / P;
    const int64_t rbeg = k0 + (int64_t)cta * chunk;
    const int64_t rend = min(n, rbeg + chunk);
    const int nr = (int)max<int64_t>(0, rend - rbeg);
    // odd column stride: row accesses (pivot / candidate rows, stride cp) are bank-conflict free
    const int64_t cp = use_smem ? (chunk | 1) : ldw;
    T* Ps = use_smem ? (T*)smem_raw : W + rbeg + k0 * ldw;
    T* ubuf = use_smem ? (T*)smem_raw + cp * nbp : (T*)smem_raw;
    __shared__ T sv[8];
    __shared__ long long si[8];
    __shared__ int sdn[8];
    __shared__ long long s_p;
    __shared__ int s_owner;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

    if (use_smem) {
        batched<8, T>(
            nr * nbp, [&](int e) -> T { const int c = e / nr, r = e - c * nr; return W[(rbeg + r) + (k0 + c) * ldw]; },
            [&](int e, T v) { const int c = e / nr, r = e - c * nr; Ps[r + c * cp] = v; });
        __syncthreads();
    }
    // publish the candidate for column j: (v, idx) of this CTA, its row, and the old row g
    auto publish = [&](int j, T v, long long idx) {
        const int64_t g = k0 + j;
        const int par = j & 1;
        if (idx != 0x7fffffffffffffffll && idx >= rbeg && idx < rend) {
            const int r = (int)(idx - rbeg);
            for (int c = threadIdx.x; c < nbp; c += blockDim.x) rowbuf[((int64_t)par * P + cta) * nbp + c] = Ps[r + c * cp];
        }
        if (g >= rbeg && g < rend) {
            const int r = (int)(g - rbeg);
            for (int c = threadIdx.x; c < nbp; c += blockDim.x) diagbuf[par * nbp + c] = Ps[r + c * cp];
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            // slots are double-buffered by column parity like rowbuf: a CTA one column ahead must
            // not overwrite a candidate another CTA has not read yet
            PSlot* sl = slots + par * 512 + cta;
            sl->v = (double)v;
            sl->idx = idx;
            // release is cumulative: the CTA's rowbuf writes (ordered by the barrier above) are published too
            asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(&sl->seq), "l"(seq_base + (unsigned long long)j + 1ull) : "memory");
        }
    };
    {
        T v;
        long long idx;
        panel_local_argmax(Ps, cp, nr, rbeg, k0, 0, v, idx, sv, si, sdn);
        publish(0, v, idx);
    }
    unsigned long long info = ~0ull;
    for (int j = 0; j < nbp; ++j) {
        const int64_t g = k0 + j;
        const int par = j & 1;
        const unsigned long long want = seq_base + (unsigned long long)j + 1ull;
        // ---- poll every slot (barrier + data in one), pick the winner
        if (warp == 0) {
            T bv = T(-1);
            long long bi = 0x7fffffffffffffffll;
            int bo = 0;
            // each lane owns up to 5 slots (P <= 160); all are polled together each round
            constexpr int kMaxPer = 5;
            bool ready[kMaxPer];
#pragma unroll
            for (int q = 0; q < kMaxPer; ++q) ready[q] = (lane + 32 * q) >= P;
            for (;;) {
                bool all = true;
#pragma unroll
                for (int q = 0; q < kMaxPer; ++q) {
                    if (!ready[q]) {
                        const unsigned long long sq = ld_relaxed64(&slots[par * 512 + lane + 32 * q].seq);
                        ready[q] = sq >= want;
                        all = all && ready[q];
                    }
                }
                if (__all_sync(0xffffffffu, all)) break;
            }
            fence_acq_rel();   // the slots' data (and the rows they guard) after the flags
#pragma unroll
            for (int q = 0; q < kMaxPer; ++q) {
                const int t = lane + 32 * q;
                if (t < P) {
                    const T cv = (T)__ldcg(&slots[par * 512 + t].v);
                    const long long ci = __ldcg(&slots[par * 512 + t].idx);
                    if (cv > bv || (cv == bv && ci < bi)) { bv = cv; bi = ci; bo = t; }
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const T v2 = __shfl_xor_sync(0xffffffffu, bv, o);
                const long long i2 = __shfl_xor_sync(0xffffffffu, bi, o);
                const int o2 = __shfl_xor_sync(0xffffffffu, bo, o);
                if (v2 > bv || (v2 == bv && i2 < bi)) { bv = v2; bi = i2; bo = o2; }
            }
            if (lane == 0) { s_p = bi; s_owner = bo; }
        }
        __syncthreads();
        const long long p = s_p;
        const int owner = s_owner;
        const bool own_p = p != g && p >= rbeg && p < rend;
        // the pivot row into ubuf; the owner of p takes the old row g (both loads in flight together)
        T* dst_p = own_p ? Ps + (p - rbeg) : nullptr;
        for (int c = threadIdx.x; c < nbp; c += blockDim.x) {
            const T u = __ldcg(&rowbuf[((int64_t)par * P + owner) * nbp + c]);
            const T dg = own_p ? __ldcg(&diagbuf[par * nbp + c]) : T(0);
            ubuf[c] = u;
            if (own_p) dst_p[c * cp] = dg;
        }
        __syncthreads();
        const T piv = ubuf[j];
        if (cta == 0 && threadIdx.x == 0) ipiv[g] = (p == 0x7fffffffffffffffll) ? g : p;
        const bool elim = piv != T(0);
        if (!elim) {                             // exact zero pivot: singular column (no swap, no elimination)
            if (info == ~0ull) info = (unsigned long long)(g + 1);
            if (own_p)                           // undo: row p keeps its own values
                for (int c = threadIdx.x; c < nbp; c += blockDim.x) dst_p[c * cp] = ubuf[c];
        } else if (g >= rbeg && g < rend) {
            const int r = (int)(g - rbeg);
            for (int c = threadIdx.x; c < nbp; c += blockDim.x) Ps[r + c * cp] = ubuf[c];
        }
        __syncthreads();
        const int64_t r0 = max<int64_t>(0, g + 1 - rbeg);
        // ---- multipliers and column j+1 of my rows > g
        if (elim) {
            const T u1 = (j + 1 < nbp) ? ubuf[j + 1] : T(0);
            for (int r = (int)r0 + threadIdx.x; r < nr; r += blockDim.x) {
                const T l = Ps[r + j * cp] / piv;
                Ps[r + j * cp] = l;
                if (j + 1 < nbp) Ps[r + (j + 1) * cp] -= l * u1;
            }
        }
        __syncthreads();
        if (j + 1 >= nbp) break;
        // ---- column j+1's candidate: finish its row (and row g+1) first, publish, then the bulk
        T v;
        long long idx;
        panel_local_argmax(Ps, cp, nr, rbeg, g + 1, j + 1, v, idx, sv, si, sdn);
        const int rc = (idx != 0x7fffffffffffffffll && idx >= rbeg && idx < rend) ? (int)(idx - rbeg) : -1;
        const int rg = (g + 1 >= rbeg && g + 1 < rend) ? (int)(g + 1 - rbeg) : -1;
        if (elim) {
            for (int c = j + 2 + threadIdx.x; c < nbp; c += blockDim.x) {
                if (rc >= 0) Ps[rc + c * cp] -= Ps[rc + j * cp] * ubuf[c];
                if (rg >= 0 && rg != rc) Ps[rg + c * cp] -= Ps[rg + j * cp] * ubuf[c];
            }
        }
        __syncthreads();
        publish(j + 1, v, idx);
        // ---- bulk rank-1 update of the remaining rows, columns j+2.. (thread = row, column phase)
        if (elim) panel_bulk_update<T>(Ps, cp, ubuf, (int)r0, nr, j, nbp, rc, rg);
        __syncthreads();
    }
    if (use_smem) {
        for (int e = threadIdx.x; e < nr * nbp; e += blockDim.x) {
            const int c = e / nr, r = e - c * nr;
            W[(rbeg + r) + (k0 + c) * ldw] = Ps[r + c * cp];
        }
    }
    if (threadIdx.x == 0 && cta == 0 && info != ~0ull) atomicMin(&st->info, info);
    if (tr_max && threadIdx.x == 0) atomicMax(tr_max, gtimer());
}

// ------------------------------------------------------------------ panel (one thread-block cluster)
// Same algorithm as lu_panel2_kernel for panels whose rows fit in the shared memory of at most
// kClMax CTAs: the per-column candidate exchange goes through distributed shared memory with
// one cluster barrier per column instead of sequence-numbered global slots (several L2 round
// trips per column).  Candidate rows / old row g are double-buffered by column parity: a CTA
// rewrites a parity buffer only after the next column's barrier, i.e. after every CTA read it.
namespace cg = cooperative_groups;
constexpr int kClMax = 8;
template <typename T>
__global__ void __launch_bounds__(kPT, 1) lu_panel_cl_kernel(T* W, int64_t ldw, int64_t n, int64_t k0, int nbp,
                                                              int64_t* ipiv, DevState* st, int prof_on) {
    cg::cluster_group cl = cg::this_cluster();
    // diagnostics (prof_on): clock64 phase totals of CTA 0 / thread 0 into st->dbg_t
    const bool prof = prof_on && blockIdx.x == 0 && threadIdx.x == 0;
    long long ph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long tp = clock64();
#define PHC(q) do { if (prof) { const long long t_ = clock64(); ph[q] += t_ - tp; tp = t_; } } while (0)
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int P = gridDim.x, cta = blockIdx.x;          // the grid is one cluster
    const int64_t m = n - k0;
    const int64_t chunk = (m + P - 1) / P;
    const int64_t rbeg = k0 + (int64_t)cta * chunk;
    const int64_t rend = min(n, rbeg + chunk);
    const int nr = (int)max<int64_t>(0, rend - rbeg);
    const int64_t cp = chunk | 1;                        // odd stride: conflict-free row accesses
    T* Ps = (T*)smem_raw;                                // chunk x nbp, column-major
    T* ubuf = Ps + cp * nbp;                             // pivot row
    T* candb = ubuf + nbp;                               // [2][nbp] my candidate row
    T* diagb = candb + 2 * nbp;                          // [2][nbp] old row g (owner of g)
    __shared__ T s_cv[2];
    __shared__ long long s_ci[2];
    __shared__ T sv[8];
    __shared__ long long si[8];
    __shared__ int sdn[8];
    __shared__ long long s_p;
    __shared__ int s_owner;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

    batched<8, T>(
        nr * nbp, [&](int e) -> T { const int c = e / nr, r = e - c * nr; return W[(rbeg + r) + (k0 + c) * ldw]; },
        [&](int e, T v) { const int c = e / nr, r = e - c * nr; Ps[r + c * cp] = v; });
    __syncthreads();
    auto publish = [&](int j, T v, long long idx) {
        const int64_t g = k0 + j;
        const int par = j & 1;
        if (idx != 0x7fffffffffffffffll && idx >= rbeg && idx < rend) {
            const int r = (int)(idx - rbeg);
            for (int c = threadIdx.x; c < nbp; c += blockDim.x) candb[par * nbp + c] = Ps[r + c * cp];
        }
        if (g >= rbeg && g < rend) {
            const int r = (int)(g - rbeg);
            for (int c = threadIdx.x; c < nbp; c += blockDim.x) diagb[par * nbp + c] = Ps[r + c * cp];
        }
        if (threadIdx.x == 0) { s_cv[par] = v; s_ci[par] = idx; }
    };
    {
        T v;
        long long idx;
        panel_local_argmax(Ps, cp, nr, rbeg, k0, 0, v, idx, sv, si, sdn);
        publish(0, v, idx);
    }
    unsigned long long info = ~0ull;
    for (int j = 0; j < nbp; ++j) {
        const int64_t g = k0 + j;
        const int par = j & 1;
        PHC(0);
        if (P > 1) cl.sync();                            // every candidate of column j is visible
        else __syncthreads();
        PHC(1);
        if (warp == 0) {
            T bv = T(-1);
            long long bi = 0x7fffffffffffffffll;
            int bo = 0;
            if (lane < P) {
                bv = *cl.map_shared_rank(&s_cv[par], lane);
                bi = *cl.map_shared_rank(&s_ci[par], lane);
                bo = lane;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const T v2 = __shfl_xor_sync(0xffffffffu, bv, o);
                const long long i2 = __shfl_xor_sync(0xffffffffu, bi, o);
                const int o2 = __shfl_xor_sync(0xffffffffu, bo, o);
                if (v2 > bv || (v2 == bv && i2 < bi)) { bv = v2; bi = i2; bo = o2; }
            }
            if (lane == 0) { s_p = bi; s_owner = bo; }
        }
        __syncthreads();
        const long long p = s_p;
        const int owner = s_owner;
        const int gown = (int)((g - k0) / chunk);
        const bool own_p = p != g && p >= rbeg && p < rend;
        const T* rc = cl.map_shared_rank(candb + par * nbp, owner);
        const T* rd = cl.map_shared_rank(diagb + par * nbp, gown);
        T* dst_p = own_p ? Ps + (p - rbeg) : nullptr;
        for (int c = threadIdx.x; c < nbp; c += blockDim.x) {
            const T u = rc[c];
            const T dg = own_p ? rd[c] : T(0);
            ubuf[c] = u;
            if (own_p) dst_p[c * cp] = dg;
        }
        __syncthreads();
        PHC(2);
        const T piv = ubuf[j];
        if (cta == 0 && threadIdx.x == 0) ipiv[g] = (p == 0x7fffffffffffffffll) ? g : p;
        const bool elim = piv != T(0);
        if (!elim) {
            if (info == ~0ull) info = (unsigned long long)(g + 1);
            if (own_p)
                for (int c = threadIdx.x; c < nbp; c += blockDim.x) dst_p[c * cp] = ubuf[c];
        } else if (g >= rbeg && g < rend) {
            const int r = (int)(g - rbeg);
            for (int c = threadIdx.x; c < nbp; c += blockDim.x) Ps[r + c * cp] = ubuf[c];
        }
        __syncthreads();
        const int64_t r0 = max<int64_t>(0, g + 1 - rbeg);
        if (elim) {
            const T u1 = (j + 1 < nbp) ? ubuf[j + 1] : T(0);
            for (int r = (int)r0 + threadIdx.x; r < nr; r += blockDim.x) {
                const T l = Ps[r + j * cp] / piv;
                Ps[r + j * cp] = l;
                if (j + 1 < nbp) Ps[r + (j + 1) * cp] -= l * u1;
            }
        }
        __syncthreads();
        PHC(3);
        if (j + 1 >= nbp) break;
        T v;
        long long idx;
        panel_local_argmax(Ps, cp, nr, rbeg, g + 1, j + 1, v, idx, sv, si, sdn);
        PHC(4);
        const int rcn = (idx != 0x7fffffffffffffffll && idx >= rbeg && idx < rend) ? (int)(idx - rbeg) : -1;
        const int rg = (g + 1 >= rbeg && g + 1 < rend) ? (int)(g + 1 - rbeg) : -1;
        if (elim) {
            for (int c = j + 2 + threadIdx.x; c < nbp; c += blockDim.x) {
                if (rcn >= 0) Ps[rcn + c * cp] -= Ps[rcn + j * cp] * ubuf[c];
                if (rg >= 0 && rg != rcn) Ps[rg + c * cp] -= Ps[rg + j * cp] * ubuf[c];
            }
        }
        __syncthreads();
        publish(j + 1, v, idx);
        PHC(5);
        if (elim) panel_bulk_update<T>(Ps, cp, ubuf, (int)r0, nr, j, nbp, rcn, rg);
        __syncthreads();
    }
    PHC(6);
#undef PHC
    if (prof)
        for (int q = 0; q < 8; ++q) st->dbg_t[q] = (unsigned long long)ph[q];
    cl.sync();                                           // no CTA exits while others may read its buffers
    for (int e = threadIdx.x; e < nr * nbp; e += blockDim.x) {
        const int c = e / nr, r = e - c * nr;
        W[(rbeg + r) + (k0 + c) * ldw] = Ps[r + c * cp];
    }
    if (threadIdx.x == 0 && cta == 0 && info != ~0ull) atomicMin(&st->info, info);
}

// ------------------------------------------------------------------ panel (leaf-blocked, one cluster)
// The panel's m rows are split over the P <= 16 CTAs of one thread-block cluster, RPT rows per
// thread (row tid + 256 i of the CTA's chunk).  The columns are factored in leaves of KLW columns
// held in REGISTERS (RPT x KLW = 64 values per thread); the rest of the panel stays in global
// memory (L2) and receives one deferred rank-KLW update per leaf.  Rows are kept ROTATED: at leaf
// step jj, a[i][k] holds leaf column (jj + k) mod KLW, so the current column is a[i][0], every
// register index is a compile-time constant and the column loop stays compact (not unrolled).
// Per column (first-max tie-break, Z15; a NaN diagonal keeps its row, as the serial sweep does):
//   warp argmax = fmax shuffle + ballot + integer min-reduction of the row index; the winning
//   lane stores its (rotated) row, the owner of row g its row g; ONE CTA barrier; every thread
//   merges the 8 warp results.  P > 1: each CTA's winner (value, index, row) -- and row g from
//   its owner -- is pushed into every CTA with st.async, which completes the receiver's mbarrier
//   transaction count: data and signal arrive together, no cluster barrier, no fence.
//   Then: swap of rows g and p (their owners), multipliers, rank-1 update in registers.
// Per leaf: the leaf's interchanges composed into one permutation of <= 2 KLW rows and applied to
// the panel's other columns; U12 = L11^{-1} A12 for the leaf's pivot rows; A22 -= L21 U12 for the
// rows below.  Result (rows interchanged within the panel, ipiv): the unblocked column sweep's up
// to rounding.
constexpr int kLfMaxP = 16;

template <typename T, int KLW>
struct LeafSmem {
    T rowbuf[2][1][KLW];                 // the CTA winner's row (rotated)
    T gbuf[2][KLW];                      // row g (rotated), CTA-local
    T crow[2][kLfMaxP][KLW];             // cluster: every CTA's candidate row
    T cgrow[2][KLW];                     // cluster: row g
    T Ub[KLW][KLW];                      // pivot rows of the leaf, natural column order
    T U12[KLW][kPW - KLW + 17];          // + padding (vector reads past the last column); odd row
                                         // stride: column accesses are bank-conflict free
    unsigned long long cvi[2][kLfMaxP][2];   // cluster: (value bits, index) per CTA
    unsigned long long mbar[2];
    T wval[2][kPT / 32];
    int widx[2][kPT / 32];
    int64_t s_piv[kPW];
    int64_t s_src[2 * KLW], s_dst[2 * KLW];
    int s_np;
};

template <typename T> AS_DEV unsigned long long t_bits(T v);
template <> AS_DEV unsigned long long t_bits<double>(double v) { return (unsigned long long)__double_as_longlong(v); }
template <> AS_DEV unsigned long long t_bits<float>(float v) { return (unsigned long long)__float_as_uint(v); }
template <typename T> AS_DEV T t_from(unsigned long long b);
template <> AS_DEV double t_from<double>(unsigned long long b) { return __longlong_as_double((long long)b); }
template <> AS_DEV float t_from<float>(unsigned long long b) { return __uint_as_float((unsigned)b); }
template <typename T>
AS_DEV void push_elem(const T* local_dst, unsigned rank, T v, unsigned rbar) {
    const unsigned ra = mapa_u32(smem_u32(local_dst), rank);
    if (sizeof(T) == 8) st_async_b64(ra, t_bits<T>(v), rbar);
    else st_async_b32(ra, (unsigned)t_bits<T>(v), rbar);
}

template <typename T, int RPT, int KLW>
__global__ void __launch_bounds__(kPT, 1) lu_panel_fast_kernel(T* W, int64_t ldw, int64_t n, int64_t k0, int nbp,
                                                                int64_t* ipiv, DevState* st, unsigned long long* tr_min,
                                                                unsigned long long* tr_max, int dbg) {
    cg::cluster_group cl = cg::this_cluster();
    if (tr_min && threadIdx.x == 0) atomicMin(tr_min, gtimer());
    const int P = (int)cl.num_blocks(), cta = (int)cl.block_rank();
    const int64_t m = n - k0;
    const int64_t chunk = (m + P - 1) / P;
    const int64_t rbeg = k0 + (int64_t)cta * chunk;
    const int64_t rend = min(n, rbeg + chunk);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    LeafSmem<T, KLW>& S = *reinterpret_cast<LeafSmem<T, KLW>*>(smem_raw);
    constexpr int URW = kPW - KLW + 17;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int kNone = 0x7fffffff;        // row positions fit in int (n <= 2^31 - 1)
    int gr[RPT];
#pragma unroll
    for (int i = 0; i < RPT; ++i) gr[i] = (rbeg + tid + (int64_t)kPT * i < rend) ? (int)(rbeg + tid + (int64_t)kPT * i) : -1;
    T a[RPT][KLW];
    auto cbar = [&]() {
        if (P > 1) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
        else __syncthreads();
    };
    if (P > 1) {
        if (tid == 0) { mbar_init(&S.mbar[0], 1); mbar_init(&S.mbar[1], 1); mbar_fence_init_cluster(); }
        cbar();
    }
    // local first-max over my rows at positions >= gmin for the current (rotated) column
    auto local_cand = [&](int gmin, T& lv, int& li) {
        lv = T(-1);
        li = kNone;
        bool dn = false;
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
            if (gr[i] >= gmin) {
                T x = a[i][0];
                x = x < T(0) ? -x : x;
                if (gr[i] == gmin && x != x) dn = true;
                if (x > lv) { lv = x; li = gr[i]; }      // rows increase with i: strict > keeps the first
            }
        }
        if (dn) { lv = T(INFINITY); li = gmin; }
    };

    unsigned long long info = ~0ull;
    int uses = 0;                             // columns processed (mbarrier phase bookkeeping)
    for (int c0 = 0; c0 < nbp; c0 += KLW) {
        const int w = min(KLW, nbp - c0);
        const int g0 = (int)(k0 + c0);
#pragma unroll
        for (int c = 0; c < KLW; ++c)
#pragma unroll
            for (int i = 0; i < RPT; ++i)
                a[i][c] = (gr[i] >= g0 && c < w) ? W[gr[i] + (k0 + c0 + c) * ldw] : T(0);
        T lv;
        int li;
        local_cand(g0, lv, li);
        if ((dbg & 8) && tid < w) S.s_piv[c0 + tid] = g0 + tid;   // ablation: no interchanges
        for (int jj = 0; jj < (dbg & 8 ? 0 : w); ++jj, ++uses) {
            const int c = c0 + jj;
            const int g = (int)(k0 + c);
            const int par = uses & 1;
            // ---- warp argmax: value by fmax shuffles, index by ballot + min-reduction
            T wm = lv;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) wm = fmax(wm, __shfl_xor_sync(0xffffffffu, wm, o));
            const unsigned wi = __reduce_min_sync(0xffffffffu, (lv == wm && li != kNone) ? (unsigned)li : (unsigned)kNone);
            if (lane == 0) { S.wval[par][warp] = wi == (unsigned)kNone ? T(-1) : wm; S.widx[par][warp] = (int)wi; }
            __syncthreads();
            // ---- CTA winner (every thread); its owner stores the row, the owner of g row g
            // (warp-uniform branches: only the owners' warps execute the row copies)
            T cv = T(-1);
            int ci = kNone;
#pragma unroll
            for (int q = 0; q < kPT / 32; ++q) {
                const T v = S.wval[par][q];
                const int ix = S.widx[par][q];
                if (v > cv || (v == cv && ix < ci)) { cv = v; ci = ix; }
            }
            const int cw = 0;
            {
                const int wc = (ci != kNone) ? (int)(((int64_t)ci - rbeg) & (kPT - 1)) >> 5 : -1;
                const int wg = (g >= rbeg && g < rend) ? (int)(((int64_t)g - rbeg) & (kPT - 1)) >> 5 : -1;
                if (warp == wc) {
#pragma unroll
                    for (int i = 0; i < RPT; ++i)
                        if (gr[i] == ci)
#pragma unroll
                            for (int k = 0; k < KLW; ++k) S.rowbuf[par][0][k] = a[i][k];
                }
                if (warp == wg) {
#pragma unroll
                    for (int i = 0; i < RPT; ++i)
                        if (gr[i] == g)
#pragma unroll
                            for (int k = 0; k < KLW; ++k) S.gbuf[par][k] = a[i][k];
                }
            }
            __syncthreads();
            int p = ci;
            const T* prow = &S.rowbuf[par][cw][0];
            const T* grw = &S.gbuf[par][0];
            if (P > 1) {
                // ---- cluster exchange: push (value, index, row) and row g into every CTA
                const unsigned bar_l = smem_u32(&S.mbar[par]);
                if (warp == 0) {
                    for (int e = lane; e < P * (KLW + 2); e += 32) {
                        const int q = e / (KLW + 2), k = e - q * (KLW + 2);
                        const unsigned rb = mapa_u32(bar_l, q);
                        if (k < KLW) push_elem<T>(&S.crow[par][cta][k], q, S.rowbuf[par][cw][k], rb);
                        else if (k == KLW) st_async_b64(mapa_u32(smem_u32(&S.cvi[par][cta][0]), q), t_bits<double>((double)cv), rb);
                        else st_async_b64(mapa_u32(smem_u32(&S.cvi[par][cta][1]), q), (unsigned long long)(unsigned)ci, rb);
                    }
                } else if (warp == 1 && g >= rbeg && g < rend) {
                    for (int e = lane; e < P * KLW; e += 32) {
                        const int q = e / KLW, k = e - q * KLW;
                        push_elem<T>(&S.cgrow[par][k], q, S.gbuf[par][k], mapa_u32(bar_l, q));
                    }
                }
                if (tid == 0) mbar_arrive_expect_tx(&S.mbar[par], (unsigned)(P * (KLW * sizeof(T) + 16) + KLW * sizeof(T)));
                const unsigned ph = (unsigned)((uses >> 1) & 1);
                while (!mbar_try_wait_cluster(&S.mbar[par], ph)) {}
                T bv = T(-1);
                int bi = kNone, bo = 0;
                for (int q = 0; q < P; ++q) {
                    const T v = (T)t_from<double>(S.cvi[par][q][0]);
                    const int ix = (int)(unsigned)S.cvi[par][q][1];
                    if (v > bv || (v == bv && ix < bi)) { bv = v; bi = ix; bo = q; }
                }
                p = bi;
                prow = &S.crow[par][bo][0];
                grw = &S.cgrow[par][0];
            }
            const T piv = prow[0];
            const bool elim = piv != T(0);
            if (tid < KLW) S.Ub[jj][(jj + tid) % KLW] = prow[tid];
            if (tid == 0) S.s_piv[c] = (p == kNone) ? g : p;
            if (!elim) {
                if (info == ~0ull) info = (unsigned long long)(g + 1);
            } else if (p != g) {
                const int wg = (g >= rbeg && g < rend) ? (int)(((int64_t)g - rbeg) & (kPT - 1)) >> 5 : -1;
                const int wp = (p >= rbeg && p < rend) ? (int)(((int64_t)p - rbeg) & (kPT - 1)) >> 5 : -1;
                if (warp == wg || warp == wp) {
#pragma unroll
                    for (int i = 0; i < RPT; ++i) {
                        if (gr[i] == g) {
#pragma unroll
                            for (int k = 0; k < KLW; ++k) a[i][k] = prow[k];
                        } else if (gr[i] == p) {
#pragma unroll
                            for (int k = 0; k < KLW; ++k) a[i][k] = grw[k];
                        }
                    }
                }
            }
            // ---- multipliers, rank-1 update (registers), rotation, next column's local candidate
            const int nlive = KLW - jj;
            T l[RPT];
#pragma unroll
            for (int i = 0; i < RPT; ++i) {
                const bool below = gr[i] > g && elim;
                l[i] = below ? a[i][0] / piv : T(0);
                if (below) a[i][0] = l[i];
            }
#pragma unroll
            for (int k = 1; k < KLW; ++k) {
                if (k < nlive) {
                    const T uk = prow[k];
#pragma unroll
                    for (int i = 0; i < RPT; ++i) a[i][k] -= l[i] * uk;
                }
            }
#pragma unroll
            for (int i = 0; i < RPT; ++i) {
                const T x0 = a[i][0];
#pragma unroll
                for (int k = 0; k < KLW - 1; ++k) a[i][k] = a[i][k + 1];
                a[i][KLW - 1] = x0;
            }
            local_cand(g + 1, lv, li);
        }
        // short leaf: finish the rotation so that a[.][c] is leaf column c again
        if (w < KLW && !(dbg & 8))
            for (int r = w; r < KLW; ++r)
#pragma unroll
                for (int i = 0; i < RPT; ++i) {
                    const T x0 = a[i][0];
#pragma unroll
                    for (int k = 0; k < KLW - 1; ++k) a[i][k] = a[i][k + 1];
                    a[i][KLW - 1] = x0;
                }
        // ---- leaf end: write back, pivots, the leaf's interchanges on the panel's other columns
#pragma unroll
        for (int cc = 0; cc < KLW; ++cc)
#pragma unroll
            for (int i = 0; i < RPT; ++i)
                if (gr[i] >= g0 && cc < w) W[gr[i] + (k0 + c0 + cc) * ldw] = a[i][cc];
        __syncthreads();
        if (cta == 0 && tid < w) ipiv[g0 + tid] = S.s_piv[c0 + tid];
        if (tid == 0) S.s_np = 0;
        __syncthreads();
        if (tid < 2 * w) {
            const int t = tid;
            int64_t x = 0;
            bool go = true;
            if (t < w) x = g0 + t;
            else {
                x = S.s_piv[c0 + t - w];
                if (x < g0 + w) go = false;
                for (int q = 0; q < t - w && go; ++q) go = S.s_piv[c0 + q] != x;
            }
            if (go) {
                int64_t pos = x;
                for (int q = 0; q < w; ++q) {
                    const int64_t r = g0 + q, tq = S.s_piv[c0 + q];
                    if (pos == r) pos = tq;
                    else if (pos == tq) pos = r;
                }
                if (pos != x) {
                    const int k = atomicAdd(&S.s_np, 1);
                    S.s_dst[k] = pos;
                    S.s_src[k] = x;
                }
            }
        }
        __syncthreads();
        {
            // a warp per column, every gather issued before any scatter; <= 2 KLW moved rows
            const int np = S.s_np;
            const int nother = nbp - w;
            constexpr int kPer = (2 * KLW + 31) / 32;
            int64_t src[kPer], dst[kPer];
#pragma unroll
            for (int u = 0; u < kPer; ++u) {
                const int k = lane + 32 * u;
                src[u] = k < np ? S.s_src[k] : 0;
                dst[u] = k < np ? S.s_dst[k] : 0;
            }
            constexpr int kCW = kPer > 2 ? 4 : 8;
            const int nw = P * (kPT / 32), w0 = cta * (kPT / 32) + warp;
            for (int t0 = 0; t0 < (dbg & 1 ? 0 : nother); t0 += nw * kCW) {
                T vv[kCW][kPer];
#pragma unroll
                for (int uu = 0; uu < kCW; ++uu) {
                    const int t = t0 + w0 + uu * nw;
                    const int col = t < c0 ? t : t + w;
#pragma unroll
                    for (int u = 0; u < kPer; ++u)
                        vv[uu][u] = (lane + 32 * u < np && t < nother) ? W[src[u] + (k0 + col) * ldw] : T(0);
                }
#pragma unroll
                for (int uu = 0; uu < kCW; ++uu) {
                    const int t = t0 + w0 + uu * nw;
                    const int col = t < c0 ? t : t + w;
#pragma unroll
                    for (int u = 0; u < kPer; ++u)
                        if (lane + 32 * u < np && t < nother) W[dst[u] + (k0 + col) * ldw] = vv[uu][u];
                }
            }
        }
        cbar();
        // ---- deferred update of the rest of the panel
        if (c0 + w < nbp && !(dbg & 2)) {
            const int c1 = c0 + w, rw = nbp - c1;
            batched<8, T>(
                KLW * rw, [&](int e) -> T { const int k = e % KLW, cc = e / KLW; return __ldcg(&W[(g0 + k) + (k0 + c1 + cc) * ldw]); },
                [&](int e, T v) { const int k = e % KLW, cc = e / KLW; S.U12[k][cc] = v; });
            __syncthreads();
            // U12 = L11^{-1} A12 (unit lower L11 = Ub) in column-oriented (axpy) form: step k
            // updates rows k+1.. of every column in parallel (a per-column serial sweep would be a
            // chain of KLW^2/2 dependent shared-memory loads)
            for (int k = 0; k + 1 < KLW; ++k) {
                const int nrow = KLW - 1 - k;
                for (int e = tid; e < nrow * rw; e += kPT) {
                    const int i2 = k + 1 + e % nrow, cc = e / nrow;
                    S.U12[i2][cc] -= S.Ub[i2][k] * S.U12[k][cc];
                }
                __syncthreads();
            }
            for (int e = tid; e < KLW * rw; e += kPT) {
                const int k = e % KLW, cc = e / KLW;
                const int64_t rk = g0 + k;
                if (rk >= rbeg && rk < rend) W[rk + (k0 + c1 + cc) * ldw] = S.U12[k][cc];
            }
            // A22 -= L21 U12 on my rows below the leaf (L21 = the leaf values in registers); batches
            // of kQ columns with the next batch's loads in flight
            constexpr int kQ = RPT >= 4 ? 2 : RPT >= 2 ? 4 : 4;
            const int lim = g0 + w;
            T nx[RPT][kQ];
            auto load = [&](int cb) {
#pragma unroll
                for (int q = 0; q < kQ; ++q)
#pragma unroll
                    for (int i = 0; i < RPT; ++i)
                        nx[i][q] = (gr[i] >= lim && cb + q < rw) ? W[gr[i] + (k0 + c1 + cb + q) * ldw] : T(0);
            };
            load(0);
            for (int cb = 0; cb < rw; cb += kQ) {
                T acc[RPT][kQ];
#pragma unroll
                for (int q = 0; q < kQ; ++q)
#pragma unroll
                    for (int i = 0; i < RPT; ++i) acc[i][q] = nx[i][q];
                if (cb + kQ < rw) load(cb + kQ);
#pragma unroll
                for (int k = 0; k < KLW; ++k) {
                    T uu[kQ];
#pragma unroll
                    for (int q = 0; q < kQ; ++q) uu[q] = S.U12[k][cb + q];
#pragma unroll
                    for (int i = 0; i < RPT; ++i)
#pragma unroll
                        for (int q = 0; q < kQ; ++q) acc[i][q] -= a[i][k] * uu[q];
                }
#pragma unroll
                for (int q = 0; q < kQ; ++q)
#pragma unroll
                    for (int i = 0; i < RPT; ++i)
                        if (gr[i] >= lim && cb + q < rw) W[gr[i] + (k0 + c1 + cb + q) * ldw] = acc[i][q];
            }
            __syncthreads();
        }
    }
    (void)URW;
    if (P > 1) cbar();                       // no CTA leaves while remote stores may target it
    if (tid == 0 && cta == 0 && info != ~0ull) atomicMin(&st->info, info);
    if (tr_max && tid == 0) atomicMax(tr_max, gtimer());
}

// ------------------------------------------------------------------ laswp
// Apply the interchanges ipiv[j0 .. j0+cnt) (in order) to columns [a0, a1) U [b0, b1) and, if
// perm != nullptr, to perm.  The cnt swaps compose into one permutation of the row set
// S = [j0, j0+cnt) U {ipiv targets}: every CTA first tracks the final position of each row of S
// through the swap sequence (one thread per row, in parallel), then one warp per column gathers
// all moved values and scatters them to their final rows -- independent accesses instead of
// cnt dependent swaps per column (column-major rows are 8-byte strided accesses either way).
constexpr int kSwapMax = 2 * kBW;
template <typename T>
__global__ void __launch_bounds__(256) laswp3_kernel(T* W, int64_t ldw, int64_t j0, int cnt, int64_t a0, int64_t a1,
                                                     int64_t b0, int64_t b1, const int64_t* ipiv, int64_t* perm) {
    __shared__ int64_t piv[kBW];
    __shared__ int64_t dst[kSwapMax], src[kSwapMax];
    __shared__ int s_np;
    if (threadIdx.x == 0) s_np = 0;
    for (int q = threadIdx.x; q < cnt; q += blockDim.x) piv[q] = ipiv[j0 + q];
    __syncthreads();
    for (int t = threadIdx.x; t < 2 * cnt; t += blockDim.x) {
        int64_t x;
        if (t < cnt) x = j0 + t;
        else {
            x = piv[t - cnt];
            if (x < j0 + cnt) continue;                       // already tracked as a block row
            bool first = true;                                // one thread per distinct external row
            for (int q = 0; q < t - cnt; ++q) first = first && (piv[q] != x);
            if (!first) continue;
        }
        int64_t pos = x;
        for (int q = 0; q < cnt; ++q) {
            const int64_t r = j0 + q, tq = piv[q];
            if (pos == r) pos = tq;
            else if (pos == tq) pos = r;
        }
        if (pos != x) {
            const int k = atomicAdd(&s_np, 1);
            dst[k] = pos;
            src[k] = x;
        }
    }
    __syncthreads();
    const int np = s_np;
    const int lane = threadIdx.x & 31;
    const int64_t na = max<int64_t>(0, a1 - a0), nb = max<int64_t>(0, b1 - b0);
    const int64_t ncols = na + nb + (perm ? 1 : 0);
    const int64_t wid = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    constexpr int kPer = kSwapMax / 32;
    for (int64_t t = wid; t < ncols; t += nw) {
        if (perm && t == ncols - 1) {
            int64_t v[kPer];
#pragma unroll
            for (int u = 0; u < kPer; ++u) { const int k = lane + 32 * u; if (k < np) v[u] = perm[src[k]]; }
            __syncwarp();
#pragma unroll
            for (int u = 0; u < kPer; ++u) { const int k = lane + 32 * u; if (k < np) perm[dst[k]] = v[u]; }
            continue;
        }
        const int64_t col = t < na ? a0 + t : b0 + (t - na);
        T* c = W + col * ldw;
        T v[kPer];
#pragma unroll
        for (int u = 0; u < kPer; ++u) { const int k = lane + 32 * u; if (k < np) v[u] = c[src[k]]; }
        __syncwarp();
#pragma unroll
        for (int u = 0; u < kPer; ++u) { const int k = lane + 32 * u; if (k < np) c[dst[k]] = v[u]; }
    }
}

// ------------------------------------------------------------------ L11^{-1}, U12 = L11^{-1} A12
// Inverse of the panel's unit-lower diagonal block (rows / columns k0 .. k0+nbp) into its Dinv0
// slot: the U12 product below and the final GETRS / GECON forward substitutions use it.  Later
// interchanges only move rows below the panel, so the block is final once the panel is.
template <typename T>
__global__ void __launch_bounds__(256) lu_linv_kernel(const T* W, int64_t ldw, int64_t k0b, int nbpb, T* Dinv) {
    // CTA h inverts the diagonal 64 x 64 block of rows k0b + 64 h .. of the panel
    const int64_t k0 = k0b + (int64_t)blockIdx.x * kB64;
    const int nbp = min(kB64, nbpb - (int)blockIdx.x * kB64);
    if (nbp <= 0) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* L = (T*)smem_raw;
    T* X = L + kB64 * kB64LD;
    T* tmp = X + kB64 * kB64LD;
    batched<8, T>(
        kB64 * kB64,
        [&](int e) -> T {
            const int r = e & 63, c = e >> 6;
            return (r > c && r < nbp) ? W[(k0 + r) + (k0 + c) * ldw] : T(0);
        },
        [&](int e, T v) { L[(e & 63) + (e >> 6) * kB64LD] = v; });
    __syncthreads();
    block_trinv64<T, true>(L, X, tmp);
    T* D = Dinv + (k0 / kB64) * (int64_t)kB64 * kB64;
    for (int e = threadIdx.x; e < kB64 * kB64; e += blockDim.x) D[e] = X[(e & 63) + (e >> 6) * kB64LD];
}

// ------------------------------------------------------------------ fused interchanges + U12
// For the trailing columns [c0, c1) of block k0 (bw <= 128 rows, one CTA per 32 columns):
//   1. the block's bw interchanges, composed into a permutation of S = block rows U targets
//      (each row of S tracked through the swap sequence in parallel, as in laswp3);
//   2. every moved value gathered from its source row before any is written;
//   3. U12 = L11^{-1} A12 on the new block rows with L11 = [La 0; Lb Lc] in 64-row halves:
//      Utop = La^{-1} Atop, Abot -= Lb Utop, Ubot = Lc^{-1} Abot (La^{-1}, Lc^{-1}: Dinv0).
// This replaces laswp + u12 + gemm + u12 on the critical path between two panels.
constexpr int kSUC = 32;
constexpr int kSULD = kBW + 1;           // column stride of the column-major row buffers
template <typename T>
__global__ void __launch_bounds__(256) swap_u12_kernel(T* W, int64_t ldw, int64_t k0, int bw, int64_t c0, int64_t c1,
                                                      const int64_t* ipiv, const T* Dinv) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* AiT = (T*)smem_raw;               // La^{-1} column-major (element (r, k) at r + 64 k)
    T* LbT = AiT + kB64 * kB64;          // Lb
    T* CiT = LbT + kB64 * kB64;          // Lc^{-1}
    T* Bn = CiT + kB64 * kB64;           // [kSUC][kSULD]: column c of the block rows after the interchanges
    T* Ex = Bn + kSUC * kSULD;           // [kSUC][kSULD]: values for the rows leaving the block
    __shared__ int64_t piv[kBW];
    __shared__ int64_t srow[2 * kBW];    // source rows: block positions 0..bw-1, then leaving rows
    __shared__ int64_t edst[kBW];
    __shared__ int s_ne;
    const int64_t cc0 = c0 + (int64_t)blockIdx.x * kSUC;
    const int nc = (int)min<int64_t>(kSUC, c1 - cc0);
    if (nc <= 0) return;
    const int p1 = min(kB64, bw), p2 = bw - p1;
    if (threadIdx.x == 0) s_ne = 0;
    for (int q = threadIdx.x; q < bw; q += blockDim.x) piv[q] = ipiv[k0 + q];
    __syncthreads();
    for (int t = threadIdx.x; t < 2 * bw; t += blockDim.x) {
        int64_t x;
        if (t < bw) x = k0 + t;
        else {
            x = piv[t - bw];
            if (x < k0 + bw) continue;
            bool first = true;
            for (int q = 0; q < t - bw; ++q) first = first && (piv[q] != x);
            if (!first) continue;
        }
        int64_t pos = x;
        for (int q = 0; q < bw; ++q) {
            const int64_t r = k0 + q, tq = piv[q];
            if (pos == r) pos = tq;
            else if (pos == tq) pos = r;
        }
        if (pos < k0 + bw) srow[pos - k0] = x;
        else { const int e = atomicAdd(&s_ne, 1); edst[e] = pos; srow[bw + e] = x; }
    }
    for (int e = threadIdx.x; e < kSUC * kSULD; e += blockDim.x) Bn[e] = T(0);   // short blocks / columns
    __syncthreads();
    const int ne = s_ne, R = bw + ne;
    // every source value before any store: consecutive threads read consecutive (mostly
    // contiguous) source rows of one column; then the triangular blocks (contiguous copies)
    batched<16, T>(
        R * nc + 3 * kB64 * kB64,
        [&](int e) -> T {
            if (e < R * nc) {
                const int c = e / R, row = e - c * R;
                return W[srow[row] + (cc0 + c) * ldw];
            }
            const int f = e - R * nc, which = f >> 12, g = f & 4095, r = g & 63, k = g >> 6;
            if (which == 0) return Dinv[(k0 / kB64) * (int64_t)kB64 * kB64 + g];
            if (p2 <= 0) return T(0);
            if (which == 1) return (r < p2) ? W[(k0 + kB64 + r) + (k0 + k) * ldw] : T(0);
            return Dinv[(k0 / kB64 + 1) * (int64_t)kB64 * kB64 + g];
        },
        [&](int e, T v) {
            if (e < R * nc) {
                const int c = e / R, row = e - c * R;
                if (row < bw) Bn[c * kSULD + row] = v;
                else Ex[c * kSULD + row - bw] = v;
            } else {
                AiT[e - R * nc] = v;                       // AiT, LbT, CiT are contiguous
            }
        });
    __syncthreads();
    // rows leaving the block
    for (int e = threadIdx.x; e < ne * nc; e += blockDim.x) {
        const int c = e / ne, row = e - c * ne;
        W[edst[row] + (cc0 + c) * ldw] = Ex[c * kSULD + row];
    }
    // thread = (row r, 8-column group g)
    const int r = threadIdx.x & 63, g = threadIdx.x >> 6;
    auto prod = [&](const T* M, int roff, T (&acc)[8]) {   // acc = M(r, :) * Bn[roff + :, g*8 ..]
#pragma unroll
        for (int u = 0; u < 8; ++u) acc[u] = T(0);
#pragma unroll 4
        for (int k = 0; k < kB64; ++k) {
            const T m = M[r + k * kB64];
#pragma unroll
            for (int u = 0; u < 8; ++u) acc[u] += m * Bn[(g * 8 + u) * kSULD + roff + k];
        }
    };
    T acc[8];
    prod(AiT, 0, acc);                                     // Utop = La^{-1} Atop
    __syncthreads();
    if (r < p1)
#pragma unroll
        for (int u = 0; u < 8; ++u) Bn[(g * 8 + u) * kSULD + r] = acc[u];
    __syncthreads();
    if (p2 > 0) {
        prod(LbT, 0, acc);                                 // Abot -= Lb Utop
        if (r < p2)
#pragma unroll
            for (int u = 0; u < 8; ++u) Bn[(g * 8 + u) * kSULD + kB64 + r] -= acc[u];
        __syncthreads();
        prod(CiT, kB64, acc);                              // Ubot = Lc^{-1} Abot
        __syncthreads();
        if (r < p2)
#pragma unroll
            for (int u = 0; u < 8; ++u) Bn[(g * 8 + u) * kSULD + kB64 + r] = acc[u];
        __syncthreads();
    }
    for (int e = threadIdx.x; e < bw * nc; e += blockDim.x) {
        const int c = e / bw, row = e - c * bw;
        W[(k0 + row) + (cc0 + c) * ldw] = Bn[c * kSULD + row];
    }
}
// ------------------------------------------------------------------ small n: one-cluster LU
// xGETRF for n <= kSmN (C1) in ONE launch: a cluster of P = ceil(n/64) CTAs, CTA c owns the
// column block [64c, 64c+64).  512 threads: thread (r, h) = row r, columns 32h .. 32h+31 of the
// block.  Per panel b (the paper's blocked GETRF order):
//   owner CTA b   its block in shared memory, factored 8 columns at a time (xGETF2 inside the
//                 group: first-max |.| pivot search by warp shuffles + one CTA barrier, the row
//                 interchange, multipliers and rank-1 steps on the group's columns held in
//                 registers; then the group's U12 rows by a column-parallel unit-lower solve and
//                 a rank-8 update of the rest of the block, pivot rows as broadcast reads); the
//                 block stays in shared memory and goes to W for the later CTAs;
//   cluster barrier
//   CTAs c > b    rows in registers: panel b's 64 interchanges as one permutation through shared
//                 memory, their own row of L_b read from W (the owner writes its block there
//                 before the cluster barrier; pivots come over DSMEM), then 8 groups of 8 rows:
//                 U12 rows by a column-parallel unit-lower solve, rank-8 update of the rows below
//                 (U12 = L11^{-1} A12, A22 -= L21 U12; two CTA barriers per group).
// At the end every CTA applies the interchanges of later panels while writing its rows to W
// (LAPACK's convention: all interchanges applied to all columns), CTA 0 writes the row
// permutation.  No grid-wide exchange, no intermediate launches: C1's factorization was ~0.7 ms
// of panel launches with one cross-CTA exchange per column.
constexpr int kSmN = 256;        // rows
constexpr int kSmT = 512;        // threads: two per row
constexpr int kSmC = 64;         // columns per CTA
constexpr int kSmH = 32;         // columns per thread in the update phase
template <typename T>
__global__ void __launch_bounds__(kSmT, 1) lu_small_kernel(T* W, int64_t ldw, int n, int64_t* ipiv, int64_t* perm,
                                                           DevState* st, int prof) {
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* Lb = (T*)smem_raw;                           // [kSmC][kSmN]: L_b copy (update) / own block (owner)
    T* ub = Lb + kSmC * kSmN;                       // [2][kSmC] pivot row (update phase)
    T* xb = ub + 2 * kSmC;                          // [2][8][8] candidate rows, [2][8] row g (group columns),
                                                    // then at xb + 272: [2][8][kSmC] U12 rows of the update groups
    __shared__ unsigned s_kh[2][kSmN / 32], s_kl[2][kSmN / 32], s_ki[2][kSmN / 32];   // warp argmax keys
    __shared__ int s_piv[kSmC];                     // this CTA's pivots (read by later CTAs)
    __shared__ int s_pb[kSmC];                      // pivots of the panel being applied
    __shared__ int s_all[kSmN];                     // all pivots (write-out)
    const int c = (int)cl.block_rank(), P = (int)cl.num_blocks();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int r = tid & (kSmN - 1), h = tid >> 8, hc = kSmH * h;
    const int cb = kSmC * c, nc = min(kSmC, n - cb);
    const bool row_ok = r < n;
#define SMPROF(slot)                                                                   \
    if (prof == 2 && tid == 0 && c == 1) {                                             \
        unsigned long long t_;                                                         \
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                         \
        st->dbg_t[slot] = t_;                                                          \
    }
    T a[kSmH];
#pragma unroll
    for (int i = 0; i < kSmH; ++i) a[i] = (row_ok && hc + i < nc) ? W[r + (int64_t)(cb + hc + i) * ldw] : T(0);
    unsigned long long info = ~0ull;

    // (the three phases as separate loops: the row registers are dead after the owner phase)
    for (int b = 0; b < c; ++b) {
        cl.sync();                                   // panel b (pivots + L_b) visible to the cluster
        {
            // ---- panel b's interchanges as one permutation of this block's rows
            SMPROF(0);
            const int* pr = cl.map_shared_rank(s_piv, b);
            if (tid < kSmC) s_pb[tid] = pr[tid];
            __syncthreads();
            const int g0 = kSmC * b;
            int dest = r;
            for (int k = 0; k < kSmC; ++k) {
                const int g = g0 + k, p = s_pb[k];
                if (dest == g) dest = p;
                else if (dest == p) dest = g;
            }
#pragma unroll
            for (int i = 0; i < kSmH; ++i) Lb[dest + (hc + i) * kSmN] = a[i];
            __syncthreads();
#pragma unroll
            for (int i = 0; i < kSmH; ++i) a[i] = Lb[r + (hc + i) * kSmN];
            __syncthreads();
            SMPROF(1);
            // ---- rows of L_b (final order now): thread (r, h) copies columns hc .. hc+31
            const T* Lr = W + (int64_t)kSmC * b * ldw;        // owner b's block, written before its barrier
            if (r > g0 && row_ok) {
                // all loads of a batch before its stores
#pragma unroll
                for (int i0 = 0; i0 < kSmH; i0 += 16) {
                    T tmp[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) tmp[i] = __ldcg(Lr + r + (int64_t)(hc + i0 + i) * ldw);
#pragma unroll
                    for (int i = 0; i < 16; ++i) Lb[r + (hc + i0 + i) * kSmN] = tmp[i];
                }
            }
            // ---- 8 groups of 8 rows: the group's U12 rows by a column-parallel unit-lower solve
            // (staged in shared memory), then a rank-8 update of the rows below (two barriers per
            // group instead of one per row)
            SMPROF(2);
            for (int k0 = 0; k0 < kSmC; k0 += 8) {
                const int gg = g0 + k0;
                T* U8 = xb + 272 + ((k0 >> 3) & 1) * (8 * kSmC);   // [8][kSmC], double-buffered
                const bool in_grp = r >= gg && r < gg + 8;
                if (in_grp) {
#pragma unroll
                    for (int i = 0; i < kSmH; ++i) U8[(r - gg) * kSmC + hc + i] = a[i];
                }
                __syncthreads();
                if (tid < kSmC) {
                    T u[8];
#pragma unroll
                    for (int t = 0; t < 8; ++t) {
                        T x = U8[t * kSmC + tid];
#pragma unroll
                        for (int s2 = 0; s2 < t; ++s2) x -= Lb[(gg + t) + (k0 + s2) * kSmN] * u[s2];
                        u[t] = x;
                        U8[t * kSmC + tid] = x;
                    }
                }
                __syncthreads();
                if (in_grp) {
#pragma unroll
                    for (int i = 0; i < kSmH; ++i) a[i] = U8[(r - gg) * kSmC + hc + i];
                } else if (r >= gg + 8 && row_ok) {
                    T lq[8];
#pragma unroll
                    for (int t = 0; t < 8; ++t) lq[t] = Lb[r + (k0 + t) * kSmN];
#pragma unroll
                    for (int t = 0; t < 8; ++t)
#pragma unroll
                        for (int i = 0; i < kSmH; ++i) a[i] -= lq[t] * U8[t * kSmC + hc + i];
                }
            }
            __syncthreads();
        }
        if (prof == 1 && tid == 0 && c < 4 && b < 4) {   // diagnostics: %globaltimer at the end of step b
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            st->dbg_t[4 * c + b] = t;
        }
    }
    {
        const int b = c;
        {
#pragma unroll
            for (int i = 0; i < kSmH; ++i) Lb[r + (hc + i) * kSmN] = a[i];
            __syncthreads();
            SMPROF(3);
            for (int j0 = 0; j0 < nc; j0 += 8) {
                if (j0 == 8) SMPROF(4);
                T q[8];
                if (h == 0) {
#pragma unroll
                    for (int t = 0; t < 8; ++t) q[t] = (j0 + t < nc) ? Lb[r + (j0 + t) * kSmN] : T(0);
                }
#pragma unroll
                for (int t = 0; t < 8; ++t) {
                    const int j = j0 + t;
                    if (j >= nc) break;
                    const int g = cb + j, par = j & 1;
                    // first-max argmax (Z15) by integer warp reductions on an order-preserving key of
                    // |a| (hi word + 1, lo word; 0 = no candidate), then the smallest row among the
                    // maxima; NaN never wins
                    unsigned kh = 0u, kl = 0u;
                    if (h == 0 && r >= g && row_ok) {
                        T x = q[t] < T(0) ? -q[t] : q[t];
                        if (x == x) {
                            if (x == T(0)) x = T(0);                // -0 -> +0
                            cand_key(x, kh, kl);
                        }
                    }
                    unsigned mh = __reduce_max_sync(0xffffffffu, kh);
                    unsigned ml = __reduce_max_sync(0xffffffffu, kh == mh ? kl : 0u);
                    unsigned mi = __reduce_min_sync(0xffffffffu, (mh != 0u && kh == mh && kl == ml) ? (unsigned)r : 0x7fffffffu);
                    // one barrier per column: the warp winner publishes its group row with its
                    // candidate, row g publishes itself (the displaced row when p != g)
                    T* CR = xb + par * 64;                      // [8 warps][8]: candidate rows
                    T* Yr = xb + 128 + par * 8;                 // row g, group columns
                    if (h == 0 && mi == (unsigned)r) {
#pragma unroll
                        for (int s2 = 0; s2 < 8; ++s2) CR[warp * 8 + s2] = q[s2];
                    }
                    if (h == 0 && r == g) {
#pragma unroll
                        for (int s2 = 0; s2 < 8; ++s2) Yr[s2] = q[s2];
                    }
                    if (lane == 0 && h == 0) { s_kh[par][warp] = mh; s_kl[par][warp] = ml; s_ki[par][warp] = mi; }
                    __syncthreads();
                    kh = lane < kSmN / 32 ? s_kh[par][lane] : 0u;
                    kl = lane < kSmN / 32 ? s_kl[par][lane] : 0u;
                    const unsigned ki = lane < kSmN / 32 ? s_ki[par][lane] : 0x7fffffffu;
                    mh = __reduce_max_sync(0xffffffffu, kh);
                    ml = __reduce_max_sync(0xffffffffu, kh == mh ? kl : 0u);
                    mi = __reduce_min_sync(0xffffffffu, (mh != 0u && kh == mh && kl == ml) ? ki : 0x7fffffffu);
                    const int ri = (int)mi;
                    const int wb = ri >> 5;                     // rows of the h = 0 warps: r = tid
                    const int p = (ri == 0x7fffffff) ? g : ri;
                    const T* X = (ri == 0x7fffffff) ? Yr : CR + wb * 8;   // pivot row, group columns
                    if (p != g && tid < kSmC && (tid < j0 || tid >= j0 + 8)) {   // the other columns, in shared memory
                        const T tt = Lb[g + tid * kSmN];
                        Lb[g + tid * kSmN] = Lb[p + tid * kSmN];
                        Lb[p + tid * kSmN] = tt;
                    }
                    if (tid == 0) s_piv[j] = p;                 // (ipiv is written after the block)
                    if (h == 0) {
                        if (p != g) {
                            if (r == g) {
#pragma unroll
                                for (int s2 = 0; s2 < 8; ++s2) q[s2] = X[s2];
                            } else if (r == p) {
#pragma unroll
                                for (int s2 = 0; s2 < 8; ++s2) q[s2] = Yr[s2];
                            }
                        }
                        const T pv = X[t];
                        if (pv == T(0)) {
                            if (info == ~0ull) info = (unsigned long long)(g + 1);   // exact zero pivot: singular
                        } else if (r > g && row_ok) {
                            const T l = q[t] / pv;
                            q[t] = l;
#pragma unroll
                            for (int s2 = t + 1; s2 < 8; ++s2) q[s2] -= l * X[s2];
                        }
                    }
                }
                if (h == 0) {
#pragma unroll
                    for (int t = 0; t < 8; ++t)
                        if (j0 + t < nc) Lb[r + (j0 + t) * kSmN] = q[t];
                }
                if (j0 == 8) SMPROF(5);
                const int j1 = min(j0 + 8, nc);
                if (j1 >= nc) break;
                __syncthreads();
                if (j0 == 8) SMPROF(6);
                // U12 rows g0 .. g0+7 of columns j1..nc-1: unit-lower solve, one thread per column
                const int g0 = cb + j0;
                if (tid >= j1 && tid < nc) {
                    T u[8];
#pragma unroll
                    for (int t = 0; t < 8; ++t) {
                        T x = Lb[(g0 + t) + tid * kSmN];
#pragma unroll
                        for (int s2 = 0; s2 < t; ++s2) x -= Lb[(g0 + t) + (j0 + s2) * kSmN] * u[s2];
                        u[t] = x;
                        Lb[(g0 + t) + tid * kSmN] = x;
                    }
                }
                __syncthreads();
                if (j0 == 8) SMPROF(7);
                // rank-8 update of the rows below the group; thread (r, h) takes 4-column chunks
                // j1 + 4h, j1 + 4h + 8, ... (four independent accumulations per chunk)
                if (r >= g0 + 8 && row_ok) {
                    T lq[8];
#pragma unroll
                    for (int t = 0; t < 8; ++t) lq[t] = Lb[r + (j0 + t) * kSmN];
                    for (int k = j1 + 4 * h; k < nc; k += 8) {
                        T x[4];
#pragma unroll
                        for (int i = 0; i < 4; ++i) x[i] = Lb[r + (k + i) * kSmN];
#pragma unroll
                        for (int t = 0; t < 8; ++t)
#pragma unroll
                            for (int i = 0; i < 4; ++i) x[i] -= lq[t] * Lb[(g0 + t) + (k + i) * kSmN];
#pragma unroll
                        for (int i = 0; i < 4; ++i)
                            if (k + i < nc) Lb[r + (k + i) * kSmN] = x[i];
                    }
                }
                __syncthreads();
            }
        }
        SMPROF(8);
        // the factored block to W for the later CTAs (read through L2: DSMEM reads of one owner by
        // all later CTAs share the owner's shared-memory port, ~20 B/clk, measured 9.6 us per panel)
        __syncthreads();
        if (tid < nc) ipiv[cb + tid] = s_piv[tid];
        if (c + 1 < P && row_ok)
            for (int i = 0; i < kSmH; ++i)
                if (hc + i < nc) W[r + (int64_t)(cb + hc + i) * ldw] = Lb[r + (hc + i) * kSmN];
        cl.sync();                                   // panel c visible to the cluster
        if (prof == 1 && tid == 0 && c < 4 && b < 4) {   // diagnostics: %globaltimer at the end of step b
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            st->dbg_t[4 * c + b] = t;
        }
    }
    for (int b = c + 1; b < P; ++b) {
        cl.sync();
        if (prof == 1 && tid == 0 && c < 4 && b < 4) {   // diagnostics: %globaltimer at the end of step b
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            st->dbg_t[4 * c + b] = t;
        }
    }
    // ---- write-out with the later panels' interchanges applied, the row permutation
    for (int q = tid; q < n; q += kSmT) s_all[q] = (int)__ldcg(ipiv + q);
    __syncthreads();
    if (row_ok) {
        int dest = r;
        for (int g = kSmC * (c + 1); g < n; ++g) {
            const int p = s_all[g];
            if (dest == g) dest = p;
            else if (dest == p) dest = g;
        }
        for (int i = 0; i < kSmH; ++i)
            if (hc + i < nc) W[dest + (int64_t)(cb + hc + i) * ldw] = Lb[r + (hc + i) * kSmN];
        if (c == 0 && h == 0) {
            int d2 = r;
            for (int g = 0; g < n; ++g) {
                const int p = s_all[g];
                if (d2 == g) d2 = p;
                else if (d2 == p) d2 = g;
            }
            perm[d2] = r;
        }
    }
    if (tid == 0 && info != ~0ull) atomicMin(&st->info, info);
    cl.sync();                                       // no CTA exits while its shared memory may be read
#undef SMPROF
}

template <typename T>
static bool small_lu_launch(const Work& w, cudaStream_t s) {
    const int n = (int)w.n;
    const int P = (n + kSmC - 1) / kSmC;
    const size_t smem = sizeof(T) * ((size_t)kSmC * kSmN + 2 * kSmC + 272 + 2 * 8 * kSmC);
    auto kern = lu_small_kernel<T>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(P);
    cfg.blockDim = dim3(kSmT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = P; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    static const int prof = getenv("AS_LU_SMALL_PROF") ? atoi(getenv("AS_LU_SMALL_PROF")) : 0;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, (T*)w.W, w.ldw, n, w.ipiv, w.perm, w.st, prof);
    if (e == cudaSuccess) return true;
    cudaGetLastError();
    return false;
}

// ------------------------------------------------------------------ host driver
struct LuStreams {
    cudaStream_t hi = nullptr;
    cudaStream_t side = nullptr;   // interchanges into the finished L columns (off the critical path)
    cudaEvent_t ev[64];
    int next = 0;
    int prio_hi = 0;
};

static LuStreams& lu_streams() {
    static thread_local LuStreams L;
    if (!L.hi) {
        int lo = 0, hi = 0;
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        L.prio_hi = hi;
        cudaStreamCreateWithPriority(&L.hi, cudaStreamNonBlocking, hi);
        cudaStreamCreateWithPriority(&L.side, cudaStreamNonBlocking, lo);
        for (auto& e : L.ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    }
    return L;
}

static int g_panel_dbg = 0;   // diagnostics: ablation mask of the register panel (lu_debug_panel_time)

// Cluster size and rows per thread of the fast panel: one CTA up to 1024 rows (RPT = 1, 2, 4
// with leaves of 64, 32, 16 columns), then up to 16 CTAs of <= 1024 rows; larger panels use the
// cooperative kernel.
template <typename T>
static bool leaf_panel_launch(const Work& w, int64_t k0, int nbp, int prio, cudaStream_t s) {
    const int64_t n = w.n, m = n - k0;
    static const int rows_env = getenv("AS_LU_LEAF_ROWS") ? atoi(getenv("AS_LU_LEAF_ROWS")) : 1024;
    static int pmax = kLfMaxP;
    if (nbp > kPW) return false;
    for (;;) {
        int P = 1;
        while (P < pmax && (m + P - 1) / P > rows_env) P *= 2;
        const int64_t chunk = (m + P - 1) / P;
        const int rpt = (int)((chunk + kPT - 1) / kPT);
        if (rpt > 4) return false;
        void* kern;
        size_t smem;
        if (rpt <= 1) { kern = (void*)lu_panel_fast_kernel<T, 1, 64>; smem = sizeof(LeafSmem<T, 64>); }
        else if (rpt <= 2) { kern = (void*)lu_panel_fast_kernel<T, 2, 32>; smem = sizeof(LeafSmem<T, 32>); }
        else { kern = (void*)lu_panel_fast_kernel<T, 4, 16>; smem = sizeof(LeafSmem<T, 16>); }
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (P > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(P);
        cfg.blockDim = dim3(kPT);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = s;
        cudaLaunchAttribute at[2];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = P; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        at[1].id = cudaLaunchAttributePriority; at[1].val.priority = prio;
        cfg.attrs = at;
        cfg.numAttrs = 2;
        LuTrace& tr = lu_trace();
        const int slot = (int)(k0 / kBW) * 4 + ((k0 % kBW) ? 2 : 1);
        unsigned long long* tmn = tr.tmin && k0 / kBW < kTraceBlocks ? tr.tmin + slot : nullptr;
        unsigned long long* tmx = tr.tmax && k0 / kBW < kTraceBlocks ? tr.tmax + slot : nullptr;
        // the cluster shape must be schedulable (checked outside the stream: a failing launch
        // would invalidate a graph capture)
        int ncl = 0;
        if (cudaOccupancyMaxActiveClusters(&ncl, kern, &cfg) == cudaSuccess && ncl > 0) {
            T* Wp = (T*)w.W;
            int64_t ldw = w.ldw;
            int64_t* ip = w.ipiv;
            DevState* stp = w.st;
            int dbg = g_panel_dbg;
            void* args[] = {&Wp, &ldw, (void*)&n, &k0, &nbp, &ip, &stp, &tmn, &tmx, &dbg};
            const cudaError_t e = cudaLaunchKernelExC(&cfg, kern, args);
            if (e == cudaSuccess) return true;
        }
        cudaGetLastError();
        if (pmax <= 1) return false;
        pmax /= 2;                          // e.g. 16-CTA clusters not available: retry with 8
    }
}

template <typename T>
static void panel_launch(const Work& w, int64_t k0, int nbp, unsigned long long seq_base, int prio, cudaStream_t s) {
    const int64_t n = w.n, m = n - k0;
    // register/cluster panel: opt-in (AS_LU_PANEL=reg) until it beats the cooperative panel
    // Panel policy.  The cluster panel occupies <= 16 SMs but is slower per column than the
    // cooperative panel (which occupies ~m/128 SMs); measured on C5 (n = 16384) the cooperative
    // panel everywhere wins (196 ms) over the cluster panel for m >= 12288 / 10240 / 8192
    // (209 / 218 / 227 ms), so the cluster panel is opt-in: AS_LU_PANEL=reg (everywhere) or
    // AS_LU_FAST_MIN_M=<m> (where the panel has >= m rows).
    static const char* pol = getenv("AS_LU_PANEL");
    static const int64_t fast_min_m = getenv("AS_LU_FAST_MIN_M") ? atoll(getenv("AS_LU_FAST_MIN_M")) : (int64_t)1 << 62;
    const bool want_fast = pol && strcmp(pol, "reg") == 0 ? true : (pol && strcmp(pol, "coop") == 0) ? false : m >= fast_min_m;
    if (want_fast && getenv("AS_LU_PANEL_OLD") == nullptr && leaf_panel_launch<T>(w, k0, nbp, prio, s)) return;
    static const int rows_per_cta = getenv("AS_LU_PANEL_ROWS") ? atoi(getenv("AS_LU_PANEL_ROWS")) : 128;
    int P = (int)std::min<int64_t>(w.num_sms, (m + rows_per_cta - 1) / rows_per_cta);
    P = std::max(P, 1);
    if (getenv("AS_LU_NO_CLUSTER") == nullptr) {
        // cluster panel when the rows fit in <= kClMax CTAs' shared memory (~200 KB each)
        int pc = 1;
        while (pc < kClMax && (size_t)((m + pc - 1) / pc) * nbp * sizeof(T) > 192 * 1024) pc *= 2;
        const int64_t ch = (m + pc - 1) / pc;
        const size_t smc = sizeof(T) * ((size_t)(ch | 1) * nbp + 5 * (size_t)nbp);
        if (smc <= 200 * 1024) {
            auto kc = lu_panel_cl_kernel<T>;
            cudaFuncSetAttribute(kc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smc);
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(pc);
            cfg.blockDim = dim3(kPT);
            cfg.dynamicSmemBytes = smc;
            cfg.stream = s;
            cudaLaunchAttribute at[2];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = pc; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
            at[1].id = cudaLaunchAttributePriority; at[1].val.priority = prio;
            cfg.attrs = at;
            cfg.numAttrs = 2;
            if (cudaLaunchKernelEx(&cfg, kc, (T*)w.W, w.ldw, n, k0, nbp, w.ipiv, w.st, (g_panel_dbg & 256) ? 1 : 0) == cudaSuccess)
                return;
            cudaGetLastError();
        }
    }
    const int64_t chunk = (m + P - 1) / P;
    size_t smem = sizeof(T) * ((chunk | 1) * nbp + nbp);
    int use_smem = 1;
    if (smem > 200 * 1024) { use_smem = 0; smem = sizeof(T) * nbp; }
    PSlot* slots = (PSlot*)w.cand;
    T* rowbuf = (T*)((char*)w.cand + sizeof(PSlot) * 1024);
    T* diagbuf = rowbuf + (int64_t)2 * 1024 * kPW;
    auto kern = lu_panel2_kernel<T>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)std::max<size_t>(smem, 1024));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(P);
    cfg.blockDim = dim3(kPT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (P > 1) { attr[na].id = cudaLaunchAttributeCooperative; attr[na].val.cooperative = 1; ++na; }
    attr[na].id = cudaLaunchAttributePriority; attr[na].val.priority = prio; ++na;
    cfg.attrs = attr;
    cfg.numAttrs = na;
    LuTrace& tr = lu_trace();
    const int slot = (int)(k0 / kBW) * 4 + ((k0 % kBW) ? 2 : 1);
    unsigned long long* tmn = tr.tmin && k0 / kBW < kTraceBlocks ? tr.tmin + slot : nullptr;
    unsigned long long* tmx = tr.tmax && k0 / kBW < kTraceBlocks ? tr.tmax + slot : nullptr;
    cudaLaunchKernelEx(&cfg, kern, (T*)w.W, w.ldw, n, k0, nbp, w.ipiv, w.st, slots, rowbuf, diagbuf, seq_base, use_smem,
                       tmn, tmx);
}

template <typename T>
static void laswp_launch(const Work& w, int64_t j0, int cnt, int64_t a0, int64_t a1, int64_t b0, int64_t b1, bool perm,
                         cudaStream_t s) {
    const int64_t ncols = std::max<int64_t>(0, a1 - a0) + std::max<int64_t>(0, b1 - b0) + (perm ? 1 : 0);
    if (ncols <= 0 || cnt <= 0) return;
    laswp3_kernel<T><<<(unsigned)std::min<int64_t>((ncols + 7) / 8, (int64_t)w.num_sms * 4), 256, 0, s>>>(
        (T*)w.W, w.ldw, j0, cnt, a0, a1, b0, b1, w.ipiv, perm ? w.perm : nullptr);
}

template <typename T>
static void linv_launch(const Work& w, int64_t k0, int nbp, cudaStream_t s) {
    const int smem = (int)(sizeof(T) * (2 * kB64 * kB64LD + 3 * 256));
    cudaFuncSetAttribute(lu_linv_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    lu_linv_kernel<T><<<(nbp + kB64 - 1) / kB64, 256, smem, s>>>((const T*)w.W, w.ldw, k0, nbp, (T*)w.Dinv0);
}

template <typename T>
static void swap_u12_launch(const Work& w, int64_t k0, int bw, int64_t c0, int64_t c1, cudaStream_t s) {
    if (c1 <= c0) return;
    const int smem = (int)(sizeof(T) * (2 * kSUC * kSULD + 3 * kB64 * kB64));
    cudaFuncSetAttribute(swap_u12_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    swap_u12_kernel<T><<<(unsigned)((c1 - c0 + kSUC - 1) / kSUC), 256, smem, s>>>((T*)w.W, w.ldw, k0, bw, c0, c1, w.ipiv,
                                                                                 (const T*)w.Dinv0);
}

template <typename T>
static void gemm_launch(const Work& w, int64_t r0, int64_t c0, int64_t k0, int64_t M, int64_t N, int64_t K, cudaStream_t s,
                        int prio, bool one_per_sm = false, int trace_slot = -1) {
    (void)prio;
    if (M <= 0 || N <= 0 || K <= 0) return;
    T* W = (T*)w.W;
    const int64_t ldw = w.ldw;
    GemmArgs g{};
    g.M = M; g.N = N; g.K = K;
    g.A = W + r0 + k0 * ldw; g.lda = ldw; g.TA = false;
    g.B = W + k0 + c0 * ldw; g.ldb = ldw; g.TB = false;
    g.C = W + r0 + c0 * ldw; g.ldc = ldw;
    g.one_per_sm = one_per_sm;
    LuTrace& tr = lu_trace();
    if (tr.tmin && trace_slot >= 0 && trace_slot < 4 * kTraceBlocks) {
        g.trace_min = tr.tmin + trace_slot;
        g.trace_max = tr.tmax + trace_slot;
    }
    launch_gemm_minus(w.dtype, g, s);
}

// Factor the block's two panels (columns k0 .. k0+bw), on stream s.
template <typename T>
static void block_panels(const Work& w, int64_t k0, int bw, int prio, cudaStream_t s) {
    const int64_t n = w.n;
    (void)n;
    // one panel per block (kPW == kBW); sequence numbers of the panel exchange grow with the block
    static_assert(kPW == kBW, "block_panels factors a block as one panel");
    panel_launch<T>(w, k0, bw, (unsigned long long)(k0 / kPW) * 256ull, prio, s);
    linv_launch<T>(w, k0, bw, s);
}

template <typename T>
static void lu_factor_t(const Work& w, cudaStream_t s) {
    const int64_t n = w.n;
    launch_copy_norm(w, true, s);
    static const bool small_off = getenv("AS_LU_SMALL_OFF") != nullptr;
    if (n <= kSmN && !small_off && small_lu_launch<T>(w, s)) {
        linv_launch<T>(w, 0, (int)n, s);                        // Dinv0: unit-L diagonal block inverses
        launch_trtri_blocks(w.dtype, w.W, w.ldw, n, w.Dinv1, true, false, w.st, true, w.args, s);
        return;
    }
    cudaMemsetAsync(w.cand, 0, sizeof(PSlot) * 1024, s);       // panel exchange slots (sequence numbers)
    if (lu_trace().tmin) {
        cudaMemsetAsync(lu_trace().tmin, 0xFF, sizeof(unsigned long long) * 4 * kTraceBlocks, s);
        cudaMemsetAsync(lu_trace().tmax, 0, sizeof(unsigned long long) * 4 * kTraceBlocks, s);
    }
    LuStreams& LS = lu_streams();
    // Look-ahead: next block's panels on a high-priority stream beside the bulk GEMM (measured
    // ~10% on C5; the gang-scheduled cooperative panel only partly overlaps).
    const bool lookahead = n >= 2048 && getenv("AS_LU_NO_LOOKAHEAD") == nullptr;
    int evi = 0;
    auto ev = [&]() { return LS.ev[(evi++) % 64]; };
    bool side_used = false;
    // first block's panels
    block_panels<T>(w, 0, (int)std::min<int64_t>(kBW, n), LS.prio_hi, s);
    for (int64_t k0 = 0; k0 < n; k0 += kBW) {
        const int bw = (int)std::min<int64_t>(kBW, n - k0);
        const int p1 = std::min(kHalf, bw);
        const int64_t kn = k0 + bw;             // next block start
        // the block's interchanges into all other columns (the panel already swapped its own):
        // the finished L columns [0, k0) on the side stream (nothing reads them before the
        // solve; the side stream keeps the blocks' order), the trailing columns [kn, n) and
        // the row permutation on the critical path
        {
            cudaEvent_t el = ev();
            cudaEventRecord(el, s);
            cudaStreamWaitEvent(LS.side, el, 0);
            laswp_launch<T>(w, k0, bw, 0, k0, 0, 0, true, LS.side);   // L columns + row permutation
            side_used = true;
        }
        if (kn >= n) break;
        // trailing columns: interchanges + U12 = L11^{-1} A12 in one kernel
        (void)p1;
        swap_u12_launch<T>(w, k0, bw, kn, n, s);
        const int64_t M = n - kn;
        const int nbw = (int)std::min<int64_t>(kBW, n - kn);
        if (lookahead && n - kn > nbw) {
            // next block's columns first (high priority), then its panels; the rest of the GEMM
            // concurrently on the main stream
            cudaEvent_t e0 = ev();
            cudaEventRecord(e0, s);
            cudaStreamWaitEvent(LS.hi, e0, 0);
            gemm_launch<T>(w, kn, kn, k0, M, nbw, bw, LS.hi, LS.prio_hi, false, (int)(k0 / kBW) * 4 + 3);
            block_panels<T>(w, kn, nbw, LS.prio_hi, LS.hi);
            gemm_launch<T>(w, kn, kn + nbw, k0, M, n - kn - nbw, bw, s, 0, getenv("AS_LU_ONE_PER_SM") != nullptr,
                           (int)(k0 / kBW) * 4 + 0);
            cudaEvent_t e1 = ev();
            cudaEventRecord(e1, LS.hi);
            cudaStreamWaitEvent(s, e1, 0);
        } else {
            gemm_launch<T>(w, kn, kn, k0, M, n - kn, bw, s, 0);
            block_panels<T>(w, kn, nbw, LS.prio_hi, s);
        }
    }
    if (side_used) {
        cudaEvent_t ej = ev();
        cudaEventRecord(ej, LS.side);
        cudaStreamWaitEvent(s, ej, 0);
    }
    // Dinv0 (unit-L diagonal block inverses) was written panel by panel
    launch_trtri_blocks(w.dtype, w.W, w.ldw, n, w.Dinv1, true, false, w.st, true, w.args, s);
}

// trace buffers for other kernels' diagnostics (triangular solves), nullptr unless AS_LU_TRACE
unsigned long long* debug_trace_buf(int which) {
    LuTrace& tr = lu_trace();
    return which == 0 ? tr.tmin : tr.tmax;
}

// host copy of the last factorization's trace (diagnostics); returns the slot count or -1
int lu_trace_copy(unsigned long long* out_min, unsigned long long* out_max, int cap) {
    LuTrace& tr = lu_trace();
    if (!tr.tmin) return -1;
    const int cnt = std::min(cap, 4 * kTraceBlocks);
    cudaDeviceSynchronize();
    cudaMemcpy(out_min, tr.tmin, sizeof(unsigned long long) * cnt, cudaMemcpyDeviceToHost);
    cudaMemcpy(out_max, tr.tmax, sizeof(unsigned long long) * cnt, cudaMemcpyDeviceToHost);
    return cnt;
}

// Diagnostics: average time (us) of one panel factorization of W (restored from Wsrc before each
// launch).  kind 0: the launch the factorization would make; kind 1: the cooperative panel.
double lu_debug_panel_time(int dtype, int kind, void* W, int64_t ldw, int64_t n, int64_t k0, int nbp, const void* Wsrc,
                           int iters, int dbg) {
    Work w{};
    w.dtype = dtype; w.n = n; w.ldw = ldw; w.W = W;
    cudaDeviceGetAttribute(&w.num_sms, cudaDevAttrMultiProcessorCount, 0);
    cudaMalloc(&w.ipiv, 8 * n);
    cudaMalloc(&w.st, sizeof(DevState));
    cudaMalloc(&w.cand, 16 * 2 * 1024 + 8 * 2 * 1024 * 128 + 8 * 2 * 128);
    cudaMemset(w.st, 0, sizeof(DevState));
    cudaMemset(&w.st->info, 0xFF, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    g_panel_dbg = dbg;
    const size_t es = dtype == AS_F64 ? 8 : 4;
    double tot = 0.0;
    for (int it = 0; it < iters; ++it) {
        cudaMemcpy(W, Wsrc, es * ldw * n, cudaMemcpyDeviceToDevice);
        cudaMemset(w.cand, 0, 16 * 2 * 1024);
        cudaEventRecord(e0, 0);
        if (dtype == AS_F64) {
            if (kind != 0 || !leaf_panel_launch<double>(w, k0, nbp, 0, 0)) {
                setenv("AS_LU_PANEL_OLD", "1", 1);
                panel_launch<double>(w, k0, nbp, 0, 0, 0);
                unsetenv("AS_LU_PANEL_OLD");
            }
        } else {
            if (kind != 0 || !leaf_panel_launch<float>(w, k0, nbp, 0, 0)) {
                setenv("AS_LU_PANEL_OLD", "1", 1);
                panel_launch<float>(w, k0, nbp, 0, 0, 0);
                unsetenv("AS_LU_PANEL_OLD");
            }
        }
        cudaEventRecord(e1, 0);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (it > 0 || iters == 1) tot += ms;
    }
    g_panel_dbg = 0;
    if (dbg & 256) {
        unsigned long long ph[16];
        cudaMemcpy(ph, w.st->dbg_t, sizeof(ph), cudaMemcpyDeviceToHost);
        fprintf(stderr, "panel phases (cycles, CTA 0, kind %d): %llu %llu %llu %llu %llu %llu %llu\n", kind, ph[0], ph[1],
                ph[2], ph[3], ph[4], ph[5], ph[6]);
    }
    const cudaError_t err = cudaGetLastError();
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(w.ipiv);
    cudaFree(w.st);
    cudaFree(w.cand);
    if (err != cudaSuccess) return -(double)err;
    return 1000.0 * tot / (iters > 1 ? iters - 1 : 1);
}

void launch_lu_factor(const Work& w, cudaStream_t s) {
    if (w.dtype == AS_F64) lu_factor_t<double>(w, s);
    else lu_factor_t<float>(w, s);
}

}  // namespace as
