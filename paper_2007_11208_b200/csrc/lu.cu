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

constexpr int kPT = 256;     // panel threads (leaf panel)
// cooperative / cluster panels: 512 threads halve the (latency-bound) bulk rank-1 update but every
// barrier-separated phase grows with the thread count: measured 337 vs 304 us (m = 128), 475 vs 442 us (m = 4096)
constexpr int kPT2 = 256;
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
AS_DEV void panel_argmax_reduce(T bv, unsigned br, int dnan, int64_t rbeg, int64_t g, T& v, long long& idx, T* sv,
                                long long* si, int* sdn) {
    // per-thread candidate (bv = |a|, br = local row or 0xffffffff, dnan = "the row at g holds a NaN")
    // -> CTA candidate.  Warp level: integer reductions on the order-preserving key + the smallest
    // row among the maxima; CTA level: every warp merges the 8 warp results the same way (one barrier).
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned kh = 0u, kl = 0u;
    if (br != 0xffffffffu) cand_key<T>(bv == T(0) ? T(0) : bv, kh, kl);   // (-0 -> +0)
    unsigned mh = __reduce_max_sync(0xffffffffu, kh);
    unsigned ml = __reduce_max_sync(0xffffffffu, kh == mh ? kl : 0u);
    const unsigned wr = __reduce_min_sync(0xffffffffu, (mh != 0u && kh == mh && kl == ml) ? br : 0xffffffffu);
    const T wm = __shfl_sync(0xffffffffu, bv, (int)(__ffs(__ballot_sync(0xffffffffu, br == wr && wr != 0xffffffffu)) - 1) & 31);
    dnan = __any_sync(0xffffffffu, dnan);
    if (lane == 0) { sv[warp] = (wr == 0xffffffffu) ? T(-1) : wm; si[warp] = (long long)wr; sdn[warp] = dnan; }
    __syncthreads();
    const int nw = (int)(blockDim.x >> 5);               // <= 32 warps: one lane per warp result
    const T v8 = lane < nw ? sv[lane] : T(-1);
    const unsigned r8 = lane < nw ? (unsigned)si[lane] : 0xffffffffu;
    const int d8 = lane < nw ? sdn[lane] : 0;
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

template <typename T>
AS_DEV void panel_local_argmax(const T* Ps, int64_t cp, int nr, int64_t rbeg, int64_t g, int col, T& v, long long& idx,
                               T* sv, long long* si, int* sdn) {
    // first max |a(r, col)| over local rows at positions >= g; NaN never wins, a NaN at row g keeps
    // g (the serial sweep's semantics).
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
    panel_argmax_reduce<T>(bv, br, dnan, rbeg, g, v, idx, sv, si, sdn);
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

// Exchange words of the cooperative panel: every 8-byte word is (seq32 << 32) | 32 payload bits, so
// a word is its own "ready" flag -- the producer needs no barrier + release fence before a flag and
// the consumer no acquire fence after it (r02: ~1 us of the 4.4 us column step).  The arena is zeroed
// per factorization (sequence numbers repeat across solves).
//   hdr   [2 parities][512 CTAs][4]: |candidate| high / low word, candidate row index (0xffffffff: none)
//   rowll [2][512][kPW][WPE]:        the CTA's candidate row
//   diagll[2][kPW][WPE]:             the row at position g (for the owner of the pivot row)
template <typename T> struct PlW { static constexpr int v = sizeof(T) / 4; };
constexpr int kPlMaxP = 512;
constexpr size_t kPlHdrWords = 2 * kPlMaxP * 4;
constexpr size_t kPlRowWords = (size_t)2 * kPlMaxP * 128 * 2;      // sized for fp64 (2 words per element)
constexpr size_t kPlDiagWords = 2 * 128 * 2;
size_t lu_cand_bytes() { return 8 * (kPlHdrWords + kPlRowWords + kPlDiagWords); }
AS_DEV void pl_put(unsigned long long* w, double x, unsigned sq) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(x), hi = (unsigned long long)sq << 32;
    asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" ::"l"(w), "l"(hi | (b >> 32)), "l"(hi | (b & 0xffffffffull)) : "memory");
}
AS_DEV void pl_put(unsigned long long* w, float x, unsigned sq) {
    asm volatile("st.volatile.global.u64 [%0], %1;" ::"l"(w), "l"(((unsigned long long)sq << 32) | __float_as_uint(x)) : "memory");
}
AS_DEV double pl_get(const unsigned long long* w, unsigned sq, double) {
    unsigned long long a, b;
    do {
        asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(w) : "memory");
    } while ((unsigned)(a >> 32) != sq || (unsigned)(b >> 32) != sq);
    return __longlong_as_double((long long)(((a & 0xffffffffull) << 32) | (b & 0xffffffffull)));
}
AS_DEV float pl_get(const unsigned long long* w, unsigned sq, float) {
    unsigned long long a;
    do {
        asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(a) : "l"(w) : "memory");
    } while ((unsigned)(a >> 32) != sq);
    return __uint_as_float((unsigned)a);
}

template <typename T>
__global__ void __launch_bounds__(kPT2, 1) lu_panel2_kernel(T* W, int64_t ldw, int64_t n, int64_t k0, int nbp,
                                                            int64_t* ipiv, DevState* st, unsigned long long* xch,
                                                            unsigned long long seq_base, int use_smem,
                                                            unsigned long long* tr_min, unsigned long long* tr_max,
                                                            unsigned poll_nap) {
    constexpr int WPE = PlW<T>::v;
    unsigned long long* hdr = xch;
    unsigned long long* rowll = xch + kPlHdrWords;
    unsigned long long* diagll = rowll + kPlRowWords;
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
    __shared__ T sv[32];
    __shared__ long long si[32];
    __shared__ int sdn[32];
    __shared__ long long s_p;
    __shared__ int s_owner;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

    if (use_smem) {
        batched<8, T>(
            nr * nbp, [&](int e) -> T { const int c = e / nr, r = e - c * nr; return W[(rbeg + r) + (k0 + c) * ldw]; },
            [&](int e, T v) { const int c = e / nr, r = e - c * nr; Ps[r + c * cp] = v; });
        __syncthreads();
    }
    // publish the candidate for column j: (|v|, idx) of this CTA, its row, and the row at position g
    auto put_hdr = [&](int j, T v, long long idx) {       // one thread
        const unsigned sq = (unsigned)(seq_base + (unsigned long long)j + 1ull);
        const unsigned long long hi = (unsigned long long)sq << 32;
        const unsigned long long vb = (unsigned long long)__double_as_longlong((double)v);
        unsigned long long* h = hdr + ((size_t)(j & 1) * kPlMaxP + cta) * 4;
        const unsigned i32 = idx == 0x7fffffffffffffffll ? 0xffffffffu : (unsigned)idx;
        asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" ::"l"(h), "l"(hi | (vb >> 32)), "l"(hi | (vb & 0xffffffffull)) : "memory");
        asm volatile("st.volatile.global.u64 [%0], %1;" ::"l"(h + 2), "l"(hi | i32) : "memory");
    };
    auto publish = [&](int j, T v, long long idx) {
        const int64_t g = k0 + j;
        const int par = j & 1;
        const unsigned sq = (unsigned)(seq_base + (unsigned long long)j + 1ull);
        if (idx != 0x7fffffffffffffffll && idx >= rbeg && idx < rend) {
            const int r = (int)(idx - rbeg);
            for (int c = threadIdx.x; c < nbp; c += blockDim.x)
                pl_put(rowll + (((size_t)par * kPlMaxP + cta) * kPW + c) * WPE, Ps[r + c * cp], sq);
        }
        if (g >= rbeg && g < rend) {
            const int r = (int)(g - rbeg);
            for (int c = threadIdx.x; c < nbp; c += blockDim.x) pl_put(diagll + ((size_t)par * kPW + c) * WPE, Ps[r + c * cp], sq);
        }
        if (threadIdx.x == 0) put_hdr(j, v, idx);
    };
    {
        T v;
        long long idx;
        panel_local_argmax(Ps, cp, nr, rbeg, k0, 0, v, idx, sv, si, sdn);
        publish(0, v, idx);
    }
    unsigned long long info = ~0ull;
    // Column step, three CTA barriers (r02: was nine): [poll] B1 [pivot row -> ubuf, the interchange's
    // two row writes] B2 [multipliers, column j+1 and each thread's candidate for it] B3 (inside the
    // reduction) [rows rc / g+1 finished and published word by word] [bulk update].  The next step's
    // B1 orders the bulk update before anything that overwrites what it reads.
    for (int j = 0; j < nbp; ++j) {
        const int64_t g = k0 + j;
        const int par = j & 1;
        const unsigned long long want = seq_base + (unsigned long long)j + 1ull;
        // ---- poll every CTA's header words (barrier + data in one), pick the winner
        const unsigned sq = (unsigned)want;
        if (warp == 0) {
            T bv = T(-1);
            long long bi = 0x7fffffffffffffffll;
            int bo = 0;
            // each lane owns up to 5 slots (P <= 160); all are polled together each round
            constexpr int kMaxPer = 5;
            bool ready[kMaxPer];
            unsigned long long h0[kMaxPer], h1[kMaxPer], h2[kMaxPer];
#pragma unroll
            for (int q = 0; q < kMaxPer; ++q) ready[q] = (lane + 32 * q) >= P;
            for (;;) {
                bool all = true;
#pragma unroll
                for (int q = 0; q < kMaxPer; ++q) {
                    if (!ready[q]) {
                        const unsigned long long* h = hdr + ((size_t)par * kPlMaxP + lane + 32 * q) * 4;
                        asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(h0[q]), "=l"(h1[q]) : "l"(h) : "memory");
                        asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(h2[q]) : "l"(h + 2) : "memory");
                        ready[q] = (unsigned)(h0[q] >> 32) == sq && (unsigned)(h1[q] >> 32) == sq && (unsigned)(h2[q] >> 32) == sq;
                        all = all && ready[q];
                    }
                }
                if (__all_sync(0xffffffffu, all)) break;
                if (poll_nap) __nanosleep(poll_nap);     // P warps spinning on the same header lines
            }
#pragma unroll
            for (int q = 0; q < kMaxPer; ++q) {
                const int t = lane + 32 * q;
                if (t < P) {
                    const T cv = (T)__longlong_as_double((long long)(((h0[q] & 0xffffffffull) << 32) | (h1[q] & 0xffffffffull)));
                    const unsigned i32 = (unsigned)h2[q];
                    const long long ci = i32 == 0xffffffffu ? 0x7fffffffffffffffll : (long long)i32;
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
        __syncthreads();                                                      // B1
        const long long p = s_p;
        const int owner = s_owner;
        const bool own_p = p != g && p >= rbeg && p < rend;
        const int g_loc = (g >= rbeg && g < rend) ? (int)(g - rbeg) : -1;
        // the pivot row into ubuf; the pivot itself first (same line, one broadcast load): an exact
        // zero pivot means no interchange and no elimination (singular column)
        const unsigned long long* prow = rowll + (((size_t)par * kPlMaxP + owner) * kPW) * WPE;
        const T piv = pl_get(prow + (size_t)j * WPE, sq, T(0));
        const bool elim = piv != T(0);
        T* dst_p = own_p ? Ps + (p - rbeg) : nullptr;
        for (int c = threadIdx.x; c < nbp; c += blockDim.x) {
            const T u = pl_get(prow + (size_t)c * WPE, sq, T(0));
            const T dg = (own_p && elim) ? pl_get(diagll + ((size_t)par * kPW + c) * WPE, sq, T(0)) : T(0);
            ubuf[c] = u;
            if (elim) {
                if (own_p) dst_p[c * cp] = dg;               // the owner of p takes the old row g
                if (g_loc >= 0) Ps[g_loc + c * cp] = u;      // the pivot row at position g
            }
        }
        if (cta == 0 && threadIdx.x == 0) ipiv[g] = (p == 0x7fffffffffffffffll) ? g : p;
        if (!elim && info == ~0ull) info = (unsigned long long)(g + 1);
        __syncthreads();                                                      // B2
        const int64_t r0 = max<int64_t>(0, g + 1 - rbeg);
        // ---- multipliers, column j+1 of my rows > g, and each thread's candidate for column j+1
        T cbv = T(-1);
        unsigned cbr = 0xffffffffu;
        int cdn = 0;
        {
            const bool more = j + 1 < nbp;
            const T u1 = more ? ubuf[j + 1] : T(0);
            for (int r = (int)r0 + threadIdx.x; r < nr; r += blockDim.x) {
                T a1 = more ? Ps[r + (j + 1) * cp] : T(0);
                if (elim) {
                    const T l = Ps[r + j * cp] / piv;
                    Ps[r + j * cp] = l;
                    if (more) { a1 -= l * u1; Ps[r + (j + 1) * cp] = a1; }
                }
                if (more) {
                    const T aa = a1 < T(0) ? -a1 : a1;
                    if (rbeg + r == g + 1 && aa != aa) cdn = 1;
                    if (aa > cbv) { cbv = aa; cbr = (unsigned)r; }   // rows increase: strict > keeps the first
                }
            }
        }
        if (j + 1 >= nbp) break;
        T v;
        long long idx;
        panel_argmax_reduce<T>(cbv, cbr, cdn, rbeg, g + 1, v, idx, sv, si, sdn);   // B3 inside
        const int rc = (idx != 0x7fffffffffffffffll && idx >= rbeg && idx < rend) ? (int)(idx - rbeg) : -1;
        const int rg = (g + 1 >= rbeg && g + 1 < rend) ? (int)(g + 1 - rbeg) : -1;
        // ---- the candidate row and row g+1: finish their update (columns j+2..) while copying them out
        {
            const int par1 = (j + 1) & 1;
            const unsigned sq1 = sq + 1u;
            const T lc = (rc >= 0 && elim) ? Ps[rc + j * cp] : T(0);
            const T lg = (rg >= 0 && elim) ? Ps[rg + j * cp] : T(0);
            unsigned long long* myrow = rowll + (((size_t)par1 * kPlMaxP + cta) * kPW) * WPE;
            unsigned long long* dgrow = diagll + ((size_t)par1 * kPW) * WPE;
            for (int c = threadIdx.x; c < nbp; c += blockDim.x) {
                const T uc = ubuf[c];
                if (rc >= 0) {
                    T a = Ps[rc + c * cp];
                    if (elim && c >= j + 2) { a -= lc * uc; Ps[rc + c * cp] = a; }
                    pl_put(myrow + (size_t)c * WPE, a, sq1);
                    if (rg == rc) pl_put(dgrow + (size_t)c * WPE, a, sq1);
                }
                if (rg >= 0 && rg != rc) {
                    T a = Ps[rg + c * cp];
                    if (elim && c >= j + 2) { a -= lg * uc; Ps[rg + c * cp] = a; }
                    pl_put(dgrow + (size_t)c * WPE, a, sq1);
                }
            }
            if (threadIdx.x == 0) put_hdr(j + 1, v, idx);      // no barrier: every word validates itself
        }
        // ---- bulk rank-1 update of the remaining rows, columns j+2.. (thread = row, column phase)
        if (elim) panel_bulk_update<T>(Ps, cp, ubuf, (int)r0, nr, j, nbp, rc, rg);
    }
    __syncthreads();
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
__global__ void __launch_bounds__(kPT2, 1) lu_panel_cl_kernel(T* W, int64_t ldw, int64_t n, int64_t k0, int nbp,
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
    // every CTA's candidate header (|v|, row), pushed into every CTA's inbox at publication: the winner
    // is then picked from local shared memory and only the winning row is read remotely (r02q: the
    // three dependent DSMEM reads of the pull version were 1865 of 7150 cycles per column at P = 8)
    __shared__ T in_cv[2][kClMax];
    __shared__ long long in_ci[2][kClMax];
    __shared__ T sv[32];
    __shared__ long long si[32];
    __shared__ int sdn[32];
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
        if ((int)threadIdx.x < P) {
            *cl.map_shared_rank(&in_cv[par][cta], threadIdx.x) = v;
            *cl.map_shared_rank(&in_ci[par][cta], threadIdx.x) = idx;
        }
    };
    {
        T v;
        long long idx;
        panel_local_argmax(Ps, cp, nr, rbeg, k0, 0, v, idx, sv, si, sdn);
        publish(0, v, idx);
    }
    unsigned long long info = ~0ull;
    // Column step: one cluster barrier and two CTA barriers (r02: was one + seven): [cluster barrier:
    // every candidate visible, the previous bulk update finished] [every warp merges the P candidates;
    // pivot row -> ubuf, the interchange's two row writes] B2 [multipliers, column j+1, candidates]
    // B3 (inside the reduction) [rows rc / g+1 finished and copied to the exchange buffers] [bulk update]
    for (int j = 0; j < nbp; ++j) {
        const int64_t g = k0 + j;
        const int par = j & 1;
        PHC(0);
        if (P > 1) cl.sync();                            // every candidate of column j is visible
        else __syncthreads();
        PHC(1);
        long long p;
        int owner;
        {
            T bv = T(-1);
            long long bi = 0x7fffffffffffffffll;
            int bo = 0;
            if (lane < P) { bv = in_cv[par][lane]; bi = in_ci[par][lane]; bo = lane; }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const T v2 = __shfl_xor_sync(0xffffffffu, bv, o);
                const long long i2 = __shfl_xor_sync(0xffffffffu, bi, o);
                const int o2 = __shfl_xor_sync(0xffffffffu, bo, o);
                if (v2 > bv || (v2 == bv && i2 < bi)) { bv = v2; bi = i2; bo = o2; }
            }
            p = bi; owner = bo;                          // identical in every lane of every warp
        }
        const int gown = (int)((g - k0) / chunk);
        const bool own_p = p != g && p >= rbeg && p < rend;
        const int g_loc = (g >= rbeg && g < rend) ? (int)(g - rbeg) : -1;
        const T* rc = cl.map_shared_rank(candb + par * nbp, owner);
        const T* rd = cl.map_shared_rank(diagb + par * nbp, gown);
        const T piv = rc[j];
        const bool elim = piv != T(0);                   // exact zero pivot: no interchange, no elimination
        T* dst_p = own_p ? Ps + (p - rbeg) : nullptr;
        for (int c = threadIdx.x; c < nbp; c += blockDim.x) {
            const T u = rc[c];
            const T dg = (own_p && elim) ? rd[c] : T(0);
            ubuf[c] = u;
            if (elim) {
                if (own_p) dst_p[c * cp] = dg;
                if (g_loc >= 0) Ps[g_loc + c * cp] = u;
            }
        }
        if (cta == 0 && threadIdx.x == 0) ipiv[g] = (p == 0x7fffffffffffffffll) ? g : p;
        if (!elim && info == ~0ull) info = (unsigned long long)(g + 1);
        __syncthreads();                                                      // B2
        PHC(2);
        const int64_t r0 = max<int64_t>(0, g + 1 - rbeg);
        T cbv = T(-1);
        unsigned cbr = 0xffffffffu;
        int cdn = 0;
        {
            const bool more = j + 1 < nbp;
            const T u1 = more ? ubuf[j + 1] : T(0);
            for (int r = (int)r0 + threadIdx.x; r < nr; r += blockDim.x) {
                T a1 = more ? Ps[r + (j + 1) * cp] : T(0);
                if (elim) {
                    const T l = Ps[r + j * cp] / piv;
                    Ps[r + j * cp] = l;
                    if (more) { a1 -= l * u1; Ps[r + (j + 1) * cp] = a1; }
                }
                if (more) {
                    const T aa = a1 < T(0) ? -a1 : a1;
                    if (rbeg + r == g + 1 && aa != aa) cdn = 1;
                    if (aa > cbv) { cbv = aa; cbr = (unsigned)r; }
                }
            }
        }
        PHC(3);
        if (j + 1 >= nbp) break;
        T v;
        long long idx;
        panel_argmax_reduce<T>(cbv, cbr, cdn, rbeg, g + 1, v, idx, sv, si, sdn);   // B3 inside
        PHC(4);
        const int rcn = (idx != 0x7fffffffffffffffll && idx >= rbeg && idx < rend) ? (int)(idx - rbeg) : -1;
        const int rg = (g + 1 >= rbeg && g + 1 < rend) ? (int)(g + 1 - rbeg) : -1;
        {
            const int par1 = (j + 1) & 1;
            const T lc = (rcn >= 0 && elim) ? Ps[rcn + j * cp] : T(0);
            const T lg = (rg >= 0 && elim) ? Ps[rg + j * cp] : T(0);
            for (int c = threadIdx.x; c < nbp; c += blockDim.x) {
                const T uc = ubuf[c];
                if (rcn >= 0) {
                    T a = Ps[rcn + c * cp];
                    if (elim && c >= j + 2) { a -= lc * uc; Ps[rcn + c * cp] = a; }
                    candb[par1 * nbp + c] = a;
                    if (rg == rcn) diagb[par1 * nbp + c] = a;
                }
                if (rg >= 0 && rg != rcn) {
                    T a = Ps[rg + c * cp];
                    if (elim && c >= j + 2) { a -= lg * uc; Ps[rg + c * cp] = a; }
                    diagb[par1 * nbp + c] = a;
                }
            }
            if ((int)threadIdx.x < P) {
                *cl.map_shared_rank(&in_cv[par1][cta], threadIdx.x) = v;
                *cl.map_shared_rank(&in_ci[par1][cta], threadIdx.x) = idx;
            }
        }
        PHC(5);
        // (the multipliers of rows rcn / rg were read above by every thread before any of its bulk
        // writes; the bulk update skips those two rows and reads only ubuf and column j)
        if (elim) panel_bulk_update<T>(Ps, cp, ubuf, (int)r0, nr, j, nbp, rcn, rg);
    }
    __syncthreads();
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

// ------------------------------------------------------------------ panel (leaf-blocked, few CTAs)
// For tall panels (m > the cluster panel's reach) beside a running trailing GEMM.  The panel's m
// rows are split over P = ceil(m / kLfRows) CTAs (32 at n = 16384).  A CTA is small enough (<= 128
// registers per thread, ~85 KB of shared memory) to share an SM with one CTA of the trailing GEMM,
// so the launch (ordinary, high priority) is placed as GEMM tiles retire -- no cluster placement,
// no gang scheduling, and the GEMM keeps every SM.  Rows stay where they are in W during the panel ("original
// order"); every CTA tracks the CURRENT position of each of its rows (pos[]) and all CTAs track which
// row sits at each of the panel's nbp positions (row_at[]), so a row interchange of xGETF2 is pure
// bookkeeping and the first-max tie-break is decided on positions exactly as in the serial sweep
// (Z15).  Columns are factored in leaves of LW columns held in shared memory:
//   per column j of the leaf: local first-max of |a| over the unpivoted rows (key |a|, then the
//     smaller position; a NaN at position g keeps g), published with the candidate's leaf row into a
//     sequence-numbered global slot; every CTA polls the P slots (barrier and data in one) and
//     merges them; bookkeeping of the interchange; multipliers and the rank-1 update of the leaf's
//     later columns, fused with the next column's local argmax;
//   per leaf: the leaf written back; U12 = L11^{-1} A12 for the leaf's pivot rows (L11 = the
//     published pivot rows, identical in every CTA); A22 -= L21 U12 for the CTA's unpivoted rows.
// At the end the <= 2 nbp rows whose position changed are moved to their final positions (two grid
// barriers around a staging copy).  ipiv is LAPACK's (position swapped with g at step g).
// Result: the unblocked column sweep's L\U and interchanges, up to rounding.
constexpr int kLfRows = 512;           // rows per CTA
constexpr int kLfMaxP = 64;            // CTAs (slots per parity)
template <typename T> struct LfLeaf;
template <> struct LfLeaf<double> { static constexpr int v = 16; };
template <> struct LfLeaf<float> { static constexpr int v = 32; };

// self-validating exchange words of the leaf panel: (seq32 << 32) | 32-bit payload
constexpr int kLlSlot = 64;                       // words per slot
constexpr int kLlWords = 4 + 32;                  // header + 32 payload words (16 doubles / 32 floats)
template <typename T> struct LlPer;
template <> struct LlPer<double> { static constexpr int v = 2; };
template <> struct LlPer<float> { static constexpr int v = 1; };
AS_DEV unsigned ll_half(double x, int h) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(x);
    return h == 0 ? (unsigned)(b >> 32) : (unsigned)b;
}
AS_DEV unsigned ll_half(float x, int) { return __float_as_uint(x); }
template <typename T> AS_DEV T ll_join(unsigned a, unsigned b);
template <> AS_DEV double ll_join<double>(unsigned a, unsigned b) {
    return __longlong_as_double((long long)(((unsigned long long)a << 32) | b));
}
template <> AS_DEV float ll_join<float>(unsigned a, unsigned) { return __uint_as_float(a); }
AS_DEV void st_relaxed64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}


template <typename T, int LW>
struct LfSmem {
    T S[kLfRows * LW];                 // leaf columns of my rows, column-major (stride kLfRows)
    T U12[LW * kPW];                   // [k][c] leaf rows of U12 for the panel's later columns
    T LU11[LW * LW];                   // [jj][c] published pivot rows of the leaf (L11 \ U11)
    T ubuf[LW];
    int pos[kLfRows];                  // current position of my row (>= 0) or -(final position) - 1
    int row_at[kPW];                   // row in W at panel position k0 + i
    int pivrow[LW];
    double cv[8];
    int cpos[8], crow[8];
    double wv;
    int wpos, wrow, wown, nmoved;
};

// lexicographic candidate order: larger |a| first, then the smaller position
template <typename T>
AS_DEV bool lf_better(T v2, int p2, T v, int p) { return v2 > v || (v2 == v && p2 < p); }

template <typename T, int LW>
__global__ void __launch_bounds__(kPT, 2) lu_panel_lf_kernel(T* W, int64_t ldw, int64_t n, int64_t k0, int nbp,
                                                             int64_t* ipiv, DevState* st, unsigned long long* llx,
                                                             T* stage, int* stage_dst, T* ubufg, unsigned* ctr,
                                                             unsigned long long seq_base,
                                                             unsigned long long* tr_min, unsigned long long* tr_max) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    LfSmem<T, LW>& sm = *(LfSmem<T, LW>*)smem_raw;
    constexpr int kLlPer = LlPer<T>::v;
    static_assert(LW * kLlPer == kLlWords - 4, "a leaf row is 32 exchange words");
    if (tr_min && threadIdx.x == 0) atomicMin(tr_min, gtimer());
    const int P = gridDim.x, cta = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t m = n - k0;
    const int chunk = (int)((m + P - 1) / P);
    const int64_t rbeg = k0 + (int64_t)cta * chunk;             // my rows of W: rbeg .. rbeg + nr
    const int nr = (int)max<int64_t>(0, min<int64_t>(n, rbeg + chunk) - rbeg);
    constexpr int RPT = kLfRows / kPT;
    for (int r = tid; r < nr; r += kPT) sm.pos[r] = (int)(rbeg + r);
    for (int i = tid; i < nbp; i += kPT) sm.row_at[i] = (int)(k0 + i);
    unsigned long long info = ~0ull;
    T bv = T(-1);                      // this thread's candidate for the next column
    int bp = 0x7fffffff, br = -1;
    bool bnan = false;                 // the row at position g holds a NaN

    // thread candidate -> CTA candidate (sm.cv[0] / cpos / crow); one barrier
    auto cta_argmax = [&](int64_t g) {
        unsigned kh = 0u, kl = 0u;
        if (br >= 0) cand_key<T>(bv, kh, kl);
        const unsigned mh = __reduce_max_sync(0xffffffffu, kh);
        const unsigned ml = __reduce_max_sync(0xffffffffu, kh == mh ? kl : 0u);
        const unsigned mp = __reduce_min_sync(0xffffffffu, (mh != 0u && kh == mh && kl == ml) ? (unsigned)bp : 0xffffffffu);
        const unsigned wl = __ballot_sync(0xffffffffu, mh != 0u && kh == mh && kl == ml && (unsigned)bp == mp);
        const int src = wl ? __ffs(wl) - 1 : 0;
        const T wv = __shfl_sync(0xffffffffu, bv, src);
        const int wr = __shfl_sync(0xffffffffu, br, src);
        const bool dn = __any_sync(0xffffffffu, bnan);
        if (lane == 0) {
            sm.cv[warp] = dn ? (double)INFINITY : (wl ? (double)wv : -1.0);
            sm.cpos[warp] = dn ? (int)g : (wl ? (int)mp : 0x7fffffff);
            sm.crow[warp] = dn ? -2 : (wl ? wr : -1);       // -2: the row at g (found below)
        }
        __syncthreads();
        if (warp == 0) {
            double v = lane < 8 ? sm.cv[lane] : -1.0;
            int pp = lane < 8 ? sm.cpos[lane] : 0x7fffffff;
            int rr = lane < 8 ? sm.crow[lane] : -1;
#pragma unroll
            for (int o = 4; o > 0; o >>= 1) {
                const double v2 = __shfl_xor_sync(0xffffffffu, v, o);
                const int p2 = __shfl_xor_sync(0xffffffffu, pp, o);
                const int r2 = __shfl_xor_sync(0xffffffffu, rr, o);
                if (lf_better(v2, p2, v, pp)) { v = v2; pp = p2; rr = r2; }
            }
            if (lane == 0) { sm.cv[0] = v; sm.cpos[0] = pp; sm.crow[0] = rr; }
        }
    };
    // local candidate of column jj (leaf-local) from scratch over my unpivoted rows
    auto scan = [&](int jj, int64_t g) {
        bv = T(-1); bp = 0x7fffffff; br = -1; bnan = false;
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
            const int r = tid + kPT * i;
            if (r < nr && sm.pos[r] >= 0) {
                T a = sm.S[r + jj * kLfRows];
                a = a < T(0) ? -a : a;
                if (a != a) { if (sm.pos[r] == g) bnan = true; continue; }
                if (lf_better(a == T(0) ? T(0) : a, sm.pos[r], bv, bp)) { bv = a == T(0) ? T(0) : a; bp = sm.pos[r]; br = r; }
            }
        }
    };

    for (int L = 0; L < nbp; L += LW) {
        const int lw = min(LW, nbp - L);
        // ---- load the leaf columns of my rows (W is in original row order during the panel)
        batched<8, T>(
            nr * lw, [&](int e) -> T { const int c = e / nr, r = e - c * nr; return __ldcg(&W[(rbeg + r) + (k0 + L + c) * ldw]); },
            [&](int e, T v) { const int c = e / nr, r = e - c * nr; sm.S[r + c * kLfRows] = v; });
        __syncthreads();
        scan(0, k0 + L);
        for (int jj = 0; jj < lw; ++jj) {
            const int j = L + jj;
            const int64_t g = k0 + j;
            const int par = j & 1;
            cta_argmax(g);
            __syncthreads();
            // ---- publish my candidate (its leaf row) and poll everyone's
            if (warp == 0) {
                int crow = sm.crow[0];
                if (crow == -2) {                     // NaN at position g: that row (mine) wins by rule
                    for (int r = 0; r < nr; ++r) if (sm.pos[r] == (int)g) { crow = r; break; }
                }
                if (P > 1) {
                    // self-validating exchange words (seq32 << 32 | payload32): no flag + data round
                    // trips, no fences per column.  Slot = [|v| hi, |v| lo, pos, row, leaf row values]
                    const unsigned sq = (unsigned)(seq_base + (unsigned long long)j + 1ull);
                    unsigned long long* mine = llx + ((int64_t)par * kLfMaxP + cta) * kLlSlot;
                    if (jj == 0) fence_acq_rel();     // my last trailing update before my first word of the leaf
                    {
                        const unsigned long long vb = (unsigned long long)__double_as_longlong(sm.cv[0]);
                        const long long rowg = crow >= 0 ? rbeg + crow : -1;
                        for (int w = lane; w < kLlWords; w += 32) {
                            unsigned pl;
                            if (w == 0) pl = (unsigned)(vb >> 32);
                            else if (w == 1) pl = (unsigned)vb;
                            else if (w == 2) pl = (unsigned)sm.cpos[0];
                            else if (w == 3) pl = (unsigned)rowg;
                            else {
                                const int e = (w - 4) / kLlPer, h = (w - 4) % kLlPer;
                                const T x = (crow >= 0 && e < lw) ? sm.S[crow + e * kLfRows] : T(0);
                                pl = ll_half(x, h);
                            }
                            st_relaxed64(mine + w, ((unsigned long long)sq << 32) | pl);
                        }
                    }
                    // phase 1: the 4 header words of every slot (lane l: word l & 3 of slots l/4 + 8k)
                    unsigned long long hw[kLfMaxP / 8];
                    bool ok[kLfMaxP / 8];
#pragma unroll
                    for (int k = 0; k < kLfMaxP / 8; ++k) ok[k] = (lane >> 2) + 8 * k >= P;
                    for (;;) {
                        bool all = true;
#pragma unroll
                        for (int k = 0; k < kLfMaxP / 8; ++k)
                            if (!ok[k]) {
                                const int q = (lane >> 2) + 8 * k;
                                hw[k] = ld_relaxed64(llx + ((int64_t)par * kLfMaxP + q) * kLlSlot + (lane & 3));
                                ok[k] = (unsigned)(hw[k] >> 32) == sq;
                                all = all && ok[k];
                            }
                        if (__all_sync(0xffffffffu, all)) break;
                    }
                    double v = -1.0;
                    int pp = 0x7fffffff, ow = 0;
                    long long rw = -1;
                    const int gb = lane & ~3;
#pragma unroll
                    for (int k = 0; k < kLfMaxP / 8; ++k) {
                        const unsigned w0 = __shfl_sync(0xffffffffu, (unsigned)hw[k], gb + 0);
                        const unsigned w1 = __shfl_sync(0xffffffffu, (unsigned)hw[k], gb + 1);
                        const unsigned w2 = __shfl_sync(0xffffffffu, (unsigned)hw[k], gb + 2);
                        const unsigned w3 = __shfl_sync(0xffffffffu, (unsigned)hw[k], gb + 3);
                        const int q = (lane >> 2) + 8 * k;
                        if (q >= P) continue;
                        const double v2 = __longlong_as_double((long long)(((unsigned long long)w0 << 32) | w1));
                        const int p2 = (int)w2;
                        if (lf_better(v2, p2, v, pp)) { v = v2; pp = p2; ow = q; rw = (long long)(int)w3; }
                    }
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) {
                        const double v2 = __shfl_xor_sync(0xffffffffu, v, o);
                        const int p2 = __shfl_xor_sync(0xffffffffu, pp, o);
                        const int o2 = __shfl_xor_sync(0xffffffffu, ow, o);
                        const long long r2 = __shfl_xor_sync(0xffffffffu, rw, o);
                        if (lf_better(v2, p2, v, pp)) { v = v2; pp = p2; ow = o2; rw = r2; }
                    }
                    // phase 2: the winner's leaf row (one word per lane)
                    {
                        const unsigned long long* src = llx + ((int64_t)par * kLfMaxP + ow) * kLlSlot + 4;
                        unsigned long long x = 0;
                        if (lane < kLlWords - 4) {
                            do { x = ld_relaxed64(src + lane); } while ((unsigned)(x >> 32) != sq);
                        }
                        const T val = ll_join<T>((unsigned)x, __shfl_down_sync(0xffffffffu, (unsigned)x, 1));
                        const int e = lane / kLlPer;
                        if (lane % kLlPer == 0 && e < lw) sm.ubuf[e] = val;
                    }
                    if (jj == lw - 1) fence_acq_rel();  // the leaf's pivot rows (A12) are read next
                    if (lane == 0) { sm.wpos = pp; sm.wrow = (int)rw; sm.wown = ow; }
                } else {
                    if (lane < lw) sm.ubuf[lane] = sm.S[crow + lane * kLfRows];
                    if (lane == 0) { sm.wpos = sm.cpos[0]; sm.wrow = (int)(rbeg + crow); sm.wown = 0; }
                }
            }
            __syncthreads();
            // ---- the interchange (bookkeeping only) and the pivot row
            const T piv = sm.ubuf[jj];
            const int p = sm.wpos, rs = sm.wrow;
            const bool elim = piv != T(0);
            if (tid == 0) {
                const int q = sm.row_at[j];            // the row currently at position g
                if (cta == 0) ipiv[g] = elim ? p : g;
                if (!elim && info == ~0ull) info = (unsigned long long)(g + 1);
                const int ps = elim ? p : (int)g;
                const int rpiv = elim ? rs : q;        // zero pivot: no interchange (the serial sweep's rule)
                sm.row_at[j] = rpiv;
                if (elim && ps - k0 < nbp && ps != g) sm.row_at[ps - k0] = q;
                if (elim && q != rpiv && q >= rbeg && q < rbeg + nr) sm.pos[q - rbeg] = ps;
                if (rpiv >= rbeg && rpiv < rbeg + nr) sm.pos[rpiv - rbeg] = -(int)g - 1;
                sm.pivrow[jj] = rpiv;
            }
            if (tid < lw) sm.LU11[jj * LW + tid] = sm.ubuf[tid];
            __syncthreads();
            // ---- multipliers, rank-1 update of the leaf's later columns, next column's candidate
            bv = T(-1); bp = 0x7fffffff; br = -1; bnan = false;
            const bool more = jj + 1 < lw;
#pragma unroll
            for (int i = 0; i < RPT; ++i) {
                const int r = tid + kPT * i;
                if (r >= nr || sm.pos[r] < 0) continue;
                T* Sr = sm.S + r;
                if (elim) {
                    const T l = Sr[jj * kLfRows] / piv;
                    Sr[jj * kLfRows] = l;
                    for (int c = jj + 1; c < lw; ++c) Sr[c * kLfRows] -= l * sm.ubuf[c];
                }
                if (more) {
                    T a = Sr[(jj + 1) * kLfRows];
                    a = a < T(0) ? -a : a;
                    if (a != a) { if (sm.pos[r] == g + 1) bnan = true; continue; }
                    if (a == T(0)) a = T(0);
                    if (lf_better(a, sm.pos[r], bv, bp)) { bv = a; bp = sm.pos[r]; br = r; }
                }
            }
        }
        __syncthreads();
        // ---- leaf done: write it back (original row order)
        batched<8, T>(
            nr * lw, [&](int e) -> T { const int c = e / nr, r = e - c * nr; return sm.S[r + c * kLfRows]; },
            [&](int e, T v) { const int c = e / nr, r = e - c * nr; W[(rbeg + r) + (k0 + L + c) * ldw] = v; });
        const int c0 = L + lw, rest = nbp - c0;
        if (rest > 0) {
            // U12 = L11^{-1} A12 on the leaf's pivot rows (their owners updated them before publishing
            // this leaf's candidates, so the acquire of the slots made them visible)
            for (int c = tid; c < rest; c += kPT) {
                T u[LW];
#pragma unroll
                for (int k = 0; k < LW; ++k)
                    if (k < lw) u[k] = __ldcg(&W[(int64_t)sm.pivrow[k] + (k0 + c0 + c) * ldw]);
#pragma unroll
                for (int k = 0; k < LW; ++k) {
                    if (k >= lw) break;
#pragma unroll
                    for (int i2 = 0; i2 < k; ++i2) u[k] -= sm.LU11[k * LW + i2] * u[i2];
                    sm.U12[k * kPW + c] = u[k];
                }
            }
            __syncthreads();
            // the leaf's U12 rows go to Ubuf (by position), NOT to the pivot rows in W: other CTAs may
            // still be reading those rows' A12 for their own (redundant) U12; the final row moves put
            // them in place.  My unpivoted rows: A22 -= L21 U12.
            if (cta == 0)
                for (int e = tid; e < lw * rest; e += kPT) {
                    const int k = e / rest, c = e - k * rest;
                    ubufg[(int64_t)(L + k) * kPW + c0 + c] = sm.U12[k * kPW + c];
                }
            // (one row at a time, 16 columns per batch: 16 independent loads in flight per thread)
            constexpr int CB = 16;
#pragma unroll 1
            for (int i = 0; i < RPT; ++i) {
                const int r = tid + kPT * i;
                if (r >= nr || sm.pos[r] < 0) continue;
                T l[LW];
#pragma unroll
                for (int k = 0; k < LW; ++k) l[k] = k < lw ? sm.S[r + k * kLfRows] : T(0);
                T* Wr = W + (rbeg + r) + (k0 + c0) * ldw;
#pragma unroll 1
                for (int c = 0; c < rest; c += CB) {
                    T a[CB];
#pragma unroll
                    for (int q = 0; q < CB; ++q) a[q] = c + q < rest ? __ldcg(&Wr[(int64_t)(c + q) * ldw]) : T(0);
#pragma unroll
                    for (int k = 0; k < LW; ++k)
#pragma unroll
                        for (int q = 0; q < CB; ++q) a[q] -= l[k] * sm.U12[k * kPW + min(c + q, kPW - 1)];
#pragma unroll
                    for (int q = 0; q < CB; ++q)
                        if (c + q < rest) Wr[(int64_t)(c + q) * ldw] = a[q];
                }
            }
        }
        __syncthreads();
    }
    // ---- final rows: every pivot row (its U part beyond its leaf from Ubuf) and every row whose
    // position changed are staged, grid barrier, scattered to their final positions
    unsigned gen = 0;
    if (P > 1) grid_barrier(ctr, ++gen, (unsigned)P);
    else __syncthreads();
    for (int r = warp; r < nr; r += kPT / 32) {
        const int ps = sm.pos[r];
        const int fin = ps >= 0 ? ps : -ps - 1;
        if (ps >= 0 && fin == (int)(rbeg + r)) continue;
        const int gi = fin - (int)k0;
        const int lend = ps >= 0 ? nbp : min(nbp, (gi / LW + 1) * LW);
        int slot = 0;
        if (lane == 0) slot = (int)atomicAdd(ctr + 1, 1u);
        slot = __shfl_sync(0xffffffffu, slot, 0);
        for (int c = lane; c < nbp; c += 32)
            stage[(int64_t)slot * kPW + c] = c < lend ? __ldcg(&W[(rbeg + r) + (k0 + c) * ldw])
                                                      : __ldcg(&ubufg[(int64_t)gi * kPW + c]);
        if (lane == 0) stage_dst[slot] = fin;
    }
    if (P > 1) grid_barrier(ctr, ++gen, (unsigned)P);
    else __syncthreads();
    const int nmv = (int)__ldcg(ctr + 1);
    for (int e = cta * kPT + tid; e < nmv * nbp; e += P * kPT) {
        const int sl = e / nbp, c = e - sl * nbp;
        W[(int64_t)__ldcg(&stage_dst[sl]) + (k0 + c) * ldw] = __ldcg(&stage[(int64_t)sl * kPW + c]);
    }
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
// ------------------------------------------------------------------ fused interchanges + U12 (v2)
// The block's full 128 x 128 inverse L11^{-1} = [La^{-1} 0; -Lc^{-1} Lb La^{-1}  Lc^{-1}] is formed once
// per block (linv128_kernel, after the panel) so that U12 = L11^{-1} A12 is ONE product per column
// tile; a CTA takes 64 trailing columns: the interchanges composed into one permutation (as above),
// every moved value gathered before any store, then U12 = L11^{-1} Bn with L11^{-1} streamed through
// L1 (4 rows x 8 columns per thread).
struct SwapPlan {
    int64_t srow[2 * kBW];   // [0, bw): source row of block position q; [bw, bw + ne): rows leaving the block
    int64_t edst[kBW];       // destination row of leaving value e
    int ne;
    int pad;
};
constexpr int kSU3C = 16;
constexpr int kSU3LD = kBW + 1;

template <typename T>
__device__ void swap_plan_build(const int64_t* ipiv, int64_t k0, int bw, SwapPlan* plan) {
    __shared__ int64_t piv[kBW];
    __shared__ int s_ne;
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
        if (pos < k0 + bw) plan->srow[pos - k0] = x;
        else { const int e = atomicAdd(&s_ne, 1); plan->edst[e] = pos; plan->srow[bw + e] = x; }
    }
    __syncthreads();
    if (threadIdx.x == 0) plan->ne = s_ne;
}

constexpr int kSU2C = 64;
constexpr int kSU2LD = kBW + 1;
template <typename T>
__global__ void __launch_bounds__(256) linv128_kernel(const T* W, int64_t ldw, int64_t k0, int bw, const T* Dinv,
                                                      T* Linv, const int64_t* ipiv, SwapPlan* plan) {
    if (blockIdx.x == kBW / 16) { swap_plan_build<T>(ipiv, k0, bw, plan); return; }   // the extra CTA
    // CTA c writes columns [16 c, 16 c + 16) of the 128 x 128 inverse; CTAs 0..3 form their slice of
    // the off-diagonal block C = -Lc^{-1} (Lb La^{-1}) (two 64 x 64 x 16 products)
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* Ci = (T*)smem_raw;                // 64 x 64
    T* Lb = Ci + kB64 * kB64;            // 64 x 64
    T* Aic = Lb + kB64 * kB64;           // 64 x 16 (La^{-1} columns of the slice)
    T* T1 = Aic + kB64 * 16;             // 64 x 16
    const int p1 = min(kB64, bw), p2 = bw - p1;
    const T* Da = Dinv + (k0 / kB64) * (int64_t)kB64 * kB64;
    const int cb = blockIdx.x * 16;      // first output column
    const bool left = cb < kB64;
    if (left && p2 > 0) {
        for (int e = threadIdx.x; e < kB64 * kB64; e += 256) {
            const int r = e & 63, c = e >> 6;
            Ci[e] = Da[kB64 * kB64 + e];
            Lb[e] = (r < p2 && c < p1) ? W[(k0 + kB64 + r) + (k0 + c) * ldw] : T(0);
        }
        for (int e = threadIdx.x; e < kB64 * 16; e += 256) Aic[e] = Da[(e & 63) + (cb + (e >> 6)) * kB64];
        __syncthreads();
        for (int e = threadIdx.x; e < kB64 * 16; e += 256) {      // T1 = Lb La^{-1}(:, slice)
            const int r = e & 63, c = e >> 6;
            T acc = T(0);
            for (int k = 0; k < kB64; ++k) acc += Lb[r + k * kB64] * Aic[k + c * kB64];
            T1[e] = acc;
        }
        __syncthreads();
    }
    for (int e = threadIdx.x; e < kBW * 16; e += 256) {
        const int r = e & (kBW - 1), c = cb + (e >> 7);
        T v;
        if (r < kB64) v = c < kB64 ? (r == c ? T(1) : Da[r + c * kB64]) : T(0);
        else if (c >= kB64) v = r == c ? T(1) : (p2 > 0 ? Da[kB64 * kB64 + (r - kB64) + (c - kB64) * kB64] : T(0));
        else if (p2 > 0) {                                          // -Lc^{-1} (Lb La^{-1})
            T acc = T(0);
            for (int k = 0; k < kB64; ++k) acc += Ci[(r - kB64) + k * kB64] * T1[k + (c - cb) * kB64];
            v = -acc;
        } else v = T(0);
        if (r >= bw || c >= bw) v = r == c ? T(1) : T(0);
        Linv[r + (int64_t)c * kBW] = v;
    }
}

template <typename T>
__global__ void __launch_bounds__(256) swap_u12v2_kernel(T* W, int64_t ldw, int64_t k0, int bw, int64_t c0, int64_t c1,
                                                        const int64_t* ipiv, const T* __restrict__ Linv) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* Bn = (T*)smem_raw;                // [kSU2C][kSU2LD]: column c of the block rows after the interchanges
    T* Ex = Bn + kSU2C * kSU2LD;         // [kSU2C][kSU2LD]: values for the rows leaving the block
    __shared__ int64_t piv[kBW];
    __shared__ int64_t srow[2 * kBW];
    __shared__ int64_t edst[kBW];
    __shared__ int s_ne;
    const int64_t cc0 = c0 + (int64_t)blockIdx.x * kSU2C;
    const int nc = (int)min<int64_t>(kSU2C, c1 - cc0);
    if (nc <= 0) return;
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
    __syncthreads();
    const int ne = s_ne, R = bw + ne;
    batched<16, T>(
        R * nc, [&](int e) -> T { const int c = e / R, row = e - c * R; return W[srow[row] + (cc0 + c) * ldw]; },
        [&](int e, T v) {
            const int c = e / R, row = e - c * R;
            if (row < bw) Bn[c * kSU2LD + row] = v;
            else Ex[c * kSU2LD + row - bw] = v;
        });
    __syncthreads();
    for (int e = threadIdx.x; e < ne * nc; e += blockDim.x) {
        const int c = e / ne, row = e - c * ne;
        W[edst[row] + (cc0 + c) * ldw] = Ex[c * kSU2LD + row];
    }
    // U12 = L11^{-1} Bn: lane -> rows lane + 32 i, warp -> columns 8 warp .. 8 warp + 7
    const int lane = threadIdx.x & 31, cg = (threadIdx.x >> 5) * 8;
    T acc[4][8];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int u = 0; u < 8; ++u) acc[i][u] = T(0);
    const int kmax = min(bw, 96 + lane + 1);            // L11^{-1} is lower triangular: k <= row
    for (int k = 0; k < kmax; ++k) {
        T l[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) l[i] = __ldg(&Linv[(lane + 32 * i) + k * kBW]);
        T bv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) bv[u] = Bn[(cg + u) * kSU2LD + k];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int u = 0; u < 8; ++u) acc[i][u] += l[i] * bv[u];
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        const int c = cg + u;
        if (c >= nc) continue;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int r = lane + 32 * i;
            if (r < bw) W[(k0 + r) + (cc0 + c) * ldw] = acc[i][u];
        }
    }
}

// ------------------------------------------------------------------ fused interchanges + U12, v3
// The composed permutation of a block's interchanges depends only on ipiv: it is formed once per
// block (the extra CTA of linv128_kernel) into a SwapPlan instead of by every CTA of every launch,
// and a CTA takes NC = 16 trailing columns (33 KB of shared memory, 6 CTAs per SM, 4x the CTAs of
// the 64-column kernel: the r02 launch list showed 57 us per launch at 64 CTAs x 132 KB, one CTA per
// SM, against ~2 us of fp64 work).  L11^{-1} is lower triangular: the product visits k in four
// blocks of 32 and row group i (rows lane + 32 i) only for i >= k / 32 (62.5 % of the FMAs).
template <typename T, int NC>
__global__ void __launch_bounds__(256) swap_u12v3_kernel(T* W, int64_t ldw, int64_t k0, int bw, int64_t c0, int64_t c1,
                                                        const SwapPlan* __restrict__ plan, const T* __restrict__ Linv,
                                                        int noswap) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* Bn = (T*)smem_raw;                // [NC][kSU3LD]: column c of the block rows after the interchanges
    T* Ex = Bn + NC * kSU3LD;            // [NC][kSU3LD]: values for the rows leaving the block
    __shared__ int64_t srow[2 * kBW];
    __shared__ int64_t edst[kBW];
    const int64_t cc0 = c0 + (int64_t)blockIdx.x * NC;
    const int nc = (int)min<int64_t>(NC, c1 - cc0);
    if (nc <= 0) return;
    // noswap: the interchanges were applied already (two-panel blocks): U12 = L11^{-1} A12 only
    const int ne = noswap ? 0 : plan->ne, R = bw + ne;
    for (int t = threadIdx.x; t < R; t += blockDim.x) srow[t] = noswap ? k0 + t : plan->srow[t];
    for (int t = threadIdx.x; t < ne; t += blockDim.x) edst[t] = plan->edst[t];
    __syncthreads();
    batched<16, T>(
        R * nc, [&](int e) -> T { const int c = e / R, row = e - c * R; return W[srow[row] + (cc0 + c) * ldw]; },
        [&](int e, T v) {
            const int c = e / R, row = e - c * R;
            if (row < bw) Bn[c * kSU3LD + row] = v;
            else Ex[c * kSU3LD + row - bw] = v;
        });
    __syncthreads();
    for (int e = threadIdx.x; e < ne * nc; e += blockDim.x) {
        const int c = e / ne, row = e - c * ne;
        W[edst[row] + (cc0 + c) * ldw] = Ex[c * kSU3LD + row];
    }
    // U12 = L11^{-1} Bn: lane -> rows lane + 32 i, warp -> columns CW warp .. CW warp + CW - 1
    constexpr int CW = NC / 8;
    const int lane = threadIdx.x & 31, cg = (threadIdx.x >> 5) * CW;
    T acc[4][CW];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int u = 0; u < CW; ++u) acc[i][u] = T(0);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int kend = min(32 * j + 32, bw);
#pragma unroll 4
        for (int k = 32 * j; k < kend; ++k) {
            T l[4], bv[CW];
#pragma unroll
            for (int i = j; i < 4; ++i) l[i] = __ldg(&Linv[(lane + 32 * i) + k * kBW]);
#pragma unroll
            for (int u = 0; u < CW; ++u) bv[u] = Bn[(cg + u) * kSU3LD + k];
#pragma unroll
            for (int i = j; i < 4; ++i)
#pragma unroll
                for (int u = 0; u < CW; ++u) acc[i][u] += l[i] * bv[u];
        }
    }
#pragma unroll
    for (int u = 0; u < CW; ++u) {
        const int c = cg + u;
        if (c >= nc) continue;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int r = lane + 32 * i;
            if (r < bw) W[(k0 + r) + (cc0 + c) * ldw] = acc[i][u];
        }
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
    cudaStream_t aux = nullptr;    // second stream of the chunked swap + U12 / trailing GEMM
    cudaEvent_t ev[64];
    cudaEvent_t evl[2];            // dataflow schedule: "block k's panel is ready" (by step parity)
    cudaEvent_t evc[4][2];         // dataflow schedule: chunk q finished step k (by step parity)
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
        cudaStreamCreateWithPriority(&L.aux, cudaStreamNonBlocking, lo);
        for (auto& e : L.ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
        for (auto& e : L.evl) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
        for (auto& r : L.evc) for (auto& e : r) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    }
    return L;
}

static int g_panel_dbg = 0;   // diagnostics: phase counters of the cluster panel (lu_debug_panel_time)

// lfbuf layout (Work::lfbuf, lf_layout): per-block counters, exchange slots, candidate rows,
// staging for the final row moves
struct LfBufs {
    unsigned* ctr;       // [2 * nblk]: grid barrier, staging count (zeroed per factorization)
    unsigned long long* llx;   // [2][kLfMaxP][kLlSlot] self-validating exchange words
    int* stage_dst;      // [2 * kPW]
    void* stage;         // [2 * kPW][kPW]
    void* ubuf;          // [kPW][kPW] U rows of the panel by position (beyond each pivot row's leaf)
    size_t zero_bytes;   // ctr + llx (zeroed per factorization: stale words of an earlier call never match)
};
static LfBufs lf_layout(void* base, int64_t n, size_t es) {
    LfBufs b{};
    const int64_t nblk = (n + kBW - 1) / kBW;
    char* p = (char*)base;
    auto take = [&](size_t bytes) { char* q = p; p += (bytes + 255) & ~(size_t)255; return q; };
    b.ctr = (unsigned*)take(sizeof(unsigned) * 2 * (size_t)nblk);
    b.llx = (unsigned long long*)take(sizeof(unsigned long long) * 2 * kLfMaxP * kLlSlot);
    b.zero_bytes = (size_t)(p - (char*)base);
    b.stage_dst = (int*)take(sizeof(int) * 2 * kPW);
    b.stage = take(es * 2 * kPW * kPW);
    b.ubuf = take(es * kPW * kPW);
    return b;
}
size_t lu_swplan_bytes(int64_t n) { return sizeof(SwapPlan) * (size_t)((n + kBW - 1) / kBW); }
size_t lu_lfbuf_bytes(int64_t n, int dtype) { return (size_t)(lf_layout(nullptr, n, dtype == AS_F64 ? 8 : 4).ubuf) +
                                                     (dtype == AS_F64 ? 8 : 4) * kPW * kPW; }

// The leaf panel: P = ceil(m / kLfRows) CTAs of one ordinary launch (see lu_panel_lf_kernel).
template <typename T>
static bool lf_panel_launch(const Work& w, int64_t k0, int nbp, unsigned long long seq_base, int prio, cudaStream_t s) {
    const int64_t n = w.n, m = n - k0;
    const int P = (int)((m + kLfRows - 1) / kLfRows);
    if (P > kLfMaxP || P > w.num_sms || nbp > kPW || !w.lfbuf) return false;
    constexpr int LW = LfLeaf<T>::v;
    auto kern = lu_panel_lf_kernel<T, LW>;
    const size_t smem = sizeof(LfSmem<T, LW>);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    LfBufs b = lf_layout(w.lfbuf, n, sizeof(T));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(P);
    cfg.blockDim = dim3(kPT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributePriority; at[0].val.priority = prio;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    LuTrace& tr = lu_trace();
    const int slot = (int)(k0 / kBW) * 4 + 1;
    unsigned long long* tmn = tr.tmin && k0 / kBW < kTraceBlocks ? tr.tmin + slot : nullptr;
    unsigned long long* tmx = tr.tmax && k0 / kBW < kTraceBlocks ? tr.tmax + slot : nullptr;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, (T*)w.W, w.ldw, n, k0, nbp, w.ipiv, w.st, b.llx,
                                             (T*)b.stage, b.stage_dst, (T*)b.ubuf, b.ctr + 2 * (k0 / kBW), seq_base, tmn,
                                             tmx);
    if (e != cudaSuccess) { cudaGetLastError(); return false; }
    return true;
}

template <typename T>
static void panel_launch(const Work& w, int64_t k0, int nbp, unsigned long long seq_base, int prio, cudaStream_t s) {
    const int64_t n = w.n, m = n - k0;
    // Panel policy: rows that fit in <= kClMax CTAs' shared memory -> one cluster (DSMEM exchange);
    // taller panels -> the leaf panel on ceil(m / 1024) CTAs (the trailing GEMM keeps the other
    // SMs); AS_LU_PANEL=coop forces the cooperative panel (m / 128 CTAs, measured slower on C5).
    const char* pol = getenv("AS_LU_PANEL");
    const bool coop = pol && strcmp(pol, "coop") == 0;
    static const int rows_per_cta = getenv("AS_LU_PANEL_ROWS") ? atoi(getenv("AS_LU_PANEL_ROWS")) : 128;
    int P = (int)std::min<int64_t>(w.num_sms, (m + rows_per_cta - 1) / rows_per_cta);
    P = std::max(P, 1);
    if (!coop && getenv("AS_LU_NO_CLUSTER") == nullptr) {
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
            cfg.blockDim = dim3(kPT2);
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
    // the leaf panel beside the big GEMMs (it leaves the SMs to them); below lf_min_m rows the GEMM of
    // a block is shorter than a leaf panel (~0.9 ms per 128 columns: latency of the per-column
    // multi-CTA exchange) and the faster cooperative panel (rows in shared memory, ~0.45 ms) wins even
    // though it occupies m/128 SMs
    static const int64_t lf_min_m = getenv("AS_LU_LF_MIN_M") ? atoll(getenv("AS_LU_LF_MIN_M")) : 12288;
    if (!coop && m > lf_min_m && lf_panel_launch<T>(w, k0, nbp, seq_base, prio, s)) return;
    const int64_t chunk = (m + P - 1) / P;
    size_t smem = sizeof(T) * ((chunk | 1) * nbp + nbp);
    int use_smem = 1;
    if (smem > 200 * 1024) { use_smem = 0; smem = sizeof(T) * nbp; }
    auto kern = lu_panel2_kernel<T>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)std::max<size_t>(smem, 1024));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(P);
    cfg.blockDim = dim3(kPT2);
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
    static const unsigned poll_nap = getenv("AS_LU_POLL_NAP") ? (unsigned)atoi(getenv("AS_LU_POLL_NAP")) : 0u;
    cudaLaunchKernelEx(&cfg, kern, (T*)w.W, w.ldw, n, k0, nbp, w.ipiv, w.st, (unsigned long long*)w.cand, seq_base,
                       use_smem, tmn, tmx, poll_nap);
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
    if (w.linv && k0 + nbp < w.n) {      // the full block inverse for the fused interchanges + U12
        const int sm2 = (int)(sizeof(T) * (2 * kB64 * kB64 + 2 * kB64 * 16));
        cudaFuncSetAttribute(linv128_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm2);
        linv128_kernel<T><<<kBW / 16 + (w.swplan ? 1 : 0), 256, sm2, s>>>(
            (const T*)w.W, w.ldw, k0, nbp, (const T*)w.Dinv0, (T*)w.linv + (k0 / kBW) * (int64_t)kBW * kBW, w.ipiv,
            w.swplan ? (SwapPlan*)w.swplan + k0 / kBW : nullptr);
    }
}

template <typename T>
static void swap_u12_launch(const Work& w, int64_t k0, int bw, int64_t c0, int64_t c1, cudaStream_t s, bool noswap = false) {
    if (c1 <= c0) return;
    if (noswap) {
        const int smem = (int)(sizeof(T) * 2 * kSU3C * kSU3LD);
        swap_u12v3_kernel<T, kSU3C><<<(unsigned)((c1 - c0 + kSU3C - 1) / kSU3C), 256, smem, s>>>(
            (T*)w.W, w.ldw, k0, bw, c0, c1, (const SwapPlan*)w.swplan + k0 / kBW,
            (const T*)w.linv + (k0 / kBW) * (int64_t)kBW * kBW, 1);
        return;
    }
    static const bool v1 = getenv("AS_LU_SWAP_V1") != nullptr;
    // the 16-column kernel (r02o, C5, same run: 163.3 ms against 170.3 with the 64-column kernel
    // everywhere and 167.2 with it on the bulk only; AS_LU_SWAP_V3_MAXC=c keeps it to launches of <= c columns)
    static const int64_t v3_maxc = getenv("AS_LU_SWAP_V3_MAXC") ? atoll(getenv("AS_LU_SWAP_V3_MAXC")) : (int64_t)1 << 40;
    if (w.linv && w.swplan && !v1 && c1 - c0 <= v3_maxc) {
        const int smem = (int)(sizeof(T) * 2 * kSU3C * kSU3LD);
        swap_u12v3_kernel<T, kSU3C><<<(unsigned)((c1 - c0 + kSU3C - 1) / kSU3C), 256, smem, s>>>(
            (T*)w.W, w.ldw, k0, bw, c0, c1, (const SwapPlan*)w.swplan + k0 / kBW,
            (const T*)w.linv + (k0 / kBW) * (int64_t)kBW * kBW, 0);
        return;
    }
    if (w.linv && !v1) {
        const int smem = (int)(sizeof(T) * 2 * kSU2C * kSU2LD);
        cudaFuncSetAttribute(swap_u12v2_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        swap_u12v2_kernel<T><<<(unsigned)((c1 - c0 + kSU2C - 1) / kSU2C), 256, smem, s>>>(
            (T*)w.W, w.ldw, k0, bw, c0, c1, w.ipiv, (const T*)w.linv + (k0 / kBW) * (int64_t)kBW * kBW);
        return;
    }
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
    cudaMemsetAsync(w.cand, 0, lu_cand_bytes(), s);            // panel exchange words (sequence numbers repeat across solves)
    if (w.lfbuf) cudaMemsetAsync(w.lfbuf, 0, lf_layout(w.lfbuf, n, sizeof(T)).zero_bytes, s);   // leaf panel counters + slots
    if (lu_trace().tmin) {
        cudaMemsetAsync(lu_trace().tmin, 0xFF, sizeof(unsigned long long) * 4 * kTraceBlocks, s);
        cudaMemsetAsync(lu_trace().tmax, 0, sizeof(unsigned long long) * 4 * kTraceBlocks, s);
    }
    LuStreams& LS = lu_streams();
    const bool lookahead = n >= 2048 && getenv("AS_LU_NO_LOOKAHEAD") == nullptr;
    int evi = 0;
    auto ev = [&]() { return LS.ev[(evi++) % 64]; };
    // AS_LU_SCHED=2: two-panel blocks with a K = 256 trailing update (below; r02v: 165.1 vs 166.1 ms on C5,
    // 147.4 vs 150.6 ms on C5f -- within run-to-run spread, kept opt-in); default: the block-synchronous
    // look-ahead schedule further down.  A dataflow schedule (fixed column chunks, one stream each, no
    // per-block join) was measured slower (179.6 vs 167.2 ms) and removed.
    static const int sched = getenv("AS_LU_SCHED") ? atoi(getenv("AS_LU_SCHED")) : 0;
    if (lookahead && sched == 2 && w.linv && w.swplan && n >= 4096) {
        // Two-panel blocks: the trailing update runs with K = 256 (DMMA GEMM 87 % of peak against 82 % at
        // K = 128, half the passes over the trailing matrix, half the joins).  Per double block
        // [k0, k0 + 256) = panels A, B:
        //   columns of B:       interchanges of A + U12(A), A22 -= L21(A) U12(A), then panel B
        //   columns of A:       interchanges of B (rows below A's block; L21(A) must be in the row order
        //                       the K = 256 update sees)
        //   trailing columns:   interchanges of A + U12(A); interchanges of B; the 128-row strip of B
        //                       -= L21(A)[rows of B] U12(A); U12(B) = L11(B)^{-1} strip; then ONE update
        //                       A22 -= [L21(A) L21(B)] [U12(A); U12(B)] on the rows below the double block.
        // Look-ahead: the next double block's panel-A columns take all of this first on the
        // high-priority stream, then panel A'; panel B' follows on the same stream as soon as the
        // first chunk of the bulk update (which holds B's columns) is done.
        auto trail = [&](int64_t k0, int wa, int wb, int64_t c0, int64_t c1, cudaStream_t st, int trace_slot) {
            if (c1 <= c0) return;
            const int64_t kb = k0 + wa;
            swap_u12_launch<T>(w, k0, wa, c0, c1, st);                       // A's interchanges + U12(A)
            if (wb > 0) {
                laswp_launch<T>(w, kb, wb, c0, c1, 0, 0, false, st);          // B's interchanges
                gemm_launch<T>(w, kb, c0, k0, wb, c1 - c0, wa, st, 0);        // strip of B's rows
                swap_u12_launch<T>(w, kb, wb, c0, c1, st, true);              // U12(B) (no interchanges)
            }
            const int64_t r0 = kb + std::max(wb, 0);
            gemm_launch<T>(w, r0, c0, k0, n - r0, c1 - c0, wa + std::max(wb, 0), st, 0, false, trace_slot);
        };
        cudaEvent_t e_start = ev();
        cudaEventRecord(e_start, s);
        cudaStreamWaitEvent(LS.hi, e_start, 0);
        cudaStreamWaitEvent(LS.side, e_start, 0);
        cudaStreamWaitEvent(LS.aux, e_start, 0);
        block_panels<T>(w, 0, (int)std::min<int64_t>(kBW, n), LS.prio_hi, LS.hi);      // panel A of block 0
        cudaEvent_t ev_b_cols = nullptr;       // "the columns of the next panels B and A' are up to date"
        cudaEvent_t ev_main_done = nullptr;    // the previous double block's bulk update is complete
        int step = 0;
        for (int64_t k0 = 0; k0 < n; k0 += 2 * kBW, ++step) {
            const int wa = (int)std::min<int64_t>(kBW, n - k0);
            const int64_t kb = k0 + wa;
            const int wb = (int)std::min<int64_t>(kBW, n - kb);          // <= 0: no panel B
            const int64_t kn = kb + std::max(wb, 0);                     // next double block
            // ---- panel B (high priority): its columns get A's interchanges, U12(A) and the K = 128 update
            if (wb > 0) {
                if (ev_b_cols) cudaStreamWaitEvent(LS.hi, ev_b_cols, 0);
                swap_u12_launch<T>(w, k0, wa, kb, kb + wb, LS.hi);
                gemm_launch<T>(w, kb, kb, k0, n - kb, wb, wa, LS.hi, LS.prio_hi);
                block_panels<T>(w, kb, wb, LS.prio_hi, LS.hi);
                laswp_launch<T>(w, kb, wb, k0, k0 + wa, 0, 0, false, LS.hi);   // B's interchanges into L21(A)
            }
            cudaEvent_t ev_p = LS.evl[step & 1];
            cudaEventRecord(ev_p, LS.hi);
            // ---- finished L columns [0, k0) and the row permutation (side stream); the previous double
            // block's bulk update still reads its L21 in the old row order: wait for it
            cudaStreamWaitEvent(LS.side, ev_p, 0);
            if (ev_main_done) cudaStreamWaitEvent(LS.side, ev_main_done, 0);
            laswp_launch<T>(w, k0, wa, 0, k0, 0, 0, true, LS.side);
            if (wb > 0) laswp_launch<T>(w, kb, wb, 0, k0, 0, 0, true, LS.side);
            if (kn >= n) break;
            // ---- look-ahead: the next panel A's columns, then panel A' (high priority)
            const int wa2 = (int)std::min<int64_t>(kBW, n - kn);
            trail(k0, wa, wb, kn, kn + wa2, LS.hi, (int)(k0 / kBW) * 4 + 3);
            block_panels<T>(w, kn, wa2, LS.prio_hi, LS.hi);
            // ---- the other trailing columns in chunks alternating between two streams; the first chunk
            // holds the next panel B's columns
            cudaStreamWaitEvent(s, ev_p, 0);
            {
                cudaEvent_t ea = LS.evc[3][step & 1];      // aux continues from the joined state of s
                cudaEventRecord(ea, s);
                cudaStreamWaitEvent(LS.aux, ea, 0);
            }
            const int64_t c0r = kn + wa2, rn = n - c0r;
            ev_b_cols = nullptr;
            if (rn > 0) {
                const int nch = rn >= 4096 ? 4 : rn >= 1024 ? 2 : 1;
                for (int i = 0; i < nch; ++i) {
                    auto bnd = [&](int q) { return q >= nch ? n : c0r + std::max<int64_t>((rn * q / nch + 63) / 64 * 64, q > 0 ? 2 * kBW : 0); };
                    const int64_t a0 = std::min<int64_t>(bnd(i), n), a1 = std::min<int64_t>(bnd(i + 1), n);
                    cudaStream_t st = (i & 1) ? LS.aux : s;
                    trail(k0, wa, wb, a0, a1, st, i == 0 ? (int)(k0 / kBW) * 4 + 0 : -1);
                    if (i == 0) { ev_b_cols = LS.evc[0][step & 1]; cudaEventRecord(ev_b_cols, st); }
                }
                cudaEvent_t eb = LS.evc[1][step & 1];
                cudaEventRecord(eb, LS.aux);
                cudaStreamWaitEvent(s, eb, 0);
            }
            ev_main_done = LS.evc[2][step & 1];
            cudaEventRecord(ev_main_done, s);
        }
        cudaEvent_t e1 = ev();
        cudaEventRecord(e1, LS.hi);
        cudaStreamWaitEvent(s, e1, 0);
        cudaEvent_t ea = ev();
        cudaEventRecord(ea, LS.aux);
        cudaStreamWaitEvent(s, ea, 0);
        cudaEvent_t ej = ev();
        cudaEventRecord(ej, LS.side);
        cudaStreamWaitEvent(s, ej, 0);
        launch_trtri_blocks(w.dtype, w.W, w.ldw, n, w.Dinv1, true, false, w.st, true, w.args, s);
        return;
    }
    // Look-ahead: next block's panels on a high-priority stream beside the bulk GEMM (measured
    // ~10% on C5; the gang-scheduled cooperative panel only partly overlaps).
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
        const int64_t M = n - kn;
        const int nbw = (int)std::min<int64_t>(kBW, n - kn);
        if (lookahead && n - kn > nbw) {
            // the next block's columns first (high priority: its swap + U12, its GEMM, its panels);
            // the other columns' swap + U12 and the bulk of the GEMM concurrently on the main stream
            // (its swap + U12 on the high-priority stream too: the bulk's first chunk does not wait for it)
            cudaEvent_t e0 = ev();
            cudaEventRecord(e0, s);
            cudaStreamWaitEvent(LS.hi, e0, 0);
            swap_u12_launch<T>(w, k0, bw, kn, kn + nbw, LS.hi);
            gemm_launch<T>(w, kn, kn, k0, M, nbw, bw, LS.hi, LS.prio_hi, false, (int)(k0 / kBW) * 4 + 3);
            block_panels<T>(w, kn, nbw, LS.prio_hi, LS.hi);
            // the other columns: swap + U12, then the bulk GEMM, in column chunks alternating between
            // two streams, so that chunk i's GEMM overlaps chunk i+1's (memory-bound) swap + U12
            const int64_t c0r = kn + nbw, rn = n - c0r;
            static const int nch_env = getenv("AS_LU_SWAP_CHUNKS") ? atoi(getenv("AS_LU_SWAP_CHUNKS")) : 4;
            const int nch = rn >= 4096 ? nch_env : rn >= 1024 ? std::min(nch_env, 2) : 1;
            if (nch <= 1) {
                swap_u12_launch<T>(w, k0, bw, c0r, n, s);
                gemm_launch<T>(w, kn, c0r, k0, M, rn, bw, s, 0, false, (int)(k0 / kBW) * 4 + 0);
            } else {
                cudaEvent_t ea = ev();
                cudaEventRecord(ea, s);
                cudaStreamWaitEvent(LS.aux, ea, 0);
                for (int i = 0; i < nch; ++i) {
                    auto bnd = [&](int q) { return q >= nch ? n : c0r + (rn * q / nch + 63) / 64 * 64; };
                    const int64_t a0 = bnd(i), a1 = bnd(i + 1);
                    cudaStream_t st = (i & 1) ? LS.aux : s;
                    swap_u12_launch<T>(w, k0, bw, a0, a1, st);
                    gemm_launch<T>(w, kn, a0, k0, M, a1 - a0, bw, st, 0, false, (int)(k0 / kBW) * 4 + 0);
                }
                cudaEvent_t eb = ev();
                cudaEventRecord(eb, LS.aux);
                cudaStreamWaitEvent(s, eb, 0);
            }
            cudaEvent_t e1 = ev();
            cudaEventRecord(e1, LS.hi);
            cudaStreamWaitEvent(s, e1, 0);
        } else {
            swap_u12_launch<T>(w, k0, bw, kn, n, s);
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
    cudaMalloc(&w.cand, lu_cand_bytes());
    const size_t lfb = lu_lfbuf_bytes(n, dtype);
    cudaMalloc(&w.lfbuf, lfb);
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
        cudaMemset(w.cand, 0, lu_cand_bytes());
        cudaMemset(w.lfbuf, 0, lf_layout(w.lfbuf, n, es).zero_bytes);
        cudaEventRecord(e0, 0);
        // kind 0: the launch the factorization makes; kind 1: the cooperative panel
        if (kind == 1) setenv("AS_LU_PANEL", "coop", 1);
        if (dtype == AS_F64) panel_launch<double>(w, k0, nbp, 0, 0, 0);
        else panel_launch<float>(w, k0, nbp, 0, 0, 0);
        if (kind == 1) unsetenv("AS_LU_PANEL");
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
    cudaFree(w.lfbuf);
    if (err != cudaSuccess) return -(double)err;
    return 1000.0 * tot / (iters > 1 ? iters - 1 : 1);
}

void launch_lu_factor(const Work& w, cudaStream_t s) {
    if (w.dtype == AS_F64) lu_factor_t<double>(w, s);
    else lu_factor_t<float>(w, s);
}

}  // namespace as
