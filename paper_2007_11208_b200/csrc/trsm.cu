// trsm.cu -- blocked triangular solves op(T) X = B (Eq. 3).
//
// K5 (TRTRS), the L/U solves of GETRS and POTRS, and every
// M / M^T application of the rcond estimators run through two kernels:
//
//  trtri_blocks_kernel: inverts the kNB x kNB diagonal blocks of the stored
//      triangle (all blocks in parallel, one CTA each) -> Dinv.
//  trsm_sf_kernel:      synchronization-free blocked substitution.  CTA
//      (step s, rhs-tile r) takes a ticket in launch order, accumulates
//      B_b - sum_{j before b} op(T)_{bj} X_j as soon as each X_j is flagged
//      complete by the CTA that produced it, multiplies by Dinv_b and
//      publishes X_b.  Ticket order guarantees that every CTA waits only on
//      CTAs that are already resident, so there is no deadlock and the
//      dependency chain is n/kNB hops long.
//
// The stored triangle (upper/lower), transpose and unit diagonal are template
// parameters; "forward" order = (lower && !trans) || (upper && trans).
#include <algorithm>
#include <cstdlib>

#include "internal.h"
#include "trsm.h"
#include "blk64.cuh"
#include "factor.h"

namespace as {

constexpr int kTsThreads = 256;
constexpr int kTsR = 8;           // max RHS columns per CTA tile (more, narrower tiles: shorter per-CTA chains)
constexpr int kLDT = kNB + 1;     // padded smem leading dimension

// ------------------------------------------------------------------ diagonal block inverse
// Dinv block b (kNB x kNB, column-major, ld kNB) = inverse of the b-th diagonal
// block of the stored triangle; padded with identity beyond n.  Upper blocks are
// inverted as (U^T)^{-1} transposed, so both cases run block_trinv64 (16 x 16
// substitutions + block diagonals) instead of 64 dependent column steps.
template <typename T, bool UPPER, bool UNIT>
__global__ void __launch_bounds__(kTsThreads) trtri_blocks_kernel(const T* __restrict__ A_, int64_t lda, int64_t n,
                                                                   T* __restrict__ Dinv, const DevState* st,
                                                                   int skip_if_singular, const DevArgs* args) {
    if (skip_if_singular && st->info != ~0ull) return;
    const T* A = A_ ? A_ : (const T*)args->A;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* Ls = (T*)smem_raw;               // kB64 x kB64LD: the block as a lower triangle
    T* Xs = Ls + kB64 * kB64LD;         // its inverse
    T* tmp = Xs + kB64 * kB64LD;        // 3 * 256 scratch
    const int b = blockIdx.x;
    const int64_t o = (int64_t)b * kNB;
    const int nb = (int)min<int64_t>(kNB, n - o);
    batched<8, T>(
        kNB * kNB,
        [&](int e) -> T {
            const int r = e % kNB, c = e / kNB;      // element (r, c) of the stored block
            if (r < nb && c < nb) {
                if (r == c) return UNIT ? T(1) : A[(o + r) + (o + c) * lda];
                const bool in_tri = UPPER ? (r < c) : (r > c);
                return in_tri ? A[(o + r) + (o + c) * lda] : T(0);
            }
            return r == c ? T(1) : T(0);
        },
        [&](int e, T v) {
            const int r = e % kNB, c = e / kNB;
            if (UPPER) Ls[c + r * kB64LD] = v;       // transpose: U^T is lower
            else Ls[r + c * kB64LD] = v;
        });
    __syncthreads();
    block_trinv64<T, UNIT>(Ls, Xs, tmp);
    T* D = Dinv + (int64_t)b * kNB * kNB;
    for (int e = threadIdx.x; e < kNB * kNB; e += blockDim.x) {
        const int r = e % kNB, c = e / kNB;
        D[r + c * kNB] = UPPER ? Xs[c + r * kB64LD] : Xs[r + c * kB64LD];
    }
}

// ------------------------------------------------------------------ sync-free blocked solve
struct TsArgs {
    const void* A; int64_t lda;      // triangle (nullptr: read args->A)
    const void* Dinv;
    void* X; int64_t ldx;            // in/out (nullptr: args->X with ldx)
    int64_t n; int nrhs;
    unsigned* sync;                  // [0] = ticket, zeroed per solve
    unsigned long long* ll;          // published X blocks, every word tagged with the solve epoch
    int slot;                        // estimator slot gate (-1: none)
    int skip_if_singular;
    unsigned long long* tr_start;    // diagnostics (AS_LU_TRACE, multi-RHS solves): per-ticket %globaltimer
    unsigned long long* tr_end;
};

// Published X blocks ("LL" words, the tag travels with the data, so one load is both the
// readiness test and the data): element (i, c) of block b, tile rt at word
// ((b * ntiles + rt) * RT + c) * kNB + i; fp64 values as two words {lo32 | epoch << 32,
// hi32 | epoch << 32} (each 8-byte word is written and read as one access), fp32 as one.
template <typename T> struct LLw { static constexpr int v = sizeof(T) / 4; };
// back-off between polls of a not-yet-published word: hundreds of spinning CTAs otherwise keep
// L2 busy with volatile loads and slow the producers down
constexpr unsigned ts_backoff_ns = 64;
AS_DEV void ll_put(unsigned long long* w, double x, unsigned ep) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(x);
    const unsigned long long hi = ((unsigned long long)ep << 32);
    asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" ::"l"(w), "l"(hi | (b & 0xffffffffull)), "l"(hi | (b >> 32))
                 : "memory");
}
AS_DEV void ll_put(unsigned long long* w, float x, unsigned ep) {
    asm volatile("st.volatile.global.u64 [%0], %1;" ::"l"(w),
                 "l"(((unsigned long long)ep << 32) | (unsigned long long)__float_as_uint(x)) : "memory");
}
AS_DEV bool ll_get(const unsigned long long* w, unsigned ep, double& x) {
    unsigned long long a, b;
    asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(w) : "memory");
    x = __longlong_as_double((long long)(((b & 0xffffffffull) << 32) | (a & 0xffffffffull)));
    return (unsigned)(a >> 32) == ep && (unsigned)(b >> 32) == ep;
}
AS_DEV bool ll_get(const unsigned long long* w, unsigned ep, float& x) {
    unsigned long long a;
    asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(a) : "l"(w) : "memory");
    x = __uint_as_float((unsigned)(a & 0xffffffffull));
    return (unsigned)(a >> 32) == ep;
}

// One 64 x 64 block times a 64 x RT tile.  RT == 1: thread (row i, k-quarter q) -> part[0]
// (the four quarters are summed through shared memory).  RT >= 4: thread (row i, column
// group g) owns columns g, g+4, ... over the full k range -> part[0 .. RT/4).
constexpr int kLDX = kNB + 1;
template <int RT> struct TsBufs { static constexpr int v = RT == 1 ? 3 : 2; };
template <int RT> struct TsPer { static constexpr int v = RT == 1 ? 1 : RT / 4; };
// RT = 4, 8: thread (row i, k-quarter g) accumulates ALL RT columns over its 16 k values (every
// block element is read once from shared memory, RT independent FMA chains), then the four
// quarters are summed through Red (4 x RT x kNB) -> part[] for columns g, g+4, ...  (one barrier).
// (A (row, column-group) split reads every block element RT/4... 4 times and was shared-memory
// bandwidth bound: 2.8 us per 64 x 64 x 8 product with three CTAs per SM.)
template <typename T, bool TRANSB, int RT>
AS_DEV void block_product(const T* __restrict__ Ms, const T* __restrict__ Xs, T (&part)[TsPer<RT>::v], int R,
                          T* __restrict__ Red) {
    const int i = threadIdx.x % kNB, g = threadIdx.x / kNB;
    constexpr int PER = TsPer<RT>::v;
#pragma unroll
    for (int u = 0; u < PER; ++u) part[u] = T(0);
    if (RT > 1 && RT <= 8) {
        T a[RT];
#pragma unroll
        for (int c = 0; c < RT; ++c) a[c] = T(0);
#pragma unroll 4
        for (int kk = 0; kk < kNB / 4; ++kk) {
            const int k = g * (kNB / 4) + kk;
            const T m = TRANSB ? Ms[k + i * kLDT] : Ms[i + k * kLDT];
#pragma unroll
            for (int c = 0; c < RT; ++c) a[c] += m * Xs[k + c * kLDX];
        }
#pragma unroll
        for (int c = 0; c < RT; ++c) Red[(g * RT + c) * kNB + i] = a[c];
        __syncthreads();
#pragma unroll
        for (int u = 0; u < PER; ++u) {
            const int c = g + 4 * u;
            if (c < R)
                part[u] = (Red[(0 * RT + c) * kNB + i] + Red[(1 * RT + c) * kNB + i]) +
                          (Red[(2 * RT + c) * kNB + i] + Red[(3 * RT + c) * kNB + i]);
        }
        return;
    }
    if (RT == 1) {
#pragma unroll 4
        for (int kk = 0; kk < kNB / 4; ++kk) {
            const int k = g * (kNB / 4) + kk;
            const T m = TRANSB ? Ms[k + i * kLDT] : Ms[i + k * kLDT];
            part[0] += m * Xs[k];
        }
    } else {
#pragma unroll 4
        for (int k = 0; k < kNB; ++k) {
            const T m = TRANSB ? Ms[k + i * kLDT] : Ms[i + k * kLDT];
#pragma unroll
            for (int u = 0; u < PER; ++u)
                if (g + 4 * u < R) part[u] += m * Xs[k + (g + 4 * u) * kLDX];
        }
    }
}

template <typename T>
AS_DEV void cp_async_elem(T* smem, const T* gmem, bool ok) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    if (sizeof(T) == 8)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(sa), "l"(gmem), "r"(ok ? 8 : 0) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(sa), "l"(gmem), "r"(ok ? 4 : 0) : "memory");
}

// Shared memory: the ring of T-block buffers (Dinv_b is staged as the last entry, off the critical
// path), the X_j tile and the k-quarter partials: 87 KB (RT = 8) / 101 KB (RT = 1), two CTAs per SM, so
// every block of an n <= 16384 solve is resident at once.
template <typename T, int RT>
constexpr size_t ts_smem() {
    return sizeof(T) * ((size_t)TsBufs<RT>::v * kNB * kLDT + (size_t)kLDX * RT +
                        (RT == 1 ? 4 * kNB : RT <= 8 ? (size_t)4 * RT * kNB : 0));
}

template <typename T, bool UPPER, bool TRANS, int RT>
__global__ void __launch_bounds__(kTsThreads) trsm_sf_kernel(TsArgs p, const DevArgs* args, const DevState* st) {
    if (p.slot >= 0 && ld_volatile_i32(&st->est_next) != p.slot) return;
    if (p.skip_if_singular && st->info != ~0ull) return;
    constexpr int PER = TsPer<RT>::v;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    // ring of NBUF T-block buffers (kNB x kLDT each).  A single-RHS solve is bound by the bytes a CTA keeps
    // in flight (one 32 KB block per L2 / HBM round trip was 0.4-0.8 us per step: r02 launch lists), so it
    // stages two blocks ahead; the multi-RHS solves stay double-buffered (two CTAs per SM).
    constexpr int NBUF = TsBufs<RT>::v;
    T* Mb0 = (T*)smem_raw;
    T* Xs = Mb0 + NBUF * kNB * kLDT;            // kLDX x RT: X_j tile (column c at c * kLDX)
    T* Red = Xs + kLDX * RT;                    // RT == 1: 4 x kNB partials
    __shared__ unsigned s_ticket;

    const T* A = (const T*)(p.A ? p.A : args->A);
    T* X = (T*)(p.X ? p.X : args->X);
    const T* Dinv = (const T*)p.Dinv;
    const int64_t n = p.n;
    const int nblk = (int)((n + kNB - 1) / kNB);
    const int ntiles = (p.nrhs + RT - 1) / RT;
    constexpr bool FWD = (!UPPER && !TRANS) || (UPPER && TRANS);

    const unsigned ep = st->epoch;
    if (threadIdx.x == 0) s_ticket = atomicAdd(&p.sync[0], 1u);
    __syncthreads();
    const unsigned t = s_ticket;
    if (p.tr_start && threadIdx.x == 0 && t < 2048) p.tr_start[t] = gtimer();
    // diagnostics: phase stamps of the (step 32, tile 0) CTA into tr_end[1024 + k]
    const bool probe = p.tr_end && threadIdx.x == 0 && t == 32u * (unsigned)((p.nrhs + RT - 1) / RT);
#define TSP(k) do { if (probe) p.tr_end[1024 + (k)] = gtimer(); } while (0)
    const int s = (int)(t / ntiles), rt = (int)(t % ntiles);
    const int b = FWD ? s : nblk - 1 - s;
    const int64_t ob = (int64_t)b * kNB;
    const int nbr = (int)min<int64_t>(kNB, n - ob);
    const int c0 = rt * RT;
    const int R = min(RT, p.nrhs - c0);
    const int i = threadIdx.x % kNB, g = threadIdx.x / kNB;

    // async staging of op(T)_{b j} (no-trans: A[b rows, j cols]; trans: A[j rows, b cols]).  Thread (row i,
    // column group g) copies elements (i, g + 4 q): one pointer increment per element on full blocks (the
    // generic index arithmetic was ~25 instructions per element, more than the product itself: ncu r02)
    auto stage = [&](T* dst, int sp) {
        const int j = FWD ? sp : nblk - 1 - sp;
        const int64_t oj = (int64_t)j * kNB;
        const int nbj = (int)min<int64_t>(kNB, n - oj);
        if (nbr == kNB && nbj == kNB) {
            const T* src = TRANS ? A + (oj + i) + (ob + g) * p.lda : A + (ob + i) + (oj + g) * p.lda;
            const unsigned sa = smem_u32(dst + i + g * kLDT);
            const int64_t step = 4 * p.lda;
#pragma unroll
            for (int q = 0; q < kNB / 4; ++q) {
                if (sizeof(T) == 8)
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa + (unsigned)(q * 4 * kLDT * sizeof(T))), "l"(src) : "memory");
                else
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa + (unsigned)(q * 4 * kLDT * sizeof(T))), "l"(src) : "memory");
                src += step;
            }
        } else {
            for (int e = threadIdx.x; e < kNB * kNB; e += kTsThreads) {
                const int r = e % kNB, c = e / kNB;
                const bool ok = TRANS ? (r < nbj && c < nbr) : (r < nbr && c < nbj);
                const T* src = !ok ? A : TRANS ? A + (oj + r) + (ob + c) * p.lda : A + (ob + r) + (oj + c) * p.lda;
                cp_async_elem(dst + r + c * kLDT, src, ok);
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    auto stage_dinv = [&](T* dst) {
        const T* D = Dinv + (int64_t)b * kNB * kNB + i + g * kNB;
        const unsigned sa = smem_u32(dst + i + g * kLDT);
#pragma unroll
        for (int q = 0; q < kNB / 4; ++q) {
            if (sizeof(T) == 8)
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa + (unsigned)(q * 4 * kLDT * sizeof(T))), "l"(D + q * 4 * kNB) : "memory");
            else
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa + (unsigned)(q * 4 * kLDT * sizeof(T))), "l"(D + q * 4 * kNB) : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    // the staged sequence: op(T) blocks of steps 0 .. s-1, then Dinv_b as "step s"; one commit group per index
    auto buf = [&](int idx) { return Mb0 + (size_t)(idx % NBUF) * kNB * kLDT; };
    auto stage_idx = [&](int idx) {
        if (idx < s) stage(buf(idx), idx);
        else if (idx == s) stage_dinv(buf(idx));
        else asm volatile("cp.async.commit_group;" ::: "memory");
    };
    T* Ds = buf(s);
#pragma unroll
    for (int q = 0; q < NBUF - 1; ++q) stage_idx(q);
    // acc = B_b for my (row, columns)
    T acc[PER];
#pragma unroll
    for (int u = 0; u < PER; ++u) {
        const int c = RT == 1 ? 0 : g + 4 * u;
        acc[u] = ((RT > 1 || g == 0) && c < R && i < nbr) ? X[(ob + i) + (c0 + c) * p.ldx] : T(0);
    }

    T part[PER];
    constexpr int NE = (kNB * RT + kTsThreads - 1) / kTsThreads;   // published words a thread fetches per step
    T xv[NE];
    bool xk[NE];
    auto spec = [&](int sp2) {
        const int j2 = FWD ? sp2 : nblk - 1 - sp2;
        const unsigned long long* src = p.ll + ((int64_t)(j2 * ntiles + rt) * RT) * kNB * LLw<T>::v;
#pragma unroll
        for (int q = 0; q < NE; ++q) {
            const int e = threadIdx.x + q * kTsThreads;
            xk[q] = e < kNB * RT && ll_get(src + (int64_t)e * LLw<T>::v, ep, xv[q]);
        }
    };
#pragma unroll
    for (int q = 0; q < NE; ++q) { xv[q] = T(0); xk[q] = false; }
    if (RT > 1 && s > 0) spec(0);   // (single RHS: measured slower, 232 vs 197 us over C3b's five transposed applies)
    for (int sp = 0; sp < s; ++sp) {
        const int j = FWD ? sp : nblk - 1 - sp;
        const int64_t oj = (int64_t)j * kNB;
        const int nbj = (int)min<int64_t>(kNB, n - oj);
        T* Ms = buf(sp);
        stage_idx(sp + NBUF - 1);               // into the buffer step sp - 1 has just released
        // X_j (tile rt): each thread spins on its own tagged words until the producer's epoch shows.  The
        // words of step sp + 1 are read speculatively one step ahead (early blocks are long published: their
        // L2 round trip then overlaps this step's barrier and product); a stale tag falls back to the spin.
        (void)oj; (void)nbj;
        if (sp + 1 == s) TSP(0);
        {
            const unsigned long long* src = p.ll + ((int64_t)(j * ntiles + rt) * RT) * kNB * LLw<T>::v;
#pragma unroll
            for (int q = 0; q < NE; ++q) {
                const int e = threadIdx.x + q * kTsThreads;
                if (e < kNB * RT) {
                    const int r = e % kNB, c = e / kNB;
                    T x = xv[q];
                    if (!xk[q])
                        while (!ll_get(src + (int64_t)e * LLw<T>::v, ep, x))
                            if (RT > 1) __nanosleep(ts_backoff_ns);   // single RHS: few pollers, latency first
                    Xs[r + c * kLDX] = x;
                }
            }
        }
        if (RT > 1 && sp + 1 < s) spec(sp + 1);
        if (sp + 1 == s) TSP(1);
        asm volatile("cp.async.wait_group %0;" ::"n"(NBUF - 1) : "memory");
        __syncthreads();
        if (sp + 1 == s) TSP(2);
        block_product<T, TRANS, RT>(Ms, Xs, part, R, Red);
        if (RT == 1) {
            Red[g * kNB + i] = part[0];
            __syncthreads();
            if (g == 0) acc[0] -= (Red[i] + Red[kNB + i]) + (Red[2 * kNB + i] + Red[3 * kNB + i]);
        } else {
#pragma unroll
            for (int u = 0; u < PER; ++u) acc[u] -= part[u];
            // Ms / Xs are reused by the next step.  RT = 4, 8: the product's own barrier (after the partial
            // sums are written) already orders every read of Ms / Xs before the next step's writes, and the
            // partials are rewritten only after the next step's first barrier: no third barrier per step
            if (RT > 8) __syncthreads();
        }
    }
    // X_b = Dinv_b * acc  (trans: Dinv_b^T)
    TSP(3);
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    TSP(4);
#pragma unroll
    for (int u = 0; u < PER; ++u) {
        const int c = RT == 1 ? 0 : g + 4 * u;
        if (RT > 1 || g == 0) Xs[i + c * kLDX] = acc[u];
    }
    __syncthreads();
    block_product<T, TRANS, RT>(Ds, Xs, part, R, Red);
    unsigned long long* dst = p.ll + ((int64_t)(b * ntiles + rt) * RT) * kNB * LLw<T>::v;
    if (RT == 1) {
        Red[g * kNB + i] = part[0];
        __syncthreads();
        if (g == 0) {
            const T x = (Red[i] + Red[kNB + i]) + (Red[2 * kNB + i] + Red[3 * kNB + i]);
            ll_put(dst + (int64_t)i * LLw<T>::v, i < nbr ? x : T(0), ep);
            if (i < nbr) X[(ob + i) + c0 * p.ldx] = x;
        }
    } else {
#pragma unroll
        for (int u = 0; u < PER; ++u) {
            const int c = g + 4 * u;
            const T x = (i < nbr && c < R) ? part[u] : T(0);
            ll_put(dst + (int64_t)(c * kNB + i) * LLw<T>::v, x, ep);
            if (i < nbr && c < R) X[(ob + i) + (c0 + c) * p.ldx] = x;
        }
    }
    TSP(5);
#undef TSP
    if (p.tr_end && threadIdx.x == 0 && t < 2048) p.tr_end[t] = gtimer();
}

// ------------------------------------------------------------------ launchers
int64_t trsm_sync_words(int64_t n, int nrhs) {
    (void)n; (void)nrhs;
    return 2;
}

// RHS tile width: 1, 4, or the wide tile (AS_TS_RT = 8 / 16 / 32 for experiments)
static int ts_wide() {
    static const int v = getenv("AS_TS_RT") ? atoi(getenv("AS_TS_RT")) : kTsR;
    return (v == 16 || v == 32) ? v : 8;
}
static int ts_rt(int nrhs) { return nrhs == 1 ? 1 : nrhs <= 4 ? 4 : ts_wide(); }

int64_t trsm_ll_words(int64_t n, int nrhs) {
    const int64_t nblk = (n + kNB - 1) / kNB;
    const int rt = ts_rt(nrhs);
    const int64_t ntiles = (nrhs + rt - 1) / rt;
    return nblk * ntiles * rt * kNB * 2;      // 2 words per element covers fp64
}

template <typename T>
static void trtri_dispatch(const T* A, int64_t lda, int64_t n, T* Dinv, bool upper, bool unit, const DevState* st,
                           bool skip, const DevArgs* args, cudaStream_t s) {
    const int nblk = (int)((n + kNB - 1) / kNB);
    const int smem = (int)(sizeof(T) * (2 * kB64 * kB64LD + 3 * 256));
    auto go = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        kern<<<nblk, kTsThreads, smem, s>>>(A, lda, n, Dinv, st, skip, args);
    };
    if (upper) {
        if (unit) go(trtri_blocks_kernel<T, true, true>);
        else go(trtri_blocks_kernel<T, true, false>);
    } else {
        if (unit) go(trtri_blocks_kernel<T, false, true>);
        else go(trtri_blocks_kernel<T, false, false>);
    }
}

void launch_trtri_blocks(int dtype, const void* A, int64_t lda, int64_t n, void* Dinv, bool upper, bool unit,
                         const DevState* st, bool skip_if_singular, const DevArgs* args, cudaStream_t s) {
    if (dtype == AS_F64) trtri_dispatch<double>((const double*)A, lda, n, (double*)Dinv, upper, unit, st, skip_if_singular, args, s);
    else trtri_dispatch<float>((const float*)A, lda, n, (float*)Dinv, upper, unit, st, skip_if_singular, args, s);
}

// A == nullptr selects args->A (the caller's matrix); X == nullptr selects args->X.
template <typename T>
static void trsm_dispatch(const TsArgs& p, bool upper, bool trans, const DevArgs* args, const DevState* st,
                          cudaStream_t s) {
    const int nblk = (int)((p.n + kNB - 1) / kNB);
    auto go = [&](auto kern, int rt, size_t smem) {
        const int ntiles = (p.nrhs + rt - 1) / rt;
        // experiment knob: AS_TS_CTAS_PER_SM=k pads shared memory so at most k CTAs share an SM
        static const int per_sm = getenv("AS_TS_CTAS_PER_SM") ? atoi(getenv("AS_TS_CTAS_PER_SM")) : 0;
        if (per_sm > 0 && rt > 1) smem = std::max<size_t>(smem, (size_t)(220 * 1024) / per_sm);
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<nblk * ntiles, kTsThreads, smem, s>>>(p, args, st);
    };
    auto by_r = [&](auto k1, auto k4, auto k8, auto k16, auto k32) {
        if (p.nrhs == 1) go(k1, 1, ts_smem<T, 1>());
        else if (p.nrhs <= 4) go(k4, 4, ts_smem<T, 4>());
        else if (ts_wide() == 16) go(k16, 16, ts_smem<T, 16>());
        else if (ts_wide() == 32) go(k32, 32, ts_smem<T, 32>());
        else go(k8, 8, ts_smem<T, 8>());
    };
#define AS_TS(U, TR) trsm_sf_kernel<T, U, TR, 1>, trsm_sf_kernel<T, U, TR, 4>, trsm_sf_kernel<T, U, TR, 8>, \
                     trsm_sf_kernel<T, U, TR, 16>, trsm_sf_kernel<T, U, TR, 32>
    if (upper) {
        if (trans) by_r(AS_TS(true, true));
        else by_r(AS_TS(true, false));
    } else {
        if (trans) by_r(AS_TS(false, true));
        else by_r(AS_TS(false, false));
    }
#undef AS_TS
}

void launch_trsm(int dtype, const void* A, int64_t lda, const void* Dinv, bool upper, bool trans, void* X,
                 int64_t ldx, int64_t n, int nrhs, SyncAlloc& sa, int slot, bool skip_if_singular,
                 const DevArgs* args, const DevState* st, cudaStream_t s) {
    TsArgs p{A, lda, Dinv, X, ldx, n, nrhs, sa.take(trsm_sync_words(n, nrhs)), sa.take_ll(trsm_ll_words(n, nrhs)), slot,
             skip_if_singular ? 1 : 0, nullptr, nullptr};
    // diagnostics only: the per-CTA timeline shares the LU trace buffers (AS_LU_TRACE) and is taken
    // only with AS_TS_TRACE as well (tools/trsm_trace.py), so that the LU timeline stays intact
    static const bool ts_trace = getenv("AS_TS_TRACE") != nullptr;
    p.tr_start = ts_trace ? debug_trace_buf(0) : nullptr;
    p.tr_end = ts_trace ? debug_trace_buf(1) : nullptr;
    if (n <= 0 || nrhs <= 0) return;
    if (dtype == AS_F64) trsm_dispatch<double>(p, upper, trans, args, st, s);
    else trsm_dispatch<float>(p, upper, trans, args, st, s);
}

}  // namespace as
