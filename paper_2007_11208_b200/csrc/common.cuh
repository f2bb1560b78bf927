// common.cuh -- shared device-side definitions of libadaptsolve (sm_100a).
// Device-resident solver state, reductions, grid barriers.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/adaptsolve.h"

#define AS_HD __host__ __device__ __forceinline__
#define AS_DEV __device__ __forceinline__

namespace as {

// typed min/max usable in host and device code (hides the CUDA overload set
// inside namespace as, so min<int64_t>(a, b) is unambiguous)
template <typename T> AS_HD T min(T a, T b) { return a < b ? a : b; }
template <typename T> AS_HD T max(T a, T b) { return a < b ? b : a; }

constexpr int kTile = 64;        // detection tile edge
constexpr int kNB = 64;          // triangular-solve / LU block size

// ------------------------------------------------------------------ solver state
// One instance lives in the plan's device workspace.  Every kernel of the
// graph reads/writes it; the host reads it back once (the single sync).
struct DevState {
    // ---- detection
    uint32_t alive;               // AS_FLAG_BANDED|LOWER|UPPER|SPD still possible
    uint32_t det_flags;           // final literal flags
    int32_t kl, ku;               // running max (atomicMax)
    unsigned long long max_diag;  // ordered bits of (double)max positive diagonal
    uint32_t pair_ticket;         // detection work queue
    uint32_t pair_kill;           // candidates killed by the tile-pair pass (alive keeps the diagonal pass's)
    uint32_t opts;                // AS_OPT_* of this plan
    int32_t force_method;
    int32_t method;               // dispatch method (after Cholesky failure: LU)
    int32_t primary;              // the primary method that produced the factor
    uint32_t flags;               // solve flags (bits 8..15)
    int64_t n;
    // ---- factor status
    unsigned long long info;      // 1 + first zero pivot (atomicMin, ~0ull = none)
    int32_t chol_failed;
    int32_t pad0;
    int64_t chol_fail_col;
    unsigned long long anorm_bits;  // ordered bits of anorm (>= 0) (atomicMax)
    double rcond;
    double thr;                   // rcond threshold
    double lsq_cut;
    int32_t max_sweeps;
    int32_t gate;                 // 1 if the gate fired (singular or rcond below threshold)
    int32_t post;                 // 0 nothing, 1 primary solve, 2 SVD fallback
    int32_t pad1;
    // ---- rcond estimator (xLACN2 state machine)
    int32_t est_next;             // next apply slot to run (-1 = done)
    int32_t est_iter;
    int32_t est_j, est_jlast;
    double est, est_old;
    // ---- fallback
    int32_t sweeps;
    int32_t rotated;              // rotations in the current sweep
    int64_t rank;
    int32_t svd_conv;
    int32_t ret;                  // AS_OK / AS_ERR_*
    unsigned long long smax_bits; // fallback sigma_max (ordered bits)
    // ---- banded path
    unsigned band_dom;            // bit0: strictly row dominant, bit1: strictly column dominant
    int32_t band_use_spike;       // partitioned solver selected
    int32_t band_fast;            // partitioned solver already produced X
    int32_t band_chain;           // narrow-band chain path selected: 1 + 4 kl + ku (kl, ku <= 3), else 0
    unsigned long long dbg_t[16]; // %globaltimer phase stamps (diagnostics)
    // ---- barriers / counters (zeroed per solve)
    uint32_t bar[4];
    uint32_t epoch;               // solve counter (kept across solves): tags the triangular-solve exchange words
    uint32_t pad3;
};

// The 25% rule of P:339 on the band capacity count(n,kl,ku) = n(kl+ku+1) - kl(kl+1)/2 - ku(ku+1)/2:
// banded <=> 4 count <= n^2, exact in 64-bit integers (Z2, Z3)
AS_HD bool band_density_ok(long long n, long long kl, long long ku) {
    unsigned long long un = (unsigned long long)n;
    unsigned long long cnt = un * (unsigned long long)(kl + ku + 1) - (unsigned long long)(kl * (kl + 1) / 2) -
                             (unsigned long long)(ku * (ku + 1) / 2);
    return 4ull * cnt <= un * un;
}

// IEEE finiteness without a library call: x - x is 0 for every finite x, NaN for NaN and +-Inf
template <typename T> AS_HD bool is_finite_val(T x) { return x - x == T(0); }

// orderable bits for non-negative doubles (IEEE bit pattern is monotone)
AS_DEV unsigned long long dbits(double v) { return (unsigned long long)__double_as_longlong(v); }
AS_DEV double dfrom(unsigned long long b) { return __longlong_as_double((long long)b); }

template <typename T> struct Eps;
template <> struct Eps<double> { static constexpr double v = 2.220446049250313080847e-16; };
template <> struct Eps<float> { static constexpr float v = 1.1920928955078125e-07f; };

// ------------------------------------------------------------------ reductions
template <typename T>
AS_DEV T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// argmax with first-index tie-break: (val, idx); NaN never wins (strict >),
// matching IxAMAX (Z15).
template <typename T>
AS_DEV void argmax_merge(T& v, long long& i, T v2, long long i2) {
    if (v2 > v || (v2 == v && i2 < i)) { v = v2; i = i2; }
}
template <typename T>
AS_DEV void warp_argmax(T& v, long long& i) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        T v2 = __shfl_xor_sync(0xffffffffu, v, o);
        long long i2 = __shfl_xor_sync(0xffffffffu, i, o);
        argmax_merge(v, i, v2, i2);
    }
}

// ------------------------------------------------------------------ memory ordering
AS_DEV unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// relaxed gpu-scope load (served by L2, no L1 invalidation per poll); pair a successful poll
// with fence_acq_rel() before reading the data it guards
AS_DEV unsigned ld_relaxed(const unsigned* p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
AS_DEV unsigned long long ld_relaxed64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
AS_DEV void fence_acq_rel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
AS_DEV void st_release(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
AS_DEV int ld_volatile_i32(const int* p) { return *(volatile const int*)p; }
AS_DEV unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Grid-wide barrier for a cooperative launch (all CTAs co-resident).
// `ctr` is a monotonically increasing counter zeroed before the launch;
// `gen` counts completed barriers of this launch (1, 2, ...).
AS_DEV void grid_barrier(unsigned* ctr, unsigned gen, unsigned nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        // arrive with release semantics (cumulative over the CTA's writes ordered by the barrier),
        // then spin with acquire loads (no sleep: the barrier is on every critical path)
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
        const unsigned target = gen * nblocks;
        while (ld_relaxed(ctr) < target) { }
        fence_acq_rel();
    }
    __syncthreads();
}

// Latency-batched element loop: each thread issues U independent loads before any of its
// stores, so a loop over global/L2 data costs ~tot / (U * blockDim) memory latencies instead of
// tot / blockDim (the kernel is latency-bound: one CTA per partition, little data per CTA).
template <int U, typename T, class Ld, class St>
AS_DEV void batched(int tot, Ld ld, St stf) {
    for (int e0 = 0; e0 < tot; e0 += U * (int)blockDim.x) {
        T v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int e = e0 + u * (int)blockDim.x + (int)threadIdx.x;
            v[u] = e < tot ? ld(e) : T(0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int e = e0 + u * (int)blockDim.x + (int)threadIdx.x;
            if (e < tot) stf(e, v[u]);
        }
    }
}


// ------------------------------------------------------------------ mbarrier / DSMEM (sm_90+)
AS_DEV unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
AS_DEV void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
AS_DEV void mbar_fence_init_cluster() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
AS_DEV void mbar_arrive_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
AS_DEV bool mbar_try_wait_cluster(unsigned long long* bar, unsigned parity) {
    unsigned ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
AS_DEV unsigned mapa_u32(unsigned addr, unsigned rank) {
    unsigned r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
// remote (DSMEM) store that completes `bytes` of the destination CTA's mbarrier transaction count
AS_DEV void st_async_b64(unsigned raddr, unsigned long long v, unsigned rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(raddr), "l"(v), "r"(rbar)
                 : "memory");
}
AS_DEV void st_async_b32(unsigned raddr, unsigned v, unsigned rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(raddr), "r"(v), "r"(rbar)
                 : "memory");
}

}  // namespace as
