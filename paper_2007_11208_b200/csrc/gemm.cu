// gemm.cu -- C -= op(A) op(B): the dense-contraction step of the blocked
// factorizations (trailing update of GETRF; SYRK/GEMM update of
// POTRF).
//
// fp64: warp-level fp64 tensor-core MMA (mma.sync.m8n8k4.f64 -> SASS DMMA;
//       tcgen05 has no f64 kind on sm_100a).  CTA tile 128x128x16, 8 warps
//       (2 x 4, warp tile 64x32 = 8x4 DMMA tiles), 3-stage cp.async pipeline,
//       shared-memory layouts padded to LD = 4 (mod 16) so every fragment load
//       is bank-conflict free.
// fp32: SIMT FFMA, same CTA tile, 8x8 register micro-tiles (tf32 tensor cores
//       would miss the fp32 accuracy bar).
//
// Requirements (checked by the launcher): all leading dimensions even and
// every operand origin 16-byte aligned (the workspace guarantees this).
#include <cstdlib>

#include "gemm.h"
#include "internal.h"

namespace as {

constexpr int GBM = 128, GBN = 128, GBK = 16, GSTAGES = 3, GTHREADS = 256;
constexpr int LDMK = GBM + 4;   // [k][m] layout, m contiguous
constexpr int LDKM = GBK + 4;   // [m][k] layout, k contiguous

AS_DEV void cp_async16(void* smem, const void* gmem, int src_bytes) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(src_bytes) : "memory");
}
AS_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
AS_DEV void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

AS_DEV void dmma884(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// Stage one BK slab of op(A) (GBM x GBK) and op(B) (GBK x GBN) into smem.
// Global element op(A)(m,k) = TA ? A[k + m*lda] : A[m + k*lda]; op(B)(k,n) = TB ? B[n + k*ldb] : B[k + n*ldb].
// smem: !TA -> As[k*LDMK + m]; TA -> As[m*LDKM + k]; !TB -> Bs[n*LDKM + k]; TB -> Bs[k*LDMK + n].
template <typename T, bool TA, bool TB>
AS_DEV void gemm_stage(T* As, T* Bs, const T* A, int64_t lda, const T* B, int64_t ldb, int64_t M, int64_t N,
                       int64_t K, int64_t m0, int64_t n0, int64_t k0) {
    constexpr int V = 16 / sizeof(T);  // elements per 16-byte chunk
    // A slab
    if (!TA) {  // GBK columns of GBM contiguous elements
        constexpr int CH = GBM / V;     // chunks per column
        for (int e = threadIdx.x; e < GBK * CH; e += GTHREADS) {
            const int kk = e / CH, mm = (e % CH) * V;
            const int64_t gk = k0 + kk, gm = m0 + mm;
            int bytes = 0;
            if (gk < K && gm < M) bytes = (int)(min<int64_t>(V, M - gm) * sizeof(T));
            const T* src = bytes ? A + gm + gk * lda : A;
            cp_async16(As + kk * LDMK + mm, src, bytes);
        }
    } else {    // GBM rows (of the transposed operand) with GBK contiguous k
        constexpr int CH = GBK / V;
        for (int e = threadIdx.x; e < GBM * CH; e += GTHREADS) {
            const int mm = e / CH, kk = (e % CH) * V;
            const int64_t gk = k0 + kk, gm = m0 + mm;
            int bytes = 0;
            if (gm < M && gk < K) bytes = (int)(min<int64_t>(V, K - gk) * sizeof(T));
            const T* src = bytes ? A + gk + gm * lda : A;
            cp_async16(As + mm * LDKM + kk, src, bytes);
        }
    }
    if (!TB) {  // GBN columns with GBK contiguous k
        constexpr int CH = GBK / V;
        for (int e = threadIdx.x; e < GBN * CH; e += GTHREADS) {
            const int nn = e / CH, kk = (e % CH) * V;
            const int64_t gk = k0 + kk, gn = n0 + nn;
            int bytes = 0;
            if (gn < N && gk < K) bytes = (int)(min<int64_t>(V, K - gk) * sizeof(T));
            const T* src = bytes ? B + gk + gn * ldb : B;
            cp_async16(Bs + nn * LDKM + kk, src, bytes);
        }
    } else {    // GBK rows with GBN contiguous n
        constexpr int CH = GBN / V;
        for (int e = threadIdx.x; e < GBK * CH; e += GTHREADS) {
            const int kk = e / CH, nn = (e % CH) * V;
            const int64_t gk = k0 + kk, gn = n0 + nn;
            int bytes = 0;
            if (gk < K && gn < N) bytes = (int)(min<int64_t>(V, N - gn) * sizeof(T));
            const T* src = bytes ? B + gn + gk * ldb : B;
            cp_async16(Bs + kk * LDMK + nn, src, bytes);
        }
    }
}



// ------------------------------------------------------------------ fp32 SIMT kernel
// Thread (ty, tx) of a 16x16 grid owns rows {ty*4..+3, 64+ty*4..+3} and
// columns {tx*4..+3, 64+tx*4..+3}.  smem: As[k][m], Bs[k][n] (both contiguous
// in the output index; loaded element-wise to allow any transpose).
constexpr int SBK = 8;
template <bool TA, bool TB>
__global__ void __launch_bounds__(GTHREADS) gemm_sgemm_kernel(GemmArgs g) {
    if (g.skip && *g.skip) return;
    const int64_t m0 = (int64_t)blockIdx.x * GBM, n0 = (int64_t)blockIdx.y * GBN;
    if (g.lower_only && n0 > m0 + GBM - 1) return;
    __shared__ __align__(16) float As[2][SBK][GBM];
    __shared__ __align__(16) float Bs[2][SBK][GBN];
    const float* A = (const float*)g.A;
    const float* B = (const float*)g.B;
    float* C = (float*)g.C;
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    float acc[8][8];   // starts as C; accumulates C - A B
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int64_t r = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + i - 4);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int64_t c = n0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + j - 4);
            acc[i][j] = (r < g.M && c < g.N) ? __ldcg(C + r + c * g.ldc) : 0.f;
        }
    }
    const int nk = (int)((g.K + SBK - 1) / SBK);
    float ra[4], rb[4];
    auto gload = [&](int kt) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int e = threadIdx.x + q * GTHREADS;   // 0..1023 over SBK x GBM
            const int kk = TA ? (e % SBK) : (e / GBM), mm = TA ? (e / SBK) : (e % GBM);
            const int64_t gk = (int64_t)kt * SBK + kk, gm = m0 + mm;
            ra[q] = (gk < g.K && gm < g.M) ? (TA ? A[gk + gm * g.lda] : A[gm + gk * g.lda]) : 0.f;
            const int kb = TB ? (e / GBN) : (e % SBK), nb = TB ? (e % GBN) : (e / SBK);
            const int64_t gkb = (int64_t)kt * SBK + kb, gn = n0 + nb;
            rb[q] = (gkb < g.K && gn < g.N) ? (TB ? B[gn + gkb * g.ldb] : B[gkb + gn * g.ldb]) : 0.f;
        }
    };
    auto sstore = [&](int buf) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int e = threadIdx.x + q * GTHREADS;
            const int kk = TA ? (e % SBK) : (e / GBM), mm = TA ? (e / SBK) : (e % GBM);
            As[buf][kk][mm] = ra[q];
            const int kb = TB ? (e / GBN) : (e % SBK), nb = TB ? (e % GBN) : (e / SBK);
            Bs[buf][kb][nb] = rb[q];
        }
    };
    gload(0);
    sstore(0);
    __syncthreads();
    for (int kt = 0; kt < nk; ++kt) {
        const int buf = kt & 1;
        if (kt + 1 < nk) gload(kt + 1);
#pragma unroll
        for (int k = 0; k < SBK; ++k) {
            float a[8], b[8];
            *(float4*)&a[0] = *(const float4*)&As[buf][k][ty * 4];
            *(float4*)&a[4] = *(const float4*)&As[buf][k][64 + ty * 4];
            *(float4*)&b[0] = *(const float4*)&Bs[buf][k][tx * 4];
            *(float4*)&b[4] = *(const float4*)&Bs[buf][k][64 + tx * 4];
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(-a[i], b[j], acc[i][j]);
        }
        if (kt + 1 < nk) sstore(buf ^ 1);
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int64_t r = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + i - 4);
        if (r >= g.M) continue;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int64_t c = n0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + j - 4);
            if (c < g.N) C[r + c * g.ldc] = acc[i][j];
        }
    }
}

// ------------------------------------------------------------------ fp32 SIMT kernel v2 (NN)
// C -= A B with A (M x K) and B (K x N) column-major, the LU trailing update's shape.  CTA tile
// 128 x 128 x 16, 256 threads, 8 x 8 register tile per thread (rows ty*4.. and 64+ty*4.., columns
// tx*4.. and 64+tx*4..: every operand read is an LDS.128), 16-byte global loads, the next k-tile's
// loads issued before the current tile's 1024 FFMAs per thread (double-buffered shared memory).
// A tile: As[k][m] straight from the m-contiguous columns; B tile: Bs[k][n] through registers
// (4 consecutive k of one column per LDG.128, stored as 4 conflict-free row writes).
namespace s2 {
constexpr int BM = 128, BN = 128, BK = 16, NT = 256;
constexpr int LDA = BM + 4, LDB = BN + 4;
}
__global__ void __launch_bounds__(s2::NT, 2) gemm_sgemm_nn_kernel(GemmArgs g) {
    using namespace s2;
    if (g.skip && *g.skip) return;
    const int64_t m0 = (int64_t)blockIdx.x * BM, n0 = (int64_t)blockIdx.y * BN;
    if (g.lower_only && n0 > m0 + BM - 1) return;
    __shared__ __align__(16) float As[2][BK][LDA];
    __shared__ __align__(16) float Bs[2][BK][LDB];
    const float* A = (const float*)g.A;
    const float* B = (const float*)g.B;
    float* C = (float*)g.C;
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const bool full = (m0 + BM <= g.M) && (n0 + BN <= g.N);
    const int nk = (int)((g.K + BK - 1) / BK);
    float4 ra[2], rb[2];
    // thread e (0..511 over 2 loads): A chunk (k = e / 32, m = 4 (e % 32)); B chunk (n = e % 128, k = 4 (e / 128))
    auto gload = [&](int kt) {
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const int e = threadIdx.x + q * NT;
            const int ka = e >> 5, ma = (e & 31) * 4;
            const int64_t gk = (int64_t)kt * BK + ka, gm = m0 + ma;
            if (gk < g.K && gm + 3 < g.M) ra[q] = __ldg((const float4*)(A + gm + gk * g.lda));
            else {
                float t[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) t[u] = (gk < g.K && gm + u < g.M) ? A[gm + u + gk * g.lda] : 0.f;
                ra[q] = make_float4(t[0], t[1], t[2], t[3]);
            }
            const int nb = e & 127, kb = (e >> 7) * 4;
            const int64_t gkb = (int64_t)kt * BK + kb, gn = n0 + nb;
            if (gn < g.N && gkb + 3 < g.K) rb[q] = __ldg((const float4*)(B + gkb + gn * g.ldb));
            else {
                float t[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) t[u] = (gn < g.N && gkb + u < g.K) ? B[gkb + u + gn * g.ldb] : 0.f;
                rb[q] = make_float4(t[0], t[1], t[2], t[3]);
            }
        }
    };
    auto sstore = [&](int buf) {
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const int e = threadIdx.x + q * NT;
            *(float4*)&As[buf][e >> 5][(e & 31) * 4] = ra[q];
            const int nb = e & 127, kb = (e >> 7) * 4;
            Bs[buf][kb + 0][nb] = rb[q].x;
            Bs[buf][kb + 1][nb] = rb[q].y;
            Bs[buf][kb + 2][nb] = rb[q].z;
            Bs[buf][kb + 3][nb] = rb[q].w;
        }
    };
    gload(0);                      // the first tile's loads in flight together with C's
    float acc[8][8];   // starts as C; accumulates C - A B
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const int64_t c = n0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + j - 4);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int64_t r = m0 + ty * 4 + 64 * h;
            if (full) {
                const float4 v = __ldcg((const float4*)(C + r + c * g.ldc));
                acc[4 * h + 0][j] = v.x; acc[4 * h + 1][j] = v.y; acc[4 * h + 2][j] = v.z; acc[4 * h + 3][j] = v.w;
            } else {
#pragma unroll
                for (int q = 0; q < 4; ++q) acc[4 * h + q][j] = (r + q < g.M && c < g.N) ? __ldcg(C + r + q + c * g.ldc) : 0.f;
            }
        }
    }
    sstore(0);
    __syncthreads();
    for (int kt = 0; kt < nk; ++kt) {
        const int buf = kt & 1;
        if (kt + 1 < nk) gload(kt + 1);
#pragma unroll
        for (int k = 0; k < BK; ++k) {
            float a[8], b[8];
            *(float4*)&a[0] = *(const float4*)&As[buf][k][ty * 4];
            *(float4*)&a[4] = *(const float4*)&As[buf][k][64 + ty * 4];
            *(float4*)&b[0] = *(const float4*)&Bs[buf][k][tx * 4];
            *(float4*)&b[4] = *(const float4*)&Bs[buf][k][64 + tx * 4];
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(-a[i], b[j], acc[i][j]);
        }
        if (kt + 1 < nk) sstore(buf ^ 1);
        __syncthreads();
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const int64_t c = n0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + j - 4);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int64_t r = m0 + ty * 4 + 64 * h;
            if (full) {
                *(float4*)(C + r + c * g.ldc) = make_float4(acc[4 * h][j], acc[4 * h + 1][j], acc[4 * h + 2][j], acc[4 * h + 3][j]);
            } else {
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if (r + q < g.M && c < g.N) C[r + q + c * g.ldc] = acc[4 * h + q][j];
            }
        }
    }
}

// ------------------------------------------------------------------ fp64 DMMA kernel v2
// CTA tile 128 x 64 x 16, 4 warps (2 x 2, warp tile 64 x 32 = 8 x 4 DMMA tiles),
// 3-stage cp.async pipeline, 2 CTAs per SM so one CTA's C read-modify-write
// epilogue overlaps the other's MMA main loop.
// tile configuration of the DMMA GEMM: k-tile BK_ and pipeline depth ST_ (the launcher's choice,
// measured in tools/gemm_bench.py); BM x BN = 128 x 64, 4 warps of 64 x 32
template <int BK_, int ST_, int NT_ = 128>
struct D2 {
    static constexpr int BM = 128, BN = 64, BK = BK_, ST = ST_, NT = NT_;
    // warp tile: MI x 4 DMMA tiles (64 x 32 with 4 warps, 32 x 32 with 8 warps: four warps per
    // scheduler instead of two to cover each other's barrier waits and C prologues)
    static constexpr int MI = NT_ == 128 ? 8 : 4;
    static constexpr int WARPS_M = BM / (8 * MI);
    static constexpr int LDA_KM = BM + 4;   // A as [k][m]
    static constexpr int LDA_MK = BK + 4;   // A as [m][k]
    static constexpr int LDB_NK = BK + 4;   // B as [n][k]
    static constexpr int LDB_KN = BN + 4;   // B as [k][n]
    static constexpr int AEL = (BK * LDA_KM > BM * LDA_MK) ? BK * LDA_KM : BM * LDA_MK;
    static constexpr int BEL = (BN * LDB_NK > BK * LDB_KN) ? BN * LDB_NK : BK * LDB_KN;
};
using d2 = D2<16, 2>;

template <bool TA, bool TB, class d2>
AS_DEV void stage_d2(double* As, double* Bs, const double* A, int64_t lda, const double* B, int64_t ldb, int64_t M,
                     int64_t N, int64_t K, int64_t m0, int64_t n0, int64_t k0) {
    constexpr int BM = d2::BM, BN = d2::BN, BK = d2::BK, NT = d2::NT;
    constexpr int LDA_KM = d2::LDA_KM, LDA_MK = d2::LDA_MK, LDB_NK = d2::LDB_NK, LDB_KN = d2::LDB_KN;
    if (!TA) {      // BK columns x BM contiguous m: chunk = 2 doubles
        for (int e = threadIdx.x; e < BK * (BM / 2); e += NT) {
            const int kk = e / (BM / 2), mm = (e % (BM / 2)) * 2;
            const int64_t gk = k0 + kk, gm = m0 + mm;
            int bytes = 0;
            if (gk < K && gm < M) bytes = (int)(min<int64_t>(2, M - gm) * 8);
            cp_async16(As + kk * LDA_KM + mm, bytes ? A + gm + gk * lda : A, bytes);
        }
    } else {
        for (int e = threadIdx.x; e < BM * (BK / 2); e += NT) {
            const int mm = e / (BK / 2), kk = (e % (BK / 2)) * 2;
            const int64_t gk = k0 + kk, gm = m0 + mm;
            int bytes = 0;
            if (gm < M && gk < K) bytes = (int)(min<int64_t>(2, K - gk) * 8);
            cp_async16(As + mm * LDA_MK + kk, bytes ? A + gk + gm * lda : A, bytes);
        }
    }
    if (!TB) {      // BN columns x BK contiguous k
        for (int e = threadIdx.x; e < BN * (BK / 2); e += NT) {
            const int nn = e / (BK / 2), kk = (e % (BK / 2)) * 2;
            const int64_t gk = k0 + kk, gn = n0 + nn;
            int bytes = 0;
            if (gn < N && gk < K) bytes = (int)(min<int64_t>(2, K - gk) * 8);
            cp_async16(Bs + nn * LDB_NK + kk, bytes ? B + gk + gn * ldb : B, bytes);
        }
    } else {
        for (int e = threadIdx.x; e < BK * (BN / 2); e += NT) {
            const int kk = e / (BN / 2), nn = (e % (BN / 2)) * 2;
            const int64_t gk = k0 + kk, gn = n0 + nn;
            int bytes = 0;
            if (gk < K && gn < N) bytes = (int)(min<int64_t>(2, N - gn) * 8);
            cp_async16(Bs + kk * LDB_KN + nn, bytes ? B + gn + gk * ldb : B, bytes);
        }
    }
}

// Interior tiles (the whole BM x BN x BK slab inside the operands): the per-thread source pointers
// are formed once per tile (stage_d2_ptrs) and every chunk is base + q * (compile-time stride) * ld,
// advanced by one k-tile per call -- ~3 instructions per 16-byte chunk instead of the ~30 of the
// bounds-checked path (r01 ncu: the staging code issued more warp instructions than the DMMAs).
template <bool TA, bool TB, class d2>
AS_DEV void stage_d2_ptrs(const double* A, int64_t lda, const double* B, int64_t ldb, int64_t m0, int64_t n0,
                          const double*& pa, const double*& pb, int& sa, int& sb) {
    constexpr int BM = d2::BM, BN = d2::BN, BK = d2::BK;
    const int t = threadIdx.x;
    if (!TA) { const int kk = t / (BM / 2), mm = (t % (BM / 2)) * 2; pa = A + m0 + mm + kk * lda; sa = kk * d2::LDA_KM + mm; }
    else     { const int mm = t / (BK / 2), kk = (t % (BK / 2)) * 2; pa = A + kk + (m0 + mm) * lda; sa = mm * d2::LDA_MK + kk; }
    if (!TB) { const int nn = t / (BK / 2), kk = (t % (BK / 2)) * 2; pb = B + kk + (n0 + nn) * ldb; sb = nn * d2::LDB_NK + kk; }
    else     { const int kk = t / (BN / 2), nn = (t % (BN / 2)) * 2; pb = B + n0 + nn + kk * ldb; sb = kk * d2::LDB_KN + nn; }
}
template <bool TA, bool TB, class d2>
AS_DEV void stage_d2_fast(double* As, double* Bs, const double* pa, int64_t lda, const double* pb, int64_t ldb, int sa,
                          int sb) {
    constexpr int BM = d2::BM, BN = d2::BN, BK = d2::BK, NT = d2::NT;
    constexpr int QA = BK * (BM / 2) / NT, QB = BN * (BK / 2) / NT;
    static_assert(BK * (BM / 2) % NT == 0 && BN * (BK / 2) % NT == 0, "chunks per thread");
    // rows of the chunk grid covered by one pass of NT threads
    constexpr int RA = TA ? NT / (BK / 2) : NT / (BM / 2);      // A: m rows (TA) or k columns (!TA) per pass
    constexpr int RB = TB ? NT / (BN / 2) : NT / (BK / 2);      // B: k rows (TB) or n columns (!TB) per pass
#pragma unroll
    for (int q = 0; q < QA; ++q)
        cp_async16(As + sa + q * RA * (TA ? d2::LDA_MK : d2::LDA_KM), pa + (int64_t)(q * RA) * lda, 16);
#pragma unroll
    for (int q = 0; q < QB; ++q)
        cp_async16(Bs + sb + q * RB * (TB ? d2::LDB_KN : d2::LDB_NK), pb + (int64_t)(q * RB) * ldb, 16);
}

template <bool TA, bool TB, class d2>
__global__ void __launch_bounds__(d2::NT, 2) gemm_dmma2_kernel(GemmArgs g) {
    constexpr int BM = d2::BM, BN = d2::BN, BK = d2::BK, ST = d2::ST, MI = d2::MI;
    constexpr int LDA_KM = d2::LDA_KM, LDA_MK = d2::LDA_MK, LDB_NK = d2::LDB_NK, LDB_KN = d2::LDB_KN;
    constexpr int AEL = d2::AEL, BEL = d2::BEL;
    if (g.skip && *g.skip) return;
    if (g.trace_min && threadIdx.x == 0) atomicMin(g.trace_min, gtimer());
    const int64_t m0 = (int64_t)blockIdx.x * BM, n0 = (int64_t)blockIdx.y * BN;
    if (g.lower_only && n0 > m0 + BM - 1) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* As = (double*)smem_raw;
    double* Bs = As + ST * AEL;
    const double* A = (const double*)g.A;
    const double* B = (const double*)g.B;
    double* C = (double*)g.C;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wm = (warp % d2::WARPS_M) * 8 * MI, wn = (warp / d2::WARPS_M) * 32;
    const int gid = lane >> 2, tig = lane & 3;
    const int nk = (int)((g.K + BK - 1) / BK);
    const bool full = (m0 + BM <= g.M) && (n0 + BN <= g.N);
    const int nkf = full ? (int)(g.K / BK) : 0;        // k-tiles [0, nkf) take the pointer-increment staging
    const double *pa, *pb;
    int sa, sb;
    stage_d2_ptrs<TA, TB, d2>(A, g.lda, B, g.ldb, m0, n0, pa, pb, sa, sb);
    const int64_t ka = TA ? (int64_t)BK : (int64_t)BK * g.lda, kb = TB ? (int64_t)BK * g.ldb : (int64_t)BK;
    auto stage = [&](int kt) {
        const int s = kt % ST;
        if (kt < nkf) {
            stage_d2_fast<TA, TB, d2>(As + s * AEL, Bs + s * BEL, pa, g.lda, pb, g.ldb, sa, sb);
            pa += ka; pb += kb;
        } else {
            stage_d2<TA, TB, d2>(As + s * AEL, Bs + s * BEL, A, g.lda, B, g.ldb, g.M, g.N, g.K, m0, n0, (int64_t)kt * BK);
        }
    };
#pragma unroll
    for (int s = 0; s < ST - 1; ++s) {
        if (s < nk) stage(s);
        cp_async_commit();
    }
    // acc starts as C (all loads in flight together, overlapping the prologue);
    // the MMAs then accumulate acc += A (-B), so the epilogue is a plain store.
    // The MMA runs on the transposed tile (first operand = B^T fragment, second = A^T fragment), so
    // a thread's two accumulator values are C(r, c), C(r + 1, c) with r = .. + 2 tig, c = .. + gid:
    // adjacent in the column-major C -> one 16-byte load / store per DMMA tile.
    double acc[MI][4][2];
#pragma unroll
    for (int i = 0; i < MI; ++i) {
        const int64_t r = m0 + wm + 8 * i + 2 * tig;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int64_t c = n0 + wn + 8 * j + gid;
            if (full) {
                const double2 v = __ldcg((const double2*)(C + r + c * g.ldc));
                acc[i][j][0] = v.x; acc[i][j][1] = v.y;
            } else {
#pragma unroll
                for (int h = 0; h < 2; ++h) acc[i][j][h] = (r + h < g.M && c < g.N) ? __ldcg(C + r + h + c * g.ldc) : 0.0;
            }
        }
    }
    for (int kt = 0; kt < nk; ++kt) {
        cp_async_wait<ST - 2>();
        __syncthreads();
        const int nxt = kt + ST - 1;
        if (nxt < nk) stage(nxt);
        cp_async_commit();
        const double* as = As + (kt % ST) * AEL;
        const double* bs = Bs + (kt % ST) * BEL;
#pragma unroll
        for (int ks = 0; ks < BK / 4; ++ks) {
            double af[MI], bf[4];
#pragma unroll
            for (int i = 0; i < MI; ++i) {
                const int m = wm + 8 * i + gid, k = ks * 4 + tig;
                af[i] = TA ? as[m * LDA_MK + k] : as[k * LDA_KM + m];
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int n = wn + 8 * j + gid, k = ks * 4 + tig;
                bf[j] = -(TB ? bs[k * LDB_KN + n] : bs[n * LDB_NK + k]);
            }
#pragma unroll
            for (int i = 0; i < MI; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], bf[j], af[i]);
        }
    }
    cp_async_wait<0>();
#pragma unroll
    for (int i = 0; i < MI; ++i) {
        const int64_t r = m0 + wm + 8 * i + 2 * tig;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int64_t c = n0 + wn + 8 * j + gid;
            if (full) {
                *(double2*)(C + r + c * g.ldc) = make_double2(acc[i][j][0], acc[i][j][1]);
            } else {
#pragma unroll
                for (int h = 0; h < 2; ++h)
                    if (r + h < g.M && c < g.N) C[r + h + c * g.ldc] = acc[i][j][h];
            }
        }
    }
    if (g.trace_max && threadIdx.x == 0) atomicMax(g.trace_max, gtimer());
}

// ------------------------------------------------------------------ fp64 tensor peak probe
// Register-resident DMMA loop (CH independent accumulator chains per warp): the fp64 tensor-core
// roofline denominator.  tools/ubench_dmma.cu swept the shapes on B200: 8 warps x 2 CTAs per SM with
// 8 chains reaches 37.1 TF/s (ncu: 99.98 % of the DMMA pipe = the 148 x 64 x 2 x 1.965 GHz nominal);
// the r01 probe's 8 warps x 4 CTAs x 16 chains sat at an anomalous 29.7 TF/s.
template <int CH>
__global__ void __launch_bounds__(256) dmma_peak_kernel(double* out, int iters) {
    double acc[CH][2];
#pragma unroll
    for (int i = 0; i < CH; ++i) acc[i][0] = acc[i][1] = 0.0;
    double a = 1.0 + 1e-9 * threadIdx.x, b = 1.0 - 1e-9 * blockIdx.x;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < CH; ++i) dmma884(acc[i][0], acc[i][1], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < CH; ++i) s += acc[i][0] + acc[i][1];
    if (s == 12345.678) out[0] = s;  // keep the work alive
}

double measure_fp64_peak(int num_sms, int iters, cudaStream_t s) {
    double* d = nullptr;
    cudaMalloc(&d, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    double best = 0.0;
    // (ctas per SM, chains): the best shapes of the sweep; the maximum is the denominator
    const int shapes[2][2] = {{2, 8}, {8, 8}};
    for (const auto& sh : shapes) {
        const int blocks = num_sms * sh[0];
        auto kern = dmma_peak_kernel<8>;
        kern<<<blocks, 256, 0, s>>>(d, 16);  // warm-up
        cudaEventRecord(e0, s);
        kern<<<blocks, 256, 0, s>>>(d, iters);
        cudaEventRecord(e1, s);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        const double flops = 2.0 * 256.0 * (double)sh[1] * (double)iters * (double)blocks * 8.0;  // 8 warps, CH mma, 256 FMA
        const double tf = flops / (ms * 1e-3) / 1e12;
        if (tf > best) best = tf;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(d);
    return best;
}

// ------------------------------------------------------------------ launcher
template <typename K>
static void launch_k(K kern, const GemmArgs& g, size_t smem, cudaStream_t s) {
    dim3 grid((unsigned)((g.M + GBM - 1) / GBM), (unsigned)((g.N + GBN - 1) / GBN));
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<grid, GTHREADS, smem, s>>>(g);
}

void launch_gemm_minus(int dtype, const GemmArgs& g, cudaStream_t s) {
    if (g.M <= 0 || g.N <= 0 || g.K <= 0) return;
    if (dtype == AS_F64) {
        // one tile configuration: 128 x 64 x 16, two stages, 4 warps of 64 x 32, two CTAs per SM.  Measured
        // against it on B200 (tools/gemm_bench.py history): three stages 74.8 %, k-tiles of 32
        // 66.8 %, both 58.6 %, a persistent 128 x 128 kernel 64.2 %, 8 warps of 32 x 32 84.6 % alone but
        // 181 vs 167 ms inside the C5 factorization (no register room left for a panel CTA on the SM)
        using C = D2<16, 2>;
        const size_t smem = sizeof(double) * C::ST * (C::AEL + C::BEL);
        auto go = [&](auto kern) {
            dim3 grid((unsigned)((g.M + C::BM - 1) / C::BM), (unsigned)((g.N + C::BN - 1) / C::BN));
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            kern<<<grid, C::NT, smem, s>>>(g);
        };
        if (!g.TA && !g.TB) go(gemm_dmma2_kernel<false, false, C>);
        else if (!g.TA && g.TB) go(gemm_dmma2_kernel<false, true, C>);
        else if (g.TA && !g.TB) go(gemm_dmma2_kernel<true, false, C>);
        else go(gemm_dmma2_kernel<true, true, C>);
    } else {
        // NN with 16-byte aligned operands (the LU trailing update): the v2 kernel
        const bool al = (((uintptr_t)g.A | (uintptr_t)g.B | (uintptr_t)g.C) & 15) == 0 && g.lda % 4 == 0 &&
                        g.ldb % 4 == 0 && g.ldc % 4 == 0;
        if (!g.TA && !g.TB && al && getenv("AS_SGEMM_V1") == nullptr) {
            dim3 grid((unsigned)((g.M + s2::BM - 1) / s2::BM), (unsigned)((g.N + s2::BN - 1) / s2::BN));
            gemm_sgemm_nn_kernel<<<grid, s2::NT, 0, s>>>(g);
        } else if (!g.TA && !g.TB) launch_k(gemm_sgemm_kernel<false, false>, g, 0, s);
        else if (!g.TA && g.TB) launch_k(gemm_sgemm_kernel<false, true>, g, 0, s);
        else if (g.TA && !g.TB) launch_k(gemm_sgemm_kernel<true, false>, g, 0, s);
        else launch_k(gemm_sgemm_kernel<true, true>, g, 0, s);
    }
}

}  // namespace as
