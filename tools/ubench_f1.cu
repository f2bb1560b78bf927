// Isolated timing of the partition band-LU step loop (band_spike.cu F1) and variants.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_f1 tools/ubench_f1.cu
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>

constexpr int K = 8, BW = 2 * K + 2, M = 183;

template <int VAR>
__global__ void f1(double* g, long long* cyc) {
    __shared__ double LUs[(M + 2 * K) * BW];
    double* LU = LUs + K * BW;
    for (int e = threadIdx.x; e < (M + 2 * K) * BW; e += blockDim.x) LUs[e] = 0.0;
    __syncthreads();
    for (int e = threadIdx.x; e < M * BW; e += blockDim.x) {
        const int r = e / BW, k = e % BW;
        if (k <= 2 * K) LU[e] = (k == K) ? 20.0 : 0.5 + 0.01 * ((r * 7 + k) % 13);
    }
    __syncthreads();
    const int m = M;
    long long t0 = clock64();
    if (threadIdx.x < 32) {
        constexpr int K1 = K + 1;
        const int lane = threadIdx.x;
        double w[K1];
#pragma unroll
        for (int q = 0; q < K1; ++q) w[q] = (lane < K1 && lane < m) ? LU[lane * BW + q - lane + K] : 0.0;
        int pl = 0;
        for (int j = 0; j < m; ++j) {
            double pr[K1];
#pragma unroll
            for (int q = 0; q < K1; ++q) pr[q] = (VAR == 2) ? w[q] : __shfl_sync(0xffffffffu, w[q], pl);
            const double inv = VAR == 1 ? pr[0] : 1.0 / pr[0];
            int d = lane - pl;
            if (d < 0) d += K1;
            const int i = j + d;
            if (lane < K1) {
                if (d == 0) {
                    if (VAR != 3) LU[j * BW + K] = inv;
#pragma unroll
                    for (int q = 1; q < K1; ++q) if (VAR != 3) LU[j * BW + K + q] = w[q];
                    const int ni = j + K1;
#pragma unroll
                    for (int q = 0; q < K1; ++q) w[q] = (q >= 1 && ni < m) ? (VAR == 4 ? 0.25 : LU[ni * BW + q - 1]) : 0.0;
                } else if (i < m) {
                    const double l = w[0] * inv;
                    if (VAR != 3) LU[i * BW + K - d] = l;
#pragma unroll
                    for (int q = 1; q < K1; ++q) w[q] -= l * pr[q];
                }
                double nxt = 0.0;
                if (VAR == 4) nxt = 0.5; else if (d == 0) { if (j + K1 < m) nxt = LU[(j + K1) * BW + K]; }
                else if (i < m) nxt = LU[i * BW + 2 * K + 1 - d];
#pragma unroll
                for (int q = 0; q < K; ++q) w[q] = w[q + 1];
                w[K] = nxt;
            }
            pl = (pl == K) ? 0 : pl + 1;
        }
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[VAR] = t1 - t0;
    for (int e = threadIdx.x; e < M * BW; e += blockDim.x) g[e] = LU[e];
}


// branch-free (predicated) formulation of the same step
__global__ void f1b(double* g, long long* cyc) {
    __shared__ double LUs[(M + 2 * K) * BW];
    double* LU = LUs + K * BW;
    for (int e = threadIdx.x; e < (M + 2 * K) * BW; e += blockDim.x) LUs[e] = 0.0;
    __syncthreads();
    for (int e = threadIdx.x; e < M * BW; e += blockDim.x) {
        const int r = e / BW, k = e % BW;
        if (k <= 2 * K) LU[e] = (k == K) ? 20.0 : 0.5 + 0.01 * ((r * 7 + k) % 13);
    }
    __syncthreads();
    const int m = M;
    long long t0 = clock64();
    if (threadIdx.x < 32) {
        constexpr int K1 = K + 1;
        const int lane = threadIdx.x;
        double w[K1];
#pragma unroll
        for (int q = 0; q < K1; ++q) w[q] = (lane < K1 && lane < m) ? LU[lane * BW + q - lane + K] : 0.0;
        int pl = 0;
        for (int j = 0; j < m; ++j) {
            double pr[K1];
#pragma unroll
            for (int q = 0; q < K1; ++q) pr[q] = __shfl_sync(0xffffffffu, w[q], pl);
            const double inv = 1.0 / pr[0];
            int d = lane - pl;
            d += (d < 0) ? K1 : 0;
            const int i = j + d;
            const bool act = lane < K1;
            const bool piv = act && d == 0;
            const bool upd = act && d != 0 && i < m;
            const double l = w[0] * inv;
            const int ni = j + K1;
            // row addresses: pivot lane writes row j, others their multiplier slot
            double* rowp = LU + (piv ? j : i) * BW;
            if (upd) rowp[K - d] = l;
            if (piv) {
                rowp[K] = inv;
#pragma unroll
                for (int q = 1; q < K1; ++q) rowp[K + q] = w[q];
            }
            const bool ld_new = piv && ni < m;
            const double* nrow = LU + (ld_new ? ni : 0) * BW;
            double wn[K1];
#pragma unroll
            for (int q = 0; q < K1; ++q) wn[q] = (ld_new && q >= 1) ? nrow[q - 1] : 0.0;
            const double nxt_p = (piv && j + K1 < m) ? LU[(j + K1) * BW + K] : 0.0;
            const double nxt_u = upd ? LU[i * BW + 2 * K + 1 - d] : 0.0;
#pragma unroll
            for (int q = 1; q < K1; ++q) w[q] = upd ? fma(-l, pr[q], w[q]) : (piv ? wn[q] : w[q]);
#pragma unroll
            for (int q = 0; q < K; ++q) w[q] = w[q + 1];
            w[K] = piv ? nxt_p : nxt_u;
            pl = (pl == K) ? 0 : pl + 1;
        }
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[5] = t1 - t0;
    for (int e = threadIdx.x; e < M * BW; e += blockDim.x) g[e] = LU[e];
}
__global__ void shfl_only(double* g, long long* cyc) {
    double w[9];
    for (int q = 0; q < 9; ++q) w[q] = g[threadIdx.x + q];
    long long t0 = clock64();
    int pl = 0;
    for (int j = 0; j < M; ++j) {
        double pr[9];
#pragma unroll
        for (int q = 0; q < 9; ++q) pr[q] = __shfl_sync(0xffffffffu, w[q], pl);
#pragma unroll
        for (int q = 0; q < 9; ++q) w[q] = fma(pr[q], 0.5, w[q]);
        pl = (pl == 8) ? 0 : pl + 1;
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[6] = t1 - t0;
    for (int q = 0; q < 9; ++q) g[threadIdx.x + q] = w[q];
}

__device__ __forceinline__ double rcp_nr(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    double e = fma(-x, r, 1.0);
    r = fma(r, e, r);
    e = fma(-x, r, 1.0);
    return fma(r, e, r);
}
// register rows, pivot row broadcast through smem (the U row store doubles as the broadcast),
// reciprocal by MUFU + 2 Newton steps.  Row layout: [L: 0..K-1 | 1/u: K | pad: K+1 | U: K+2..2K+1]
template <int VAR>
__global__ void f1c(double* g, long long* cyc) {
    __shared__ __align__(16) double LUs[(M + 2 * K) * BW];
    double* LU = LUs + K * BW;
    for (int e = threadIdx.x; e < (M + 2 * K) * BW; e += blockDim.x) LUs[e] = 0.0;
    __syncthreads();
    // same values as f1 (A(r, r + c) for c = k - K), stored in the new layout
    for (int e = threadIdx.x; e < M * BW; e += blockDim.x) {
        const int r = e / BW, k = e % BW;
        if (k <= 2 * K) {
            const double v = (k == K) ? 20.0 : 0.5 + 0.01 * ((r * 7 + k) % 13);
            const int slot = k <= K ? k : k + 1;
            LU[r * BW + slot] = v;
        }
    }
    __syncthreads();
    const int m = M;
    long long t0 = clock64();
    if (threadIdx.x < 32) {
        constexpr int K1 = K + 1;
        const int lane = threadIdx.x;
        // lane l (1..K) holds row j+l at columns j..j+K (after step j-1); slot of A(i, c): c - i + K (L/diag) or +1 (U)
        auto slot = [](int dc) { return dc <= 0 ? dc + K : dc + K + 1; };
        double w[K1];
        const int l = lane;
        const int i0 = l;   // row at step 0
#pragma unroll
        for (int q = 0; q < K1; ++q) w[q] = (l >= 1 && l <= K && i0 < m) ? LU[i0 * BW + slot(q - i0)] : 0.0;
        for (int j = 0; j < m; ++j) {
            // lane 1 holds row j (the pivot, completed by step j-1) -> publish U(j, j..j+K)
            if (lane == 1) {
                // w[0] = u_jj, w[1..K] = U(j, j+1..j+K)
                const double inv = VAR == 1 ? 1.0 / w[0] : rcp_nr(w[0]);
                double* row = LU + j * BW;
                row[K] = inv;
#pragma unroll
                for (int q = 1; q < K1; ++q) row[K + 1 + q] = w[q];
            }
            __syncwarp();
            const double* prow = LU + j * BW;
            const double inv = prow[K];
            double pr[K1];
#pragma unroll
            for (int q = 1; q < K1; ++q) pr[q] = prow[K + 1 + q];
            // rows j+1..j+K: lanes 2..K+1 hold them (lane l holds row j + l - 1) -> after the step, shift lanes down
            const int i = j + lane - 1;
            double wn[K1];
#pragma unroll
            for (int q = 0; q < K1; ++q) wn[q] = w[q];
            if (lane >= 2 && lane <= K1 && i < m) {
                const double lm = w[0] * inv;
                LU[i * BW + K - (lane - 1)] = lm;
#pragma unroll
                for (int q = 1; q < K1; ++q) wn[q] = fma(-lm, pr[q], w[q]);
            }
            // row i moves to lane l-1 and to columns j+1..j+K+1 (entering column: original A(i, j+K+1))
            double nx = 0.0;
            if (lane >= 2 && lane <= K1 && i < m) nx = LU[i * BW + slot(j + K + 1 - i)];
            if (lane == K1 + 0) { }
            double sh[K1];
#pragma unroll
            for (int q = 0; q < K; ++q) sh[q] = __shfl_down_sync(0xffffffffu, wn[q + 1], 1);
            const double shn = __shfl_down_sync(0xffffffffu, nx, 1);
#pragma unroll
            for (int q = 0; q < K; ++q) w[q] = sh[q];
            w[K] = shn;
            // the new bottom row j+K+1 enters at lane K: columns j+1..j+K+1
            const int ni = j + K1;
            if (lane == K) {
#pragma unroll
                for (int q = 0; q < K1; ++q) w[q] = (ni < m) ? LU[ni * BW + slot(j + 1 + q - ni)] : 0.0;
            }
        }
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[7 + VAR] = t1 - t0;
    // back to the f1 layout for comparison
    for (int e = threadIdx.x; e < M * BW; e += blockDim.x) {
        const int r = e / BW, k = e % BW;
        if (k <= 2 * K) g[M * BW + e] = LU[r * BW + (k <= K ? k : k + 1)];
    }
}
int main() {
    double* g;
    long long* c;
    cudaMalloc(&g, 2 * sizeof(double) * M * BW);
    cudaMalloc(&c, 128);
    for (int it = 0; it < 3; ++it) {
        f1<0><<<1, 256>>>(g, c);
        f1<1><<<1, 256>>>(g, c);
        f1<2><<<1, 256>>>(g, c);
        f1<3><<<1, 256>>>(g, c);
        f1<4><<<1, 256>>>(g, c);
        f1b<<<1, 256>>>(g, c);
        shfl_only<<<1, 32>>>(g, c);
        cudaDeviceSynchronize();
        long long h[7];
        cudaMemcpy(h, c, 56, cudaMemcpyDeviceToHost);
        printf("branch-free %.1f cyc/step, shfl-only %.1f cyc/step\n", (double)h[5] / M, (double)h[6] / M);
        f1<0><<<1, 256>>>(g, c);
        f1c<0><<<1, 256>>>(g, c);
        cudaDeviceSynchronize();
        long long hc[9];
        cudaMemcpy(hc, c, 72, cudaMemcpyDeviceToHost);
        static double hg[2 * M * BW];
        cudaMemcpy(hg, g, sizeof(hg), cudaMemcpyDeviceToHost);
        double md = 0;
        for (int e = 0; e < M * BW; ++e) { const int k = e % BW; if (k <= 2 * K) md = fmax(md, fabs(hg[e] - hg[M * BW + e]) / (fabs(hg[e]) + 1e-300)); }
        printf("smem-broadcast + rcp-NR: %.1f cyc/step, max rel diff vs f1 %.3e\n", (double)hc[7] / M, md);
        printf("F1 cyc/step: base %.1f | no div %.1f | no shfl %.1f | no st %.1f | no ld %.1f\n", (double)h[0] / M,
               (double)h[1] / M, (double)h[2] / M, (double)h[3] / M, (double)h[4] / M);
    }
    return 0;
}
