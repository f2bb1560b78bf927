// blk64.cuh -- 64 x 64 block kernels-in-a-CTA used by the factorizations (256 threads).
//
//  block_trinv64   X = L^{-1} for a lower-triangular 64 x 64 block in shared memory
//                  (unit or non-unit diagonal): the four 16 x 16 diagonal blocks are
//                  inverted by substitution (one lane per column, two blocks per warp),
//                  the off-diagonal blocks follow by diagonals,
//                  X_ij = -X_ii sum_{k=j}^{i-1} L_ik X_kj,
//                  so the dependency chain is 16 substitution steps + 3 block products
//                  instead of 64 barrier-separated column steps.
//  tile_mul64      C = A op(B) for 64 x 64 tiles in shared memory, 4 x 4 register tile per
//                  thread (the in-place L21 / U12 products of Cholesky and LU).
#pragma once
#include "common.cuh"

namespace as {

constexpr int kB64 = 64;
constexpr int kB64LD = kB64 + 1;     // padded column stride of the 64 x 64 smem blocks

// Lane c (< 16) of the calling warp writes column c of the inverse of the 16 x 16 lower block
// at L (column-major, ld) to X (ld ldx).  The other 16 lanes of the warp handle a second block
// (L2 -> X2) when given.
template <typename T, bool UNIT>
AS_DEV void warp_trinv16(const T* L, T* X, const T* L2, T* X2, int ld) {
    const int lane = threadIdx.x & 31;
    const int c = lane & 15;
    const T* M = lane < 16 ? L : L2;
    T* Out = lane < 16 ? X : X2;
    if (M == nullptr) return;
    T rd[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) rd[j] = UNIT ? T(1) : T(1) / M[j + j * ld];
    T x[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        T s = (j == c) ? T(1) : T(0);
#pragma unroll
        for (int k = 0; k < j; ++k) s -= M[j + k * ld] * x[k];
        x[j] = s * rd[j];
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) Out[j + c * ld] = (j >= c) ? x[j] : T(0);
}

// X = L^{-1}, both 64 x 64 column-major with ld kB64LD in shared memory (X must not alias L);
// tmp: 3 * 256 elements of shared scratch.  The strictly upper parts of X are zeroed.
template <typename T, bool UNIT>
AS_DEV void block_trinv64(const T* L, T* X, T* tmp) {
    const int warp = threadIdx.x >> 5;
    // diagonal blocks: warps 0, 1 take two blocks each
    if (warp < 2) {
        const int b0 = 2 * warp, b1 = 2 * warp + 1;
        warp_trinv16<T, UNIT>(L + 16 * b0 * (kB64LD + 1), X + 16 * b0 * (kB64LD + 1), L + 16 * b1 * (kB64LD + 1),
                              X + 16 * b1 * (kB64LD + 1), kB64LD);
    }
    // strictly upper blocks of X are zero
    for (int e = threadIdx.x; e < kB64 * kB64; e += blockDim.x) {
        const int r = e & 63, cc = e >> 6;
        if ((r >> 4) < (cc >> 4)) X[r + cc * kB64LD] = T(0);
    }
    __syncthreads();
    // block diagonals d = 1, 2, 3: outputs (i, j = i - d), i = d..3
    for (int d = 1; d <= 3; ++d) {
        const int nout = 4 - d;
        // phase 1: tmp_o = sum_{k=j}^{i-1} L_ik X_kj   (16 x 16 each)
        for (int e = threadIdx.x; e < nout * 256; e += blockDim.x) {
            const int o = e >> 8, r = e & 15, cc = (e >> 4) & 15;
            const int i = d + o, j = o;
            T s = T(0);
            for (int k = j; k < i; ++k) {
#pragma unroll
                for (int q = 0; q < 16; ++q)
                    s += L[(16 * i + r) + (16 * k + q) * kB64LD] * X[(16 * k + q) + (16 * j + cc) * kB64LD];
            }
            tmp[o * 256 + r + 16 * cc] = s;
        }
        __syncthreads();
        // phase 2: X_ij = -X_ii tmp_o
        for (int e = threadIdx.x; e < nout * 256; e += blockDim.x) {
            const int o = e >> 8, r = e & 15, cc = (e >> 4) & 15;
            const int i = d + o, j = o;
            T s = T(0);
#pragma unroll
            for (int q = 0; q < 16; ++q) s += X[(16 * i + r) + (16 * i + q) * kB64LD] * tmp[o * 256 + q + 16 * cc];
            X[(16 * i + r) + (16 * j + cc) * kB64LD] = -s;
        }
        __syncthreads();
    }
}

// acc (this thread's 4 x 4 tile, rows 4 tr.., cols 4 tc..) = sum_k A(r, k) B'(k, c) over k < kk,
// with As[k * lda + r] and Bs[k * ldb + c] (both "k-major") in shared memory.
template <typename T>
AS_DEV void tile_mul64(const T* As, int lda, const T* Bs, int ldb, int kk, T (&acc)[4][4]) {
    const int tr = threadIdx.x & 15, tc = threadIdx.x >> 4;
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[p][q] = T(0);
    for (int k = 0; k < kk; ++k) {
        T av[4], bv[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) { av[q] = As[k * lda + 4 * tr + q]; bv[q] = Bs[k * ldb + 4 * tc + q]; }
#pragma unroll
        for (int p = 0; p < 4; ++p)
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[p][q] += av[p] * bv[q];
    }
}

}  // namespace as
