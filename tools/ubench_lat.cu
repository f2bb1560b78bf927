// Latency microbenchmarks (one warp, dependent chains) for the band-solve step model.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_lat tools/ubench_lat.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int N = 4096;

__global__ void k_dfma(double* out, double a, double b, long long* cyc) {
    double x = out[threadIdx.x];
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) x = fma(x, a, b);
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_dadd(double* out, double a, long long* cyc) {
    double x = out[threadIdx.x];
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) x = x + a;
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_ddiv(double* out, double a, long long* cyc) {
    double x = out[threadIdx.x];
    long long t0 = clock64();
#pragma unroll 4
    for (int i = 0; i < N / 16; ++i) x = a / x;
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[0] = (t1 - t0) * 16;
}
__global__ void k_drcp(double* out, double a, long long* cyc) {
    double x = out[threadIdx.x];
    long long t0 = clock64();
#pragma unroll 4
    for (int i = 0; i < N / 16; ++i) x = __drcp_rn(x) * a;
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[0] = (t1 - t0) * 16;
}
__global__ void k_shfl(double* out, int src, long long* cyc) {
    double x = out[threadIdx.x];
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) x = __shfl_sync(0xffffffffu, x, (src + i) & 31);
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_lds(double* out, long long* cyc) {
    __shared__ int nxt[1024];
    for (int i = threadIdx.x; i < 1024; i += 32) nxt[i] = (i * 17 + 5) & 1023;
    __syncwarp();
    int p = threadIdx.x;
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) p = nxt[p];
    long long t1 = clock64();
    out[threadIdx.x] = p;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
// store then reload the same smem address (the old per-step pattern)
__global__ void k_stld(double* out, double a, long long* cyc) {
    __shared__ double v[1024];
    double x = out[threadIdx.x];
    volatile double* vp = v;
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) { vp[threadIdx.x] = x; x = vp[threadIdx.x] + a; }
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}


// throughput of independent ops from ONE warp: 16 independent chains, N/16 steps each
__global__ void k_shfl_tp(double* out, long long* cyc) {
    double x[16];
    for (int q = 0; q < 16; ++q) x[q] = out[threadIdx.x] + q;
    long long t0 = clock64();
    for (int i = 0; i < N / 16; ++i) {
#pragma unroll
        for (int q = 0; q < 16; ++q) x[q] = __shfl_sync(0xffffffffu, x[q], (i + q) & 31);
    }
    long long t1 = clock64();
    double s = 0; for (int q = 0; q < 16; ++q) s += x[q];
    out[threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_shfl32_tp(double* out, long long* cyc) {
    float x[16];
    for (int q = 0; q < 16; ++q) x[q] = out[threadIdx.x] + q;
    long long t0 = clock64();
    for (int i = 0; i < N / 16; ++i) {
#pragma unroll
        for (int q = 0; q < 16; ++q) x[q] = __shfl_sync(0xffffffffu, x[q], (i + q) & 31);
    }
    long long t1 = clock64();
    float s = 0; for (int q = 0; q < 16; ++q) s += x[q];
    out[threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_lds_tp(double* out, long long* cyc) {
    __shared__ double v[256];
    for (int i = threadIdx.x; i < 256; i += 32) v[i] = i;
    __syncwarp();
    double acc[16];
    for (int q = 0; q < 16; ++q) acc[q] = 0;
    int base = threadIdx.x & 1;
    long long t0 = clock64();
    for (int i = 0; i < N / 16; ++i) {
#pragma unroll
        for (int q = 0; q < 16; ++q) acc[q] += v[(base + i * 16 + q) & 255];   // broadcast-ish loads
    }
    long long t1 = clock64();
    double s = 0; for (int q = 0; q < 16; ++q) s += acc[q];
    out[threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_dfma_tp(double* out, long long* cyc) {
    double x[16];
    for (int q = 0; q < 16; ++q) x[q] = out[threadIdx.x] + q;
    long long t0 = clock64();
    for (int i = 0; i < N / 16; ++i) {
#pragma unroll
        for (int q = 0; q < 16; ++q) x[q] = fma(x[q], 1.0000001, 1e-9);
    }
    long long t1 = clock64();
    double s = 0; for (int q = 0; q < 16; ++q) s += x[q];
    out[threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}


__global__ void k_shfl_chain(double* out, long long* cyc) {
    double x = out[threadIdx.x];
    long long t0 = clock64();
#pragma unroll 8
    for (int i = 0; i < N / 16; ++i) { x = __shfl_sync(0xffffffffu, x, threadIdx.x ^ 1); x = x + 1.0; }
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[0] = (t1 - t0) * 16;
}
__global__ void k_shfl32_chain(double* out, long long* cyc) {
    float x = out[threadIdx.x];
    long long t0 = clock64();
#pragma unroll 8
    for (int i = 0; i < N / 16; ++i) { x = __shfl_sync(0xffffffffu, x, threadIdx.x ^ 1); x = x + 1.0f; }
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[0] = (t1 - t0) * 16;
}
__global__ void k_lds_chain(double* out, long long* cyc) {
    __shared__ double v[64];
    for (int i = threadIdx.x; i < 64; i += 32) v[i] = 0.0;
    __syncwarp();
    double x = out[threadIdx.x];
    long long t0 = clock64();
#pragma unroll 8
    for (int i = 0; i < N / 16; ++i) { x = v[(int)x & 63] + 1.0; }
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[0] = (t1 - t0) * 16;
}
int main() {
    double* d;
    long long* c;
    cudaMalloc(&d, 1024 * sizeof(double));
    cudaMalloc(&c, 64);
    cudaMemset(d, 0, 1024 * sizeof(double));
    long long h;
    auto rep = [&](const char* name) {
        cudaDeviceSynchronize();
        cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("%-8s %.2f cyc/op\n", name, (double)h / N);
    };
    for (int it = 0; it < 2; ++it) {
        k_dfma<<<1, 32>>>(d, 1.0000001, 1e-9, c); rep("dfma");
        k_dadd<<<1, 32>>>(d, 1e-9, c); rep("dadd");
        cudaMemset(d, 0x3f, 1024 * sizeof(double));
        k_ddiv<<<1, 32>>>(d, 1.5, c); rep("ddiv");
        k_drcp<<<1, 32>>>(d, 1.5, c); rep("drcp");
        k_shfl<<<1, 32>>>(d, 3, c); rep("shfl64");
        k_lds<<<1, 32>>>(d, c); rep("lds");
        k_stld<<<1, 32>>>(d, 1e-9, c); rep("st+ld");
        k_shfl_tp<<<1, 32>>>(d, c); rep("shfl64 tp");
        k_shfl32_tp<<<1, 32>>>(d, c); rep("shfl32 tp");
        k_lds_tp<<<1, 32>>>(d, c); rep("lds64 tp");
        k_dfma_tp<<<1, 32>>>(d, c); rep("dfma tp");
        cudaMemset(d, 0, 1024 * sizeof(double));
        k_shfl_chain<<<1, 32>>>(d, c); rep("shfl64+dadd chain");
        k_shfl32_chain<<<1, 32>>>(d, c); rep("shfl32+fadd chain");
        k_lds_chain<<<1, 32>>>(d, c); rep("lds64+f2i+dadd chain");
    }
    return 0;
}
