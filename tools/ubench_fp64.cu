// FP64 FMA throughput / latency probe (SIMT DFMA vs the DMMA measured by as_measure_fp64_peak).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubench_fp64 tools/ubench_fp64.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>
__global__ void k_tput(double* out, double a, double b, int iters) {
    double x[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = out[threadIdx.x] + c;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int c = 0; c < CH; ++c) x[c] = fma(x[c], a, b);
    double s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += x[c];
    if (s == 1.2345) out[threadIdx.x] = s;
}
__global__ void k_lat(double* out, double a, double b, int iters, long long* cyc) {
    double x = out[threadIdx.x];
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) x = fma(x, a, b);
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
// one "column step" skeleton: warp argmax (double, int) + CTA merge through shared memory
__global__ void k_step(double* out, int iters, long long* cyc) {
    __shared__ double rv[8];
    __shared__ int ri[8];
    double v = out[threadIdx.x];
    int idx = threadIdx.x;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        double bv = fabs(v);
        int bi = idx;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double v2 = __shfl_xor_sync(0xffffffffu, bv, o);
            const int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
            if (v2 > bv || (v2 == bv && i2 < bi)) { bv = v2; bi = i2; }
        }
        if ((threadIdx.x & 31) == 0) { rv[threadIdx.x >> 5] = bv; ri[threadIdx.x >> 5] = bi; }
        __syncthreads();
        bv = rv[threadIdx.x & 7];
        bi = ri[threadIdx.x & 7];
#pragma unroll
        for (int o = 4; o > 0; o >>= 1) {
            const double v2 = __shfl_xor_sync(0xffffffffu, bv, o);
            const int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
            if (v2 > bv || (v2 == bv && i2 < bi)) { bv = v2; bi = i2; }
        }
        v = v * 0.999 + bv * 1e-6;
        idx = bi;
        __syncthreads();
    }
    long long t1 = clock64();
    out[threadIdx.x] = v + idx;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_bar(double* out, int iters, long long* cyc) {
    double v = out[threadIdx.x];
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) { v = v * 0.999 + 1e-6; __syncthreads(); }
    long long t1 = clock64();
    out[threadIdx.x] = v;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
    double* d; long long* c;
    cudaMalloc(&d, 1 << 20); cudaMalloc(&c, 64); cudaMemset(d, 0, 1 << 20);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int tpb : {128, 256, 512, 1024}) {
        const int iters = 4096;
        k_tput<8><<<sms, tpb>>>(d, 0.999, 1e-3, iters);
        cudaEventRecord(e0);
        k_tput<8><<<sms * 2, tpb>>>(d, 0.999, 1e-3, iters);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        const double fl = 2.0 * 8 * iters * (double)tpb * sms * 2;
        printf("DFMA tput tpb=%4d: %.2f TFLOP/s (%.1f DFMA/clk/SM at 1.965 GHz)\n", tpb, fl / ms / 1e9,
               fl / 2 / (ms * 1e-3) / sms / 1.965e9);
    }
    k_lat<<<1, 32>>>(d, 0.999, 1e-3, 4096, c);
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("DFMA dependent latency: %.1f cycles\n", h / 4096.0);
    for (int tpb : {128, 256}) {
        k_step<<<1, tpb>>>(d, 1024, c);
        cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("argmax step (tpb %d): %.1f cycles/iter\n", tpb, h / 1024.0);
        k_bar<<<1, tpb>>>(d, 1024, c);
        cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("syncthreads loop (tpb %d): %.1f cycles/iter\n", tpb, h / 1024.0);
    }
    return 0;
}
