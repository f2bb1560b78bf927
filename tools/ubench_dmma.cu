// fp64 tensor-core (DMMA) throughput probe: which register loop reaches the pipe's peak on B200?
// Variants: mma.sync m8n8k4 with CH independent accumulator chains and W warps per CTA,
// m16n8k16 (8 DMMA.8x8x4 per instruction), and a DMMA + DFMA mix (do the two pipes add?).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_dmma tools/ubench_dmma.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void mma884(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
__device__ __forceinline__ void mma16816(double (&d)[4], const double (&a)[8], const double (&b)[4]) {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, "
                 "{%12,%13,%14,%15}, {%0,%1,%2,%3};"
                 : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
                 : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                   "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

template <int CH>
__global__ void k884(double* out, int iters) {
    double acc[CH][2];
#pragma unroll
    for (int i = 0; i < CH; ++i) acc[i][0] = acc[i][1] = 0.0;
    double a = 1.0 + 1e-9 * threadIdx.x, b = 1.0 - 1e-9 * blockIdx.x;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < CH; ++i) mma884(acc[i][0], acc[i][1], a, b);
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < CH; ++i) s += acc[i][0] + acc[i][1];
    if (s == 12345.678) out[0] = s;
}

template <int CH>
__global__ void k16816(double* out, int iters) {
    double acc[CH][4];
    double a[8], b[4];
#pragma unroll
    for (int i = 0; i < CH; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = 1.0 + 1e-9 * (threadIdx.x + i);
#pragma unroll
    for (int i = 0; i < 4; ++i) b[i] = 1.0 - 1e-9 * (blockIdx.x + i);
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < CH; ++i) mma16816(acc[i], a, b);
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < CH; ++i) s += acc[i][0] + acc[i][1] + acc[i][2] + acc[i][3];
    if (s == 12345.678) out[0] = s;
}

// half the warps DMMA, half DFMA
template <int CH>
__global__ void kmix(double* out, int iters) {
    const int warp = threadIdx.x >> 5;
    double s = 0.0;
    if (warp & 1) {
        double acc[CH][2];
#pragma unroll
        for (int i = 0; i < CH; ++i) acc[i][0] = acc[i][1] = 0.0;
        double a = 1.0 + 1e-9 * threadIdx.x, b = 1.0 - 1e-9 * blockIdx.x;
        for (int it = 0; it < iters; ++it)
#pragma unroll
            for (int i = 0; i < CH; ++i) mma884(acc[i][0], acc[i][1], a, b);
#pragma unroll
        for (int i = 0; i < CH; ++i) s += acc[i][0] + acc[i][1];
    } else {
        double x[16];
#pragma unroll
        for (int c = 0; c < 16; ++c) x[c] = threadIdx.x + c;
        const double a = 0.999999, b = 1e-7;
        for (int it = 0; it < iters * 2; ++it)
#pragma unroll
            for (int c = 0; c < 16; ++c) x[c] = fma(x[c], a, b);
#pragma unroll
        for (int c = 0; c < 16; ++c) s += x[c];
    }
    if (s == 12345.678) out[0] = s;
}

template <typename K>
static double run(K kern, int blocks, int threads, int iters, double flop_per_iter_thread_block) {
    double* d;
    cudaMalloc(&d, 8);
    kern<<<blocks, threads>>>(d, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    kern<<<blocks, threads>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaFree(d);
    return flop_per_iter_thread_block * iters * blocks / (ms * 1e-3) / 1e12;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int it = 20000;
    // m8n8k4: 256 FMA = 512 flop per mma per warp
    for (int warps : {4, 8, 16}) {
        for (int bps : {1, 2, 4, 8}) {
            if (warps * bps > 64) continue;
            const double f8 = 512.0 * 8 * warps, f16 = 512.0 * 16 * warps, f32 = 512.0 * 32 * warps;
            printf("m8n8k4 warps/cta=%2d ctas/sm=%d  CH=8 %6.2f  CH=16 %6.2f  CH=32 %6.2f TF/s\n", warps, bps,
                   run(k884<8>, sms * bps, 32 * warps, it, f8), run(k884<16>, sms * bps, 32 * warps, it, f16),
                   run(k884<32>, sms * bps, 32 * warps, it / 2, f32));
        }
    }
    // m16n8k16: 16*8*16 = 2048 FMA = 4096 flop per mma
    for (int warps : {4, 8, 16})
        for (int bps : {1, 2, 4}) {
            if (warps * bps > 64) continue;
            printf("m16n8k16 warps/cta=%2d ctas/sm=%d CH=2 %6.2f  CH=4 %6.2f TF/s\n", warps, bps,
                   run(k16816<2>, sms * bps, 32 * warps, it / 4, 4096.0 * 2 * warps),
                   run(k16816<4>, sms * bps, 32 * warps, it / 8, 4096.0 * 4 * warps));
        }
    // mix: half warps DMMA (CH=16, 512 flop each), half DFMA (16 chains x 2 iters, 32 lanes x 2 flop)
    for (int bps : {2, 4}) {
        const int warps = 8;
        const double f = (warps / 2) * (512.0 * 16) + (warps / 2) * (32.0 * 2 * 16 * 2);
        printf("mix DMMA+DFMA warps/cta=8 ctas/sm=%d: %6.2f TF/s combined\n", bps, run(kmix<16>, sms * bps, 256, it, f));
    }
    return 0;
}
