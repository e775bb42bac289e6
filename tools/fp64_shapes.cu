// Microbenchmark: fp64 tensor-core throughput per mma.sync shape (m8n8k4,
// m16n8k4, m16n8k8, m16n8k16) and DMMA + DFMA issued concurrently by
// different warps of one CTA (does the FP64 FMA pipe add to the DMMA pipe?).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_shapes tools/fp64_shapes.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void mma884(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}
__device__ __forceinline__ void mma1684(double (&c)[4], double a0, double a1, double b) {
    asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                 : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3]) : "d"(a0), "d"(a1), "d"(b));
}
__device__ __forceinline__ void mma1688(double (&c)[4], const double (&a)[4], const double (&b)[2]) {
    asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
                 : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}
__device__ __forceinline__ void mma16816(double (&c)[4], const double (&a)[8], const double (&b)[4]) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, "
        "{%0,%1,%2,%3};"
        : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
        : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]), "d"(b[0]), "d"(b[1]),
          "d"(b[2]), "d"(b[3]));
}

template <int SHAPE>
__global__ void mma_k(double* out, int iters) {
    double x = threadIdx.x * 1e-3, y = 1.0 + threadIdx.x * 1e-4;
    double s = 0;
    if (SHAPE == 0) {
        double c[8][2] = {};
        for (int i = 0; i < iters; i++)
#pragma unroll
            for (int j = 0; j < 8; j++) mma884(c[j], x, y);
        for (int j = 0; j < 8; j++) s += c[j][0] + c[j][1];
    } else if (SHAPE == 1) {
        double c[8][4] = {};
        for (int i = 0; i < iters; i++)
#pragma unroll
            for (int j = 0; j < 8; j++) mma1684(c[j], x, y, y);
        for (int j = 0; j < 8; j++) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
    } else if (SHAPE == 2) {
        double c[8][4] = {};
        double a[4] = {x, y, x, y}, b[2] = {y, x};
        for (int i = 0; i < iters; i++)
#pragma unroll
            for (int j = 0; j < 8; j++) mma1688(c[j], a, b);
        for (int j = 0; j < 8; j++) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
    } else {
        double c[8][4] = {};
        double a[8] = {x, y, x, y, x, y, x, y}, b[4] = {y, x, y, x};
        for (int i = 0; i < iters; i++)
#pragma unroll
            for (int j = 0; j < 8; j++) mma16816(c[j], a, b);
        for (int j = 0; j < 8; j++) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// warps with (warp % 2 == 0) run DMMA m8n8k4, the others DFMA chains
__global__ void mixed_k(double* out, int iters, int dfma_iters) {
    const int warp = threadIdx.x >> 5;
    double s = 0;
    if (warp % 2 == 0) {
        double x = threadIdx.x * 1e-3, y = 1.0 + threadIdx.x * 1e-4;
        double c[8][2] = {};
        for (int i = 0; i < iters; i++)
#pragma unroll
            for (int j = 0; j < 8; j++) mma884(c[j], x, y);
        for (int j = 0; j < 8; j++) s += c[j][0] + c[j][1];
    } else {
        double a[8];
        for (int j = 0; j < 8; j++) a[j] = threadIdx.x * 1e-9 + j;
        const double b = 1.0000001, c = 1e-12;
        for (int i = 0; i < dfma_iters; i++)
#pragma unroll
            for (int j = 0; j < 8; j++) a[j] = fma(a[j], b, c);
        for (int j = 0; j < 8; j++) s += a[j];
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out;
    cudaMalloc(&out, sizeof(double) * sms * 8 * 1024);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int grid = sms * 4, thr = 256, iters = 4000;
    const double flop_per[4] = {2.0 * 8 * 8 * 4, 2.0 * 16 * 8 * 4, 2.0 * 16 * 8 * 8, 2.0 * 16 * 8 * 16};
    const char* names[4] = {"m8n8k4", "m16n8k4", "m16n8k8", "m16n8k16"};
    void (*ks[4])(double*, int) = {mma_k<0>, mma_k<1>, mma_k<2>, mma_k<3>};
    for (int s = 0; s < 4; ++s) {
        ks[s]<<<grid, thr>>>(out, 50);
        cudaDeviceSynchronize();
        cudaEventRecord(e0);
        ks[s]<<<grid, thr>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double fl = flop_per[s] * 8.0 * iters * grid * (thr / 32);
        printf("%-9s %.2f TFLOP/s (%s)\n", names[s], fl / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
    // mixed: half the warps DMMA, half DFMA; report both rates over the common time
    for (int dfi : {4000, 8000, 16000}) {
        mixed_k<<<grid, thr>>>(out, 50, 50);
        cudaDeviceSynchronize();
        cudaEventRecord(e0);
        mixed_k<<<grid, thr>>>(out, iters, dfi);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double fl_mma = flop_per[0] * 8.0 * iters * grid * (thr / 64);
        const double fl_fma = 2.0 * 8.0 * dfi * grid * thr / 2;
        printf("mixed dfma_iters=%d: %.3f ms, DMMA %.2f + DFMA %.2f = %.2f TFLOP/s\n", dfi, ms, fl_mma / ms / 1e9,
               fl_fma / ms / 1e9, (fl_mma + fl_fma) / ms / 1e9);
    }
    return 0;
}
