// Microbenchmark: tcgen05 INT8 tensor-core throughput on one B200 (kind::i8,
// cta_group::1, M = 128, N = 256, K = 32, s32 accumulators in TMEM), one CTA
// per SM, one elected thread issuing back-to-back MMAs from shared-memory
// operands (K-major, no swizzle), completion through tcgen05.commit ->
// mbarrier.  Plus the DMMA fp64 peak for the ratio that bounds an Ozaki-style
// fp64 emulation ("next").
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/i8_tc_peak tools/i8_tc_peak.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x)                                                                         \
    do {                                                                              \
        cudaError_t e = (x);                                                          \
        if (e != cudaSuccess) {                                                       \
            printf("CUDA error %s at line %d\n", cudaGetErrorString(e), __LINE__);    \
            return 1;                                                                 \
        }                                                                             \
    } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// SM100 shared-memory matrix descriptor: start >> 4 [0,14), LBO >> 4 [16,30),
// SBO >> 4 [32,46), version 1 [46,48), swizzle none (0) [61,64).
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}

constexpr int M = 128, N = 256, K = 32;  // one kind::i8 MMA
// instruction descriptor: c = s32 (2) [4,6), a = s8 (1) [7,10), b = s8 (1) [10,13),
// K-major A and B, N >> 3 [17,23), M >> 4 [24,29)
constexpr uint32_t kIdesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);

__global__ void __launch_bounds__(128) i8_mma_kernel(int iters, unsigned long long* cycles, int* sink) {
    __shared__ __align__(1024) int8_t a[M * K];
    __shared__ __align__(1024) int8_t b[N * K];
    __shared__ uint32_t tmem_base;
    __shared__ __align__(8) unsigned long long bar;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < M * K; i += blockDim.x) a[i] = (int8_t)((i * 7) & 63);
    for (int i = tid; i < N * K; i += blockDim.x) b[i] = (int8_t)((i * 5) & 63);
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                     "r"(256));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;");  // operands written by generic stores, read by the tensor core
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tmem_base;
    // K-major canonical layout without swizzle: core matrices of 8 rows x 16 B;
    // LBO = next core matrix along K (128 B), SBO = next 8-row group (K * 8 B)
    const uint64_t da = smem_desc(smem_u32(a), 128, K * 8), db = smem_desc(smem_u32(b), 128, K * 8);
    unsigned long long t0 = 0, t1 = 0;
    if (tid == 0) {
        t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            asm volatile(
                "{\n\t.reg .pred p;\n\t"
                "setp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                "l"(da), "l"(db), "r"(kIdesc), "r"(i > 0 ? 1 : 0));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(&bar)));
        asm volatile(
            "{\n\t.reg .pred P1;\nWAIT:\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t"
            "@!P1 bra WAIT;\n\t}" ::"r"(smem_u32(&bar)));
        t1 = clock64();
        cycles[blockIdx.x] = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    // read one accumulator word back so the work is observable
    if (warp == 0) {
        uint32_t v;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(tmem));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        if (tid == 0) sink[blockIdx.x] = (int)v;
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
    }
}

__global__ void dmma_k(double* out, int iters) {
    double acc[8][2] = {};
    double x = threadIdx.x * 1e-3, y = 1.0 + threadIdx.x * 1e-4;
    for (int i = 0; i < iters; i++)
#pragma unroll
        for (int j = 0; j < 8; j++)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(acc[j][0]), "+d"(acc[j][1])
                         : "d"(x), "d"(y));
    double s = 0;
    for (int j = 0; j < 8; j++) s += acc[j][0] + acc[j][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    int sms = 0, clk = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
    unsigned long long* cycles;
    int* sink;
    CK(cudaMalloc(&cycles, sizeof(unsigned long long) * sms));
    CK(cudaMalloc(&sink, sizeof(int) * sms));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 20000;
    i8_mma_kernel<<<sms, 128>>>(100, cycles, sink);
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0));
    i8_mma_kernel<<<sms, 128>>>(iters, cycles, sink);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long c0 = 0;
    CK(cudaMemcpy(&c0, cycles, sizeof(c0), cudaMemcpyDeviceToHost));
    const double ops = 2.0 * M * N * K * (double)iters * sms;
    printf("tcgen05 kind::i8 M%d N%d K%d: %.1f TOPS (event-timed, %d SMs), %.1f clk per MMA on SM 0\n", M, N, K,
           ops / (ms * 1e-3) / 1e12, sms, (double)c0 / iters);

    double* out;
    CK(cudaMalloc(&out, sizeof(double) * sms * 4 * 256));
    dmma_k<<<sms * 4, 256>>>(out, 50);
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0));
    dmma_k<<<sms * 4, 256>>>(out, 5000);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    const double fl = 2.0 * 8 * 8 * 4 * 8.0 * 5000 * sms * 4 * (256 / 32);
    printf("DMMA fp64: %.2f TFLOP/s\n", fl / (ms * 1e-3) / 1e12);
    return 0;
}
