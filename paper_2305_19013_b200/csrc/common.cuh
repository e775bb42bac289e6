// Shared helpers for the ekcg B200 kernels (sm_100a, fp64).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define EKCG_OK 0
#define EKCG_EINVAL -1
#define EKCG_ELAUNCH -2

// Global launch counter (read by bench.py through ekcg_launch_count()).
extern unsigned long long g_ekcg_launches;

// Every device-loop kernel takes an optional `live` flag.  The engine's
// finalize kernel clears it when the solve stops (converged / maxiter /
// breakdown), so iterations enqueued ahead of the host's status check
// retire as empty launches.  nullptr means "always run".
// Programmatic dependent launch: a kernel launched with the PDL attribute may
// start while its predecessor on the stream drains; griddepcontrol.wait
// blocks until the predecessor's writes are visible (a no-op otherwise), and
// launch_dependents lets the successor's CTAs be scheduled early.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

#ifndef EKCG_PDL_TRIGGER
#define EKCG_PDL_TRIGGER 0  // early launch_dependents measured 1 % slower (tools/ab_lib.py)
#endif

#define EKCG_GATE(live)                         \
    do {                                        \
        pdl_wait();                             \
        if (EKCG_PDL_TRIGGER) pdl_trigger();    \
        if ((live) != nullptr && *(live) == 0)  \
            return;                             \
    } while (0)

// <<<>>> replacement that adds the programmatic-dependent-launch attribute
// (back-to-back launch floor 5.2 -> 3.2 us on B200).
template <typename... KArgs, typename... Args>
static inline cudaError_t launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                                   Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

static inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// ---------------------------------------------------------------------------
// Per-device launch set-up.  The library holds no tunable state: every kernel
// choice and split count is a function of the call's arguments and of the
// device it runs on.  What is cached is per device ordinal -- the SM count
// and, per kernel instance, the raised dynamic shared-memory limit and its
// occupancy -- so a process driving several GPUs sets each one up.
// ---------------------------------------------------------------------------
constexpr int kEkcgMaxDevices = 64;

static inline int ekcg_device() {
    int d = 0;
    if (cudaGetDevice(&d) != cudaSuccess || d < 0 || d >= kEkcgMaxDevices) {
        cudaGetLastError();
        d = 0;
    }
    return d;
}

static inline int device_sms() {
    static int sms[kEkcgMaxDevices];
    const int d = ekcg_device();
    if (sms[d] == 0) {
        int v = 148;
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d) != cudaSuccess || v < 1) {
            cudaGetLastError();
            v = 148;
        }
        sms[d] = v;
    }
    return sms[d];
}

// Resident CTAs per SM of `fn` at (threads, smem) on the current device, after
// raising its dynamic shared-memory limit there; 0 when it cannot launch.
// `cache` is a per-kernel-instance array of kEkcgMaxDevices ints (static at the call site).
template <typename F>
static inline int kernel_occupancy(F fn, int threads, size_t smem, int* cache) {
    const int d = ekcg_device();
    if (cache[d] == 0) {
        int occ = 0;
        if (smem > 48 * 1024 &&
            cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
                cudaSuccess) {
            cudaGetLastError();
        } else if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)fn, threads, smem) !=
                   cudaSuccess) {
            cudaGetLastError();
            occ = 0;
        }
        cache[d] = occ + 1;  // 1 = set up, cannot launch
    }
    return cache[d] - 1;
}

static inline int launch_status() {
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? EKCG_OK : EKCG_ELAUNCH;
}

static inline unsigned grid_for(long long work, int block, long long cap = 148LL * 32) {
    long long g = (work + block - 1) / block;
    if (g < 1) g = 1;
    if (g > cap) g = cap;
    return (unsigned)g;
}

// IEEE round-to-nearest products/sums that nvcc may not contract into FMA.
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }

// m8n8k4 fp64 tensor-core MMA (SASS: DMMA.8x8x4).  acc[0..1] += A(8x4) * B(4x8).
// Fragment ownership (lane = threadIdx.x % 32):
//   A: row lane>>2, col lane&3;   B: row (k) lane&3, col (n) lane>>2;
//   C: row lane>>2, cols 2*(lane&3) + {0,1}.
// 4 doubles with one 256-bit access (LDG.E.ENL2.256 / STG.E.ENL2.256 on sm_100a; 32-B aligned)
__device__ __forceinline__ void ld4_256(const double* p, double (&v)[4]) {
    asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
                 : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3])
                 : "l"(p));
}
__device__ __forceinline__ void st4_256(double* p, const double (&v)[4]) {
    asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(v[0]), "d"(v[1]), "d"(v[2]), "d"(v[3])
                 : "memory");
}

__device__ __forceinline__ void dmma_8x8x4(double (&acc)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(acc[0]), "+d"(acc[1])
                 : "d"(a), "d"(b));
}

// Small control block shared by the device-side iteration loop.
struct EkcgCtrl {
    int live;          // 1 while the solve runs
    int status;        // 0 running, 1 converged, 2 maxiter, 3 breakdown, 4 stagnated
    int k_done;        // completed iterations (history length - 1)
    int brk_kind;      // 0 none, 1 zero column, 2 pivot
    int brk_col;
    int brk_iter;
    int best_k;
    int pad;
    double brk_pivot;
    double brk_scale;
    double rho0;
    double tol_abs;    // tol * rho0
    double best_rho;
    double last_rho;
};
