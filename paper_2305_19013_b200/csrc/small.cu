// Single-CTA kernels for the m x m Gram factorizations and the device-side
// iteration bookkeeping (stop test, stagnation guard, breakdown flags).
//
// Cholesky follows the row-oriented form of cholesky_small (linalg.py:164-184):
//   piv_j = B_jj - R[:j,j].R[:j,j];  breakdown if !finite(piv) or piv <= tol*max|diag B|
//   R_jj = sqrt(piv);  R[j,k] = (B_jk - R[:j,j].R[:j,k]) / R_jj   (k > j)
// and the triangular solves of trsm_right_inv (linalg.py:187-196) become a
// multiply by the explicit upper inverse S = R^-1 (applied by ekcg_block_update).
#include <math.h>
#include "common.cuh"
#include "ekcg_b200.h"

unsigned long long g_ekcg_launches = 0;

#include "factor.cuh"

namespace {

using namespace ekcg_dev;
constexpr int kSmallThreads = 256;

__global__ void __launch_bounds__(kSmallThreads)
prechol_kernel(const double* __restrict__ Graw, int m, double* __restrict__ S0, EkcgCtrl* ctrl,
               int iteration, double tol) {
    pdl_wait();
    if (ctrl->live == 0) return;
    extern __shared__ double sm[];
    double* G = sm;
    for (int e = threadIdx.x; e < m * m; e += blockDim.x) G[e] = Graw[e];
    __syncthreads();
    prechol_body(G, G + m * m, G + 2 * m * m, m, S0, ctrl, iteration, tol);
}

__global__ void __launch_bounds__(kSmallThreads)
cholinv_kernel(const double* __restrict__ Gin, int m, double* __restrict__ Sout, EkcgCtrl* ctrl, int iteration,
               double tol) {
    pdl_wait();
    if (ctrl->live == 0) return;
    extern __shared__ double sm[];
    double* G = sm;
    for (int e = threadIdx.x; e < m * m; e += blockDim.x) G[e] = Gin[e];
    __syncthreads();
    cholinv_body(G, G + m * m, G + 2 * m * m, m, Sout, ctrl, iteration, tol);
}

__global__ void __launch_bounds__(kSmallThreads)
cholesky_kernel(const double* __restrict__ Bin, int m, double tol, double* __restrict__ Rout,
                double* __restrict__ info) {
    pdl_wait();
    extern __shared__ double sm[];
    double* B = sm;
    double* R = B + m * m;
    __shared__ double piv, scale;
    for (int e = threadIdx.x; e < m * m; e += blockDim.x) B[e] = Bin[e];
    __syncthreads();
    int fail = chol_rows(B, R, m, tol, piv, scale);
    for (int e = threadIdx.x; e < m * m; e += blockDim.x) Rout[e] = R[e];
    if (threadIdx.x == 0) {
        info[0] = fail >= 0 ? 1.0 : 0.0;
        info[1] = fail >= 0 ? (double)fail : -1.0;
        info[2] = fail >= 0 ? piv : 0.0;
        info[3] = scale;
    }
}

__global__ void start_kernel(EkcgCtrl* ctrl, const double* __restrict__ rho2, double tol,
                             double* __restrict__ history) {
    pdl_wait();
    double rho0 = sqrt(*rho2);
    history[0] = rho0;
    ctrl->rho0 = rho0;
    ctrl->tol_abs = tol * rho0;
    ctrl->best_rho = rho0;
    ctrl->best_k = 0;
    ctrl->last_rho = rho0;
    ctrl->k_done = 0;
    ctrl->brk_kind = 0;
    ctrl->brk_col = -1;
    ctrl->brk_iter = 0;
    ctrl->brk_pivot = 0.0;
    ctrl->brk_scale = 0.0;
    if (rho0 == 0.0) {
        ctrl->status = 1;
        ctrl->live = 0;
    } else {
        ctrl->status = 0;
        ctrl->live = 1;
    }
}

// solvers.py:398-415 (history append, stagnation guard) and :357 (loop test).
__global__ void finish_kernel(EkcgCtrl* ctrl, const double* __restrict__ rho2, int k, int kmax,
                              int stagnation_window, double* __restrict__ history) {
    pdl_wait();
    if (ctrl->live == 0) return;
    finish_body(ctrl, *rho2, k, kmax, stagnation_window, history);
}

__global__ void store_norm_kernel(const double* __restrict__ rho2, double* __restrict__ checks, int slot,
                                  const int* __restrict__ live) {
    EKCG_GATE(live);
    checks[slot] = sqrt(*rho2);
}

bool set_smem(const void* fn, size_t bytes) {
    return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) == cudaSuccess;
}

}  // namespace

extern "C" int ekcg_prechol(const double* Graw, int m, double* S0, void* ctrl, int iteration, double tol,
                            void* stream) {
    if (m < 1 || m > kMaxM || ctrl == nullptr) return EKCG_EINVAL;
    size_t smem = 3 * sizeof(double) * m * m;
    if (!set_smem((const void*)prechol_kernel, smem)) return EKCG_ELAUNCH;
    launch_k(prechol_kernel, 1, kSmallThreads, smem, as_stream(stream), Graw, m, S0, (EkcgCtrl*)ctrl, iteration, tol);
    ++g_ekcg_launches;
    return launch_status();
}

extern "C" int ekcg_cholinv(const double* G, int m, double* S, void* ctrl, int iteration, double tol,
                            void* stream) {
    if (m < 1 || m > kMaxM || ctrl == nullptr) return EKCG_EINVAL;
    size_t smem = 3 * sizeof(double) * m * m;
    if (!set_smem((const void*)cholinv_kernel, smem)) return EKCG_ELAUNCH;
    launch_k(cholinv_kernel, 1, kSmallThreads, smem, as_stream(stream), G, m, S, (EkcgCtrl*)ctrl, iteration, tol);
    ++g_ekcg_launches;
    return launch_status();
}

extern "C" int ekcg_cholesky(const double* B, int m, double tol, double* R, double* info, void* stream) {
    if (m < 1 || m > kMaxM) return EKCG_EINVAL;
    size_t smem = 2 * sizeof(double) * m * m;
    if (!set_smem((const void*)cholesky_kernel, smem)) return EKCG_ELAUNCH;
    launch_k(cholesky_kernel, 1, kSmallThreads, smem, as_stream(stream), B, m, tol, R, info);
    ++g_ekcg_launches;
    return launch_status();
}

extern "C" int ekcg_ctrl_bytes(void) { return (int)sizeof(EkcgCtrl); }

extern "C" int ekcg_start(void* ctrl, const double* rho2, double tol, double* history, void* stream) {
    if (ctrl == nullptr || rho2 == nullptr || history == nullptr) return EKCG_EINVAL;
    launch_k(start_kernel, 1, 1, 0, as_stream(stream), (EkcgCtrl*)ctrl, rho2, tol, history);
    ++g_ekcg_launches;
    return launch_status();
}

extern "C" int ekcg_finish(void* ctrl, const double* rho2, int k, int kmax, int stagnation_window,
                           double* history, void* stream) {
    if (ctrl == nullptr) return EKCG_EINVAL;
    launch_k(finish_kernel, 1, 1, 0, as_stream(stream), (EkcgCtrl*)ctrl, rho2, k, kmax, stagnation_window, history);
    ++g_ekcg_launches;
    return launch_status();
}

extern "C" int ekcg_store_norm(const double* rho2, double* checks, int slot, const int* live, void* stream) {
    if (slot < 0) return EKCG_EINVAL;
    launch_k(store_norm_kernel, 1, 1, 0, as_stream(stream), rho2, checks, slot, live);
    ++g_ekcg_launches;
    return launch_status();
}

extern "C" unsigned long long ekcg_launch_count(void) { return g_ekcg_launches; }
