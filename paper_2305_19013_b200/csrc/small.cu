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

namespace {

constexpr int kSmallThreads = 256;
constexpr int kMaxM = 64;

// Cholesky of the symmetric m x m matrix in smem B (row-major); R (smem) gets
// the upper factor.  Returns -1 on success, else the failing column (and the
// pivot/scale through the references).  All threads participate.
__device__ int chol_rows(const double* B, double* R, int m, double tol, double& piv_out,
                         double& scale_out) {
    __shared__ double s_piv;
    __shared__ int s_fail;
    const int tid = threadIdx.x;
    for (int e = tid; e < m * m; e += blockDim.x) R[e] = 0.0;
    if (tid == 0) {
        double sc = 0.0;
        for (int j = 0; j < m; ++j) sc = fmax(sc, fabs(B[j * m + j]));
        scale_out = sc;
        s_fail = -1;
    }
    __syncthreads();
    const double scale = scale_out;
    for (int j = 0; j < m; ++j) {
        if (tid == 0) {
            double dot = 0.0;
            for (int i = 0; i < j; ++i) dot += R[i * m + j] * R[i * m + j];
            double piv = B[j * m + j] - dot;
            if (!isfinite(piv) || piv <= tol * scale) {
                s_fail = j;
                s_piv = piv;
            } else {
                R[j * m + j] = sqrt(piv);
            }
        }
        __syncthreads();
        if (s_fail >= 0) {
            piv_out = s_piv;
            return s_fail;
        }
        const double rjj = R[j * m + j];
        for (int k = j + 1 + tid; k < m; k += blockDim.x) {
            double dot = 0.0;
            for (int i = 0; i < j; ++i) dot += R[i * m + j] * R[i * m + k];
            R[j * m + k] = (B[j * m + k] - dot) / rjj;
        }
        __syncthreads();
    }
    return -1;
}

// S = R^-1 for upper-triangular R: one thread per column, back substitution.
__device__ void tri_inverse(const double* R, double* S, int m) {
    for (int e = threadIdx.x; e < m * m; e += blockDim.x) S[e] = 0.0;
    __syncthreads();
    for (int c = threadIdx.x; c < m; c += blockDim.x) {
        S[c * m + c] = 1.0 / R[c * m + c];
        for (int i = c - 1; i >= 0; --i) {
            double s = 0.0;
            for (int k = i + 1; k <= c; ++k) s += R[i * m + k] * S[k * m + c];
            S[i * m + c] = -s / R[i * m + i];
        }
    }
    __syncthreads();
}

__device__ void record_breakdown(EkcgCtrl* ctrl, int kind, int col, double piv, double scale, int iteration) {
    ctrl->brk_kind = kind;
    ctrl->brk_col = col;
    ctrl->brk_pivot = piv;
    ctrl->brk_scale = scale;
    ctrl->brk_iter = iteration;
    ctrl->status = 3;
    ctrl->live = 0;
}

__global__ void __launch_bounds__(kSmallThreads)
prechol_kernel(const double* __restrict__ Graw, int m, double* __restrict__ S0, EkcgCtrl* ctrl,
               int iteration, double tol) {
    if (ctrl->live == 0) return;
    extern __shared__ double sm[];
    double* B = sm;
    double* R = B + m * m;
    double* S = R + m * m;
    __shared__ double nrm[kMaxM];
    __shared__ int dead;
    __shared__ double piv, scale;
    const int tid = threadIdx.x;
    if (tid == 0) dead = -1;
    __syncthreads();
    // column norms (aortho.py:74-79): a zero column is a breakdown
    for (int j = tid; j < m; j += blockDim.x) nrm[j] = sqrt(Graw[j * m + j]);
    __syncthreads();
    if (tid == 0) {
        for (int j = 0; j < m; ++j)
            if (nrm[j] == 0.0) { dead = j; break; }
        if (dead >= 0) record_breakdown(ctrl, 1, dead, 0.0, 0.0, iteration);
    }
    __syncthreads();
    if (dead >= 0) return;
    // G0 = sym(D^-1 Graw D^-1)  (aortho.py:21-22,105)
    for (int e = tid; e < m * m; e += blockDim.x) {
        int a = e / m, b = e % m;
        double gab = Graw[a * m + b] / nrm[a] / nrm[b];
        double gba = Graw[b * m + a] / nrm[b] / nrm[a];
        B[e] = 0.5 * (gab + gba);
    }
    __syncthreads();
    int fail = chol_rows(B, R, m, tol, piv, scale);
    if (fail >= 0) {
        if (tid == 0) record_breakdown(ctrl, 2, fail, piv, scale, iteration);
        return;
    }
    tri_inverse(R, S, m);
    for (int e = tid; e < m * m; e += blockDim.x) S0[e] = S[e] / nrm[e / m];
}

__global__ void __launch_bounds__(kSmallThreads)
cholinv_kernel(const double* __restrict__ G, int m, double* __restrict__ Sout, EkcgCtrl* ctrl, int iteration,
               double tol) {
    if (ctrl->live == 0) return;
    extern __shared__ double sm[];
    double* B = sm;
    double* R = B + m * m;
    double* S = R + m * m;
    __shared__ double piv, scale;
    const int tid = threadIdx.x;
    for (int e = tid; e < m * m; e += blockDim.x) {
        int a = e / m, b = e % m;
        B[e] = 0.5 * (G[a * m + b] + G[b * m + a]);
    }
    __syncthreads();
    int fail = chol_rows(B, R, m, tol, piv, scale);
    if (fail >= 0) {
        if (tid == 0) record_breakdown(ctrl, 2, fail, piv, scale, iteration);
        return;
    }
    tri_inverse(R, S, m);
    for (int e = tid; e < m * m; e += blockDim.x) Sout[e] = S[e];
}

__global__ void __launch_bounds__(kSmallThreads)
cholesky_kernel(const double* __restrict__ Bin, int m, double tol, double* __restrict__ Rout,
                double* __restrict__ info) {
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
    if (ctrl->live == 0) return;
    double rho = sqrt(*rho2);
    history[k] = rho;
    ctrl->k_done = k;
    ctrl->last_rho = rho;
    if (rho < ctrl->best_rho) {
        ctrl->best_rho = rho;
        ctrl->best_k = k;
    } else if (stagnation_window > 0 && k - ctrl->best_k >= stagnation_window) {
        ctrl->status = 4;
        ctrl->live = 0;
        return;
    }
    if (!(rho > ctrl->tol_abs)) {
        ctrl->status = 1;
        ctrl->live = 0;
    } else if (k + 1 > kmax) {
        ctrl->status = 2;
        ctrl->live = 0;
    }
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
    prechol_kernel<<<1, kSmallThreads, smem, as_stream(stream)>>>(Graw, m, S0, (EkcgCtrl*)ctrl, iteration, tol);
    ++g_ekcg_launches;
    return launch_status();
}

extern "C" int ekcg_cholinv(const double* G, int m, double* S, void* ctrl, int iteration, double tol,
                            void* stream) {
    if (m < 1 || m > kMaxM || ctrl == nullptr) return EKCG_EINVAL;
    size_t smem = 3 * sizeof(double) * m * m;
    if (!set_smem((const void*)cholinv_kernel, smem)) return EKCG_ELAUNCH;
    cholinv_kernel<<<1, kSmallThreads, smem, as_stream(stream)>>>(G, m, S, (EkcgCtrl*)ctrl, iteration, tol);
    ++g_ekcg_launches;
    return launch_status();
}

extern "C" int ekcg_cholesky(const double* B, int m, double tol, double* R, double* info, void* stream) {
    if (m < 1 || m > kMaxM) return EKCG_EINVAL;
    size_t smem = 2 * sizeof(double) * m * m;
    if (!set_smem((const void*)cholesky_kernel, smem)) return EKCG_ELAUNCH;
    cholesky_kernel<<<1, kSmallThreads, smem, as_stream(stream)>>>(B, m, tol, R, info);
    ++g_ekcg_launches;
    return launch_status();
}

extern "C" int ekcg_ctrl_bytes(void) { return (int)sizeof(EkcgCtrl); }

extern "C" int ekcg_start(void* ctrl, const double* rho2, double tol, double* history, void* stream) {
    if (ctrl == nullptr || rho2 == nullptr || history == nullptr) return EKCG_EINVAL;
    start_kernel<<<1, 1, 0, as_stream(stream)>>>((EkcgCtrl*)ctrl, rho2, tol, history);
    ++g_ekcg_launches;
    return launch_status();
}

extern "C" int ekcg_finish(void* ctrl, const double* rho2, int k, int kmax, int stagnation_window,
                           double* history, void* stream) {
    if (ctrl == nullptr || k < 1) return EKCG_EINVAL;
    finish_kernel<<<1, 1, 0, as_stream(stream)>>>((EkcgCtrl*)ctrl, rho2, k, kmax, stagnation_window, history);
    ++g_ekcg_launches;
    return launch_status();
}

extern "C" int ekcg_store_norm(const double* rho2, double* checks, int slot, const int* live, void* stream) {
    if (slot < 0) return EKCG_EINVAL;
    store_norm_kernel<<<1, 1, 0, as_stream(stream)>>>(rho2, checks, slot, live);
    ++g_ekcg_launches;
    return launch_status();
}

extern "C" unsigned long long ekcg_launch_count(void) { return g_ekcg_launches; }
