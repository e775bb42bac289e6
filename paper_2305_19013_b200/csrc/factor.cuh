// Device-side m x m factorizations and iteration bookkeeping shared by the
// single-CTA kernels (small.cu) and the fused kernels' last-CTA epilogues
// (fused.cu).  All functions are called by every thread of one CTA.
//
// Cholesky follows the row-oriented form of cholesky_small (linalg.py:164-184):
//   piv_j = B_jj - R[:j,j].R[:j,j];  breakdown if !finite(piv) or piv <= tol*max|diag B|
//   R_jj = sqrt(piv);  R[j,k] = (B_jk - R[:j,j].R[:j,k]) / R_jj   (k > j)
// and the triangular solves of trsm_right_inv (linalg.py:187-196) become a
// multiply by the explicit upper inverse S = R^-1.
#pragma once
#include <math.h>
#include "common.cuh"

namespace ekcg_dev {

constexpr int kMaxM = 64;


// Cholesky of the symmetric m x m matrix in smem B (row-major); R (smem) gets
// the upper factor.  Returns -1 on success, else the failing column (and the
// pivot/scale through the references).  All threads participate.
__device__ inline int chol_rows(const double* B, double* R, int m, double tol, double& piv_out,
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
__device__ inline void tri_inverse(const double* R, double* S, int m) {
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

// Fixed-width fast path (M = 8, 16, 32): right-looking Cholesky with a
// CTA-parallel trailing update (two barriers per column), then S = R^-1 with
// one thread per column, the column kept in registers (fully unrolled).  A is
// the symmetric input (smem, overwritten); R and S (smem) get the factor and
// its inverse.  Same breakdown test as chol_rows.  Returns -1 or the column.
template <int M>
__device__ inline int chol_inv_fixed(double* A, double* R, double* S, double tol, double& piv_out,
                                     double& scale_out) {
    __shared__ double s_rinv[M];
    __shared__ double s_scale;
    const int tid = threadIdx.y * blockDim.x + threadIdx.x, nthr = blockDim.x * blockDim.y;
    for (int e = tid; e < M * M; e += nthr) R[e] = 0.0;
    if (tid == 0) {
        double sc = 0.0;
#pragma unroll
        for (int j = 0; j < M; ++j) sc = fmax(sc, fabs(A[j * M + j]));
        s_scale = sc;
    }
    __syncthreads();
    const double scale = s_scale;
    scale_out = scale;
#pragma unroll 1
    for (int j = 0; j < M; ++j) {
        const double piv = A[j * M + j];
        if (!isfinite(piv) || piv <= tol * scale) {
            piv_out = piv;
            return j;
        }
        const double rjj = sqrt(piv);
        for (int k = j + 1 + tid; k < M; k += nthr) R[j * M + k] = A[j * M + k] / rjj;
        if (tid == 0) {
            R[j * M + j] = rjj;
            s_rinv[j] = 1.0 / rjj;
        }
        __syncthreads();
        const int L = M - j - 1;
        for (int e = tid; e < L * L; e += nthr) {
            const int i = j + 1 + e / L, k = j + 1 + e % L;
            A[i * M + k] -= R[j * M + i] * R[j * M + k];
        }
        __syncthreads();
    }
    if (tid < M) {
        const int c = tid;
        double col[M];
#pragma unroll
        for (int i = M - 1; i >= 0; --i) {
            double s = 0.0;
#pragma unroll
            for (int k = i + 1; k < M; ++k) s += (k <= c) ? R[i * M + k] * col[k] : 0.0;
            col[i] = (i > c) ? 0.0 : (i == c) ? s_rinv[c] : -s * s_rinv[i];
        }
#pragma unroll
        for (int i = 0; i < M; ++i) S[i * M + c] = col[i];
    }
    __syncthreads();
    return -1;
}

// Cholesky + explicit inverse of the symmetric m x m matrix in A (smem,
// overwritten): R, S = R^-1 into smem.  -1 or the failing column.
__device__ inline int chol_inverse(double* A, double* R, double* S, int m, double tol, double& piv, double& scale) {
    switch (m) {
        case 8: return chol_inv_fixed<8>(A, R, S, tol, piv, scale);
        case 16: return chol_inv_fixed<16>(A, R, S, tol, piv, scale);
        case 32: return chol_inv_fixed<32>(A, R, S, tol, piv, scale);
        default: {
            const int fail = chol_rows(A, R, m, tol, piv, scale);
            if (fail < 0) tri_inverse(R, S, m);
            return fail;
        }
    }
}

__device__ inline void record_breakdown(EkcgCtrl* ctrl, int kind, int col, double piv, double scale, int iteration) {
    if (iteration <= 0) iteration = ctrl->k_done + 1;  // graph replay: iteration read on the device
    ctrl->brk_kind = kind;
    ctrl->brk_col = col;
    ctrl->brk_pivot = piv;
    ctrl->brk_scale = scale;
    ctrl->brk_iter = iteration;
    ctrl->status = 3;
    ctrl->live = 0;
}


// Pre-CholQR factor from the raw Gram G = W^T W (smem, m x m, overwritten):
// column norms D (aortho.py:74-79), G0 = sym(D^-1 G D^-1), R0 = chol(G0),
// S0 = D^-1 R0^-1 written to global S0out.  R, S: smem scratch (m*m each).
__device__ inline void prechol_body(double* G, double* R, double* S, int m, double* S0out, EkcgCtrl* ctrl,
                                    int iteration, double tol) {
    __shared__ double nrm[kMaxM];
    __shared__ int dead;
    __shared__ double piv, scale;
    const int tid = threadIdx.x;
    if (tid == 0) dead = -1;
    for (int j = tid; j < m; j += blockDim.x) nrm[j] = sqrt(G[j * m + j]);
    __syncthreads();
    if (tid == 0) {
        for (int j = 0; j < m; ++j)
            if (nrm[j] == 0.0) { dead = j; break; }
        if (dead >= 0) record_breakdown(ctrl, 1, dead, 0.0, 0.0, iteration);
    }
    __syncthreads();
    if (dead >= 0) return;
    // G0 = sym(D^-1 G D^-1) into R (as scratch), then back into G
    for (int e = tid; e < m * m; e += blockDim.x) {
        int a = e / m, b = e % m;
        double gab = G[a * m + b] / nrm[a] / nrm[b];
        double gba = G[b * m + a] / nrm[b] / nrm[a];
        R[e] = 0.5 * (gab + gba);
    }
    __syncthreads();
    for (int e = tid; e < m * m; e += blockDim.x) G[e] = R[e];
    __syncthreads();
    int fail = chol_inverse(G, R, S, m, tol, piv, scale);
    if (fail >= 0) {
        if (tid == 0) record_breakdown(ctrl, 2, fail, piv, scale, iteration);
        return;
    }
    for (int e = tid; e < m * m; e += blockDim.x) S0out[e] = S[e] / nrm[e / m];
}

// A-CholQR factor: R = chol(sym(G)), S = R^-1 written to global Sout.  G
// (smem, m x m) is overwritten.
__device__ inline void cholinv_body(double* G, double* R, double* S, int m, double* Sout, EkcgCtrl* ctrl,
                                    int iteration, double tol) {
    __shared__ double piv, scale;
    const int tid = threadIdx.x;
    for (int e = tid; e < m * m; e += blockDim.x) {
        int a = e / m, b = e % m;
        R[e] = 0.5 * (G[a * m + b] + G[b * m + a]);
    }
    __syncthreads();
    for (int e = tid; e < m * m; e += blockDim.x) G[e] = R[e];
    __syncthreads();
    int fail = chol_inverse(G, R, S, m, tol, piv, scale);
    if (fail >= 0) {
        if (tid == 0) record_breakdown(ctrl, 2, fail, piv, scale, iteration);
        return;
    }
    for (int e = tid; e < m * m; e += blockDim.x) Sout[e] = S[e];
}

// End of iteration k (solvers.py:398-415, :357), single thread.
__device__ inline void finish_body(EkcgCtrl* ctrl, double rho2, int k, int kmax, int stagnation_window,
                                   double* history) {
    if (k <= 0) k = ctrl->k_done + 1;  // graph replay: iteration read on the device
    double rho = sqrt(rho2);
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
    if (rho <= ctrl->tol_abs) {
        ctrl->status = 1;
        ctrl->live = 0;
    } else if (!(rho > ctrl->tol_abs) || k + 1 > kmax) {
        // NaN residual: the reference's loop test `history[-1] > tol * rho0` is false, so it stops, and
        // `history[-1] <= tol * rho0` is false too, so the status is "maxiter" (solvers.py:357,417)
        ctrl->status = 2;
        ctrl->live = 0;
    }
}

// "Last CTA" arrival for deterministic in-kernel reductions: every CTA has
// written its partial; the CTA that increments the counter last returns true
// (after a fence) and then sums all partials in fixed order.  It also resets
// the counter for the next launch.
__device__ inline bool last_cta_arrive(unsigned int* counter) {
    __shared__ bool is_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0 && threadIdx.y == 0) {
        unsigned total = gridDim.x * gridDim.y;
        unsigned prev = atomicAdd(counter, 1u);
        is_last = (prev == total - 1);
        if (is_last) *counter = 0u;
    }
    __syncthreads();
    if (is_last) __threadfence();
    return is_last;
}

// Like last_cta_arrive for `expected` arrivals on `counter` (a group of CTAs);
// the last one gets true and resets the counter.
__device__ inline bool last_arrive(unsigned int* counter, unsigned expected) {
    __shared__ bool is_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0 && threadIdx.y == 0) {
        unsigned prev = atomicAdd(counter, 1u);
        is_last = (prev == expected - 1);
        if (is_last) *counter = 0u;
    }
    __syncthreads();
    if (is_last) __threadfence();
    return is_last;
}

// out[j] = sum_{p < P} partials[p*len + j] (fixed order, L2-coherent loads), by one CTA.
__device__ inline void cta_sum_partials(const double* partials, int P, int len, double* out) {
    const int nthr = blockDim.x * blockDim.y;
    const int tid = threadIdx.y * blockDim.x + threadIdx.x;
    for (int j = tid; j < len; j += nthr) {
        double s = __ldcg(partials + j);
        for (int p = 1; p < P; ++p) s += __ldcg(partials + (long long)p * len + j);
        out[j] = s;
    }
    __syncthreads();
}

// Deterministic high-MLP sum of P partial vectors by one CTA: thread j sums
// p = 0..P-1 into 16 interleaved accumulators, then combines them in order.
__device__ inline void cta_sum_partials_mlp(const double* partials, int P, int len, double* out) {
    const int nthr = blockDim.x * blockDim.y;
    const int tid = threadIdx.y * blockDim.x + threadIdx.x;
    for (int j = tid; j < len; j += nthr) {
        double acc[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) acc[q] = 0.0;
        int p = 0;
        for (; p + 16 <= P; p += 16) {
#pragma unroll
            for (int q = 0; q < 16; ++q) acc[q] += __ldcg(partials + (long long)(p + q) * len + j);
        }
        for (int q = 0; p < P; ++p, ++q) acc[q] += __ldcg(partials + (long long)p * len + j);
        double s = acc[0];
#pragma unroll
        for (int q = 1; q < 16; ++q) s += acc[q];
        out[j] = s;
    }
    __syncthreads();
}

}  // namespace ekcg_dev
