// Fused iteration kernels: each removes whole passes over an n x m block and
// the separate reduce / factor launches of the unfused sequence.
//
//   ekcg_update_prechol  W'' = W' - sum Q_i C_i (CGS2 pass 2, aortho.py:93-94)
//                        + Graw = W''^T W'' + Pre-CholQR factor S0 (aortho.py:104-106)
//   ekcg_update_vec      W_k = W0 S (trsm_right_inv, linalg.py:187-196)
//                        + alpha = W_k^T r (solvers.py:394)
//   ekcg_stencil_cholinv G = W0^T (A W0) without writing A W0 + A-CholQR
//                        factor S (aortho.py:107-109)
//   ekcg_stencil_xr      AW_k = A W_k (written) + x += W_k alpha, r -= AW_k alpha,
//                        |r|^2 and the end-of-iteration bookkeeping (solvers.py:394-415)
//
// Split-K partial sums are reduced inside the kernel by the last CTA to arrive
// (an integer ticket, then a fixed-order sum), so results stay bit-identical
// from run to run.  That CTA also runs the m x m factorization.
#include "common.cuh"
#include "ekcg_b200.h"
#include "factor.cuh"
#include "stencil.cuh"

namespace {

using namespace ekcg_dev;

// smem row stride (doubles) so the 4 rows of an mma k-step land 8 banks apart
__host__ __device__ constexpr int pad_stride(int M) { return M == 8 ? 20 : M + 4; }

constexpr int kFusedCtas = 148 * 2;

// acc[ta][tb] += A^T B over the k-steps [k0, k1) (stride ks) of a row tile in
// smem: A rows TA[r][a0 + .], B rows TB[r][b0 + .] with row stride lds.
template <int NA, int NB>
__device__ __forceinline__ void smem_gram(const double* TA, const double* TB, int lds, int a0, int b0, int k0,
                                          int k1, int ks, int lane, double (&acc)[NA][NB][2]) {
    const int lr = lane & 3, lc = lane >> 2;
    for (int k = k0; k < k1; k += ks) {
        const int r = 4 * k + lr;
        double af[NA], bf[NB];
#pragma unroll
        for (int ta = 0; ta < NA; ++ta) af[ta] = TA[r * lds + a0 + 8 * ta + lc];
#pragma unroll
        for (int tb = 0; tb < NB; ++tb) bf[tb] = TB[r * lds + b0 + 8 * tb + lc];
#pragma unroll
        for (int ta = 0; ta < NA; ++ta)
#pragma unroll
            for (int tb = 0; tb < NB; ++tb) dmma_8x8x4(acc[ta][tb], af[ta], bf[tb]);
    }
}

// ---------------------------------------------------------------------------
// Block update with epilogue.  CTA tile = 4 warps x 8*MR rows; every warp of
// the CTA walks the same tiles so the epilogue can use __syncthreads.
//   EPI 1: Graw partial of the output rows (staged in smem) -> prechol -> S0
//   EPI 2: alpha partial = out^T vec -> alpha
// ---------------------------------------------------------------------------
template <int M, int MR, int EPI>
__global__ void __launch_bounds__(128)
update_epi_kernel(const double* const* __restrict__ Qs, int ldq, int d, const double* __restrict__ C,
                  const double* Win, int ldwi, double* Wout, int ldwo, double beta, double sign, long long n,
                  const double* __restrict__ vec, double* __restrict__ partials, unsigned int* counter,
                  double* out, EkcgCtrl* ctrl, int iteration, double tol) {
    pdl_wait();
    if (ctrl->live == 0) return;
    extern __shared__ double sm[];
    constexpr int NT = M / 8;
    constexpr int KK = M / 4;
    constexpr int LDS = pad_stride(M);
    constexpr int RT = 32 * MR;
    constexpr bool SPLITK = (M <= 16);
    constexpr int GT = SPLITK ? NT : NT / 2;  // Gram tiles per warp and axis
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int lr = lane & 3, lc = lane >> 2;
    const int ga0 = SPLITK ? 0 : (warp % 2) * (M / 2);
    const int gb0 = SPLITK ? 0 : (warp / 2) * (M / 2);

    double gacc[GT][GT][2];
    double vacc[NT][2];
#pragma unroll
    for (int a = 0; a < GT; ++a)
#pragma unroll
        for (int b = 0; b < GT; ++b) gacc[a][b][0] = gacc[a][b][1] = 0.0;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) vacc[nt][0] = vacc[nt][1] = 0.0;

    const long long tiles = (n + RT - 1) / RT;
    for (long long tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
        const long long rbase = tile * RT + warp * 8 * MR;
        double acc[MR][NT][2];
#pragma unroll
        for (int mr = 0; mr < MR; ++mr)
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) acc[mr][nt][0] = acc[mr][nt][1] = 0.0;
        for (int i = 0; i < d; ++i) {
            const double* __restrict__ Q = Qs[i];
            const double* __restrict__ Ci = C + (long long)i * M * M;
#pragma unroll
            for (int kk = 0; kk < KK; ++kk) {
                double bfr[NT];
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) bfr[nt] = __ldg(Ci + (4 * kk + lr) * M + 8 * nt + lc);
                double afr[MR];
#pragma unroll
                for (int mr = 0; mr < MR; ++mr) {
                    long long r = rbase + 8 * mr + lc;
                    afr[mr] = (r < n) ? __ldg(Q + r * ldq + 4 * kk + lr) : 0.0;
                }
#pragma unroll
                for (int mr = 0; mr < MR; ++mr)
#pragma unroll
                    for (int nt = 0; nt < NT; ++nt) dmma_8x8x4(acc[mr][nt], afr[mr], bfr[nt]);
            }
        }
#pragma unroll
        for (int mr = 0; mr < MR; ++mr) {
            const long long r = rbase + 8 * mr + lc;
            const int trow = warp * 8 * MR + 8 * mr + lc;
            const double vr = (EPI == 2 && r < n) ? vec[r] : 0.0;
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
                const int b = 8 * nt + 2 * lr;
                double o0 = 0.0, o1 = 0.0;
                if (r < n) {
                    o0 = sign * acc[mr][nt][0];
                    o1 = sign * acc[mr][nt][1];
                    if (beta != 0.0) {
                        o0 = beta * Win[r * ldwi + b] + o0;
                        o1 = beta * Win[r * ldwi + b + 1] + o1;
                    }
                    Wout[r * ldwo + b] = o0;
                    Wout[r * ldwo + b + 1] = o1;
                }
                if (EPI == 1) {
                    sm[trow * LDS + b] = o0;
                    sm[trow * LDS + b + 1] = o1;
                } else {
                    vacc[nt][0] += o0 * vr;
                    vacc[nt][1] += o1 * vr;
                }
            }
        }
        if (EPI == 1) {
            __syncthreads();
            if (SPLITK) smem_gram<GT, GT>(sm, sm, LDS, 0, 0, warp, RT / 4, 4, lane, gacc);
            else smem_gram<GT, GT>(sm, sm, LDS, ga0, gb0, 0, RT / 4, 1, lane, gacc);
            __syncthreads();
        }
    }

    // ---- CTA partial ----
    if (EPI == 1) {
        double* red = sm;  // SPLITK: [4][M*M]; else [M*M] (quadrants are disjoint)
#pragma unroll
        for (int ta = 0; ta < GT; ++ta)
#pragma unroll
            for (int tb = 0; tb < GT; ++tb) {
                const int a = ga0 + 8 * ta + lc, b = gb0 + 8 * tb + 2 * lr;
                const int base = SPLITK ? warp * M * M : 0;
                red[base + a * M + b] = gacc[ta][tb][0];
                red[base + a * M + b + 1] = gacc[ta][tb][1];
            }
        __syncthreads();
        for (int o = threadIdx.x; o < M * M; o += blockDim.x) {
            double s = red[o];
            if (SPLITK)
                for (int w = 1; w < 4; ++w) s += red[w * M * M + o];
            partials[(long long)blockIdx.x * M * M + o] = s;
        }
    } else {
        __shared__ double vred[4][M];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                double v = vacc[nt][h];
                v += __shfl_xor_sync(0xffffffffu, v, 4);
                v += __shfl_xor_sync(0xffffffffu, v, 8);
                v += __shfl_xor_sync(0xffffffffu, v, 16);
                if (lc == 0) vred[warp][8 * nt + 2 * lr + h] = v;
            }
        __syncthreads();
        for (int o = threadIdx.x; o < M; o += blockDim.x)
            partials[(long long)blockIdx.x * M + o] = ((vred[0][o] + vred[1][o]) + vred[2][o]) + vred[3][o];
    }

    if (last_cta_arrive(counter)) {
        if (EPI == 1) {
            double* G = sm;
            cta_sum_partials_mlp(partials, gridDim.x, M * M, G);
            prechol_body(G, G + M * M, G + 2 * M * M, M, out, ctrl, iteration, tol);
        } else {
            cta_sum_partials_mlp(partials, gridDim.x, M, out);
        }
    }
}

// ---------------------------------------------------------------------------
// Stencil epilogues.  Block = (G, R) threads, G = M / VEC threads per row.
// ---------------------------------------------------------------------------

// G = W0^T (A W0) partials from smem row tiles, then cholinv by the last CTA.
template <int VEC, int M>
__global__ void __launch_bounds__(256)
stencil_cholinv_kernel(EkcgStencil s, UniformFaces uf, const double* __restrict__ X, int ldx,
                       double* __restrict__ partials, unsigned int* counter, double* Sout, EkcgCtrl* ctrl,
                       int iteration, double tol, int finalize) {
    pdl_wait();
    if (ctrl->live == 0) return;
    extern __shared__ double sm[];
    constexpr int G = M / VEC;
    constexpr int R = 256 / G;
    constexpr int LDS = pad_stride(M);
    constexpr int NT = M / 8;
    constexpr int KSTEPS = R / 4;
    // warp -> (tile group, k lane): M<=16 all tiles per warp; M=32 4 groups of
    // 2x2 tiles; M=64 8 groups of 4x2 tiles.
    constexpr int GA = (M <= 16) ? NT : 4 / ((M == 32) ? 2 : 1);
    constexpr int GBT = (M <= 16) ? NT : 2;
    constexpr int NGROUPS = (M <= 16) ? 1 : (M == 32 ? 4 : 8);
    constexpr int KL = 8 / NGROUPS;  // warps sharing a group split the k-steps
    double* TX = sm;             // [R][LDS]  W0 rows
    double* TY = sm + R * LDS;   // [R][LDS]  (A W0) rows
    const int warp = (threadIdx.y * blockDim.x + threadIdx.x) >> 5;
    const int lane = (threadIdx.y * blockDim.x + threadIdx.x) & 31;
    const int grp = warp % NGROUPS, kl = warp / NGROUPS;
    constexpr int AGROUPS = (M <= 16) ? 1 : M / (8 * GA);
    const int a0 = (grp % AGROUPS) * 8 * GA;
    const int b0 = (grp / AGROUPS) * 8 * GBT;
    double gacc[GA][GBT][2];
#pragma unroll
    for (int a = 0; a < GA; ++a)
#pragma unroll
        for (int b = 0; b < GBT; ++b) gacc[a][b][0] = gacc[a][b][1] = 0.0;

    const long long n = s.row_end;
    const int c0 = threadIdx.x * VEC;
    const int ty = threadIdx.y;
    for (long long base = s.row_begin + (long long)blockIdx.x * R; base < n; base += (long long)gridDim.x * R) {
        const long long i = base + ty;
        double y[VEC];
        if (i < n) {
            long long off[7];
            double val[7];
            int dpos;
            const int cnt = stencil_row(s, uf, i, off, val, dpos);
            stencil_apply_row<VEC>(X, ldx, c0, M, off, val, cnt, y);
#pragma unroll
            for (int v = 0; v < VEC; ++v) TX[ty * LDS + c0 + v] = __ldg(X + i * ldx + c0 + v);
        } else {
#pragma unroll
            for (int v = 0; v < VEC; ++v) {
                y[v] = 0.0;
                TX[ty * LDS + c0 + v] = 0.0;
            }
        }
#pragma unroll
        for (int v = 0; v < VEC; ++v) TY[ty * LDS + c0 + v] = y[v];
        __syncthreads();
        smem_gram<GA, GBT>(TX, TY, LDS, a0, b0, kl, KSTEPS, KL, lane, gacc);
        __syncthreads();
    }
    // CTA partial: red[kl][M*M] (groups own disjoint outputs), fixed-order sum over kl
    double* red = sm;
    const int lr = lane & 3, lc = lane >> 2;
#pragma unroll
    for (int ta = 0; ta < GA; ++ta)
#pragma unroll
        for (int tb = 0; tb < GBT; ++tb) {
            const int a = a0 + 8 * ta + lc, b = b0 + 8 * tb + 2 * lr;
            red[kl * M * M + a * M + b] = gacc[ta][tb][0];
            red[kl * M * M + a * M + b + 1] = gacc[ta][tb][1];
        }
    __syncthreads();
    const int tid = threadIdx.y * blockDim.x + threadIdx.x;
    for (int o = tid; o < M * M; o += 256) {
        double sacc = red[o];
        for (int k = 1; k < KL; ++k) sacc += red[k * M * M + o];
        partials[(long long)blockIdx.x * M * M + o] = sacc;
    }
    if (last_cta_arrive(counter)) {
        if (!finalize) {
            cta_sum_partials_mlp(partials, gridDim.x * gridDim.y, M * M, Sout);  // local G
        } else {
            double* Gm = sm;
            cta_sum_partials_mlp(partials, gridDim.x * gridDim.y, M * M, Gm);
            cholinv_body(Gm, Gm + M * M, Gm + 2 * M * M, M, Sout, ctrl, iteration, tol);
        }
    }
}

// AW = A W (written), x += W alpha, r -= AW alpha, |r|^2; the last CTA
// finishes the iteration (or just stores |r|^2 when do_finish == 0).
template <int VEC>
__global__ void __launch_bounds__(256)
stencil_xr_kernel(EkcgStencil s, UniformFaces uf, const double* __restrict__ X, int ldx, double* __restrict__ Y,
                  int ldy, int m, const double* __restrict__ alpha, double* __restrict__ x, double* __restrict__ r,
                  double* __restrict__ partials, unsigned int* counter, EkcgCtrl* ctrl, int k, int kmax,
                  int stagnation_window, double* __restrict__ history, int do_finish, double* rho2_out) {
    pdl_wait();
    if (ctrl->live == 0) return;
    __shared__ double sa[64];
    __shared__ double wsum[8];
    const int tid = threadIdx.y * blockDim.x + threadIdx.x;
    for (int a = tid; a < m; a += 256) sa[a] = alpha[a];
    __syncthreads();
    const int G = blockDim.x;
    const long long n = s.row_end;
    const int c0 = threadIdx.x * VEC;
    double sq = 0.0;
    for (long long base = s.row_begin + (long long)blockIdx.x * blockDim.y; base < n;
         base += (long long)gridDim.x * blockDim.y) {
        const long long i = base + threadIdx.y;
        double dx = 0.0, dr = 0.0;
        if (i < n) {
            long long off[7];
            double val[7];
            int dpos;
            const int cnt = stencil_row(s, uf, i, off, val, dpos);
            double y[VEC];
            stencil_apply_row<VEC>(X, ldx, c0, m, off, val, cnt, y);
            if (VEC >= 2 && c0 + VEC <= m) {
#pragma unroll
                for (int h = 0; h < VEC / 2; ++h)
                    reinterpret_cast<double2*>(Y + i * ldy + c0)[h] = make_double2(y[2 * h], y[2 * h + 1]);
            } else {
                for (int v = 0; v < VEC && c0 + v < m; ++v) Y[i * ldy + c0 + v] = y[v];
            }
#pragma unroll
            for (int v = 0; v < VEC; ++v) {
                if (c0 + v < m) {
                    dx += __ldg(X + i * ldx + c0 + v) * sa[c0 + v];
                    dr += y[v] * sa[c0 + v];
                }
            }
        }
        // the G threads of a row are consecutive lanes
        for (int o = G / 2; o > 0; o >>= 1) {
            dx += __shfl_xor_sync(0xffffffffu, dx, o);
            dr += __shfl_xor_sync(0xffffffffu, dr, o);
        }
        if (i < n && threadIdx.x == 0) {
            x[i] = x[i] + dx;
            const double rn = r[i] - dr;
            r[i] = rn;
            sq += rn * rn;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
    if ((tid & 31) == 0) wsum[tid >> 5] = sq;
    __syncthreads();
    if (tid == 0) {
        double t = wsum[0];
        for (int w = 1; w < 8; ++w) t += wsum[w];
        partials[blockIdx.x] = t;
    }
    if (last_cta_arrive(counter)) {
        __shared__ double tot;
        if (tid < 32) {
            double acc = 0.0;
            for (int p = tid; p < (int)gridDim.x; p += 32) acc += __ldcg(partials + p);
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            if (tid == 0) tot = acc;
        }
        __syncthreads();
        if (tid == 0) {
            if (do_finish) finish_body(ctrl, tot, k, kmax, stagnation_window, history);
            else *rho2_out = tot;
        }
    }
}

bool set_smem(const void* fn, size_t bytes) {
    if (bytes <= 48 * 1024) return true;
    return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) == cudaSuccess;
}

template <int M, int MR, int EPI>
int launch_update_epi(const double* const* Qs, int ldq, int d, const double* C, const double* Win, int ldwi,
                      double* Wout, int ldwo, double beta, double sign, long long n, const double* vec,
                      double* partials, unsigned int* counter, double* out, EkcgCtrl* ctrl, int iteration,
                      double tol, cudaStream_t st) {
    constexpr int LDS = pad_stride(M);
    constexpr int RT = 32 * MR;
    size_t smem = 0;
    if (EPI == 1) {
        size_t need = (size_t)RT * LDS;
        if ((size_t)4 * M * M > need) need = 4 * M * M;
        if ((size_t)3 * M * M > need) need = 3 * M * M;
        smem = need * sizeof(double);
    }
    auto fn = update_epi_kernel<M, MR, EPI>;
    if (!set_smem((const void*)fn, smem)) return EKCG_ELAUNCH;
    long long tiles = (n + RT - 1) / RT;
    int grid = (int)(tiles < kFusedCtas ? tiles : kFusedCtas);
    launch_k(fn, grid, 128, smem, st, Qs, ldq, d, C, Win, ldwi, Wout, ldwo, beta, sign, n, vec, partials, counter, out,
                                ctrl, iteration, tol);
    return EKCG_OK;
}

template <int VEC, int M>
int launch_stencil_cholinv(const EkcgStencil& s, const UniformFaces& uf, long long n, const double* X, int ldx,
                           double* partials, unsigned int* counter, double* Sout, EkcgCtrl* ctrl, int iteration,
                           double tol, int finalize, cudaStream_t st) {
    constexpr int G = M / VEC;
    constexpr int R = 256 / G;
    constexpr int LDS = pad_stride(M);
    constexpr int NGROUPS = (M <= 16) ? 1 : (M == 32 ? 4 : 8);
    constexpr int KL = 8 / NGROUPS;
    size_t need = (size_t)2 * R * LDS;
    if ((size_t)KL * M * M > need) need = (size_t)KL * M * M;
    if ((size_t)3 * M * M > need) need = 3 * M * M;
    size_t smem = need * sizeof(double);
    auto fn = stencil_cholinv_kernel<VEC, M>;
    if (!set_smem((const void*)fn, smem)) return EKCG_ELAUNCH;
    long long blocks = (n + R - 1) / R;
    int grid = (int)(blocks < kFusedCtas ? blocks : kFusedCtas);
    launch_k(fn, grid, dim3(G, R), smem, st, s, uf, X, ldx, partials, counter, Sout, ctrl, iteration, tol, finalize);
    return EKCG_OK;
}

}  // namespace

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
extern "C" int ekcg_fused_partials(long long n, int m) {
    (void)n;
    return (kFusedCtas + 64) * (m * m > 1 ? m * m : 1);  // + group sums of the two-level reduction
}

extern "C" int ekcg_update_prechol(const double* const* Qs, int ldq, int d, const double* C, const double* Win,
                                   int ldwi, double* Wout, int ldwo, int m, long long n, double* partials,
                                   unsigned int* counter, double* S0, void* ctrl, int iteration, double tol,
                                   void* stream) {
    if (d < 1 || ldq < m || ldwi < m || ldwo < m || n < 1 || ctrl == nullptr) return EKCG_EINVAL;
    EkcgCtrl* c = (EkcgCtrl*)ctrl;
    cudaStream_t st = as_stream(stream);
    int rc;
    switch (m) {
        case 8: rc = launch_update_epi<8, 4, 1>(Qs, ldq, d, C, Win, ldwi, Wout, ldwo, 1.0, -1.0, n, nullptr, partials, counter, S0, c, iteration, tol, st); break;
        case 16: rc = launch_update_epi<16, 4, 1>(Qs, ldq, d, C, Win, ldwi, Wout, ldwo, 1.0, -1.0, n, nullptr, partials, counter, S0, c, iteration, tol, st); break;
        case 32: rc = launch_update_epi<32, 4, 1>(Qs, ldq, d, C, Win, ldwi, Wout, ldwo, 1.0, -1.0, n, nullptr, partials, counter, S0, c, iteration, tol, st); break;
        case 64: rc = launch_update_epi<64, 2, 1>(Qs, ldq, d, C, Win, ldwi, Wout, ldwo, 1.0, -1.0, n, nullptr, partials, counter, S0, c, iteration, tol, st); break;
        default: return EKCG_EINVAL;
    }
    if (rc != EKCG_OK) return rc;
    ++g_ekcg_launches;
    return launch_status();
}

extern "C" int ekcg_update_vec(const double* const* Qs, int ldq, const double* S, double* Wout, int ldwo, int m,
                               long long n, const double* vec, double* partials, unsigned int* counter,
                               double* vout, void* ctrl, void* stream) {
    if (ldq < m || ldwo < m || n < 1 || ctrl == nullptr) return EKCG_EINVAL;
    EkcgCtrl* c = (EkcgCtrl*)ctrl;
    cudaStream_t st = as_stream(stream);
    int rc;
    switch (m) {
        case 8: rc = launch_update_epi<8, 4, 2>(Qs, ldq, 1, S, nullptr, m, Wout, ldwo, 0.0, 1.0, n, vec, partials, counter, vout, c, 0, 0.0, st); break;
        case 16: rc = launch_update_epi<16, 4, 2>(Qs, ldq, 1, S, nullptr, m, Wout, ldwo, 0.0, 1.0, n, vec, partials, counter, vout, c, 0, 0.0, st); break;
        case 32: rc = launch_update_epi<32, 4, 2>(Qs, ldq, 1, S, nullptr, m, Wout, ldwo, 0.0, 1.0, n, vec, partials, counter, vout, c, 0, 0.0, st); break;
        case 64: rc = launch_update_epi<64, 2, 2>(Qs, ldq, 1, S, nullptr, m, Wout, ldwo, 0.0, 1.0, n, vec, partials, counter, vout, c, 0, 0.0, st); break;
        default: return EKCG_EINVAL;
    }
    if (rc != EKCG_OK) return rc;
    ++g_ekcg_launches;
    return launch_status();
}

extern "C" int ekcg_stencil_cholinv(const EkcgStencil* desc, const double* X, int ldx, int m, double* partials,
                                    unsigned int* counter, double* S, void* ctrl, int iteration, double tol,
                                    int finalize, void* stream) {
    EkcgStencil s;
    UniformFaces uf;
    long long n;
    int rc = prepare_stencil(desc, s, uf, n);
    if (rc != EKCG_OK) return rc;
    if (ldx != m || ((reinterpret_cast<uintptr_t>(X) & 15) != 0) || ctrl == nullptr) return EKCG_EINVAL;
    EkcgCtrl* c = (EkcgCtrl*)ctrl;
    cudaStream_t st = as_stream(stream);
    n = s.row_end - s.row_begin;
    if (launch_march_cholinv(s, uf, X, ldx, m, partials, counter, S, c, iteration, tol, finalize, kFusedCtas, st) ==
        EKCG_OK) {
        ++g_ekcg_launches;
        return launch_status();
    }
    switch (m) {
        case 8: rc = launch_stencil_cholinv<4, 8>(s, uf, n, X, ldx, partials, counter, S, c, iteration, tol, finalize, st); break;
        case 16: rc = launch_stencil_cholinv<4, 16>(s, uf, n, X, ldx, partials, counter, S, c, iteration, tol, finalize, st); break;
        case 32: rc = launch_stencil_cholinv<4, 32>(s, uf, n, X, ldx, partials, counter, S, c, iteration, tol, finalize, st); break;
        case 64: rc = launch_stencil_cholinv<4, 64>(s, uf, n, X, ldx, partials, counter, S, c, iteration, tol, finalize, st); break;
        default: return EKCG_EINVAL;
    }
    if (rc != EKCG_OK) return rc;
    ++g_ekcg_launches;
    return launch_status();
}

extern "C" int ekcg_stencil_xr(const EkcgStencil* desc, const double* X, int ldx, double* Y, int ldy, int m,
                               const double* alpha, double* x, double* r, double* partials, unsigned int* counter,
                               void* ctrl, int k, int kmax, int stagnation_window, double* history, int do_finish,
                               double* rho2_out, void* stream) {
    EkcgStencil s;
    UniformFaces uf;
    long long n;
    int rc = prepare_stencil(desc, s, uf, n);
    if (rc != EKCG_OK) return rc;
    if (m < 1 || m > 64 || ldx < m || ldy < m || ctrl == nullptr) return EKCG_EINVAL;
    EkcgCtrl* c = (EkcgCtrl*)ctrl;
    cudaStream_t st = as_stream(stream);
    const bool aligned = (ldx % 2 == 0) && (ldy % 2 == 0) && ((reinterpret_cast<uintptr_t>(X) & 15) == 0) &&
                         ((reinterpret_cast<uintptr_t>(Y) & 15) == 0);
    if (launch_march_xr(s, uf, X, ldx, Y, ldy, m, alpha, x, r, partials, counter, c, k, kmax, stagnation_window,
                        history, do_finish, rho2_out, kFusedCtas, st) == EKCG_OK) {
        ++g_ekcg_launches;
        return launch_status();
    }
    int vec = 1;
    if (aligned && m % 4 == 0) vec = 4;
    else if (aligned && m % 2 == 0) vec = 2;
    int g = (m + vec - 1) / vec;
    int gp = 1;
    while (gp < g) gp <<= 1;  // threads per row: power of two so a row's lanes are shuffle-aligned
    if (gp > 32) return EKCG_EINVAL;
    dim3 block(gp, 256 / gp);
    n = s.row_end - s.row_begin;
    long long blocks = (n + block.y - 1) / block.y;
    int grid = (int)(blocks < kFusedCtas ? blocks : kFusedCtas);
    if (vec == 4)
        launch_k(stencil_xr_kernel<4>, grid, block, 0, st, s, uf, X, ldx, Y, ldy, m, alpha, x, r, partials, counter, c, k,
                                                    kmax, stagnation_window, history, do_finish, rho2_out);
    else if (vec == 2)
        launch_k(stencil_xr_kernel<2>, grid, block, 0, st, s, uf, X, ldx, Y, ldy, m, alpha, x, r, partials, counter, c, k,
                                                    kmax, stagnation_window, history, do_finish, rho2_out);
    else
        launch_k(stencil_xr_kernel<1>, grid, block, 0, st, s, uf, X, ldx, Y, ldy, m, alpha, x, r, partials, counter, c, k,
                                                    kmax, stagnation_window, history, do_finish, rho2_out);
    ++g_ekcg_launches;
    return launch_status();
}
