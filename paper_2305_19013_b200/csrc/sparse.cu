// Sparse operator kernels: T^t split, bit-exact CSR SpMM, bit-exact grid stencil SpMM.
//
// Bit-exactness contract (reference linalg.py:133-152): numpy's
// `np.add.reduceat(values[:,None] * X[col_idx], row_ptr[:-1], axis=0)` forms each
// product p_j = fl(v_j * x_cj) separately and sums a row as
//     y_i = p_0 + pairwise(p_1, ..., p_k)
// where `pairwise` is numpy's pairwise summation (sequential below 8 terms,
// 8-way blocked up to 128, recursive halving above).  The kernels below
// reproduce that association with __dmul_rn/__dadd_rn (no FMA contraction).
#include "common.cuh"
#include "ekcg_b200.h"

// ---------------------------------------------------------------------------
// Launch shape shared by the row-wise kernels: blockDim = (G, R) with G threads
// per row (one per column group) and R rows per block, grid-striding over
// rows -- no 64-bit integer division in the index math.
// ---------------------------------------------------------------------------
struct RowLaunch {
    dim3 grid, block;
};

static RowLaunch row_launch(long long n, int groups) {
    if (groups > 256) groups = 256;
    int rows = 256 / groups;
    if (rows < 1) rows = 1;
    long long blocks = (n + rows - 1) / rows;
    long long cap = 148LL * 16;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    return {dim3((unsigned)blocks), dim3(groups, rows)};
}

#define ROW_LOOP(row, n)                                                                  \
    for (long long row = (long long)blockIdx.x * blockDim.y + threadIdx.y; row < (n);   \
         row += (long long)gridDim.x * blockDim.y)

// ---------------------------------------------------------------------------
// T^t split: W[i, j] = (owner[i] == j) ? v[i] : +0.0  (partition.py:48-55)
// ---------------------------------------------------------------------------
__global__ void split_kernel(const double* __restrict__ v, const int* __restrict__ owner,
                             double* __restrict__ W, long long n, int t, int ldw,
                             const int* __restrict__ live) {
    EKCG_GATE(live);
    ROW_LOOP(i, n) {
        const int own = owner[i];
        const double vi = v[i];
        for (int j = threadIdx.x; j < t; j += blockDim.x) W[i * ldw + j] = (own == j) ? vi : 0.0;
    }
}

// W = split(v) + Wprev * diag(beta)  (MSDO-CG candidate, solvers.py:378-382)
__global__ void split_axpy_kernel(const double* __restrict__ v, const int* __restrict__ owner,
                                  const double* __restrict__ Wprev, int ldp,
                                  const double* __restrict__ beta, double beta_sign,
                                  double* __restrict__ W, long long n, int t, int ldw,
                                  const int* __restrict__ live) {
    EKCG_GATE(live);
    ROW_LOOP(i, n) {
        const int own = owner[i];
        const double vi = v[i];
        for (int j = threadIdx.x; j < t; j += blockDim.x) {
            double s = (own == j) ? vi : 0.0;
            double bj = beta_sign * beta[j];
            W[i * ldw + j] = add_rn(s, mul_rn(Wprev[i * ldp + j], bj));
        }
    }
}

// ---------------------------------------------------------------------------
// numpy pairwise summation of the row tail p_1..p_cnt for one column.
// ---------------------------------------------------------------------------
__device__ __noinline__ double tail_pairwise(const int* __restrict__ ci, const double* __restrict__ vv,
                                             long long lo, long long cnt,
                                             const double* __restrict__ X, int ldx, int col) {
    if (cnt < 8) {
        double acc = -0.0;
        for (long long q = 0; q < cnt; ++q)
            acc = add_rn(acc, mul_rn(vv[lo + q], X[(long long)ci[lo + q] * ldx + col]));
        return acc;
    }
    if (cnt <= 128) {
        double r[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = mul_rn(vv[lo + j], X[(long long)ci[lo + j] * ldx + col]);
        long long q = 8;
        long long stop = cnt - (cnt % 8);
        for (; q < stop; q += 8) {
#pragma unroll
            for (int j = 0; j < 8; ++j)
                r[j] = add_rn(r[j], mul_rn(vv[lo + q + j], X[(long long)ci[lo + q + j] * ldx + col]));
        }
        double acc = add_rn(add_rn(add_rn(r[0], r[1]), add_rn(r[2], r[3])),
                            add_rn(add_rn(r[4], r[5]), add_rn(r[6], r[7])));
        for (; q < cnt; ++q)
            acc = add_rn(acc, mul_rn(vv[lo + q], X[(long long)ci[lo + q] * ldx + col]));
        return acc;
    }
    long long half = cnt / 2;
    half -= half % 8;
    double left = tail_pairwise(ci, vv, lo, half, X, ldx, col);
    double right = tail_pairwise(ci, vv, lo + half, cnt - half, X, ldx, col);
    return add_rn(left, right);
}

// Threads (column, row) of a 2-D block; rows of stencil-like matrices are
// short, so the common branch is the sequential (< 8 term) tail, kept inline.
__global__ void csr_spmm_kernel(const long long* __restrict__ rp, const int* __restrict__ ci,
                                const double* __restrict__ vv, const double* __restrict__ X, int ldx,
                                double* __restrict__ Y, int ldy, long long n, int m,
                                const int* __restrict__ live) {
    EKCG_GATE(live);
    ROW_LOOP(i, n) {
        const long long lo = rp[i], hi = rp[i + 1];
        for (int c = threadIdx.x; c < m; c += blockDim.x) {
            double y;
            if (hi <= lo) {
                y = 0.0;  // unreachable for validated SPD matrices (diagonal present)
            } else {
                double p0 = mul_rn(vv[lo], X[(long long)ci[lo] * ldx + c]);
                long long cnt = hi - lo - 1;
                if (cnt == 0) {
                    y = p0;
                } else if (cnt < 8) {
                    double acc = mul_rn(vv[lo + 1], X[(long long)ci[lo + 1] * ldx + c]);
                    for (long long q = 2; q <= cnt; ++q)
                        acc = add_rn(acc, mul_rn(vv[lo + q], X[(long long)ci[lo + q] * ldx + c]));
                    y = add_rn(p0, acc);
                } else {
                    y = add_rn(p0, tail_pairwise(ci, vv, lo + 1, cnt, X, ldx, c));
                }
            }
            Y[i * ldy + c] = y;
        }
    }
}

// ---------------------------------------------------------------------------
// Grid stencil: the operator `_diffusion_matrix(shape, kappa)` assembles
// (generators.py:25-60), generalised with per-axis coefficients c_axis
// (c = 1 reproduces the reference exactly).  Node kappa comes from a tile
// field (tile edge 1 = a full node field; null field = constant kappa).
// Face between lo/hi nodes: c * (2*k_lo*k_hi/(k_lo+k_hi)); Dirichlet boundary
// faces add c * k_node.  The diagonal accumulates, per axis from slowest to
// fastest: +face_hi, +face_lo, +boundary(first), +boundary(last) -- the order
// of the np.add.at calls in generators.py:46-53.  Row entries in column order:
// z-, y-, x-, diag, x+, y+, z+.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double harmonic_face(double c, double klo, double khi) {
    // generators.py:45 -- `2.0 * ka * kb / (ka + kb)` evaluated left to right.
    double h = __ddiv_rn(mul_rn(mul_rn(2.0, klo), khi), add_rn(klo, khi));
    return mul_rn(c, h);
}

// Per-launch constants for a uniform-kappa grid: faces and boundary terms per
// axis are the same everywhere, computed once on the device by the first
// thread that needs them would cost a barrier; the host passes them instead
// (same IEEE operations, so the same bits as harmonic_face()).
struct UniformFaces {
    double fz, fy, fx;  // c * 2k^2/(2k)
    double bz, by, bx;  // c * k
};

template <int VEC>
__global__ void __launch_bounds__(256)
stencil_spmm_kernel(EkcgStencil s, UniformFaces uf, const double* __restrict__ X, int ldx,
                    double* __restrict__ Y, int ldy, int m, const int* __restrict__ live) {
    EKCG_GATE(live);
    const unsigned nx = s.nx, ny = s.ny, nz = s.nz;
    const long long nxy = (long long)nx * ny;
    const long long n = nxy * nz;
    const bool three = (s.dim == 3);
    const bool uniform = (s.kfield == nullptr);
    const int c0 = threadIdx.x * VEC;
    ROW_LOOP(i, n) {
        const unsigned iu = (unsigned)i;
        const unsigned x = iu % nx;
        const unsigned rest = iu / nx;
        const unsigned y = rest % ny;
        const unsigned z = rest / ny;

        double fzl = 0.0, fzh = 0.0, fyl = 0.0, fyh = 0.0, fxl = 0.0, fxh = 0.0;
        double diag = 0.0;
        if (uniform) {
            if (three) {
                if (z < nz - 1) { fzh = uf.fz; diag = add_rn(diag, fzh); }
                if (z > 0)      { fzl = uf.fz; diag = add_rn(diag, fzl); }
                if (z == 0)      diag = add_rn(diag, uf.bz);
                if (z == nz - 1) diag = add_rn(diag, uf.bz);
            }
            if (y < ny - 1) { fyh = uf.fy; diag = add_rn(diag, fyh); }
            if (y > 0)      { fyl = uf.fy; diag = add_rn(diag, fyl); }
            if (y == 0)      diag = add_rn(diag, uf.by);
            if (y == ny - 1) diag = add_rn(diag, uf.by);
            if (x < nx - 1) { fxh = uf.fx; diag = add_rn(diag, fxh); }
            if (x > 0)      { fxl = uf.fx; diag = add_rn(diag, fxl); }
            if (x == 0)      diag = add_rn(diag, uf.bx);
            if (x == nx - 1) diag = add_rn(diag, uf.bx);
        } else {
            // tile coordinates of the node; a neighbour is in the adjacent tile
            // exactly when the step crosses a tile edge
            const unsigned txi = x / (unsigned)s.tx, tyi = y / (unsigned)s.ty, tzi = z / (unsigned)s.tz;
            const unsigned rx = x - txi * s.tx, ry = y - tyi * s.ty, rz = z - tzi * s.tz;
            const long long fx = s.fx, fxy = (long long)s.fx * s.fy;
            const double* __restrict__ F = s.kfield;
            const long long tc = tzi * fxy + tyi * fx + txi;
            const double kc = F[tc];
            if (three) {
                if (z < nz - 1) { fzh = harmonic_face(s.cz, kc, F[tc + (rz + 1 == (unsigned)s.tz ? fxy : 0)]); diag = add_rn(diag, fzh); }
                if (z > 0)      { fzl = harmonic_face(s.cz, F[tc - (rz == 0 ? fxy : 0)], kc); diag = add_rn(diag, fzl); }
                if (z == 0)      diag = add_rn(diag, mul_rn(s.cz, kc));
                if (z == nz - 1) diag = add_rn(diag, mul_rn(s.cz, kc));
            }
            if (y < ny - 1) { fyh = harmonic_face(s.cy, kc, F[tc + (ry + 1 == (unsigned)s.ty ? fx : 0)]); diag = add_rn(diag, fyh); }
            if (y > 0)      { fyl = harmonic_face(s.cy, F[tc - (ry == 0 ? fx : 0)], kc); diag = add_rn(diag, fyl); }
            if (y == 0)      diag = add_rn(diag, mul_rn(s.cy, kc));
            if (y == ny - 1) diag = add_rn(diag, mul_rn(s.cy, kc));
            if (x < nx - 1) { fxh = harmonic_face(s.cx, kc, F[tc + (rx + 1 == (unsigned)s.tx ? 1 : 0)]); diag = add_rn(diag, fxh); }
            if (x > 0)      { fxl = harmonic_face(s.cx, F[tc - (rx == 0 ? 1 : 0)], kc); diag = add_rn(diag, fxl); }
            if (x == 0)      diag = add_rn(diag, mul_rn(s.cx, kc));
            if (x == nx - 1) diag = add_rn(diag, mul_rn(s.cx, kc));
        }

        // row entries in ascending column order: z-, y-, x-, diag, x+, y+, z+
        long long off[7];
        double val[7];
        int cnt = 0;
        if (three && z > 0)      { off[cnt] = i - nxy; val[cnt++] = -fzl; }
        if (y > 0)               { off[cnt] = i - nx;  val[cnt++] = -fyl; }
        if (x > 0)               { off[cnt] = i - 1;   val[cnt++] = -fxl; }
        off[cnt] = i; val[cnt++] = diag;
        if (x < nx - 1)          { off[cnt] = i + 1;   val[cnt++] = -fxh; }
        if (y < ny - 1)          { off[cnt] = i + nx;  val[cnt++] = -fyh; }
        if (three && z < nz - 1) { off[cnt] = i + nxy; val[cnt++] = -fzh; }

        if (VEC >= 2 && c0 + VEC <= m) {
            // vector path: VEC/2 double2 loads per neighbour row (16 B aligned)
            constexpr int H = VEC >= 2 ? VEC / 2 : 1;
            double2 acc[H], p0[H];
#pragma unroll
            for (int h = 0; h < VEC / 2; ++h) {
                double2 a = __ldg(reinterpret_cast<const double2*>(X + off[0] * ldx + c0) + h);
                double2 b = __ldg(reinterpret_cast<const double2*>(X + off[1] * ldx + c0) + h);
                p0[h] = make_double2(mul_rn(val[0], a.x), mul_rn(val[0], a.y));
                acc[h] = make_double2(mul_rn(val[1], b.x), mul_rn(val[1], b.y));
            }
            for (int q = 2; q < cnt; ++q) {
#pragma unroll
                for (int h = 0; h < VEC / 2; ++h) {
                    double2 a = __ldg(reinterpret_cast<const double2*>(X + off[q] * ldx + c0) + h);
                    acc[h].x = add_rn(acc[h].x, mul_rn(val[q], a.x));
                    acc[h].y = add_rn(acc[h].y, mul_rn(val[q], a.y));
                }
            }
#pragma unroll
            for (int h = 0; h < VEC / 2; ++h)
                reinterpret_cast<double2*>(Y + i * ldy + c0)[h] =
                    make_double2(add_rn(p0[h].x, acc[h].x), add_rn(p0[h].y, acc[h].y));
        } else {
            for (int c = c0; c < c0 + VEC && c < m; ++c) {
                double p0 = mul_rn(val[0], __ldg(X + off[0] * ldx + c));
                double acc = mul_rn(val[1], __ldg(X + off[1] * ldx + c));
                for (int q = 2; q < cnt; ++q) acc = add_rn(acc, mul_rn(val[q], __ldg(X + off[q] * ldx + c)));
                Y[i * ldy + c] = add_rn(p0, acc);
            }
        }
    }
}

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
static double host_face(double c, double k) {
    volatile double two_k = 2.0 * k;
    volatile double num = two_k * k;
    volatile double den = k + k;
    volatile double h = num / den;
    return c * h;
}

extern "C" int ekcg_split(const double* v, const int* owner, double* W, long long n, int t, int ldw,
                          const int* live, void* stream) {
    if (n < 0 || t < 1 || ldw < t) return EKCG_EINVAL;
    if (n == 0) return EKCG_OK;
    RowLaunch L = row_launch(n, t < 32 ? t : 32);
    split_kernel<<<L.grid, L.block, 0, as_stream(stream)>>>(v, owner, W, n, t, ldw, live);
    ++g_ekcg_launches;
    return launch_status();
}

extern "C" int ekcg_split_axpy(const double* v, const int* owner, const double* Wprev, int ldp,
                               const double* beta, double beta_sign, double* W, long long n, int t,
                               int ldw, const int* live, void* stream) {
    if (n < 0 || t < 1 || ldw < t || ldp < t) return EKCG_EINVAL;
    if (n == 0) return EKCG_OK;
    RowLaunch L = row_launch(n, t < 32 ? t : 32);
    split_axpy_kernel<<<L.grid, L.block, 0, as_stream(stream)>>>(v, owner, Wprev, ldp, beta, beta_sign, W, n, t,
                                                                 ldw, live);
    ++g_ekcg_launches;
    return launch_status();
}

extern "C" int ekcg_spmm_csr(const long long* row_ptr, const int* col_idx, const double* values,
                             const double* X, int ldx, double* Y, int ldy, long long n, int m,
                             const int* live, void* stream) {
    if (n < 0 || m < 1 || ldx < m || ldy < m) return EKCG_EINVAL;
    if (n == 0) return EKCG_OK;
    RowLaunch L = row_launch(n, m < 64 ? m : 64);
    csr_spmm_kernel<<<L.grid, L.block, 0, as_stream(stream)>>>(row_ptr, col_idx, values, X, ldx, Y, ldy, n, m,
                                                               live);
    ++g_ekcg_launches;
    return launch_status();
}

extern "C" int ekcg_spmm_stencil(const EkcgStencil* desc, const double* X, int ldx, double* Y, int ldy,
                                 int m, const int* live, void* stream) {
    if (desc == nullptr || m < 1 || ldx < m || ldy < m) return EKCG_EINVAL;
    EkcgStencil s = *desc;
    if (s.dim != 2 && s.dim != 3) return EKCG_EINVAL;
    if (s.dim == 2) s.nz = 1;
    if (s.nx < 2 || s.ny < 2 || (s.dim == 3 && s.nz < 2)) return EKCG_EINVAL;
    if (s.kfield != nullptr && (s.tx < 1 || s.ty < 1 || s.tz < 1 || s.fx < 1 || s.fy < 1)) return EKCG_EINVAL;
    long long n = (long long)s.nx * s.ny * s.nz;
    if (n >= (1LL << 32)) return EKCG_EINVAL;
    UniformFaces uf{};
    if (s.kfield == nullptr) {
        uf.fz = host_face(s.cz, s.kconst);
        uf.fy = host_face(s.cy, s.kconst);
        uf.fx = host_face(s.cx, s.kconst);
        uf.bz = s.cz * s.kconst;
        uf.by = s.cy * s.kconst;
        uf.bx = s.cx * s.kconst;
    }
    cudaStream_t st = as_stream(stream);
    const bool aligned = (ldx % 2 == 0) && (ldy % 2 == 0) && ((reinterpret_cast<uintptr_t>(X) & 15) == 0) &&
                         ((reinterpret_cast<uintptr_t>(Y) & 15) == 0);
    if (aligned && m % 4 == 0) {
        RowLaunch L = row_launch(n, m / 4);
        stencil_spmm_kernel<4><<<L.grid, L.block, 0, st>>>(s, uf, X, ldx, Y, ldy, m, live);
    } else if (aligned && m % 2 == 0) {
        RowLaunch L = row_launch(n, m / 2);
        stencil_spmm_kernel<2><<<L.grid, L.block, 0, st>>>(s, uf, X, ldx, Y, ldy, m, live);
    } else {
        RowLaunch L = row_launch(n, m);
        stencil_spmm_kernel<1><<<L.grid, L.block, 0, st>>>(s, uf, X, ldx, Y, ldy, m, live);
    }
    ++g_ekcg_launches;
    return launch_status();
}
