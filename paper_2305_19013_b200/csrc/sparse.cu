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
#include "stencil.cuh"

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
    long long cap = (long long)device_sms() * 16;
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

// W[i, j] += Wprev[i, j] * (beta_sign * beta[j])  (preconditioned MSDO candidate,
// solvers.py:378-382 with candidate_split = M^-1 split(r) already in W)
__global__ void axpy_cols_kernel(double* __restrict__ W, int ldw, const double* __restrict__ Wprev, int ldp,
                                 const double* __restrict__ beta, double beta_sign, long long n, int t,
                                 const int* __restrict__ live) {
    EKCG_GATE(live);
    ROW_LOOP(i, n) {
        for (int j = threadIdx.x; j < t; j += blockDim.x)
            W[i * ldw + j] = add_rn(W[i * ldw + j], mul_rn(Wprev[i * ldp + j], beta_sign * beta[j]));
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

// Vectorized CSR SpMM: G = m / VEC threads per row, VEC contiguous columns per
// thread (16-B loads of X / stores of Y for VEC >= 2).  Rows with at most 8
// entries (every stencil-like row) load all their (col, value) pairs and X
// gathers up front, predicated, so up to 8 independent gathers per thread are
// in flight; the sum is then formed in the reference association
// p0 + (((p1 + p2) + p3) + ...).  Longer rows take numpy's pairwise tail per
// column (tail_pairwise).  Bitwise equal to csr_spmm_kernel.
template <int VEC>
__device__ __forceinline__ void load_xvec(const double* __restrict__ X, long long off, double (&v)[VEC]) {
    if (VEC == 1) {
        v[0] = __ldg(X + off);
    } else {
#pragma unroll
        for (int h = 0; h < VEC / 2; ++h) {
            const double2 t = __ldg(reinterpret_cast<const double2*>(X + off) + h);
            v[2 * h] = t.x;
            v[2 * h + 1] = t.y;
        }
    }
}

template <int VEC>
__global__ void __launch_bounds__(256, VEC == 4 ? 2 : 3)
csr_spmm_vec_kernel(const long long* __restrict__ rp, const int* __restrict__ ci, const double* __restrict__ vv,
                    const double* __restrict__ X, int ldx, double* __restrict__ Y, int ldy, long long n,
                    const int* __restrict__ live) {
    EKCG_GATE(live);
    const int c0 = threadIdx.x * VEC;
    ROW_LOOP(i, n) {
        const long long lo = __ldg(rp + i), hi = __ldg(rp + i + 1);
        const long long cnt = hi - lo - 1;  // tail length after p0
        double y[VEC];
        if (hi <= lo) {
#pragma unroll
            for (int v = 0; v < VEC; ++v) y[v] = 0.0;  // unreachable for validated SPD matrices
        } else if (cnt < 8) {
            int cq[8];
            double aq[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                cq[q] = q <= cnt ? __ldg(ci + lo + q) : 0;
                aq[q] = q <= cnt ? __ldg(vv + lo + q) : 0.0;
            }
            double xq[8][VEC] = {};  // defined on every path: keeps the gathers in registers
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                if (q <= cnt) load_xvec<VEC>(X, (long long)cq[q] * ldx + c0, xq[q]);
            }
#pragma unroll
            for (int v = 0; v < VEC; ++v) {
                const double p0 = mul_rn(aq[0], xq[0][v]);
                if (cnt == 0) {
                    y[v] = p0;
                } else {
                    double acc = mul_rn(aq[1], xq[1][v]);
#pragma unroll
                    for (int q = 2; q < 8; ++q)
                        if (q <= cnt) acc = add_rn(acc, mul_rn(aq[q], xq[q][v]));
                    y[v] = add_rn(p0, acc);
                }
            }
        } else {
            const double a0 = __ldg(vv + lo);
            const long long x0 = (long long)__ldg(ci + lo) * ldx;
            for (int v = 0; v < VEC; ++v)
                y[v] = add_rn(mul_rn(a0, __ldg(X + x0 + c0 + v)), tail_pairwise(ci, vv, lo + 1, cnt, X, ldx, c0 + v));
        }
        if (VEC == 1) {
            Y[i * ldy + c0] = y[0];
        } else {
#pragma unroll
            for (int h = 0; h < VEC / 2; ++h)
                reinterpret_cast<double2*>(Y + i * ldy + c0)[h] = make_double2(y[2 * h], y[2 * h + 1]);
        }
    }
}

// One short row (CNT + 1 <= 8 entries) for 4 columns: all gathers issued up
// front, then `pre` (the next row's loads), then the sum in the reference
// association p0 + (((p1 + p2) + p3) + ...).  CNT is a template argument so the
// gathers are unpredicated and exactly as many as the row has.
template <int CNT, bool W256, class Pre>
__device__ __forceinline__ void csr_short_row(const int (&cq)[8], const double (&aq)[8],
                                              const double* __restrict__ X, int ldx, int c0, double (&y)[4],
                                              Pre&& pre) {
    double xq[CNT + 1][4];
#pragma unroll
    for (int q = 0; q <= CNT; ++q) {
        if (W256)
            ld4_256(X + (long long)cq[q] * ldx + c0, xq[q]);
        else
            load_xvec<4>(X, (long long)cq[q] * ldx + c0, xq[q]);
    }
    pre();
#pragma unroll
    for (int v = 0; v < 4; ++v) {
        const double p0 = mul_rn(aq[0], xq[0][v]);
        if (CNT == 0) {
            y[v] = p0;
        } else {
            double acc = mul_rn(aq[1], xq[1][v]);
#pragma unroll
            for (int q = 2; q <= CNT; ++q) acc = add_rn(acc, mul_rn(aq[q], xq[q][v]));
            y[v] = add_rn(p0, acc);
        }
    }
}

// Software-pipelined form of csr_spmm_vec_kernel<4> for m = 4G, G in {4, 8, 16,
// 32} threads per row, persistent grid.  A row costs three dependent memory
// latencies (row pointers -> (col, value) pairs -> X gathers); here, while the
// gathers of row i are in flight, the thread group already holds the pairs of
// its next row and loads the row pointers of the one after, so a row costs
// about one.  The group keeps the next row's pairs distributed (entry q in
// thread q % G, slot q / G) and shuffles them in when the row becomes current;
// short rows dispatch on their length to an unpredicated body.  Same products
// and association as csr_spmm_vec_kernel (bitwise equal).
template <int G, bool W256>
__global__ void __launch_bounds__(256, 2)
csr_spmm_pf_kernel(const long long* __restrict__ rp, const int* __restrict__ ci, const double* __restrict__ vv,
                   const double* __restrict__ X, int ldx, double* __restrict__ Y, int ldy, long long n,
                   const int* __restrict__ live) {
    static_assert(G == 4 || G == 8 || G == 16 || G == 32, "G is a power of two in [4, 32]");
    constexpr int S = G >= 8 ? 1 : 2;  // slots per thread
    constexpr int R = 256 / G;         // rows per block
    EKCG_GATE(live);
    const int g = threadIdx.x;
    const int c0 = g * 4;
    const int lane = (threadIdx.x + threadIdx.y * G) & 31;
    const int base = lane & ~(G - 1);  // first lane of the group
    const long long stride = (long long)gridDim.x * R;
    long long i = (long long)blockIdx.x * R + threadIdx.y;
    long long iw = i - lane / G;  // the warp's first row: the loop is warp-uniform so shuffles see every lane
    long long lo = 0, hi = 0, nlo = 0, nhi = 0;
    if (i < n) {
        lo = __ldg(rp + i);
        hi = __ldg(rp + i + 1);
    }
    if (i + stride < n) {
        nlo = __ldg(rp + i + stride);
        nhi = __ldg(rp + i + stride + 1);
    }
    int cs[S];
    double as[S];
    // this thread's share of a short row: entries g (+ G)
    auto load_share = [&](long long l, long long h) {
        const long long cnt = h - l - 1;
#pragma unroll
        for (int s = 0; s < S; ++s) {
            const int q = g + s * G;
            const bool ok = h > l && cnt < 8 && q <= cnt;
            cs[s] = ok ? __ldg(ci + l + q) : 0;
            as[s] = ok ? __ldg(vv + l + q) : 0.0;
        }
    };
    load_share(lo, hi);
    for (; iw < n; i += stride, iw += stride) {
        const long long cnt = hi - lo - 1;
        int cq[8];
        double aq[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            if (q / G < S) {
                cq[q] = __shfl_sync(0xffffffffu, cs[q / G < S ? q / G : 0], base + (q % G));
                aq[q] = __shfl_sync(0xffffffffu, as[q / G < S ? q / G : 0], base + (q % G));
            }
        }
        long long plo = 0, phi = 0;
        auto pre = [&]() {  // next row's pairs and the row pointers of the one after
            load_share(nlo, nhi);
            if (i + 2 * stride < n) {
                plo = __ldg(rp + i + 2 * stride);
                phi = __ldg(rp + i + 2 * stride + 1);
            }
        };
        double y[4];
        switch (hi <= lo ? -1 : (cnt < 8 ? (int)cnt : 8)) {
            case 0: csr_short_row<0, W256>(cq, aq, X, ldx, c0, y, pre); break;
            case 1: csr_short_row<1, W256>(cq, aq, X, ldx, c0, y, pre); break;
            case 2: csr_short_row<2, W256>(cq, aq, X, ldx, c0, y, pre); break;
            case 3: csr_short_row<3, W256>(cq, aq, X, ldx, c0, y, pre); break;
            case 4: csr_short_row<4, W256>(cq, aq, X, ldx, c0, y, pre); break;
            case 5: csr_short_row<5, W256>(cq, aq, X, ldx, c0, y, pre); break;
            case 6: csr_short_row<6, W256>(cq, aq, X, ldx, c0, y, pre); break;
            case 7: csr_short_row<7, W256>(cq, aq, X, ldx, c0, y, pre); break;
            case 8: {
                pre();
                const double a0 = __ldg(vv + lo);
                const long long x0 = (long long)__ldg(ci + lo) * ldx;
                for (int v = 0; v < 4; ++v)
                    y[v] = add_rn(mul_rn(a0, __ldg(X + x0 + c0 + v)),
                                  tail_pairwise(ci, vv, lo + 1, cnt, X, ldx, c0 + v));
                break;
            }
            default:  // empty row, or past the end
                pre();
#pragma unroll
                for (int v = 0; v < 4; ++v) y[v] = 0.0;
        }
        if (i < n) {
            if (W256) {
                st4_256(Y + i * ldy + c0, y);
            } else {
                reinterpret_cast<double2*>(Y + i * ldy + c0)[0] = make_double2(y[0], y[1]);
                reinterpret_cast<double2*>(Y + i * ldy + c0)[1] = make_double2(y[2], y[3]);
            }
        }
        lo = nlo;
        hi = nhi;
        nlo = plo;
        nhi = phi;
    }
}

template <int G, bool W256>
static void launch_csr_pf(const long long* rp, const int* ci, const double* vv, const double* X, int ldx, double* Y,
                          int ldy, long long n, const int* live, cudaStream_t st) {
    static int cache[kEkcgMaxDevices];
    int occ = kernel_occupancy(csr_spmm_pf_kernel<G, W256>, 256, 0, cache);
    if (occ < 1) occ = 1;
    constexpr int R = 256 / G;
    long long blocks = (n + R - 1) / R, cap = (long long)occ * device_sms();
    if (blocks > cap) blocks = cap;
    launch_k(csr_spmm_pf_kernel<G, W256>, dim3((unsigned)blocks), dim3(G, R), 0, st, rp, ci, vv, X, ldx, Y, ldy, n, live);
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
template <int VEC>
__global__ void __launch_bounds__(256)
stencil_spmm_kernel(EkcgStencil s, UniformFaces uf, const double* __restrict__ X, int ldx,
                    double* __restrict__ Y, int ldy, int m, const int* __restrict__ live) {
    EKCG_GATE(live);
    const int c0 = threadIdx.x * VEC;
    for (long long i = s.row_begin + (long long)blockIdx.x * blockDim.y + threadIdx.y; i < s.row_end;
         i += (long long)gridDim.x * blockDim.y) {
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
    }
}

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
extern "C" int ekcg_split(const double* v, const int* owner, double* W, long long n, int t, int ldw,
                          const int* live, void* stream) {
    if (n < 0 || t < 1 || ldw < t) return EKCG_EINVAL;
    if (n == 0) return EKCG_OK;
    RowLaunch L = row_launch(n, t < 32 ? t : 32);
    launch_k(split_kernel, L.grid, L.block, 0, as_stream(stream), v, owner, W, n, t, ldw, live);
    ++g_ekcg_launches;
    return launch_status();
}

extern "C" int ekcg_split_axpy(const double* v, const int* owner, const double* Wprev, int ldp,
                               const double* beta, double beta_sign, double* W, long long n, int t,
                               int ldw, const int* live, void* stream) {
    if (n < 0 || t < 1 || ldw < t || ldp < t) return EKCG_EINVAL;
    if (n == 0) return EKCG_OK;
    RowLaunch L = row_launch(n, t < 32 ? t : 32);
    launch_k(split_axpy_kernel, L.grid, L.block, 0, as_stream(stream), v, owner, Wprev, ldp, beta, beta_sign, W, n, t,
                                                                 ldw, live);
    ++g_ekcg_launches;
    return launch_status();
}

extern "C" int ekcg_axpy_cols(double* W, int ldw, const double* Wprev, int ldp, const double* beta,
                              double beta_sign, long long n, int t, const int* live, void* stream) {
    if (n < 0 || t < 1 || ldw < t || ldp < t) return EKCG_EINVAL;
    if (n == 0) return EKCG_OK;
    RowLaunch L = row_launch(n, t < 32 ? t : 32);
    launch_k(axpy_cols_kernel, L.grid, L.block, 0, as_stream(stream), W, ldw, Wprev, ldp, beta, beta_sign, n, t, live);
    ++g_ekcg_launches;
    return launch_status();
}

// CSR kernel forms (ekcg_spmm_csr_kernel): every form computes each row as p0 + pairwise(p1..pk) with
// separately rounded products, so they agree bit for bit; the automatic choice is the fastest that applies.
enum CsrForm { kCsrAuto = 0, kCsrPipelined = 1, kCsrPipelined128 = 2, kCsrVec4 = 3, kCsrVec2 = 4, kCsrScalar = 5 };

static int spmm_csr_impl(int form, const long long* row_ptr, const int* col_idx, const double* values,
                         const double* X, int ldx, double* Y, int ldy, long long n, int m, const int* live,
                         cudaStream_t st) {
    if (n < 0 || m < 1 || ldx < m || ldy < m || form < kCsrAuto || form > kCsrScalar) return EKCG_EINVAL;
    if (n == 0) return EKCG_OK;
    const bool al16 = ((reinterpret_cast<uintptr_t>(X) | reinterpret_cast<uintptr_t>(Y)) & 15) == 0 &&
                      ldx % 2 == 0 && ldy % 2 == 0;
    const bool al32 = ((reinterpret_cast<uintptr_t>(X) | reinterpret_cast<uintptr_t>(Y)) & 31) == 0 &&
                      ldx % 4 == 0 && ldy % 4 == 0;
    const int G = m / 4;
    const bool pf_ok = m % 4 == 0 && (G == 4 || G == 8 || G == 16 || G == 32) && al16;
    const bool v4_ok = m % 4 == 0 && m / 4 <= 256 && al16;
    const bool v2_ok = m % 2 == 0 && m / 2 <= 256 && al16;
    if (form == kCsrAuto) form = pf_ok ? kCsrPipelined : v4_ok ? kCsrVec4 : v2_ok ? kCsrVec2 : kCsrScalar;
    if (form == kCsrPipelined || form == kCsrPipelined128) {
        if (!pf_ok) return EKCG_EINVAL;
        if (form == kCsrPipelined && al32) {  // 256-bit X gathers / Y stores
            if (G == 4) launch_csr_pf<4, true>(row_ptr, col_idx, values, X, ldx, Y, ldy, n, live, st);
            else if (G == 8) launch_csr_pf<8, true>(row_ptr, col_idx, values, X, ldx, Y, ldy, n, live, st);
            else if (G == 16) launch_csr_pf<16, true>(row_ptr, col_idx, values, X, ldx, Y, ldy, n, live, st);
            else launch_csr_pf<32, true>(row_ptr, col_idx, values, X, ldx, Y, ldy, n, live, st);
        } else {
            if (G == 4) launch_csr_pf<4, false>(row_ptr, col_idx, values, X, ldx, Y, ldy, n, live, st);
            else if (G == 8) launch_csr_pf<8, false>(row_ptr, col_idx, values, X, ldx, Y, ldy, n, live, st);
            else if (G == 16) launch_csr_pf<16, false>(row_ptr, col_idx, values, X, ldx, Y, ldy, n, live, st);
            else launch_csr_pf<32, false>(row_ptr, col_idx, values, X, ldx, Y, ldy, n, live, st);
        }
    } else if (form == kCsrVec4) {
        if (!v4_ok) return EKCG_EINVAL;
        RowLaunch L = row_launch(n, m / 4);
        launch_k(csr_spmm_vec_kernel<4>, L.grid, L.block, 0, st, row_ptr, col_idx, values, X, ldx, Y, ldy, n, live);
    } else if (form == kCsrVec2) {
        if (!v2_ok) return EKCG_EINVAL;
        RowLaunch L = row_launch(n, m / 2);
        launch_k(csr_spmm_vec_kernel<2>, L.grid, L.block, 0, st, row_ptr, col_idx, values, X, ldx, Y, ldy, n, live);
    } else if (m == 1) {
        RowLaunch L = row_launch(n, 1);
        launch_k(csr_spmm_vec_kernel<1>, L.grid, L.block, 0, st, row_ptr, col_idx, values, X, ldx, Y, ldy, n, live);
    } else {
        RowLaunch L = row_launch(n, m < 64 ? m : 64);
        launch_k(csr_spmm_kernel, L.grid, L.block, 0, st, row_ptr, col_idx, values, X, ldx, Y, ldy, n, m, live);
    }
    ++g_ekcg_launches;
    return launch_status();
}

extern "C" int ekcg_spmm_csr(const long long* row_ptr, const int* col_idx, const double* values,
                             const double* X, int ldx, double* Y, int ldy, long long n, int m,
                             const int* live, void* stream) {
    return spmm_csr_impl(kCsrAuto, row_ptr, col_idx, values, X, ldx, Y, ldy, n, m, live, as_stream(stream));
}

extern "C" int ekcg_spmm_csr_kernel(int form, const long long* row_ptr, const int* col_idx, const double* values,
                                    const double* X, int ldx, double* Y, int ldy, long long n, int m,
                                    const int* live, void* stream) {
    return spmm_csr_impl(form, row_ptr, col_idx, values, X, ldx, Y, ldy, n, m, live, as_stream(stream));
}

// Per-node coefficient rows of a kfield operator (ekcg_stencil_coefs): the same stencil_coef arithmetic the
// kernels run on the fly (descriptor without a table), stored once.
__global__ void __launch_bounds__(256)
stencil_coef_build_kernel(EkcgStencil s, UniformFaces uf, double* __restrict__ coef, long long n) {
    const int S = (s.dim == 3) ? 8 : 6;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const unsigned x = (unsigned)(i % s.nx);
        const long long rest = i / s.nx;
        const unsigned y = (unsigned)(rest % s.ny), z = (unsigned)(rest / s.ny);
        double v[7];
        if (s.dim == 3) stencil_coef(s, uf, x, y, z, v);
        else stencil_coef(s, uf, x, (unsigned)rest, 0u, v);
        double* r = coef + S * i;
        if (s.dim == 3) {
            for (int q = 0; q < 7; ++q) r[q] = v[q];
            r[7] = 0.0;
        } else {
            for (int q = 0; q < 5; ++q) r[q] = v[q + 1];
            r[5] = 0.0;
        }
    }
}

extern "C" int ekcg_stencil_coefs(const EkcgStencil* desc, double* coef, void* stream) {
    EkcgStencil s;
    UniformFaces uf;
    long long n;
    int rc = prepare_stencil(desc, s, uf, n);
    if (rc != EKCG_OK) return rc;
    if (s.kfield == nullptr || coef == nullptr || (reinterpret_cast<uintptr_t>(coef) & 15)) return EKCG_EINVAL;
    s.coef = nullptr;  // compute every row on the fly
    const long long blocks = (n + 255) / 256;
    const unsigned grid = (unsigned)(blocks < (long long)device_sms() * 16 ? blocks : (long long)device_sms() * 16);
    launch_k(stencil_coef_build_kernel, grid, 256, 0, as_stream(stream), s, uf, coef, n);
    ++g_ekcg_launches;
    return launch_status();
}

// Stencil kernel forms (ekcg_spmm_stencil_kernel): 0 automatic (the TMA plane march above
// kMarchMinWork block entries, else the row-parallel kernel), 1 the plane march at any size, 2 the
// row-parallel kernel.  Both kernels reproduce the generator's CSR association, so they agree bit for bit.
static int spmm_stencil_impl(int form, const EkcgStencil* desc, const double* X, int ldx, double* Y, int ldy,
                             int m, const int* live, cudaStream_t st) {
    if (m < 1 || ldx < m || ldy < m || form < 0 || form > 2) return EKCG_EINVAL;
    EkcgStencil s;
    UniformFaces uf;
    long long n;
    int rc = prepare_stencil(desc, s, uf, n);
    if (rc != EKCG_OK) return rc;
    const bool aligned = (ldx % 2 == 0) && (ldy % 2 == 0) && ((reinterpret_cast<uintptr_t>(X) & 15) == 0) &&
                         ((reinterpret_cast<uintptr_t>(Y) & 15) == 0);
    n = s.row_end - s.row_begin;
    if (form != 2) {
        const long long min_work = form == 1 ? 0 : kMarchMinWork;
        if (launch_stencil_march(s, uf, X, ldx, Y, ldy, m, live, st, min_work) == EKCG_OK) {
            ++g_ekcg_launches;
            return launch_status();
        }
        if (form == 1) return EKCG_EINVAL;
    }
    if (aligned && m % 4 == 0) {
        RowLaunch L = row_launch(n, m / 4);
        launch_k(stencil_spmm_kernel<4>, L.grid, L.block, 0, st, s, uf, X, ldx, Y, ldy, m, live);
    } else if (aligned && m % 2 == 0) {
        RowLaunch L = row_launch(n, m / 2);
        launch_k(stencil_spmm_kernel<2>, L.grid, L.block, 0, st, s, uf, X, ldx, Y, ldy, m, live);
    } else {
        RowLaunch L = row_launch(n, m);
        launch_k(stencil_spmm_kernel<1>, L.grid, L.block, 0, st, s, uf, X, ldx, Y, ldy, m, live);
    }
    ++g_ekcg_launches;
    return launch_status();
}

extern "C" int ekcg_spmm_stencil(const EkcgStencil* desc, const double* X, int ldx, double* Y, int ldy,
                                 int m, const int* live, void* stream) {
    return spmm_stencil_impl(0, desc, X, ldx, Y, ldy, m, live, as_stream(stream));
}

extern "C" int ekcg_spmm_stencil_kernel(int form, const EkcgStencil* desc, const double* X, int ldx, double* Y,
                                        int ldy, int m, const int* live, void* stream) {
    return spmm_stencil_impl(form, desc, X, ldx, Y, ldy, m, live, as_stream(stream));
}
