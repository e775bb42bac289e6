// Structured-grid stencil rows (the `_diffusion_matrix` operator of
// generators.py:25-60) shared by the plain and fused stencil kernels.
//
// Face between lo/hi nodes: c * (2*k_lo*k_hi/(k_lo+k_hi)); Dirichlet boundary
// faces add c * k_node.  The diagonal accumulates, per axis from slowest to
// fastest: +face_hi, +face_lo, +boundary(first), +boundary(last) -- the order
// of the np.add.at calls in generators.py:46-53.  Row entries come out in
// ascending column order (z-, y-, x-, diag, x+, y+, z+) and a row is summed as
// p0 + (((p1 + p2) + p3) + ...) with separately rounded products: bitwise the
// reference spmm on the assembled CSR (linalg.py:141-152).
#pragma once
#include "common.cuh"
#include "ekcg_b200.h"

__device__ __forceinline__ double harmonic_face(double c, double klo, double khi) {
    // generators.py:45 -- `2.0 * ka * kb / (ka + kb)` evaluated left to right.
    double h = __ddiv_rn(mul_rn(mul_rn(2.0, klo), khi), add_rn(klo, khi));
    return mul_rn(c, h);
}

// a / b for the tile edges: a shift when b is a power of two (every tile field
// here; the test is uniform across the launch), else the integer division.
__device__ __forceinline__ unsigned tile_div(unsigned a, int b) {
    const unsigned ub = (unsigned)b;
    return (ub & (ub - 1)) == 0 ? (a >> (__ffs(b) - 1)) : a / ub;
}

// Per-launch constants for a uniform-kappa grid (computed by the host with the
// same IEEE operations as harmonic_face, so the same bits).
struct UniformFaces {
    double fz, fy, fx;  // c * 2k^2/(2k)
    double bz, by, bx;  // c * k
    double dint;        // diagonal of an interior node: ((((fz + fz) + fy) + fy) + fx) + fx
};

// Face coefficient between a node (kappa kc, tile index tc) and a neighbour
// `off` tiles away: a division only when the neighbour is in another tile (or
// no per-tile self-harmonic table is given); harmonic_face(c, k, k) equals
// c * kself[tile] bitwise (same IEEE operations, evaluated on the host).
__device__ __forceinline__ double face_lo(const EkcgStencil& s, double c, const double* F, long long tc, double kc,
                                         bool cross, long long off, const double* hcross) {
    if (!cross && s.kself != nullptr) return mul_rn(c, __ldg(s.kself + tc));
    if (cross && hcross != nullptr) return __ldg(hcross + tc - off);  // host-built, same IEEE operations
    return harmonic_face(c, __ldg(F + tc - (cross ? off : 0)), kc);
}
__device__ __forceinline__ double face_hi(const EkcgStencil& s, double c, const double* F, long long tc, double kc,
                                         bool cross, long long off, const double* hcross) {
    if (!cross && s.kself != nullptr) return mul_rn(c, __ldg(s.kself + tc));
    if (cross && hcross != nullptr) return __ldg(hcross + tc);
    return harmonic_face(c, kc, __ldg(F + tc + (cross ? off : 0)));
}

// Coefficients of the node (x, y, z): v[0..6] = z-, y-, x-, diag, x+, y+, z+
// (absent neighbours: 0) and the presence mask (bit q = slot q present).
// Per-node coefficient row (2-D: slots 1..5, 3-D: slots 0..6) from the table built by ekcg_stencil_coefs.
__device__ __forceinline__ void coef_row(const EkcgStencil& s, long long i, double (&v)[7]) {
    if (s.dim == 3) {
        const double2* r = reinterpret_cast<const double2*>(s.coef + 8 * i);
        const double2 a = __ldg(r), b = __ldg(r + 1), c = __ldg(r + 2), d = __ldg(r + 3);
        v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y; v[4] = c.x; v[5] = c.y; v[6] = d.x;
    } else {
        const double2* r = reinterpret_cast<const double2*>(s.coef + 6 * i);
        const double2 a = __ldg(r), b = __ldg(r + 1), c = __ldg(r + 2);
        v[0] = 0.0; v[1] = a.x; v[2] = a.y; v[3] = b.x; v[4] = b.y; v[5] = c.x; v[6] = 0.0;
    }
}

__device__ __forceinline__ unsigned stencil_mask(const EkcgStencil& s, unsigned x, unsigned y, unsigned z) {
    const bool three = (s.dim == 3);
    unsigned mk = 1u << 3;
    if (three && z > 0)          mk |= 1u << 0;
    if (y > 0)                   mk |= 1u << 1;
    if (x > 0)                   mk |= 1u << 2;
    if (x < s.nx - 1)            mk |= 1u << 4;
    if (y < s.ny - 1)            mk |= 1u << 5;
    if (three && z < s.nz - 1)   mk |= 1u << 6;
    return mk;
}

__device__ __forceinline__ unsigned stencil_coef(const EkcgStencil& s, const UniformFaces& uf, unsigned x,
                                                 unsigned y, unsigned z, double (&v)[7]) {
    const unsigned nx = s.nx, ny = s.ny, nz = s.nz;
    const bool three = (s.dim == 3);
    if (s.coef != nullptr) {
        coef_row(s, three ? ((long long)z * ny + y) * nx + x : (long long)y * nx + x, v);
        return stencil_mask(s, x, y, z);
    }
    double fzl = 0.0, fzh = 0.0, fyl = 0.0, fyh = 0.0, fxl = 0.0, fxh = 0.0;
    double diag = 0.0;
    if (s.kfield == nullptr) {
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
        const unsigned txi = tile_div(x, s.tx), tyi = tile_div(y, s.ty), tzi = tile_div(z, s.tz);
        const unsigned rx = x - txi * s.tx, ry = y - tyi * s.ty, rz = z - tzi * s.tz;
        const long long fx = s.fx, fxy = (long long)s.fx * s.fy;
        const double* __restrict__ F = s.kfield;
        const long long tc = tzi * fxy + tyi * fx + txi;
        const double kc = __ldg(F + tc);
        if (three) {
            if (z < nz - 1) { fzh = face_hi(s, s.cz, F, tc, kc, rz + 1 == (unsigned)s.tz, fxy, s.hz); diag = add_rn(diag, fzh); }
            if (z > 0)      { fzl = face_lo(s, s.cz, F, tc, kc, rz == 0, fxy, s.hz); diag = add_rn(diag, fzl); }
            if (z == 0)      diag = add_rn(diag, mul_rn(s.cz, kc));
            if (z == nz - 1) diag = add_rn(diag, mul_rn(s.cz, kc));
        }
        if (y < ny - 1) { fyh = face_hi(s, s.cy, F, tc, kc, ry + 1 == (unsigned)s.ty, fx, s.hy); diag = add_rn(diag, fyh); }
        if (y > 0)      { fyl = face_lo(s, s.cy, F, tc, kc, ry == 0, fx, s.hy); diag = add_rn(diag, fyl); }
        if (y == 0)      diag = add_rn(diag, mul_rn(s.cy, kc));
        if (y == ny - 1) diag = add_rn(diag, mul_rn(s.cy, kc));
        if (x < nx - 1) { fxh = face_hi(s, s.cx, F, tc, kc, rx + 1 == (unsigned)s.tx, 1, s.hx); diag = add_rn(diag, fxh); }
        if (x > 0)      { fxl = face_lo(s, s.cx, F, tc, kc, rx == 0, 1, s.hx); diag = add_rn(diag, fxl); }
        if (x == 0)      diag = add_rn(diag, mul_rn(s.cx, kc));
        if (x == nx - 1) diag = add_rn(diag, mul_rn(s.cx, kc));
    }
    v[0] = -fzl; v[1] = -fyl; v[2] = -fxl; v[3] = diag; v[4] = -fxh; v[5] = -fyh; v[6] = -fzh;
    unsigned mk = 1u << 3;
    if (three && z > 0)      mk |= 1u << 0;
    if (y > 0)               mk |= 1u << 1;
    if (x > 0)               mk |= 1u << 2;
    if (x < nx - 1)          mk |= 1u << 4;
    if (y < ny - 1)          mk |= 1u << 5;
    if (three && z < nz - 1) mk |= 1u << 6;
    return mk;
}

// Row i of the operator: neighbour offsets and values in column order.
// Returns the entry count; `dpos` gets the position of the diagonal entry.
__device__ __forceinline__ int stencil_row(const EkcgStencil& s, const UniformFaces& uf, long long i,
                                           long long (&off)[7], double (&val)[7], int& dpos) {
    const unsigned nx = s.nx, ny = s.ny, nz = s.nz;
    const long long nxy = (long long)nx * ny;
    const bool three = (s.dim == 3);
    const unsigned iu = (unsigned)i;
    const unsigned x = iu % nx;
    const unsigned rest = iu / nx;
    const unsigned y = rest % ny;
    const unsigned z = rest / ny;

    double fzl = 0.0, fzh = 0.0, fyl = 0.0, fyh = 0.0, fxl = 0.0, fxh = 0.0;
    double diag = 0.0;
    if (s.coef != nullptr) {
        double v[7];
        coef_row(s, i, v);
        fzl = -v[0]; fyl = -v[1]; fxl = -v[2]; diag = v[3]; fxh = -v[4]; fyh = -v[5]; fzh = -v[6];
    } else if (s.kfield == nullptr) {
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
        // tile coordinates of the node; a neighbour lies in the adjacent tile
        // exactly when the step crosses a tile edge
        const unsigned txi = tile_div(x, s.tx), tyi = tile_div(y, s.ty), tzi = tile_div(z, s.tz);
        const unsigned rx = x - txi * s.tx, ry = y - tyi * s.ty, rz = z - tzi * s.tz;
        const long long fx = s.fx, fxy = (long long)s.fx * s.fy;
        const double* __restrict__ F = s.kfield;
        const long long tc = tzi * fxy + tyi * fx + txi;
        const double kc = __ldg(F + tc);
        if (three) {
            if (z < nz - 1) { fzh = face_hi(s, s.cz, F, tc, kc, rz + 1 == (unsigned)s.tz, fxy, s.hz); diag = add_rn(diag, fzh); }
            if (z > 0)      { fzl = face_lo(s, s.cz, F, tc, kc, rz == 0, fxy, s.hz); diag = add_rn(diag, fzl); }
            if (z == 0)      diag = add_rn(diag, mul_rn(s.cz, kc));
            if (z == nz - 1) diag = add_rn(diag, mul_rn(s.cz, kc));
        }
        if (y < ny - 1) { fyh = face_hi(s, s.cy, F, tc, kc, ry + 1 == (unsigned)s.ty, fx, s.hy); diag = add_rn(diag, fyh); }
        if (y > 0)      { fyl = face_lo(s, s.cy, F, tc, kc, ry == 0, fx, s.hy); diag = add_rn(diag, fyl); }
        if (y == 0)      diag = add_rn(diag, mul_rn(s.cy, kc));
        if (y == ny - 1) diag = add_rn(diag, mul_rn(s.cy, kc));
        if (x < nx - 1) { fxh = face_hi(s, s.cx, F, tc, kc, rx + 1 == (unsigned)s.tx, 1, s.hx); diag = add_rn(diag, fxh); }
        if (x > 0)      { fxl = face_lo(s, s.cx, F, tc, kc, rx == 0, 1, s.hx); diag = add_rn(diag, fxl); }
        if (x == 0)      diag = add_rn(diag, mul_rn(s.cx, kc));
        if (x == nx - 1) diag = add_rn(diag, mul_rn(s.cx, kc));
    }

    int cnt = 0;
    if (three && z > 0)      { off[cnt] = i - nxy; val[cnt++] = -fzl; }
    if (y > 0)               { off[cnt] = i - nx;  val[cnt++] = -fyl; }
    if (x > 0)               { off[cnt] = i - 1;   val[cnt++] = -fxl; }
    dpos = cnt;
    off[cnt] = i; val[cnt++] = diag;
    if (x < nx - 1)          { off[cnt] = i + 1;   val[cnt++] = -fxh; }
    if (y < ny - 1)          { off[cnt] = i + nx;  val[cnt++] = -fyh; }
    if (three && z < nz - 1) { off[cnt] = i + nxy; val[cnt++] = -fzh; }
    return cnt;
}

// y[c0 .. c0+VEC) of row i (VEC even and 16-B aligned rows use double2 loads).
template <int VEC>
__device__ __forceinline__ void stencil_apply_row(const double* __restrict__ X, int ldx, int c0, int m,
                                                  const long long (&off)[7], const double (&val)[7], int cnt,
                                                  double (&y)[VEC]) {
    if (VEC >= 2 && c0 + VEC <= m) {
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
        for (int h = 0; h < VEC / 2; ++h) {
            y[2 * h] = add_rn(p0[h].x, acc[h].x);
            y[2 * h + 1] = add_rn(p0[h].y, acc[h].y);
        }
    } else {
#pragma unroll
        for (int v = 0; v < VEC; ++v) {
            const int c = c0 + v;
            if (c >= m) {
                y[v] = 0.0;
                continue;
            }
            double p0 = mul_rn(val[0], __ldg(X + off[0] * ldx + c));
            double acc = mul_rn(val[1], __ldg(X + off[1] * ldx + c));
            for (int q = 2; q < cnt; ++q) acc = add_rn(acc, mul_rn(val[q], __ldg(X + off[q] * ldx + c)));
            y[v] = add_rn(p0, acc);
        }
    }
}

static inline double host_face(double c, double k) {
    volatile double two_k = 2.0 * k;
    volatile double num = two_k * k;
    volatile double den = k + k;
    volatile double h = num / den;
    return c * h;
}

// Validate / normalise a descriptor and fill the uniform-face constants.
static inline int prepare_stencil(const EkcgStencil* desc, EkcgStencil& s, UniformFaces& uf, long long& n) {
    if (desc == nullptr) return EKCG_EINVAL;
    s = *desc;
    if (s.dim != 2 && s.dim != 3) return EKCG_EINVAL;
    if (s.dim == 2) s.nz = 1;
    if (s.nx < 2 || s.ny < 2 || (s.dim == 3 && s.nz < 2)) return EKCG_EINVAL;
    if (s.kfield != nullptr && (s.tx < 1 || s.ty < 1 || s.tz < 1 || s.fx < 1 || s.fy < 1)) return EKCG_EINVAL;
    n = (long long)s.nx * s.ny * s.nz;
    if (n >= (1LL << 32)) return EKCG_EINVAL;
    if (s.row_end <= 0) {
        s.row_begin = 0;
        s.row_end = n;
    }
    if (s.row_begin < 0 || s.row_begin >= s.row_end || s.row_end > n) return EKCG_EINVAL;
    // the per-node table only stands in for a kfield operator's coefficients (16-B aligned rows)
    if (s.kfield == nullptr || (reinterpret_cast<uintptr_t>(s.coef) & 15)) s.coef = nullptr;
    uf = UniformFaces{};
    if (s.kfield == nullptr) {
        uf.fz = host_face(s.cz, s.kconst);
        uf.fy = host_face(s.cy, s.kconst);
        uf.fx = host_face(s.cx, s.kconst);
        uf.bz = s.cz * s.kconst;
        uf.by = s.cy * s.kconst;
        uf.bx = s.cx * s.kconst;
        volatile double d = 0.0;
        if (s.dim == 3) {
            d = d + uf.fz;
            d = d + uf.fz;
        }
        d = d + uf.fy;
        d = d + uf.fy;
        d = d + uf.fx;
        d = d + uf.fx;
        uf.dint = d;
    }
    return EKCG_OK;
}

// Below this many block entries (rows x columns) the row-parallel kernels finish sooner than the
// plane march, which is latency-bound on small grids (a few CTAs, serial plane steps).
constexpr long long kMarchMinWork = 1LL << 21;
// Plane-marching stencil SpMM (stencil_march.cu) over at least min_work block entries; EKCG_EINVAL when it
// does not apply.
int launch_stencil_march(const EkcgStencil& s, const UniformFaces& uf, const double* X, int ldx, double* Y, int ldy,
                         int m, const int* live, cudaStream_t st, long long min_work);
// Fused plane-marching kernels for m = 16 (stencil_march.cu); EKCG_EINVAL when they do not apply.
int launch_march_cholinv(const EkcgStencil& s, const UniformFaces& uf, const double* X, int ldx, int m,
                         double* partials, unsigned int* counter, double* S, EkcgCtrl* ctrl, int iteration, double tol,
                         int finalize, int max_ctas, cudaStream_t st);
int launch_march_xr(const EkcgStencil& s, const UniformFaces& uf, const double* X, int ldx, double* Y, int ldy, int m,
                    const double* alpha, double* x, double* r, double* partials, unsigned int* counter, EkcgCtrl* ctrl,
                    int k, int kmax, int stag, double* history, int do_finish, double* rho2_out, int max_ctas,
                    cudaStream_t st);
