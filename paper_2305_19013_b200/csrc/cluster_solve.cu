// A whole truncated-window SRE-CG / SRE-CG2 solve (solvers.py:319-428) in ONE
// kernel on ONE thread-block cluster, for problems small enough that every
// block lives in L2 and an iteration of separate launches is latency-bound
// (BASELINE config 1: n = 10,000, t = 8 -- ~10 launches of 8-18 us each).
//
// The cluster's CTAs own contiguous row ranges.  Row-local work (split, CGS2
// updates, W S products, x / r updates) needs no exchange.  Each Gram-type
// reduction (CGS2 coefficients, W^T W, W0^T A W0, W^T r, |r|^2) is summed per
// warp (DMMA tiles) and per CTA in fixed order, then every CTA pushes its
// partial into every peer's shared memory with st.async (a distributed-shared-
// memory store that completes on the receiver's mbarrier) and each CTA adds the
// received partials in rank order: a one-way ~0.2 us exchange instead of a
// barrier, and all CTAs hold bit-identical sums -- so they factor the m x m
// matrices redundantly and take the same decisions (breakdown, stop test) with
// no host round trip and no atomics (reruns are bit-identical).  Two cluster
// barriers per iteration publish W0 and W_k to the operator rows of the
// neighbouring CTAs, which read their halo rows from L2 (ld.global.cg); they
// also bound how far CTAs drift apart, which is what makes the receive
// buffers (one per reduction of an iteration) safe to reuse.
//
// Arithmetic: the operator rows keep the reference association
// p0 + (((p1 + p2) + ...)) with separately rounded products (bitwise spmm,
// linalg.py:141-152); the m x m factors follow factor.cuh (right-looking
// Cholesky with the reference's breakdown test, explicit upper inverse), run by
// one warp with reciprocal multiplies.
#include <cooperative_groups.h>

#include "common.cuh"
#include "ekcg_b200.h"
#include "stencil.cuh"
#include "tma.cuh"

namespace cg = cooperative_groups;

namespace {

constexpr int kNT = 256;       // threads per CTA (measured: 128 / 512 / 1024 are 20-40 % slower at config 1)
constexpr int kNW = kNT / 32;  // warps per CTA
constexpr int kMaxCl = 16;     // CTAs per cluster
constexpr int kMaxWin = 4;     // retained blocks: <= 4 for m <= 8, <= 2 for m <= 16
constexpr size_t kSmemCap = 225 * 1024;  // dynamic shared memory (227 KB per CTA less the static part)
// one receive buffer + mbarrier per reduction of an iteration
enum { R_PASS1 = 0, R_PASS2, R_GRAW, R_G, R_ALPHA, R_RHO, R_CHECK, R_COUNT };

struct Args {
    EkcgStencil s;
    UniformFaces uf;
    const long long* rp;  // CSR (rp != nullptr) or the stencil descriptor
    const int* ci;
    const double* vv;
    long long n;
    int t, window, kmax, every;
    const int* owner;
    const double* b;
    double* x;
    double* r;
    double* blocks;  // 2 window + 3 blocks of `span` doubles + one n-vector
    long long span;
    EkcgCtrl* ctrl;
    double* history;
    double* checks;
    double chol_tol;
    long long* ticks;  // optional diagnostics: per-phase SM-cycle totals of CTA 0 (20 entries)
};

// Shared-memory layout (in doubles), a function of P1 = window m^2 and P2 = m^2.
struct Layout {
    int wpart;           // [kNW][P1] warp partials
    int recv[R_COUNT];   // [cl][len] received CTA partials per reduction
    int len[R_COUNT];
    int C, G, R, S, S0;  // coefficient block and m x m factor scratch
    int alpha, red, misc;
    int total;
};

__host__ __device__ inline Layout make_layout(int window, int m, int cl) {
    Layout L;
    const int P1 = window * m * m, P2 = m * m;
    int o = 0;
    L.wpart = o;
    o += kNW * P1;
    const int lens[R_COUNT] = {P1, P1, P2, P2, 16, 2, 2};
    for (int i = 0; i < R_COUNT; ++i) {
        L.len[i] = lens[i];
        L.recv[i] = o;
        o += cl * lens[i];
    }
    L.C = o;
    o += P1;
    L.G = o;
    o += 256;
    L.R = o;
    o += 256;
    L.S = o;
    o += 256;
    L.S0 = o;
    o += 256;
    L.alpha = o;
    o += 16;
    L.red = o;
    o += kNW;
    L.misc = o;
    o += 32;  // mbarriers (R_COUNT x 8 B) and the block pointer lists
    L.total = o;
    return L;
}

struct Ctx {
    double* sm;
    const Layout* Lp;  // in shared memory (indexed by reduction id)
    unsigned long long* bar;  // R_COUNT mbarriers
    const double** qp;        // retained Q blocks, oldest first
    const double** aqp;       // retained A Q blocks
    const double** one;       // a one-block list
    unsigned rank, cl;
    unsigned parity;          // bit i: phase parity of bar[i]
};

// ---- cluster exchange ------------------------------------------------------
__device__ __forceinline__ unsigned mapa_u32(unsigned local, unsigned rank) {
    unsigned r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
    return r;
}
// 8-byte store into a peer's shared memory that completes (8 bytes) on the peer's mbarrier
__device__ __forceinline__ void st_async_f64(unsigned raddr, double v, unsigned rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(raddr),
                 "l"(__double_as_longlong(v)), "r"(rbar)
                 : "memory");
}

// Sum of the CTAs' partial vectors (length len) of reduction `reg`, identical in every CTA:
// exchange_begin arms this CTA's mbarrier for cl * len doubles; exchange_send pushes this CTA's
// partial of element e into every CTA's receive buffer (slot = this rank); exchange_finish waits
// for all cl partials and sums them in a fixed pairwise order into out[e] (times sign), ending
// with a CTA barrier.
__device__ __forceinline__ void exchange_begin(Ctx& c, int reg, int len) {
    if (threadIdx.x == 0) mbar_expect_tx(c.bar + reg, c.cl * (unsigned)len * 8u);
}
__device__ __forceinline__ void exchange_send(Ctx& c, int reg, int len, int e, double v) {
    double* rbuf = c.sm + c.Lp->recv[reg];
    const unsigned la = smem_u32(rbuf + c.rank * len + e), lb = smem_u32(c.bar + reg);
#pragma unroll
    for (unsigned rk = 0; rk < kMaxCl; ++rk)
        if (rk < c.cl) st_async_f64(mapa_u32(la, rk), v, mapa_u32(lb, rk));
}
__device__ __forceinline__ void exchange_finish(Ctx& c, int reg, int len, double* out, double sign) {
    const double* rbuf = c.sm + c.Lp->recv[reg];
    mbar_wait(c.bar + reg, (c.parity >> reg) & 1u);
    c.parity ^= 1u << reg;
    for (int e = threadIdx.x; e < len; e += kNT) {
        double p[kMaxCl];
#pragma unroll
        for (unsigned rk = 0; rk < kMaxCl; ++rk) p[rk] = rk < c.cl ? rbuf[rk * len + e] : 0.0;
        // fixed pairwise tree (absent ranks add +0.0): the same order in every CTA, 4 dependent adds
#pragma unroll
        for (int st = 1; st < kMaxCl; st *= 2)
#pragma unroll
            for (int rk = 0; rk + st < kMaxCl; rk += 2 * st) p[rk] += p[rk + st];
        out[e] = sign * p[0];
    }
    __syncthreads();
}

// ---- operator rows ---------------------------------------------------------
// Entries of row i in column order: neighbour row indices and values.
template <bool CSR>
__device__ __forceinline__ int op_row(const Args& a, long long i, long long (&off)[8], double (&val)[8]) {
    if (CSR) {
        const long long lo = __ldg(a.rp + i), hi = __ldg(a.rp + i + 1);
        const int cnt = (int)(hi - lo);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            if (q < cnt) {
                off[q] = __ldg(a.ci + lo + q);
                val[q] = __ldg(a.vv + lo + q);
            }
        }
        return cnt;
    } else {
        long long o7[7];
        double v7[7];
        int dpos;
        const int cnt = stencil_row(a.s, a.uf, i, o7, v7, dpos);
#pragma unroll
        for (int q = 0; q < 7; ++q) {
            off[q] = o7[q];
            val[q] = v7[q];
        }
        return cnt;
    }
}

// One item = one row x VW columns: all of the row's loads in flight together, then the reference
// association p0 + (((p1 + p2) + ...)) per column.
template <bool CSR, int VW>
__device__ __forceinline__ void apply_items(const Args& a, const double* X, int ldx, double* Y, int ldy, int m, long long r0,
                            long long r1) {
    const unsigned groups = (unsigned)(m / VW);
    const unsigned items = (unsigned)(r1 - r0) * groups;
    const bool pow2 = (groups & (groups - 1)) == 0;
    const int sh = __ffs((int)groups) - 1;
    for (unsigned it = threadIdx.x; it < items; it += kNT) {
        const unsigned rl = pow2 ? (it >> sh) : it / groups;
        const long long row = r0 + rl;
        const int c = (int)(it - rl * groups) * VW;
        if (!CSR) {
            // grid stencil: coefficients in slot order z-, y-, x-, diag, x+, y+, z+ with a presence mask
            // (stencil_coef: uniform faces, tile field or per-node table), fixed neighbour offsets, every
            // present entry loaded up front, then p0 + (((p1 + p2) + ...)) over the present entries in
            // order -- no per-row branches, so interior and boundary rows of a warp take the same path
            const unsigned nx = a.s.nx, ny = a.s.ny;
            const unsigned iu = (unsigned)row;
            const unsigned x = iu % nx, rest = iu / nx;
            const bool three = a.s.dim == 3;
            const unsigned y = three ? rest % ny : rest, z = three ? rest / ny : 0u;
            double cf[7];
            const unsigned mk = stencil_coef(a.s, a.uf, x, y, z, cf);
            const double* xc = X + row * ldx + c;
            const long long sy = (long long)nx * ldx, sz = sy * ny;
            const long long offs[7] = {-sz, -sy, -(long long)ldx, 0, (long long)ldx, sy, sz};
            double v[7][VW];
#pragma unroll
            for (int e = 0; e < 7; ++e) {
#pragma unroll
                for (int j = 0; j < VW; ++j) v[e][j] = 0.0;
                if (mk & (1u << e)) {
                    const double* src = xc + offs[e];
                    if (VW == 1) {
                        v[e][0] = __ldcg(src);
                    } else {
#pragma unroll
                        for (int h = 0; h < VW / 2; ++h) {
                            const double2 t2 = __ldcg(reinterpret_cast<const double2*>(src) + h);
                            v[e][2 * h] = t2.x;
                            v[e][(2 * h + 1) % VW] = t2.y;
                        }
                    }
                }
            }
            double p0[VW], acc[VW];
#pragma unroll
            for (int j = 0; j < VW; ++j) p0[j] = acc[j] = 0.0;
            int seen = 0;
#pragma unroll
            for (int e = 0; e < 7; ++e) {
                const bool on = (mk >> e) & 1u;
#pragma unroll
                for (int j = 0; j < VW; ++j) {
                    const double pr = mul_rn(cf[e], v[e][j]);
                    p0[j] = (on && seen == 0) ? pr : p0[j];
                    acc[j] = (on && seen == 1) ? pr : ((on && seen > 1) ? add_rn(acc[j], pr) : acc[j]);
                }
                seen += on ? 1 : 0;
            }
            double* dst = Y + row * ldy + c;
            if (VW == 1) {
                dst[0] = seen > 1 ? add_rn(p0[0], acc[0]) : p0[0];
            } else {
#pragma unroll
                for (int h = 0; h < VW / 2; ++h)
                    reinterpret_cast<double2*>(dst)[h] =
                        make_double2(add_rn(p0[2 * h], acc[2 * h]), add_rn(p0[(2 * h + 1) % VW], acc[(2 * h + 1) % VW]));
            }
            continue;
        }
        long long off[8];
        double val[8];
        const int cnt = op_row<CSR>(a, row, off, val);
        double xv[8][VW];
#pragma unroll
        for (int q = 0; q < 8; ++q)
            if (q < cnt) {
                const double* src = X + off[q] * ldx + c;
                if (VW == 1) {
                    xv[q][0] = __ldcg(src);
                } else {
#pragma unroll
                    for (int h = 0; h < VW / 2; ++h) {
                        const double2 v = __ldcg(reinterpret_cast<const double2*>(src) + h);
                        xv[q][2 * h] = v.x;
                        xv[q][(2 * h + 1) % VW] = v.y;
                    }
                }
            }
        double y[VW];
#pragma unroll
        for (int j = 0; j < VW; ++j) {
            y[j] = 0.0;
            if (cnt > 0) {
                const double p0 = mul_rn(val[0], xv[0][j]);
                if (cnt == 1) {
                    y[j] = p0;
                } else {
                    double acc = mul_rn(val[1], xv[1][j]);
#pragma unroll
                    for (int q = 2; q < 8; ++q)
                        if (q < cnt) acc = add_rn(acc, mul_rn(val[q], xv[q][j]));
                    y[j] = add_rn(p0, acc);
                }
            }
        }
        double* dst = Y + row * ldy + c;
        if (VW == 1) {
            dst[0] = y[0];
        } else {
#pragma unroll
            for (int h = 0; h < VW / 2; ++h)
                reinterpret_cast<double2*>(dst)[h] = make_double2(y[2 * h], y[(2 * h + 1) % VW]);
        }
    }
}

// Y[rows r0..r1) = A X for m columns; X rows of other CTAs come from L2 (ld.global.cg).
template <bool CSR>
__device__ __forceinline__ void apply_local(const Args& a, const double* X, int ldx, double* Y, int ldy, int m, long long r0,
                            long long r1) {
    const bool even = (ldx % 2 == 0) && (ldy % 2 == 0);
    if (even && m % 4 == 0) apply_items<CSR, 4>(a, X, ldx, Y, ldy, m, r0, r1);
    else if (even && m % 2 == 0) apply_items<CSR, 2>(a, X, ldx, Y, ldy, m, r0, r1);
    else apply_items<CSR, 1>(a, X, ldx, Y, ldy, m, r0, r1);
}

// ---- reductions -------------------------------------------------------------
// fp64 tensor-core tile product (SASS DMMA.8x8x4); not volatile, so the loads of the next row chunks are
// scheduled ahead of it.  Fragments (lane = 4 g + q): A[g][q], B[q][g], C[g][2 q + {0, 1}].
__device__ __forceinline__ void dmma(double (&acc)[2], double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
        : "+d"(acc[0]), "+d"(acc[1])
        : "d"(a), "d"(b));
}

// out[i m1 m2 + a m2 + b] = sign * sum over ALL rows of X_i[row, a] Y[row, b]  (i < d <= 4 / MT), identical
// in every CTA.  Each warp sums 4-row chunks of the CTA's rows with DMMA tiles (A = X_i^T, B = Y: both
// fragments are element (row base + q, column 8 t + g)); the warps' tiles are added in warp order and the
// CTA partials exchanged (exchange_sum).
template <int MT>
__device__ __forceinline__ void gram_all(Ctx& c, const double* const* X, int d, int ldx, int m1, const double* Y, int ldy, int m2,
                         long long r0, long long r1, int reg, double* out, double sign = 1.0, bool defer = false) {
    constexpr int DMAX = 4 / MT;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, q = lane & 3;
    const int E = m1 * m2, P = d * E;
    double* wpart = c.sm + c.Lp->wpart;
    double acc[DMAX][MT][MT][2];
#pragma unroll
    for (int i = 0; i < DMAX; ++i)
#pragma unroll
        for (int ta = 0; ta < MT; ++ta)
#pragma unroll
            for (int tb = 0; tb < MT; ++tb) acc[i][ta][tb][0] = acc[i][ta][tb][1] = 0.0;
    const double* Xi[DMAX];
#pragma unroll
    for (int i = 0; i < DMAX; ++i) Xi[i] = (i < d) ? X[i] : nullptr;
#pragma unroll 8
    for (long long base = r0 + 4 * warp; base < r1; base += 4 * kNW) {
        const long long row = base + q;
        const bool in = row < r1;
        double yb[MT], xa[DMAX][MT];
#pragma unroll
        for (int tb = 0; tb < MT; ++tb) yb[tb] = (in && 8 * tb + g < m2) ? Y[row * ldy + 8 * tb + g] : 0.0;
#pragma unroll
        for (int i = 0; i < DMAX; ++i)
#pragma unroll
            for (int ta = 0; ta < MT; ++ta)
                xa[i][ta] = (i < d && in && 8 * ta + g < m1) ? Xi[i][row * ldx + 8 * ta + g] : 0.0;
#pragma unroll
        for (int i = 0; i < DMAX; ++i)
            if (i < d) {
#pragma unroll
                for (int ta = 0; ta < MT; ++ta)
#pragma unroll
                    for (int tb = 0; tb < MT; ++tb) dmma(acc[i][ta][tb], xa[i][ta], yb[tb]);
            }
    }
#pragma unroll
    for (int i = 0; i < DMAX; ++i)
        if (i < d) {
#pragma unroll
            for (int ta = 0; ta < MT; ++ta)
#pragma unroll
                for (int tb = 0; tb < MT; ++tb)
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int ar = 8 * ta + g, bc = 8 * tb + 2 * q + h;
                        if (ar < m1 && bc < m2) wpart[warp * P + i * E + ar * m2 + bc] = acc[i][ta][tb][h];
                    }
        }
    __syncthreads();
    // up to 2 elements per thread (P <= window m^2 <= 2 kNT), each exchanged under the same barrier phase
    exchange_begin(c, reg, P);
    for (int e = threadIdx.x; e < P; e += kNT) {
        double pw[kNW];
#pragma unroll
        for (int w = 0; w < kNW; ++w) pw[w] = wpart[w * P + e];
#pragma unroll
        for (int st = 1; st < kNW; st *= 2)
#pragma unroll
            for (int w = 0; w + st < kNW; w += 2 * st) pw[w] += pw[w + st];
        exchange_send(c, reg, P, e, pw[0]);
    }
    if (!defer) exchange_finish(c, reg, P, out, sign);  // deferred: the caller finishes after independent work
}

// Fixed-order sum of one value per thread over the CTA, then over the cluster: identical in every CTA.
__device__ __forceinline__ double scalar_all(Ctx& c, double v, int reg) {
    double* red = c.sm + c.Lp->red;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0) {
        s = red[0];
#pragma unroll
        for (int w = 1; w < kNW; ++w) s += red[w];
    }
    double* out = c.sm + c.Lp->recv[reg] + c.cl;  // the region's second half (len 2: only the first receives)
    exchange_begin(c, reg, 1);
    if (threadIdx.x == 0) exchange_send(c, reg, 1, 0, s);
    exchange_finish(c, reg, 1, out, 1.0);
    return *out;
}

// ---- row-local block operations ---------------------------------------------
// Wout = (init ? Win : 0) + sum_i Q_i C_i on the CTA's rows, C_i (m x m, row-major, in shared memory)
// already carrying the sign; in place allowed (a chunk's loads all precede its stores, and no other
// chunk touches its rows).  DMMA tiles: A = Q_i[8 rows][4 k], B = C_i[4 k][8 n], accumulator = the W
// tile.  U chunks of 8 rows are loaded together, then multiplied, then stored.
template <int MT>
__device__ __forceinline__ void update_local(const double* Win, bool init, const double* const* Q, int d, const double* C,
                             double* Wout, int m, long long r0, long long r1) {
    constexpr int DMAX = 4 / MT, KS = 2 * MT, U = 4;  // d <= DMAX, m <= 8 MT: KS k-steps of 4
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, q = lane & 3;
    const bool vec = (m % 2 == 0);
    const double* Qi[DMAX];
#pragma unroll
    for (int i = 0; i < DMAX; ++i) Qi[i] = (i < d) ? Q[i] : nullptr;
    for (long long base0 = r0 + 8 * warp; base0 < r1; base0 += 8 * kNW * U) {
        double acc[U][MT][2], av[U][DMAX][KS];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long long row = base0 + (long long)u * 8 * kNW + g;
            const bool in = row < r1;
#pragma unroll
            for (int tn = 0; tn < MT; ++tn) {
                const int cc = 8 * tn + 2 * q;
                acc[u][tn][0] = acc[u][tn][1] = 0.0;
                if (init && in) {
                    if (vec && cc < m) {
                        const double2 w = *reinterpret_cast<const double2*>(Win + row * m + cc);
                        acc[u][tn][0] = w.x;
                        acc[u][tn][1] = w.y;
                    } else {
                        if (cc < m) acc[u][tn][0] = Win[row * m + cc];
                        if (cc + 1 < m) acc[u][tn][1] = Win[row * m + cc + 1];
                    }
                }
            }
#pragma unroll
            for (int i = 0; i < DMAX; ++i)
#pragma unroll
                for (int ks = 0; ks < KS; ++ks) {
                    const int kk = 4 * ks + q;
                    av[u][i][ks] = (i < d && in && kk < m) ? Qi[i][row * m + kk] : 0.0;
                }
        }
#pragma unroll
        for (int i = 0; i < DMAX; ++i)
            if (i < d) {
                const double* ci = C + i * m * m;
#pragma unroll
                for (int ks = 0; ks < KS; ++ks) {
                    const int kk = 4 * ks + q;
                    if (4 * ks < m) {
#pragma unroll
                        for (int tn = 0; tn < MT; ++tn) {
                            const int nn = 8 * tn + g;
                            const double bv = (kk < m && nn < m) ? ci[kk * m + nn] : 0.0;
#pragma unroll
                            for (int u = 0; u < U; ++u) dmma(acc[u][tn], av[u][i][ks], bv);
                        }
                    }
                }
            }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long long row = base0 + (long long)u * 8 * kNW + g;
            if (row < r1) {
#pragma unroll
                for (int tn = 0; tn < MT; ++tn) {
                    const int cc = 8 * tn + 2 * q;
                    if (vec && cc < m) {
                        *reinterpret_cast<double2*>(Wout + row * m + cc) = make_double2(acc[u][tn][0], acc[u][tn][1]);
                    } else {
                        if (cc < m) Wout[row * m + cc] = acc[u][tn][0];
                        if (cc + 1 < m) Wout[row * m + cc + 1] = acc[u][tn][1];
                    }
                }
            }
        }
    }
}

// ---- m x m factors (warp 0 of every CTA, identical inputs) ----------------------
// Right-looking Cholesky of the symmetric m x m matrix A (smem, overwritten) with the breakdown test of
// cholesky_small (linalg.py:164-184: pivot not finite or <= tol * max |diag|), then S = R^-1 (upper,
// zeros below the diagonal) with one lane per column held in registers.  Called by one whole warp.
// Returns -1 or the failing column.
template <int MB>
__device__ __forceinline__ int warp_chol_inverse(double* A, double* R, double* S, double* rinv, int m, double tol, double& piv_out,
                                 double& scale_out) {
    const int lane = threadIdx.x & 31;
    double sc = lane < m ? fabs(A[lane * m + lane]) : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sc = fmax(sc, __shfl_xor_sync(0xffffffffu, sc, o));
    scale_out = sc;
    for (int e = lane; e < m * m; e += 32) R[e] = 0.0;
    __syncwarp();
    for (int j = 0; j < m; ++j) {
        const double piv = A[j * m + j];
        if (!isfinite(piv) || piv <= tol * sc) {
            piv_out = piv;
            return j;
        }
        // 1 / sqrt(piv) and sqrt(piv) = piv / sqrt(piv) from one rsqrt (~1 ulp each): the dependent
        // sqrt -> divide chain of the launch-per-phase kernels is what an 8 x 8 factor spends its time in
        const double ri = rsqrt(piv);
        const double rjj = piv * ri;
        if (lane > j && lane < m) R[j * m + lane] = A[j * m + lane] * ri;
        if (lane == j) {
            R[j * m + j] = rjj;
            rinv[j] = ri;
        }
        __syncwarp();
        const int L = m - j - 1;
        for (int e = lane; e < L * L; e += 32) {
            const int i = j + 1 + e / L, k = j + 1 + e % L;
            A[i * m + k] -= R[j * m + i] * R[j * m + k];
        }
        __syncwarp();
    }
    if (lane < m) {
        const int cc = lane;
        double col[MB];
#pragma unroll
        for (int i = MB - 1; i >= 0; --i) {
            double s = 0.0;
#pragma unroll
            for (int k = i + 1; k < MB; ++k) s += (k <= cc && k < m && i < m) ? R[i * m + k] * col[k] : 0.0;
            col[i] = (i > cc || i >= m) ? 0.0 : (i == cc) ? rinv[cc] : -s * rinv[i];
        }
#pragma unroll
        for (int i = 0; i < MB; ++i)
            if (i < m) S[i * m + cc] = col[i];
    }
    __syncwarp();
    return -1;
}

// m = 8: the same factor with the matrix held in registers by one warp (lane 4 i + q owns A[i][2 q],
// A[i][2 q + 1]: the DMMA accumulator layout) and the column steps exchanged by shuffles -- no shared-
// memory round trips inside the column loop.  PRE: Pre-CholQR (column norms D from the raw diagonal, the
// factor of sym(D^-1 G D^-1), output D^-1 R^-1); else the plain factor of sym(G), output R^-1.
// Called by one whole warp; returns 0 ok / 1 zero column / 2 pivot breakdown.
template <bool PRE>
__device__ __forceinline__ int warp_factor8(const double* G, double* Rs, double* Sout, double* rinv, double* inrm,
                                            double tol, int& col, double& piv_out, double& scale_out) {
    const int lane = threadIdx.x & 31, i = lane >> 2, q = lane & 3, k0 = 2 * q;
    double a0 = 0.5 * (G[i * 8 + k0] + G[k0 * 8 + i]);
    double a1 = 0.5 * (G[i * 8 + k0 + 1] + G[(k0 + 1) * 8 + i]);
    if (PRE) {
        const int j = lane & 7;
        const double dg = G[j * 8 + j];
        const unsigned zero = __ballot_sync(0xffffffffu, lane < 8 && dg == 0.0);
        if (zero) {
            col = __ffs((int)zero) - 1;
            piv_out = 0.0;
            scale_out = 0.0;
            return 1;
        }
        const double ir = rsqrt(dg);  // NaN for a negative / NaN diagonal: the first pivot test then fails
        if (lane < 8) inrm[lane] = ir;
        const double ii = __shfl_sync(0xffffffffu, ir, i);
        const double ik0 = __shfl_sync(0xffffffffu, ir, k0);
        const double ik1 = __shfl_sync(0xffffffffu, ir, k0 + 1);
        a0 *= ii * ik0;
        a1 *= ii * ik1;
    }
    double sc = (k0 == i) ? fabs(a0) : ((k0 + 1 == i) ? fabs(a1) : 0.0);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sc = fmax(sc, __shfl_xor_sync(0xffffffffu, sc, o));
    scale_out = sc;
    double r0 = 0.0, r1 = 0.0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const double piv = __shfl_sync(0xffffffffu, (j & 1) ? a1 : a0, 4 * j + (j >> 1));
        if (!isfinite(piv) || piv <= tol * sc) {
            col = j;
            piv_out = piv;
            return 2;
        }
        const double ri = rsqrt(piv);
        const double rjj = piv * ri;
        const double ajk0 = __shfl_sync(0xffffffffu, a0, 4 * j + q);  // A[j][2 q], A[j][2 q + 1]
        const double ajk1 = __shfl_sync(0xffffffffu, a1, 4 * j + q);
        const double t0 = __shfl_sync(0xffffffffu, a0, 4 * j + (i >> 1));  // A[j][i]
        const double t1 = __shfl_sync(0xffffffffu, a1, 4 * j + (i >> 1));
        const double rji = ((i & 1) ? t1 : t0) * ri;
        if (i == j) {
            r0 = k0 > j ? a0 * ri : (k0 == j ? rjj : 0.0);
            r1 = k0 + 1 > j ? a1 * ri : (k0 + 1 == j ? rjj : 0.0);
        }
        if (i > j) {
            a0 -= rji * (ajk0 * ri);
            a1 -= rji * (ajk1 * ri);
        }
        if (lane == 0) rinv[j] = ri;
    }
    Rs[i * 8 + k0] = r0;
    Rs[i * 8 + k0 + 1] = r1;
    __syncwarp();
    if (lane < 8) {
        const int cc = lane;
        double colv[8];
#pragma unroll
        for (int r = 7; r >= 0; --r) {
            double acc = 0.0;
#pragma unroll
            for (int k = r + 1; k < 8; ++k) acc += (k <= cc) ? Rs[r * 8 + k] * colv[k] : 0.0;
            colv[r] = (r > cc) ? 0.0 : (r == cc) ? rinv[cc] : -acc * rinv[r];
        }
#pragma unroll
        for (int r = 0; r < 8; ++r) Sout[r * 8 + cc] = PRE ? colv[r] * inrm[r] : colv[r];
    }
    __syncwarp();
    return 0;
}

// Pre-CholQR factor S0 = D^-1 chol(sym(D^-1 G D^-1))^-1 (aortho.py:74-79, 104-106) from G = W^T W.
// 0 ok, 1 zero column, 2 pivot breakdown (col / piv / scale describe it).
template <int MB>
__device__ __forceinline__ int prechol_local(Ctx& c, int m, double tol, int& col, double& piv, double& scale) {
    __shared__ int res[2];
    __shared__ double resd[2];
    __shared__ double nrm[16], inrm[16], rinv[16];
    double* G = c.sm + c.Lp->G;
    double* R = c.sm + c.Lp->R;
    double* S = c.sm + c.Lp->S;
    double* S0 = c.sm + c.Lp->S0;
    if (MB == 8 && m == 8) {
        if (threadIdx.x < 32) {
            int bad = -1;
            double pv = 0.0, scv = 0.0;
            const int kind = warp_factor8<true>(G, R, S0, rinv, inrm, tol, bad, pv, scv);
            if (threadIdx.x == 0) {
                res[0] = kind;
                res[1] = bad;
                resd[0] = pv;
                resd[1] = scv;
            }
        }
    } else if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        int kind = 0, bad = -1;
        double pv = 0.0, scv = 0.0;
        if (lane < m) {
            const double gjj = G[lane * m + lane];
            const double ir = gjj > 0.0 ? rsqrt(gjj) : 0.0;
            nrm[lane] = gjj > 0.0 ? gjj * ir : sqrt(gjj);  // 0 (zero column) or NaN pass through
            inrm[lane] = ir;
        }
        __syncwarp();
        int dead = -1;
        for (int j = m - 1; j >= 0; --j)
            if (nrm[j] == 0.0) dead = j;
        if (dead >= 0) {
            kind = 1;
            bad = dead;
        } else {
            for (int e = lane; e < m * m; e += 32) {
                const int a = e / m, b = e % m;
                const double gab = G[a * m + b] * inrm[a] * inrm[b];
                const double gba = G[b * m + a] * inrm[b] * inrm[a];
                R[e] = 0.5 * (gab + gba);
            }
            __syncwarp();
            for (int e = lane; e < m * m; e += 32) G[e] = R[e];
            __syncwarp();
            const int fail = warp_chol_inverse<MB>(G, R, S, rinv, m, tol, pv, scv);
            if (fail >= 0) {
                kind = 2;
                bad = fail;
            } else {
                for (int e = lane; e < m * m; e += 32) S0[e] = S[e] * inrm[e / m];
            }
        }
        if (lane == 0) {
            res[0] = kind;
            res[1] = bad;
            resd[0] = pv;
            resd[1] = scv;
        }
    }
    __syncthreads();
    col = res[1];
    piv = resd[0];
    scale = resd[1];
    return res[0];
}

// A-CholQR factor S = chol(sym G)^-1 (aortho.py:107-109).
template <int MB>
__device__ __forceinline__ int cholinv_local(Ctx& c, int m, double tol, int& col, double& piv, double& scale) {
    __shared__ int res[2];
    __shared__ double resd[2];
    __shared__ double rinv[16];
    double* G = c.sm + c.Lp->G;
    double* R = c.sm + c.Lp->R;
    double* S = c.sm + c.Lp->S;
    if (MB == 8 && m == 8) {
        if (threadIdx.x < 32) {
            __shared__ double unused_inrm[8];
            int bad = -1;
            double pv = 0.0, scv = 0.0;
            const int kind = warp_factor8<false>(G, R, S, rinv, unused_inrm, tol, bad, pv, scv);
            if (threadIdx.x == 0) {
                res[0] = kind;
                res[1] = bad;
                resd[0] = pv;
                resd[1] = scv;
            }
        }
    } else if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        double pv = 0.0, scv = 0.0;
        for (int e = lane; e < m * m; e += 32) {
            const int a = e / m, b = e % m;
            R[e] = 0.5 * (G[a * m + b] + G[b * m + a]);
        }
        __syncwarp();
        for (int e = lane; e < m * m; e += 32) G[e] = R[e];
        __syncwarp();
        const int fail = warp_chol_inverse<MB>(G, R, S, rinv, m, tol, pv, scv);
        if (lane == 0) {
            res[0] = fail >= 0 ? 2 : 0;
            res[1] = fail;
            resd[0] = pv;
            resd[1] = scv;
        }
    }
    __syncthreads();
    col = res[1];
    piv = resd[0];
    scale = resd[1];
    return res[0];
}

// CSR operators: true when no row of the matrix holds more than 8 entries (the operator rows keep 8 in
// registers) -- agreed across the cluster, so every CTA takes the same branch.
__device__ __forceinline__ bool rows_fit(Ctx& c, const Args& a, long long r0, long long r1) {
    double bad = 0.0;
    for (long long row = r0 + threadIdx.x; row < r1; row += kNT)
        if (__ldg(a.rp + row + 1) - __ldg(a.rp + row) > 8) bad = 1.0;
    return scalar_all(c, bad, R_ALPHA) == 0.0;  // a region no later exchange reuses before a cluster barrier
}

// M > 0: the block width is exactly M (compile-time index math); M == 0: runtime width a.t <= 8 MT.
template <bool CSR, int MT, int M>
__global__ void __launch_bounds__(kNT, 1) cluster_solve_kernel(const Args a) {
    extern __shared__ __align__(16) double smem[];
    cg::cluster_group cluster = cg::this_cluster();
    const int tid = threadIdx.x;
    const long long n = a.n;
    const int m = M > 0 ? M : a.t, win = a.window;
    Ctx c;
    c.sm = smem;
    __shared__ Layout s_layout;
    if (tid == 0) s_layout = make_layout(win, m, (int)cluster.num_blocks());
    __syncthreads();
    c.Lp = &s_layout;
    c.bar = reinterpret_cast<unsigned long long*>(smem + c.Lp->misc);
    c.qp = reinterpret_cast<const double**>(smem + c.Lp->misc + R_COUNT);
    c.aqp = c.qp + kMaxWin;
    c.one = c.aqp + kMaxWin;
    c.rank = cluster.block_rank();
    c.cl = cluster.num_blocks();
    c.parity = 0;
    const unsigned rank = c.rank, cl = c.cl;
    // contiguous row ranges in multiples of 8 rows (whole DMMA row tiles per CTA)
    const long long per = ((n + cl - 1) / cl + 7) / 8 * 8;
    const long long r0 = min(n, (long long)rank * per), r1 = min(n, r0 + per);
    const bool lead = (rank == 0 && tid == 0);
    const bool prof = lead && a.ticks != nullptr;
    long long tick = prof ? clock64() : 0;
#define PHASE(id)                        \
    if (prof) {                          \
        const long long now = clock64(); \
        a.ticks[id] += now - tick;       \
        tick = now;                      \
    }

    if (tid == 0) {
        for (int i = 0; i < R_COUNT; ++i) mbar_init(c.bar + i, 1);
        mbar_fence_init();
    }
    cluster.sync();  // every CTA's mbarriers exist before any peer signals them

    pdl_wait();
    EkcgCtrl* ctrl = a.ctrl;
    bool run = ctrl->live != 0;  // rho0 == 0: nothing to do (same value in every CTA)
    const double tol_abs = ctrl->tol_abs;
    double best_rho = ctrl->best_rho;
    int best_k = ctrl->best_k;
    if (CSR && run && !rows_fit(c, a, r0, r1)) {  // a row with more than 8 entries: refuse (status 5)
        if (lead) {
            ctrl->status = 5;
            ctrl->live = 0;
        }
        run = false;
    }

    double* WA = a.blocks + 2LL * win * a.span;
    double* WB = WA + a.span;
    double* WC = WB + a.span;
    double* tmpv = WC + a.span;
    double* Csm = smem + c.Lp->C;
    double* Gs = smem + c.Lp->G;
    double* alpha = smem + c.Lp->alpha;

    int d = 0, since = 0, newest = -1;
    int status = 0, brk_kind = 0, brk_col = -1;
    double brk_piv = 0.0, brk_scale = 0.0, rho = ctrl->last_rho;
    int k = 1;
    for (; run; ++k) {
        const int slot = since % win;
        double* Qnew = a.blocks + (long long)slot * a.span;
        double* AQnew = a.blocks + (long long)(win + slot) * a.span;
        if (tid < d) {  // retained blocks, oldest first
            const int sl = ((since - d + tid) % win + win) % win;
            c.qp[tid] = a.blocks + (long long)sl * a.span;
            c.aqp[tid] = a.blocks + (long long)(win + sl) * a.span;
        }
        // ---- candidate (solvers.py:366-371): split(r) for an empty store, else the cached A W_{k-1} ----
        const double* W;
        if (d == 0) {
            const unsigned items = (unsigned)(r1 - r0) * (unsigned)m;
            for (unsigned it = tid; it < items; it += kNT) {
                const long long row = r0 + it / (unsigned)m;
                const int col = (int)(it % (unsigned)m);
                WA[row * m + col] = (a.owner[row] == col) ? a.r[row] : 0.0;
            }
            W = WA;
        } else {
            W = a.blocks + (long long)(win + newest) * a.span;
        }
        __syncthreads();
        PHASE(0);
        // ---- CGS2 against the retained blocks (aortho.py:89-95): C = [A Q_i]^T W, W <- W - sum Q_i C_i ----
        for (int pas = 0; pas < 2 && d > 0; ++pas) {
            gram_all<MT>(c, c.aqp, d, m, m, W, m, m, r0, r1, pas == 0 ? R_PASS1 : R_PASS2, Csm, -1.0);
            PHASE(1);
            update_local<MT>(W, true, c.qp, d, Csm, WA, m, r0, r1);
            W = WA;
            __syncthreads();
            PHASE(3);
        }
        // ---- Pre-CholQR (aortho.py:98-106): Graw = W^T W, W0 = W S0 ----
        if (tid == 0) c.one[0] = WA;
        __syncthreads();
        gram_all<MT>(c, c.one, 1, m, m, WA, m, m, r0, r1, R_GRAW, Gs);
        PHASE(4);
        brk_kind = prechol_local<8 * MT>(c, m, a.chol_tol, brk_col, brk_piv, brk_scale);
        if (brk_kind != 0) {
            status = 3;
            break;
        }
        PHASE(6);
        update_local<MT>(nullptr, false, c.one, 1, smem + c.Lp->S0, WB, m, r0, r1);
        cluster.sync();  // W0 rows visible to the neighbours' operator rows
        PHASE(7);
        // ---- A-CholQR (aortho.py:107-110): G = W0^T A W0, W_k = W0 S ----
        apply_local<CSR>(a, WB, m, WC, m, m, r0, r1);
        if (tid == 0) c.one[0] = WB;
        __syncthreads();
        PHASE(8);
        gram_all<MT>(c, c.one, 1, m, m, WC, m, m, r0, r1, R_G, Gs);
        PHASE(9);
        brk_kind = cholinv_local<8 * MT>(c, m, a.chol_tol, brk_col, brk_piv, brk_scale);
        if (brk_kind != 0) {
            status = 3;
            break;
        }
        PHASE(11);
        update_local<MT>(nullptr, false, c.one, 1, smem + c.Lp->S, Qnew, m, r0, r1);
        cluster.sync();  // W_k rows visible to the neighbours' operator rows
        PHASE(12);
        // ---- alpha = W_k^T r (solvers.py:394): partials sent now, summed after A W_k (which does not
        // need alpha), so the exchange is hidden behind the operator rows ----
        if (tid == 0) c.one[0] = Qnew;
        __syncthreads();
        gram_all<MT>(c, c.one, 1, m, m, a.r, 1, 1, r0, r1, R_ALPHA, alpha, 1.0, true);
        PHASE(13);
        apply_local<CSR>(a, Qnew, m, AQnew, m, m, r0, r1);
        exchange_finish(c, R_ALPHA, m, alpha, 1.0);  // ends with a CTA barrier: A W_k rows written
        PHASE(15);
        // ---- x += W alpha, r -= A W alpha, |r|^2 (solvers.py:395-398) ----
        {
            double part = 0.0;
            for (long long row = r0 + tid; row < r1; row += kNT) {
                const double* w = Qnew + row * m;
                const double* aw = AQnew + row * m;
                double wv[8 * MT], awv[8 * MT];
#pragma unroll
                for (int cc = 0; cc < 8 * MT; ++cc) {
                    wv[cc] = cc < m ? w[cc] : 0.0;
                    awv[cc] = cc < m ? aw[cc] : 0.0;
                }
                double dx = 0.0, dr = 0.0;
#pragma unroll
                for (int cc = 0; cc < 8 * MT; ++cc)
                    if (cc < m) {
                        dx = fma(wv[cc], alpha[cc], dx);
                        dr = fma(awv[cc], alpha[cc], dr);
                    }
                a.x[row] += dx;
                const double rn = a.r[row] - dr;
                a.r[row] = rn;
                part = fma(rn, rn, part);
            }
            PHASE(16);
            rho = sqrt(scalar_all(c, part, R_RHO));
            PHASE(17);
        }
        newest = slot;
        ++since;
        if (d < win) ++d;
        // ---- true-residual drift log every `every` iterations (solvers.py:401-402) ----
        if (k % a.every == 0) {
            cluster.sync();  // every CTA's x rows written
            apply_local<CSR>(a, a.x, 1, tmpv, 1, 1, r0, r1);
            __syncthreads();
            double part = 0.0;
            for (long long row = r0 + tid; row < r1; row += kNT) {
                const double e = a.b[row] - tmpv[row];
                part = fma(e, e, part);
            }
            const double tr2 = scalar_all(c, part, R_CHECK);
            if (lead) a.checks[k / a.every - 1] = sqrt(tr2);
        }
        PHASE(18);
        // ---- end of iteration (solvers.py:357, 398-415; finish_body of factor.cuh) ----
        if (lead) a.history[k] = rho;
        if (rho < best_rho) {
            best_rho = rho;
            best_k = k;
        }
        if (rho <= tol_abs) {
            status = 1;
            break;
        }
        if (!(rho > tol_abs) || k + 1 > a.kmax) {
            status = 2;
            break;
        }
    }
    if (lead && run) {
        if (status == 3) {
            ctrl->brk_kind = brk_kind;
            ctrl->brk_col = brk_col;
            ctrl->brk_pivot = brk_piv;
            ctrl->brk_scale = brk_scale;
            ctrl->brk_iter = k;
            ctrl->k_done = k - 1;
        } else {
            ctrl->k_done = k;
            ctrl->last_rho = rho;
        }
        ctrl->best_rho = best_rho;
        ctrl->best_k = best_k;
        ctrl->status = status;
        ctrl->live = 0;
    }
    cluster.sync();  // no CTA exits while a peer may still write into its shared memory
#undef PHASE
}

template <bool CSR, int MT, int M>
int launch_cluster(const Args& a, cudaStream_t st) {
    auto fn = cluster_solve_kernel<CSR, MT, M>;
    static size_t ready[kEkcgMaxDevices];  // dynamic shared memory the kernel is set up for, per device
    const int dev = ekcg_device();
    // the largest cluster whose receive buffers fit and that the device can place (16 needs the
    // non-portable opt-in; 8 is portable)
    for (int cl = kMaxCl; cl >= 1; cl >>= 1) {
        const size_t smem = sizeof(double) * (size_t)make_layout(a.window, a.t, cl).total;
        if (smem > kSmemCap) continue;
        if (ready[dev] < smem) {
            if (cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
                    cudaSuccess ||
                cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) !=
                    cudaSuccess) {
                cudaGetLastError();
                return EKCG_ELAUNCH;
            }
            ready[dev] = smem;
        }
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(cl);
        cfg.blockDim = dim3(kNT);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute attr[2];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = cl;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[1].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 2;
        int clusters = 0;
        if (cudaOccupancyMaxActiveClusters(&clusters, (const void*)fn, &cfg) != cudaSuccess || clusters < 1) {
            cudaGetLastError();
            continue;
        }
        if (cudaLaunchKernelEx(&cfg, fn, a) == cudaSuccess) {
            ++g_ekcg_launches;
            return EKCG_OK;
        }
        cudaGetLastError();
    }
    return EKCG_ELAUNCH;
}

template <bool CSR>
int launch_cluster_m(const Args& a, cudaStream_t st) {
    if (a.t == 8) return launch_cluster<CSR, 1, 8>(a, st);
    if (a.t == 16) return launch_cluster<CSR, 2, 16>(a, st);
    return a.t < 8 ? launch_cluster<CSR, 1, 0>(a, st) : launch_cluster<CSR, 2, 0>(a, st);
}


// ---------------------------------------------------------------------------
// Classical CG (solvers.py:199-258, unpreconditioned: z = r) on the same cluster machinery: one cluster
// barrier (p visible to the neighbours' operator rows) and two scalar exchanges (p^T A p, |r|^2) per
// iteration.  The launch-per-phase `cg` reads three scalars back to the host every iteration.
// ---------------------------------------------------------------------------
struct CgArgs {
    Args op;        // operator, n, kmax, x, r, ctrl, history (t = window = 1)
    double* p;      // n
    double* ap;     // n
};

template <bool CSR>
__global__ void __launch_bounds__(kNT, 1) cluster_cg_kernel(const CgArgs ca) {
    extern __shared__ __align__(16) double smem[];
    const Args& a = ca.op;
    cg::cluster_group cluster = cg::this_cluster();
    const int tid = threadIdx.x;
    const long long n = a.n;
    __shared__ Layout s_layout;
    if (tid == 0) s_layout = make_layout(1, 1, (int)cluster.num_blocks());
    __syncthreads();
    Ctx c;
    c.sm = smem;
    c.Lp = &s_layout;
    c.bar = reinterpret_cast<unsigned long long*>(smem + c.Lp->misc);
    c.qp = c.aqp = c.one = nullptr;
    c.rank = cluster.block_rank();
    c.cl = cluster.num_blocks();
    c.parity = 0;
    const long long per = (n + c.cl - 1) / c.cl;
    const long long r0 = min(n, (long long)c.rank * per), r1 = min(n, r0 + per);
    const bool lead = (c.rank == 0 && tid == 0);
    if (tid == 0) {
        for (int i = 0; i < R_COUNT; ++i) mbar_init(c.bar + i, 1);
        mbar_fence_init();
    }
    cluster.sync();

    pdl_wait();
    EkcgCtrl* ctrl = a.ctrl;
    bool run = ctrl->live != 0;  // rho0 == 0: converged before the first iteration
    const double tol_abs = ctrl->tol_abs;
    if (CSR && run && !rows_fit(c, a, r0, r1)) {
        if (lead) {
            ctrl->status = 5;
            ctrl->live = 0;
        }
        run = false;
    }
    double* __restrict__ p = ca.p;
    double* __restrict__ ap = ca.ap;
    double rz = 0.0, rho = ctrl->last_rho, pAp = 0.0;
    int status = 0, k = 1;
    if (run) {
        double part = 0.0;
        for (long long row = r0 + tid; row < r1; row += kNT) {
            const double rv = a.r[row];
            p[row] = rv;  // p = z = r
            part = fma(rv, rv, part);
        }
        rz = scalar_all(c, part, R_CHECK);  // r . z
    }
    for (; run; ++k) {
        cluster.sync();  // every CTA's p rows written
        apply_local<CSR>(a, p, 1, ap, 1, 1, r0, r1);
        __syncthreads();
        double part = 0.0;
        for (long long row = r0 + tid; row < r1; row += kNT) part = fma(p[row], ap[row], part);
        pAp = scalar_all(c, part, R_CHECK);  // (two-slot scalar regions: R_CHECK, R_RHO)
        if (pAp <= 0.0) {  // nonpositive curvature (solvers.py:228-231)
            status = 3;
            break;
        }
        const double alpha = rz / pAp;
        part = 0.0;
        for (long long row = r0 + tid; row < r1; row += kNT) {
            a.x[row] = fma(alpha, p[row], a.x[row]);
            const double rn = fma(-alpha, ap[row], a.r[row]);
            a.r[row] = rn;
            part = fma(rn, rn, part);
        }
        const double rz_new = scalar_all(c, part, R_RHO);
        rho = sqrt(rz_new);
        if (lead) a.history[k] = rho;
        if (rho <= tol_abs) {
            status = 1;
            break;
        }
        if (!(rho > tol_abs) || k + 1 > a.kmax) {
            status = 2;
            break;
        }
        const double beta = rz_new / rz;
        rz = rz_new;
        for (long long row = r0 + tid; row < r1; row += kNT) p[row] = fma(beta, p[row], a.r[row]);
    }
    if (lead && run) {
        if (status == 3) {
            ctrl->brk_kind = 3;
            ctrl->brk_pivot = pAp;
            ctrl->brk_iter = k;
            ctrl->k_done = k - 1;
        } else {
            ctrl->k_done = k;
            ctrl->last_rho = rho;
        }
        ctrl->status = status;
        ctrl->live = 0;
    }
    cluster.sync();
}

template <bool CSR>
int launch_cluster_cg(const CgArgs& ca, cudaStream_t st) {
    auto fn = cluster_cg_kernel<CSR>;
    static bool ready[kEkcgMaxDevices];
    const int dev = ekcg_device();
    if (!ready[dev]) {
        if (cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
            cudaGetLastError();
            return EKCG_ELAUNCH;
        }
        ready[dev] = true;
    }
    for (int cl = kMaxCl; cl >= 1; cl >>= 1) {
        const size_t smem = sizeof(double) * (size_t)make_layout(1, 1, cl).total;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(cl);
        cfg.blockDim = dim3(kNT);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute attr[2];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = cl;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[1].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 2;
        int clusters = 0;
        if (cudaOccupancyMaxActiveClusters(&clusters, (const void*)fn, &cfg) != cudaSuccess || clusters < 1) {
            cudaGetLastError();
            continue;
        }
        if (cudaLaunchKernelEx(&cfg, fn, ca) == cudaSuccess) {
            ++g_ekcg_launches;
            return EKCG_OK;
        }
        cudaGetLastError();
    }
    return EKCG_ELAUNCH;
}

}  // namespace

extern "C" int ekcg_cluster_solve_fits(long long n, int t, int window) {
    if (n < 1 || t < 1 || t > 16 || window < 1) return 0;
    const int mt = t <= 8 ? 1 : 2;  // 8-wide DMMA tiles per block dimension
    if (window * mt > kMaxWin || window * t * t > 2 * kNT || n * t > (1LL << 22)) return 0;
    return sizeof(double) * (size_t)make_layout(window, t, 4).total <= kSmemCap ? 1 : 0;  // at least 4 CTAs
}

extern "C" int ekcg_cluster_solve(const EkcgStencil* desc, const long long* row_ptr, const int* col_idx,
                                  const double* values, long long n, int t, int window, int kmax, int every,
                                  const int* owner, const double* b, double* x, double* r, double* blocks,
                                  long long span, void* ctrl, double* history, double* checks, double chol_tol,
                                  long long* phase_ticks, void* stream) {
    if (!ekcg_cluster_solve_fits(n, t, window) || kmax < 1 || every < 1 || span < n * t) return EKCG_EINVAL;
    if (owner == nullptr || b == nullptr || x == nullptr || r == nullptr || blocks == nullptr || ctrl == nullptr ||
        history == nullptr || checks == nullptr)
        return EKCG_EINVAL;
    Args a = {};
    a.n = n;
    a.t = t;
    a.window = window;
    a.kmax = kmax;
    a.every = every;
    a.owner = owner;
    a.b = b;
    a.x = x;
    a.r = r;
    a.blocks = blocks;
    a.span = span;
    a.ctrl = (EkcgCtrl*)ctrl;
    a.history = history;
    a.checks = checks;
    a.chol_tol = chol_tol;
    a.ticks = phase_ticks;
    if (desc != nullptr) {
        long long ns = 0;
        if (prepare_stencil(desc, a.s, a.uf, ns) != EKCG_OK || ns != n) return EKCG_EINVAL;
        if (a.s.row_begin != 0 || a.s.row_end != n) return EKCG_EINVAL;
        return launch_cluster_m<false>(a, as_stream(stream));
    }
    if (row_ptr == nullptr || col_idx == nullptr || values == nullptr) return EKCG_EINVAL;
    a.rp = row_ptr;
    a.ci = col_idx;
    a.vv = values;
    return launch_cluster_m<true>(a, as_stream(stream));
}

extern "C" int ekcg_cluster_cg(const EkcgStencil* desc, const long long* row_ptr, const int* col_idx,
                               const double* values, long long n, int kmax, double* x, double* r, double* scratch,
                               void* ctrl, double* history, void* stream) {
    if (n < 1 || n > (1LL << 22) || kmax < 1) return EKCG_EINVAL;
    if (x == nullptr || r == nullptr || scratch == nullptr || ctrl == nullptr || history == nullptr)
        return EKCG_EINVAL;
    CgArgs ca = {};
    Args& a = ca.op;
    a.n = n;
    a.t = 1;
    a.window = 1;
    a.kmax = kmax;
    a.every = 1;
    a.x = x;
    a.r = r;
    a.ctrl = (EkcgCtrl*)ctrl;
    a.history = history;
    ca.p = scratch;
    ca.ap = scratch + n;
    if (desc != nullptr) {
        long long ns = 0;
        if (prepare_stencil(desc, a.s, a.uf, ns) != EKCG_OK || ns != n) return EKCG_EINVAL;
        if (a.s.row_begin != 0 || a.s.row_end != n) return EKCG_EINVAL;
        return launch_cluster_cg<false>(ca, as_stream(stream));
    }
    if (row_ptr == nullptr || col_idx == nullptr || values == nullptr) return EKCG_EINVAL;
    a.rp = row_ptr;
    a.ci = col_idx;
    a.vv = values;
    return launch_cluster_cg<true>(ca, as_stream(stream));
}
