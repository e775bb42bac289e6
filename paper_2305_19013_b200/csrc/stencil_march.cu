// Plane-marching stencil SpMM on TMA: Y = A X for the grid operator.
//
// A CTA owns a TX x TY tile of (x, y) grid columns and KC block columns and
// marches along the slowest grid axis (z in 3-D, y in 2-D).  Each plane of
// the tile plus a one-node ring is one TMA box [1][TY+2][TX+2][KC] of the
// tensor view X[z][y][x][col]; NS stages are in flight, completion tracked by
// one mbarrier per stage.  Out-of-grid ring nodes, the planes before the
// first and after the last, and columns >= m are zero-filled by the TMA unit
// (they are never read: absent stencil entries are skipped by mask).  Every X
// row comes from HBM once; only the tile ring is re-read, through L2.
//
// Same coefficients, the same column-ordered entries and the same
// p0 + (((p1 + p2) + ...)) association with separately rounded products as
// the row-parallel kernel (sparse.cu), so the result is bitwise the reference
// spmm on the assembled CSR (linalg.py:141-152).
#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "ekcg_b200.h"
#include "stencil.cuh"
#include "tma.cuh"
#include "factor.cuh"

namespace {

using namespace ekcg_dev;


// Tile shapes: 3-D TX x TY in (x, y); 2-D a TX segment of the x axis.  NS
// stages; NS - 2 planes are loaded ahead of the one being computed.
template <int DIM_, int KC_, int TX_, int TY_, int NS_>
struct March {
    static constexpr int DIM = DIM_, KC = KC_, TX = TX_, TY = TY_, NS = NS_, AHEAD = NS_ - 2;
    static constexpr int PX = TX + 2, PY = (DIM == 3) ? TY + 2 : 1, OY = (DIM == 3) ? 1 : 0;
    static constexpr int LANES = KC / 4;  // 4 doubles per item
    static constexpr int ITEMS = TX * TY * LANES;
    static constexpr int NT = ITEMS < 256 ? ITEMS : 256;
    static constexpr int IPT = ITEMS / NT;
    static constexpr int BOX = PX * PY * KC;                 // doubles per TMA box
    static constexpr int STAGE = ((BOX * 8 + 127) / 128) * 16;  // stage stride: 128-B aligned TMA destinations
    static constexpr size_t SMEM = sizeof(double) * STAGE * NS;
    static constexpr int MINB = (int)((227 * 1024) / (SMEM + 1024)) < 8 ? (int)((227 * 1024) / (SMEM + 1024)) : 8;
    static_assert(ITEMS % NT == 0, "items per thread");
};

template <class P>
__device__ __forceinline__ void march_apply(const double (&v)[7], unsigned mk, bool interior, const double* pm,
                                            const double* pc, const double* pp, int ix, int iy, int ig,
                                            double (&o)[4], int& ha, int& hb);

// A X for one item: node (x0+ix, y0+iy) of plane w, columns 4 ig .. 4 ig+3 of
// the chunk, from the staged planes pm / pc / pp (previous, current, next).
// o[0..1] are columns 4 ig + ha (+1), o[2..3] columns 4 ig + hb (+1).
template <class P>
__device__ __forceinline__ void march_node(const EkcgStencil& s, const UniformFaces& uf, const double* pm,
                                           const double* pc, const double* pp, int x0, int y0, int ix, int iy, int ig,
                                           int w, unsigned nx, unsigned ny, unsigned nw, double (&o)[4], int& ha,
                                           int& hb) {
    constexpr int DIM = P::DIM, KC = P::KC;
    const unsigned x = x0 + ix, y = y0 + iy;
    const bool interior = x > 0 && x + 1 < nx && w > 0 && (unsigned)w + 1 < nw &&
                          (DIM == 2 || (y > 0 && y + 1 < ny));
    double v[7];
    unsigned mk;
    if (interior && s.kfield == nullptr) {
        v[0] = -uf.fz; v[1] = -uf.fy; v[2] = -uf.fx; v[3] = uf.dint;
        v[4] = -uf.fx; v[5] = -uf.fy; v[6] = -uf.fz;
        mk = (DIM == 3) ? 0x7fu : 0x3eu;
    } else {
        mk = (DIM == 3) ? stencil_coef(s, uf, x, y, (unsigned)w, v)
                        : stencil_coef(s, uf, x, (unsigned)w, 0u, v);
    }
    march_apply<P>(v, mk, interior, pm, pc, pp, ix, iy, ig, o, ha, hb);
}

// The products and sums of one item from its coefficient row v (slot order z-, y-, x-, diag, x+, y+, z+),
// presence mask mk and the staged planes: p0 + (((p1 + p2) + ...)) over the present entries in order.
template <class P>
__device__ __forceinline__ void march_apply(const double (&v)[7], unsigned mk, bool interior, const double* pm,
                                            const double* pc, const double* pp, int ix, int iy, int ig,
                                            double (&o)[4], int& ha, int& hb) {
    constexpr int DIM = P::DIM, KC = P::KC;
    const int hc = ((iy + P::OY) * P::PX + ix + 1) * KC + 4 * ig;
    // neighbour slices in entry order z-, y-, x-, diag, x+, y+, z+ (2-D: the march axis is y)
    const double* nb[7];
    if (DIM == 3) {
        nb[0] = pm + hc; nb[1] = pc + hc - P::PX * KC; nb[2] = pc + hc - KC; nb[3] = pc + hc;
        nb[4] = pc + hc + KC; nb[5] = pc + hc + P::PX * KC; nb[6] = pp + hc;
    } else {
        nb[0] = pc; nb[1] = pm + hc; nb[2] = pc + hc - KC; nb[3] = pc + hc;
        nb[4] = pc + hc + KC; nb[5] = pp + hc; nb[6] = pc;
    }
    // the two 16-B halves of the item's 4 columns: for KC = 16 odd nodes
    // take the upper 8 columns first, so a quarter warp (2 nodes x 4
    // lanes) reads 128 distinct bytes per LDS.128 -- no bank conflicts
    const int sw = (KC == 16) ? ((ix & 1) ? 8 : 0) : 0;
    ha = (2 * ig + sw) % KC - 4 * ig;
    hb = (2 * ig + KC / 2 + sw) % KC - 4 * ig;
    if (interior) {
        // all entries present: straight-line p0 + ((p1 + p2) + ...)
        constexpr int e0 = (DIM == 3) ? 0 : 1, e1 = (DIM == 3) ? 6 : 5;
        double p0[4], acc[4];
        {
            const double2 a = *reinterpret_cast<const double2*>(nb[e0] + ha);
            const double2 b = *reinterpret_cast<const double2*>(nb[e0] + hb);
            p0[0] = mul_rn(v[e0], a.x); p0[1] = mul_rn(v[e0], a.y);
            p0[2] = mul_rn(v[e0], b.x); p0[3] = mul_rn(v[e0], b.y);
        }
        {
            const double2 a = *reinterpret_cast<const double2*>(nb[e0 + 1] + ha);
            const double2 b = *reinterpret_cast<const double2*>(nb[e0 + 1] + hb);
            acc[0] = mul_rn(v[e0 + 1], a.x); acc[1] = mul_rn(v[e0 + 1], a.y);
            acc[2] = mul_rn(v[e0 + 1], b.x); acc[3] = mul_rn(v[e0 + 1], b.y);
        }
#pragma unroll
        for (int e = e0 + 2; e <= e1; ++e) {
            const double2 a = *reinterpret_cast<const double2*>(nb[e] + ha);
            const double2 b = *reinterpret_cast<const double2*>(nb[e] + hb);
            acc[0] = add_rn(acc[0], mul_rn(v[e], a.x)); acc[1] = add_rn(acc[1], mul_rn(v[e], a.y));
            acc[2] = add_rn(acc[2], mul_rn(v[e], b.x)); acc[3] = add_rn(acc[3], mul_rn(v[e], b.y));
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) o[j] = add_rn(p0[j], acc[j]);
    } else {
        double p0[4] = {0.0, 0.0, 0.0, 0.0}, acc[4] = {0.0, 0.0, 0.0, 0.0};
        int seen = 0;
#pragma unroll
        for (int e = 0; e < 7; ++e) {
            if (!(mk & (1u << e))) continue;
            const double2 a = *reinterpret_cast<const double2*>(nb[e] + ha);
            const double2 b = *reinterpret_cast<const double2*>(nb[e] + hb);
            const double pr[4] = {mul_rn(v[e], a.x), mul_rn(v[e], a.y), mul_rn(v[e], b.x), mul_rn(v[e], b.y)};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if (seen == 0) p0[j] = pr[j];
                else if (seen == 1) acc[j] = pr[j];
                else acc[j] = add_rn(acc[j], pr[j]);
            }
            ++seen;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) o[j] = add_rn(p0[j], acc[j]);
    }
}

template <class P>
__global__ void __launch_bounds__(P::NT, P::MINB)
stencil_march_kernel(const __grid_constant__ CUtensorMap tmap, EkcgStencil s, UniformFaces uf,
                     double* __restrict__ Y, int ldy, int m, int w_begin, int w_end, int wchunk,
                     const int* __restrict__ live) {
    EKCG_GATE(live);
    constexpr int DIM = P::DIM, KC = P::KC, kNS = P::NS, kAhead = P::AHEAD;
    extern __shared__ __align__(128) double smem[];
    __shared__ __align__(8) unsigned long long bar[kNS];

    const int tid = threadIdx.x;
    const unsigned nx = s.nx, ny = s.ny;
    const unsigned tiles_x = (nx + P::TX - 1) / P::TX;
    const int x0 = (int)((blockIdx.x % tiles_x) * P::TX);
    const int y0 = (DIM == 3) ? (int)((blockIdx.x / tiles_x) * P::TY) : 0;
    const int c0 = blockIdx.y * KC;
    const int wb = w_begin + blockIdx.z * wchunk;
    const int we = min(w_end, wb + wchunk);
    if (wb >= we) return;
    const int nq = we - wb + 2;  // planes wb-1 .. we
    const unsigned nw = (DIM == 3) ? s.nz : ny;

    if (tid == 0) {
#pragma unroll
        for (int q = 0; q < kNS; ++q) mbar_init(&bar[q], 1);
        mbar_fence_init();
    }
    __syncthreads();
    auto issue = [&](int q) {
        const int slot = q % kNS;
        mbar_expect_tx(&bar[slot], (unsigned)(P::BOX * sizeof(double)));
        const int z = wb - 1 + q;
        if (DIM == 3) tma_load_4d(smem + slot * P::STAGE, &tmap, &bar[slot], c0, x0 - 1, y0 - 1, z);
        else tma_load_3d(smem + slot * P::STAGE, &tmap, &bar[slot], c0, x0 - 1, z);
    };
    if (tid == 0)
        for (int q = 0; q <= kAhead && q < nq; ++q) issue(q);

    // per-item node coordinates (fixed over the march)
    int ix[P::IPT], iy[P::IPT], ig[P::IPT];
    bool act[P::IPT];
#pragma unroll
    for (int it = 0; it < P::IPT; ++it) {
        const int item = tid + it * P::NT;
        const int nd = item / P::LANES;
        ig[it] = item % P::LANES;
        ix[it] = nd % P::TX;
        iy[it] = nd / P::TX;
        act[it] = (x0 + ix[it] < (int)nx) && (DIM == 2 || y0 + iy[it] < (int)ny) && (c0 + 4 * ig[it] + 4 <= m);
    }

    // Tile fields with the host-built tables (kself, hx, hy, hz): the march axis (y in 2-D, z in 3-D) is shared
    // by the whole CTA, so the tile layer and the position inside it are CTA-uniform -- a node's tile lookups
    // and its in-plane faces are redone only when the march enters a new tile layer (a uniform branch), and a
    // plane costs two selects for the march-axis faces and the diagonal's add chain instead of the full
    // stencil_coef (tile divisions, 64-bit index math, face bookkeeping: ~60 % of this kernel's instructions
    // were integer / control in ncu) or a 64-B table row per node.  Same IEEE operations in the same order as
    // stencil_coef, so the same bits.
    // (preferred over the per-node table when both are present: config 3 0.294 -> 0.246 ms; operators built
    // from a CSR matrix have only the table)
    const bool fastf = P::IPT == 1 && s.kfield != nullptr && s.kself != nullptr && s.hx != nullptr &&
                       s.hy != nullptr && (DIM == 2 || s.hz != nullptr);
    const int f_tw = (DIM == 3) ? s.tz : s.ty;           // tile edge along the march axis
    const int f_sw = (DIM == 3) ? s.fx * s.fy : s.fx;    // field stride of one tile layer
    int f_rw = 0, f_tc = 0;
    double f_kc = 0.0, f_fwin = 0.0, f_fxl = 0.0, f_fxh = 0.0, f_fyl = 0.0, f_fyh = 0.0;
    bool f_xlo = false, f_xhi = false, f_xlc = false, f_xhc = false;
    bool f_ylo = false, f_yhi = false, f_ylc = false, f_yhc = false;
    if (fastf) {
        const unsigned x = (unsigned)(x0 + ix[0]);
        const unsigned txi = tile_div(x, s.tx);
        const unsigned rx = x - txi * (unsigned)s.tx;
        f_xlo = x > 0;
        f_xhi = x + 1 < nx;
        f_xlc = rx == 0;
        f_xhc = rx + 1 == (unsigned)s.tx;
        unsigned tyi = 0;
        if (DIM == 3) {
            const unsigned y = (unsigned)(y0 + iy[0]);
            tyi = tile_div(y, s.ty);
            const unsigned ry = y - tyi * (unsigned)s.ty;
            f_ylo = y > 0;
            f_yhi = y + 1 < ny;
            f_ylc = ry == 0;
            f_yhc = ry + 1 == (unsigned)s.ty;
        }
        const unsigned twi = tile_div((unsigned)wb, f_tw);
        f_rw = wb - (int)(twi * (unsigned)f_tw);
        f_tc = (DIM == 3) ? ((int)twi * s.fy + (int)tyi) * s.fx + (int)txi : (int)twi * s.fx + (int)txi;
    }
    auto tile_layer = [&]() {  // the node's constants inside tile f_tc
        f_kc = __ldg(s.kfield + f_tc);
        const double ks = __ldg(s.kself + f_tc);
        f_fwin = mul_rn(DIM == 3 ? s.cz : s.cy, ks);
        const double fxin = mul_rn(s.cx, ks);
        f_fxl = f_xlo ? (f_xlc ? __ldg(s.hx + f_tc - 1) : fxin) : 0.0;
        f_fxh = f_xhi ? (f_xhc ? __ldg(s.hx + f_tc) : fxin) : 0.0;
        if (DIM == 3) {
            const double fyin = mul_rn(s.cy, ks);
            f_fyl = f_ylo ? (f_ylc ? __ldg(s.hy + f_tc - s.fx) : fyin) : 0.0;
            f_fyh = f_yhi ? (f_yhc ? __ldg(s.hy + f_tc) : fyin) : 0.0;
        }
    };
    if (fastf && act[0]) tile_layer();

    for (int w = wb; w < we; ++w) {
        const int q = w - wb + 1;
        // one thread observes the TMA completions; the CTA barrier then both
        // publishes plane q+1 and retires every read of step q-1, so the
        // stage of plane q+AHEAD-NS (<= q-2) can be refilled
        if (tid == 0) {
            if (w == wb) {
                mbar_wait(&bar[(q - 1) % kNS], ((q - 1) / kNS) & 1);
                mbar_wait(&bar[q % kNS], (q / kNS) & 1);
            }
            mbar_wait(&bar[(q + 1) % kNS], ((q + 1) / kNS) & 1);
        }
        __syncthreads();
        if (tid == 0 && q + kAhead < nq) {
            fence_proxy_async_smem();  // the CTA's generic reads of the stage (ordered by the barrier) before the refill
            issue(q + kAhead);
        }
        const double* pm = smem + ((q - 1) % kNS) * P::STAGE;
        const double* pc = smem + (q % kNS) * P::STAGE;
        const double* pp = smem + ((q + 1) % kNS) * P::STAGE;
#pragma unroll
        for (int it = 0; it < P::IPT; ++it) {
            if (!act[it]) continue;
            const unsigned x = x0 + ix[it], y = y0 + iy[it];
            double o[4];
            int ha, hb;
            if (fastf) {
                // march-axis faces: the tile-interior value, or the host-built cross-tile face on the layer's edges
                const double* __restrict__ hw = (DIM == 3) ? s.hz : s.hy;
                const double cw = (DIM == 3) ? s.cz : s.cy;
                const bool wlo = w > 0, whi = (unsigned)w + 1 < nw;
                const double fwh = whi ? (f_rw + 1 == f_tw ? __ldg(hw + f_tc) : f_fwin) : 0.0;
                const double fwl = wlo ? (f_rw == 0 ? __ldg(hw + f_tc - f_sw) : f_fwin) : 0.0;
                double diag = 0.0;  // the add order of stencil_coef: slowest axis first; +hi, +lo, +first, +last
                if (whi) diag = add_rn(diag, fwh);
                if (wlo) diag = add_rn(diag, fwl);
                if (!wlo) diag = add_rn(diag, mul_rn(cw, f_kc));
                if (!whi) diag = add_rn(diag, mul_rn(cw, f_kc));
                if (DIM == 3) {
                    if (f_yhi) diag = add_rn(diag, f_fyh);
                    if (f_ylo) diag = add_rn(diag, f_fyl);
                    if (!f_ylo) diag = add_rn(diag, mul_rn(s.cy, f_kc));
                    if (!f_yhi) diag = add_rn(diag, mul_rn(s.cy, f_kc));
                }
                if (f_xhi) diag = add_rn(diag, f_fxh);
                if (f_xlo) diag = add_rn(diag, f_fxl);
                if (!f_xlo) diag = add_rn(diag, mul_rn(s.cx, f_kc));
                if (!f_xhi) diag = add_rn(diag, mul_rn(s.cx, f_kc));
                double v[7];
                unsigned mk = (1u << 3) | (f_xlo ? 1u << 2 : 0u) | (f_xhi ? 1u << 4 : 0u);
                if (DIM == 3) {
                    v[0] = -fwl; v[1] = -f_fyl; v[2] = -f_fxl; v[3] = diag; v[4] = -f_fxh; v[5] = -f_fyh; v[6] = -fwh;
                    mk |= (wlo ? 1u : 0u) | (f_ylo ? 1u << 1 : 0u) | (f_yhi ? 1u << 5 : 0u) | (whi ? 1u << 6 : 0u);
                } else {
                    v[0] = 0.0; v[1] = -fwl; v[2] = -f_fxl; v[3] = diag; v[4] = -f_fxh; v[5] = -fwh; v[6] = 0.0;
                    mk |= (wlo ? 1u << 1 : 0u) | (whi ? 1u << 5 : 0u);
                }
                march_apply<P>(v, mk, mk == ((DIM == 3) ? 0x7fu : 0x3eu), pm, pc, pp, ix[it], iy[it], ig[it], o, ha, hb);
            } else {
                march_node<P>(s, uf, pm, pc, pp, x0, y0, ix[it], iy[it], ig[it], w, nx, ny, nw, o, ha, hb);
            }
            const long long row = (DIM == 3) ? ((long long)w * ny + y) * nx + x : (long long)w * nx + x;
            double* yr = Y + row * ldy + c0 + 4 * ig[it];
            *reinterpret_cast<double2*>(yr + ha) = make_double2(o[0], o[1]);
            *reinterpret_cast<double2*>(yr + hb) = make_double2(o[2], o[3]);
        }
        if (fastf && ++f_rw == f_tw) {  // the next plane starts a new tile layer (CTA-uniform)
            f_rw = 0;
            f_tc += f_sw;
            if (w + 1 < we && act[0]) tile_layer();
        }
    }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
        else
            cudaGetLastError();
    }
    return fn;
}

template <class P>
bool make_plane_map(const EkcgStencil& s, const double* X, int ldx, int m, CUtensorMap& map) {
    constexpr int DIM = P::DIM, KC = P::KC;
    auto encode = encode_fn();
    if (encode == nullptr) return false;
    cuuint64_t dims[4], strides[3];
    cuuint32_t box[4], estr[4] = {1, 1, 1, 1};
    dims[0] = (cuuint64_t)m;
    dims[1] = (cuuint64_t)s.nx;
    strides[0] = (cuuint64_t)ldx * sizeof(double);
    box[0] = KC;
    box[1] = P::PX;
    if (DIM == 3) {
        dims[2] = (cuuint64_t)s.ny;
        dims[3] = (cuuint64_t)s.nz;
        strides[1] = strides[0] * s.nx;
        strides[2] = strides[1] * s.ny;
        box[2] = P::PY;
        box[3] = 1;
    } else {
        dims[2] = (cuuint64_t)s.ny;
        strides[1] = strides[0] * s.nx;
        box[2] = 1;
    }
    return encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, DIM + 1, const_cast<double*>(X), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <class P>
int launch_march(const EkcgStencil& s, const UniformFaces& uf, const double* X, int ldx, double* Y, int ldy, int m,
                 int wb, int we, const int* live, cudaStream_t st) {
    constexpr int DIM = P::DIM, KC = P::KC;
    CUtensorMap map;
    if (!make_plane_map<P>(s, X, ldx, m, map)) return EKCG_EINVAL;

    static int cache[kEkcgMaxDevices];
    const int occ = kernel_occupancy(stencil_march_kernel<P>, P::NT, P::SMEM, cache);
    if (occ < 1) return EKCG_EINVAL;
    const long long resident = (long long)occ * device_sms();
    const long long tiles = (DIM == 3) ? (long long)((s.nx + P::TX - 1) / P::TX) * ((s.ny + P::TY - 1) / P::TY)
                                       : (long long)((s.nx + P::TX - 1) / P::TX);
    const int colchunks = (m + KC - 1) / KC;
    const long long per_chunk = tiles * colchunks;
    // Split the march axis into w chunks so that the grid fills whole waves of the resident slots:
    // the launch takes about waves(w) x (planes per CTA + the 2 halo planes each chunk re-reads), so a
    // grid of 2.6 waves (what "two waves, rounded up" gave configs 3 and 5) idles 14 % of the slot-time
    // in its last wave.  Marches of at least 8 planes; ties go to the finer split.
    const int planes = we - wb;
    long long wmax = planes / 8;
    if (wmax < 1) wmax = 1;
    if (wmax > 64) wmax = 64;
    long long wchunks = 1, best_cost = -1;
    for (long long w = 1; w <= wmax; ++w) {
        const long long per_cta = (planes + w - 1) / w;
        const long long ctas = per_chunk * ((planes + per_cta - 1) / per_cta);
        const long long waves = (ctas + resident - 1) / resident;
        const long long cost = waves * (per_cta + 2);
        if (best_cost < 0 || cost <= best_cost) {
            best_cost = cost;
            wchunks = w;
        }
    }
    const int wchunk = (int)((planes + wchunks - 1) / wchunks);
    dim3 grid((unsigned)tiles, colchunks, (planes + wchunk - 1) / wchunk);
    launch_k(stencil_march_kernel<P>, grid, P::NT, P::SMEM, st, map, s, uf, Y, ldy, m, wb, we, wchunk, live);
    return EKCG_OK;
}

// ---------------------------------------------------------------------------
// Fused plane-marching kernels for 16-column blocks (one column chunk), a
// persistent grid walking (tile, plane-chunk) work items:
//   EPI_GRAM: G = X^T (A X) -- A X goes to a shared tile, never to HBM; the
//             DMMA consumes X from the staged plane and A X from the tile --
//             then the last CTA sums the CTA partials (fixed order) and
//             factors G (A-CholQR: S = chol(sym G)^-1), or stores G.
//   EPI_XR:   Y = A X written; x += X alpha, r -= Y alpha, |r|^2 partials;
//             the last CTA finishes the iteration (or stores |r|^2).
// ---------------------------------------------------------------------------
constexpr int EPI_GRAM = 1, EPI_XR = 2;
constexpr int kRedGroup = 16;  // CTAs per first-level group of the in-kernel Gram reduction

struct FusedArgs {
    double* partials;
    unsigned int* counter;
    EkcgCtrl* ctrl;
    int iteration;
    double tol;
    int finalize;
    double* out;  // S (finalize) or G
    // xr
    double* Y;
    int ldy;
    const double* alpha;
    double* x;
    double* r;
    int k, kmax, stag;
    double* history;
    int do_finish;
    double* rho2_out;
};

template <class P, int EPI>
__global__ void __launch_bounds__(P::NT, 2)
stencil_march_fused_kernel(const __grid_constant__ CUtensorMap tmap, EkcgStencil s, UniformFaces uf, int w_begin,
                           int w_end, int wchunk, int items, FusedArgs fa) {
    pdl_wait();
    if (fa.ctrl->live == 0) return;
    constexpr int DIM = P::DIM, KC = P::KC, kNS = P::NS, kAhead = P::AHEAD, NODES = P::TX * P::TY;
    static_assert(KC == 16 && P::IPT == 1 && P::NT == 256 && NODES == 64, "16 columns, 64-node tiles");
    extern __shared__ __align__(128) double smem[];
    __shared__ __align__(8) unsigned long long bar[kNS];
    __shared__ __align__(16) double sa[16];
    double* tileY = smem + kNS * P::STAGE;  // [NODES][16] A X of the current plane (EPI_GRAM)

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned nx = s.nx, ny = s.ny;
    const unsigned nw = (DIM == 3) ? s.nz : ny;
    const unsigned tiles_x = (nx + P::TX - 1) / P::TX;
    const int planes = w_end - w_begin;
    const int wchunks = (planes + wchunk - 1) / wchunk;
    if (tid == 0) {
#pragma unroll
        for (int q = 0; q < kNS; ++q) mbar_init(&bar[q], 1);
        mbar_fence_init();
    }
    if (EPI == EPI_XR && tid < 16) sa[tid] = fa.alpha[tid];
    __syncthreads();

    const int nd = tid >> 2, ig = tid & 3;
    const int ix = nd % P::TX, iy = nd / P::TX;
    const int lr = lane & 3, lc = lane >> 2;
    double gacc[2][2][2] = {{{0.0, 0.0}, {0.0, 0.0}}, {{0.0, 0.0}, {0.0, 0.0}}};
    double sq = 0.0;
    long long qg = 0;  // planes issued by this CTA so far (ring position and mbarrier phase)

    for (int item = blockIdx.x; item < items; item += gridDim.x) {
        const int tile = item / wchunks, wc = item % wchunks;
        const int x0 = (int)((tile % tiles_x) * P::TX);
        const int y0 = (DIM == 3) ? (int)((tile / tiles_x) * P::TY) : 0;
        const int wb = w_begin + wc * wchunk;
        const int we = min(w_end, wb + wchunk);
        const int nq = we - wb + 2;
        __syncthreads();  // the previous item's reads are done before its stages are refilled
        auto issue = [&](int q) {
            const long long g = qg + q;
            const int slot = (int)(g % kNS);
            mbar_expect_tx(&bar[slot], (unsigned)(P::BOX * sizeof(double)));
            const int z = wb - 1 + q;
            if (DIM == 3) tma_load_4d(smem + slot * P::STAGE, &tmap, &bar[slot], 0, x0 - 1, y0 - 1, z);
            else tma_load_3d(smem + slot * P::STAGE, &tmap, &bar[slot], 0, x0 - 1, z);
        };
        if (tid == 0) {
            fence_proxy_async_smem();  // the previous item's generic reads of the stages before the refills
            for (int q = 0; q <= kAhead && q < nq; ++q) issue(q);
        }
        const bool act = (x0 + ix < (int)nx) && (DIM == 2 || y0 + iy < (int)ny);
        for (int w = wb; w < we; ++w) {
            const int q = w - wb + 1;
            if (tid == 0) {
                if (w == wb) {
                    mbar_wait(&bar[(qg + q - 1) % kNS], (unsigned)(((qg + q - 1) / kNS) & 1));
                    mbar_wait(&bar[(qg + q) % kNS], (unsigned)(((qg + q) / kNS) & 1));
                }
                mbar_wait(&bar[(qg + q + 1) % kNS], (unsigned)(((qg + q + 1) / kNS) & 1));
            }
            __syncthreads();
            if (tid == 0 && q + kAhead < nq) {
                fence_proxy_async_smem();  // the CTA's generic reads of the stage (ordered by the barrier) before the refill
                issue(q + kAhead);
            }
            const double* pm = smem + ((qg + q - 1) % kNS) * P::STAGE;
            const double* pc = smem + ((qg + q) % kNS) * P::STAGE;
            const double* pp = smem + ((qg + q + 1) % kNS) * P::STAGE;
            double o[4] = {0.0, 0.0, 0.0, 0.0};
            int ha = 0, hb = 0;
            if (act) march_node<P>(s, uf, pm, pc, pp, x0, y0, ix, iy, ig, w, nx, ny, nw, o, ha, hb);
            else {
                const int sw = (ix & 1) ? 8 : 0;
                ha = (2 * ig + sw) % KC - 4 * ig;
                hb = (2 * ig + KC / 2 + sw) % KC - 4 * ig;
            }
            if (EPI == EPI_GRAM) {
                double* ty = tileY + nd * KC + 4 * ig;
                *reinterpret_cast<double2*>(ty + ha) = make_double2(o[0], o[1]);
                *reinterpret_cast<double2*>(ty + hb) = make_double2(o[2], o[3]);
                __syncwarp();
                // G += X^T (A X) over the warp's own 8 nodes (two k-steps, no CTA barrier:
                // warp w wrote tileY rows 8w..8w+7); lane (i, k) reads columns 2i, 2i+1 of
                // node k (interleaved tiles t: column 2i + t)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int node = 8 * warp + 4 * h + lr;
                    const int hx = node % P::TX, hy = node / P::TX;
                    const double2 a = *reinterpret_cast<const double2*>(
                        pc + ((hy + P::OY) * P::PX + hx + 1) * KC + 2 * lc);
                    const double2 b = *reinterpret_cast<const double2*>(tileY + node * KC + 2 * lc);
                    dmma_8x8x4(gacc[0][0], a.x, b.x);
                    dmma_8x8x4(gacc[0][1], a.x, b.y);
                    dmma_8x8x4(gacc[1][0], a.y, b.x);
                    dmma_8x8x4(gacc[1][1], a.y, b.y);
                }
            } else {
                // every lane takes part in the shuffles; inactive nodes contribute zeros
                const unsigned x = x0 + ix, y = y0 + iy;
                const long long row = (DIM == 3) ? ((long long)w * ny + y) * nx + x : (long long)w * nx + x;
                double xv = 0.0, rv = 0.0, dx = 0.0, dr = 0.0;
                if (act) {
                    if (ig == 0) {
                        xv = fa.x[row];
                        rv = fa.r[row];
                    }
                    double* yr = fa.Y + row * fa.ldy + 4 * ig;
                    *reinterpret_cast<double2*>(yr + ha) = make_double2(o[0], o[1]);
                    *reinterpret_cast<double2*>(yr + hb) = make_double2(o[2], o[3]);
                    const double* xc = pc + ((iy + P::OY) * P::PX + ix + 1) * KC + 4 * ig;
                    const double2 w0 = *reinterpret_cast<const double2*>(xc + ha);
                    const double2 w1 = *reinterpret_cast<const double2*>(xc + hb);
                    const int ca = 4 * ig + ha, cb = 4 * ig + hb;
                    dx = w0.x * sa[ca] + w0.y * sa[ca + 1] + w1.x * sa[cb] + w1.y * sa[cb + 1];
                    dr = o[0] * sa[ca] + o[1] * sa[ca + 1] + o[2] * sa[cb] + o[3] * sa[cb + 1];
                }
                dx += __shfl_xor_sync(0xffffffffu, dx, 1);
                dr += __shfl_xor_sync(0xffffffffu, dr, 1);
                dx += __shfl_xor_sync(0xffffffffu, dx, 2);
                dr += __shfl_xor_sync(0xffffffffu, dr, 2);
                if (act && ig == 0) {
                    fa.x[row] = xv + dx;
                    const double rn = rv - dr;
                    fa.r[row] = rn;
                    sq += rn * rn;
                }
            }
        }
        qg += nq;
    }

    // CTA partial, fixed order, then the last CTA's epilogue
    __syncthreads();
    if (EPI == EPI_GRAM) {
        double* red = smem;  // [8 warps][256]
#pragma unroll
        for (int ta = 0; ta < 2; ++ta)
#pragma unroll
            for (int tb = 0; tb < 2; ++tb)
#pragma unroll
                for (int e = 0; e < 2; ++e)
                    red[warp * 256 + (2 * lc + ta) * 16 + 2 * (2 * lr + e) + tb] = gacc[ta][tb][e];
        __syncthreads();
        {
            double v = red[tid];
#pragma unroll
            for (int w = 1; w < 8; ++w) v += red[w * 256 + tid];
            fa.partials[(long long)blockIdx.x * 256 + tid] = v;
        }
        // two-level fixed-order reduction: the last CTA of each group of kRedGroup
        // consecutive CTAs sums the group's partials (one round of loads), the
        // last group to finish sums the group sums -- instead of one CTA reading
        // every partial (counter[1 + g]: group g, counter[0]: groups done)
        const int ngroups = (int)((gridDim.x + kRedGroup - 1) / kRedGroup);
        const int g = (int)(blockIdx.x / kRedGroup);
        const int p0 = g * kRedGroup, p1 = min((int)gridDim.x, p0 + kRedGroup);
        if (last_arrive(fa.counter + 1 + g, (unsigned)(p1 - p0))) {
            double v = __ldcg(fa.partials + (long long)p0 * 256 + tid);
            for (int p = p0 + 1; p < p1; ++p) v += __ldcg(fa.partials + (long long)p * 256 + tid);
            fa.partials[((long long)gridDim.x + g) * 256 + tid] = v;
            if (last_arrive(fa.counter, (unsigned)ngroups)) {
                double* Gm = smem + 8 * 256;
                cta_sum_partials_mlp(fa.partials + (long long)gridDim.x * 256, ngroups, 256, Gm);
                if (fa.finalize) cholinv_body(Gm, Gm + 256, Gm + 512, 16, fa.out, fa.ctrl, fa.iteration, fa.tol);
                else
                    for (int e = tid; e < 256; e += 256) fa.out[e] = Gm[e];
            }
        }
    } else {
        __shared__ double wsum[8];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
        if (lane == 0) wsum[warp] = sq;
        __syncthreads();
        if (tid == 0) {
            double t = wsum[0];
            for (int w = 1; w < 8; ++w) t += wsum[w];
            fa.partials[blockIdx.x] = t;
        }
        if (last_cta_arrive(fa.counter)) {
            __shared__ double tot;
            if (tid < 32) {
                double acc = 0.0;
                for (int p = tid; p < (int)gridDim.x; p += 32) acc += __ldcg(fa.partials + p);
                for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
                if (tid == 0) tot = acc;
            }
            __syncthreads();
            if (tid == 0) {
                if (fa.do_finish) finish_body(fa.ctrl, tot, fa.k, fa.kmax, fa.stag, fa.history);
                else *fa.rho2_out = tot;
            }
        }
    }
}

template <class P, int EPI>
int launch_march_fused(const EkcgStencil& s, const UniformFaces& uf, const double* X, int max_ctas,
                       const FusedArgs& fa, cudaStream_t st, int items_per_cta = 1, int min_planes = 4) {
    constexpr int DIM = P::DIM;
    const long long plane = (DIM == 3) ? (long long)s.nx * s.ny : (long long)s.nx;
    if (s.row_begin % plane != 0 || s.row_end % plane != 0) return EKCG_EINVAL;
    const int wb = (int)(s.row_begin / plane), we = (int)(s.row_end / plane);
    CUtensorMap map;
    if (!make_plane_map<P>(s, X, 16, 16, map)) return EKCG_EINVAL;
    constexpr size_t smem = P::SMEM + sizeof(double) * 64 * 16;
    static_assert(P::SMEM >= sizeof(double) * 11 * 256, "reduction scratch fits the stages");
    static int cache[kEkcgMaxDevices];
    const int occ = kernel_occupancy(stencil_march_fused_kernel<P, EPI>, P::NT, smem, cache);
    if (occ < 1) return EKCG_EINVAL;
    const long long resident = (long long)occ * device_sms();
    const long long tiles = (DIM == 3) ? (long long)((s.nx + P::TX - 1) / P::TX) * ((s.ny + P::TY - 1) / P::TY)
                                       : (long long)((s.nx + P::TX - 1) / P::TX);
    int grid = resident < max_ctas ? resident : max_ctas;
    // plane chunks: about items_per_cta work items per resident CTA, marches of >= min_planes planes
    const int planes = we - wb;
    long long wchunks = ((long long)grid * items_per_cta + tiles - 1) / tiles;
    if (wchunks > planes / min_planes) wchunks = planes / min_planes;
    if (wchunks < 1) wchunks = 1;
    const int wchunk = (int)((planes + wchunks - 1) / wchunks);
    wchunks = (planes + wchunk - 1) / wchunk;
    const long long items = tiles * wchunks;
    if (items < grid) grid = (int)items;
    launch_k(stencil_march_fused_kernel<P, EPI>, grid, P::NT, smem, st, map, s, uf, wb, we, wchunk, (int)items, fa);
    return EKCG_OK;
}

}  // namespace

// Launch the plane-marching kernel when it applies (m % 4 == 0, 16-byte
// aligned rows, whole planes in the row range); EKCG_EINVAL otherwise, and
// the caller takes the row-parallel kernel.
int launch_stencil_march(const EkcgStencil& s, const UniformFaces& uf, const double* X, int ldx, double* Y, int ldy,
                         int m, const int* live, cudaStream_t st, long long min_work) {
    if (m % 4 != 0 || ldx % 2 != 0 || ldy % 2 != 0 || (reinterpret_cast<uintptr_t>(X) & 15) ||
        (reinterpret_cast<uintptr_t>(Y) & 15))
        return EKCG_EINVAL;
    const long long plane = (s.dim == 3) ? (long long)s.nx * s.ny : (long long)s.nx;
    if (s.row_begin % plane != 0 || s.row_end % plane != 0) return EKCG_EINVAL;
    // small grids: the march is latency-bound (a few CTAs, serial plane steps);
    // the row-parallel kernel finishes sooner
    if ((s.row_end - s.row_begin) * (long long)m < min_work) return EKCG_EINVAL;
    const int wb = (int)(s.row_begin / plane), we = (int)(s.row_end / plane);
    const int kc = (m % 16 == 0) ? 16 : (m % 8 == 0) ? 8 : 4;
    if (s.dim == 3) {
        if (kc == 16) return launch_march<March<3, 16, 16, 4, 4>>(s, uf, X, ldx, Y, ldy, m, wb, we, live, st);
        if (kc == 8) return launch_march<March<3, 8, 16, 8, 6>>(s, uf, X, ldx, Y, ldy, m, wb, we, live, st);
        return launch_march<March<3, 4, 16, 16, 6>>(s, uf, X, ldx, Y, ldy, m, wb, we, live, st);
    }
    if (kc == 16) return launch_march<March<2, 16, 64, 1, 6>>(s, uf, X, ldx, Y, ldy, m, wb, we, live, st);
    if (kc == 8) return launch_march<March<2, 8, 128, 1, 6>>(s, uf, X, ldx, Y, ldy, m, wb, we, live, st);
    return launch_march<March<2, 4, 128, 1, 6>>(s, uf, X, ldx, Y, ldy, m, wb, we, live, st);
}

// Fused plane-marching kernels for m = 16 (EKCG_EINVAL when they do not apply:
// the caller takes the row-parallel fused kernels).  Gram partials reduced in
// groups of 3 CTAs, 2 levels (tools/kernel_times.py --fused).

int launch_march_cholinv(const EkcgStencil& s, const UniformFaces& uf, const double* X, int ldx, int m,
                         double* partials, unsigned int* counter, double* S, EkcgCtrl* ctrl, int iteration, double tol,
                         int finalize, int max_ctas, cudaStream_t st) {
    if (m != 16 || ldx != 16 || (reinterpret_cast<uintptr_t>(X) & 15) ||
        (s.row_end - s.row_begin) * 16 < kMarchMinWork)
        return EKCG_EINVAL;
    FusedArgs fa{};
    fa.partials = partials;
    fa.counter = counter;
    fa.ctrl = ctrl;
    fa.iteration = iteration;
    fa.tol = tol;
    fa.finalize = finalize;
    fa.out = S;
    if (s.dim == 3) return launch_march_fused<March<3, 16, 16, 4, 4>, EPI_GRAM>(s, uf, X, max_ctas, fa, st, 3, 2);
    return launch_march_fused<March<2, 16, 64, 1, 4>, EPI_GRAM>(s, uf, X, max_ctas, fa, st);
}

int launch_march_xr(const EkcgStencil& s, const UniformFaces& uf, const double* X, int ldx, double* Y, int ldy, int m,
                    const double* alpha, double* x, double* r, double* partials, unsigned int* counter, EkcgCtrl* ctrl,
                    int k, int kmax, int stag, double* history, int do_finish, double* rho2_out, int max_ctas,
                    cudaStream_t st) {
    if (m != 16 || ldx != 16 || ldy % 2 != 0 || (reinterpret_cast<uintptr_t>(X) & 15) ||
        (reinterpret_cast<uintptr_t>(Y) & 15) || (s.row_end - s.row_begin) * 16 < kMarchMinWork)
        return EKCG_EINVAL;
    FusedArgs fa{};
    fa.partials = partials;
    fa.counter = counter;
    fa.ctrl = ctrl;
    fa.Y = Y;
    fa.ldy = ldy;
    fa.alpha = alpha;
    fa.x = x;
    fa.r = r;
    fa.k = k;
    fa.kmax = kmax;
    fa.stag = stag;
    fa.history = history;
    fa.do_finish = do_finish;
    fa.rho2_out = rho2_out;
    if (s.dim == 3) return launch_march_fused<March<3, 16, 16, 4, 4>, EPI_XR>(s, uf, X, max_ctas, fa, st, 3, 2);
    return launch_march_fused<March<2, 16, 64, 1, 4>, EPI_XR>(s, uf, X, max_ctas, fa, st);
}
