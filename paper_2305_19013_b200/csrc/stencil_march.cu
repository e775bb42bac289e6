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

namespace {

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
        if (tid == 0 && q + kAhead < nq) issue(q + kAhead);
        const double* pm = smem + ((q - 1) % kNS) * P::STAGE;
        const double* pc = smem + (q % kNS) * P::STAGE;
        const double* pp = smem + ((q + 1) % kNS) * P::STAGE;
#pragma unroll
        for (int it = 0; it < P::IPT; ++it) {
            if (!act[it]) continue;
            const unsigned x = x0 + ix[it], y = y0 + iy[it];
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
            const int hc = ((iy[it] + P::OY) * P::PX + ix[it] + 1) * KC + 4 * ig[it];
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
            const int sw = (KC == 16) ? ((ix[it] & 1) ? 8 : 0) : 0;
            const int ha = (2 * ig[it] + sw) % KC - 4 * ig[it];
            const int hb = (2 * ig[it] + KC / 2 + sw) % KC - 4 * ig[it];
            double o[4];
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
            const long long row = (DIM == 3) ? ((long long)w * ny + y) * nx + x : (long long)w * nx + x;
            double* yr = Y + row * ldy + c0 + 4 * ig[it];
            *reinterpret_cast<double2*>(yr + ha) = make_double2(o[0], o[1]);
            *reinterpret_cast<double2*>(yr + hb) = make_double2(o[2], o[3]);
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
int launch_march(const EkcgStencil& s, const UniformFaces& uf, const double* X, int ldx, double* Y, int ldy, int m,
                 int wb, int we, const int* live, cudaStream_t st) {
    constexpr int DIM = P::DIM, KC = P::KC;
    auto encode = encode_fn();
    if (encode == nullptr) return EKCG_EINVAL;
    CUtensorMap map;
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
    CUresult r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, DIM + 1, const_cast<double*>(X), dims, strides, box,
                        estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return EKCG_EINVAL;

    static int resident = 0;
    if (resident == 0) {
        cudaFuncSetAttribute(stencil_march_kernel<P>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)P::SMEM);
        int occ = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, stencil_march_kernel<P>, P::NT, P::SMEM) !=
                cudaSuccess || occ < 1) {
            cudaGetLastError();
            occ = 1;
        }
        int dev = 0, sms = 148;
        if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        resident = occ * sms;
    }
    const long long tiles = (DIM == 3) ? (long long)((s.nx + P::TX - 1) / P::TX) * ((s.ny + P::TY - 1) / P::TY)
                                       : (long long)((s.nx + P::TX - 1) / P::TX);
    const int colchunks = (m + KC - 1) / KC;
    const long long per_chunk = tiles * colchunks;
    // enough CTAs for two waves of the resident slots; a march of at least 8 planes
    long long wchunks = (2LL * resident + per_chunk - 1) / per_chunk;
    const int planes = we - wb;
    if (wchunks > planes / 8) wchunks = planes / 8;
    if (wchunks < 1) wchunks = 1;
    const int wchunk = (int)((planes + wchunks - 1) / wchunks);
    dim3 grid((unsigned)tiles, colchunks, (planes + wchunk - 1) / wchunk);
    stencil_march_kernel<P><<<grid, P::NT, P::SMEM, st>>>(map, s, uf, Y, ldy, m, wb, we, wchunk, live);
    return EKCG_OK;
}

}  // namespace

// Launch the plane-marching kernel when it applies (m % 4 == 0, 16-byte
// aligned rows, whole planes in the row range); EKCG_EINVAL otherwise, and
// the caller takes the row-parallel kernel.
int launch_stencil_march(const EkcgStencil& s, const UniformFaces& uf, const double* X, int ldx, double* Y, int ldy,
                         int m, const int* live, cudaStream_t st) {
    if (m % 4 != 0 || ldx % 2 != 0 || ldy % 2 != 0 || (reinterpret_cast<uintptr_t>(X) & 15) ||
        (reinterpret_cast<uintptr_t>(Y) & 15))
        return EKCG_EINVAL;
    const long long plane = (s.dim == 3) ? (long long)s.nx * s.ny : (long long)s.nx;
    if (s.row_begin % plane != 0 || s.row_end % plane != 0) return EKCG_EINVAL;
    const int wb = (int)(s.row_begin / plane), we = (int)(s.row_end / plane);
    const int kc = (m % 16 == 0) ? 16 : (m % 8 == 0) ? 8 : 4;
    if (s.dim == 3) {
        if (kc == 16) {
            switch (g_march_variant) {
                case 1: return launch_march<March<3, 16, 16, 8, 6>>(s, uf, X, ldx, Y, ldy, m, wb, we, live, st);
                case 2: return launch_march<March<3, 16, 16, 4, 8>>(s, uf, X, ldx, Y, ldy, m, wb, we, live, st);
                case 3: return launch_march<March<3, 16, 32, 4, 6>>(s, uf, X, ldx, Y, ldy, m, wb, we, live, st);
                case 4: return launch_march<March<3, 16, 16, 4, 6>>(s, uf, X, ldx, Y, ldy, m, wb, we, live, st);
                case 5: return launch_march<March<3, 16, 16, 4, 4>>(s, uf, X, ldx, Y, ldy, m, wb, we, live, st);
                case 6: return launch_march<March<3, 16, 32, 8, 4>>(s, uf, X, ldx, Y, ldy, m, wb, we, live, st);
                default: return launch_march<March<3, 16, 16, 8, 4>>(s, uf, X, ldx, Y, ldy, m, wb, we, live, st);
            }
        }
        if (kc == 8) return launch_march<March<3, 8, 16, 8, 6>>(s, uf, X, ldx, Y, ldy, m, wb, we, live, st);
        return launch_march<March<3, 4, 16, 16, 6>>(s, uf, X, ldx, Y, ldy, m, wb, we, live, st);
    }
    if (kc == 16) return launch_march<March<2, 16, 64, 1, 6>>(s, uf, X, ldx, Y, ldy, m, wb, we, live, st);
    if (kc == 8) return launch_march<March<2, 8, 128, 1, 6>>(s, uf, X, ldx, Y, ldy, m, wb, we, live, st);
    return launch_march<March<2, 4, 128, 1, 6>>(s, uf, X, ldx, Y, ldy, m, wb, we, live, st);
}
