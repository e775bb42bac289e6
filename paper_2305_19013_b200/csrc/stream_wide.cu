// Streamed DMMA kernels for wide blocks (m = 32 Gram, m = 32 / 64 update).
//
// Same producer/consumer scheme as the 16-column kernels (stream.cu): one
// producer warp moves contiguous row slabs of the row-major blocks into an
// NS-slot shared-memory ring with 1-D bulk copies (TMA engine, mbarrier
// completion) and four consumer warps run the fp64 DMMA m8n8k4 on fragments
// read from shared memory, so the loads in flight are bounded by the ring,
// not by registers.  At m >= 32 the CGS2 products are FP64-bound (m/4 flop
// per byte vs a machine balance of ~5.7), so these kernels are judged by the
// DMMA pipe, not by HBM: the ring keeps the tensor pipe fed instead of
// stalling on global loads (tools/kernel_times.py).
//
//   gram_wide_stream_kernel   C_i = X_i^T Y over a row chunk, GB blocks per
//                             CTA sharing each Y slab (split-K partials,
//                             reduced in fixed order by ekcg_reduce)
//   update_wide_stream_kernel Wout = beta Win + sign sum_i Q_i C_i with every
//                             C_i resident in shared memory (padded rows)
//
// No floating-point atomics: reruns are bit-identical.
#include "common.cuh"
#include "ekcg_b200.h"
#include "tma.cuh"

namespace {

// ---------------------------------------------------------------------------
// Gram: lane (i, k) of a consumer warp reads columns 16h + 2i, 16h + 2i + 1
// of slab row k (one 16-B load per h), which feed the interleaved 8-wide
// tiles 2h and 2h + 1 (tile t, element i = column 16 (t / 2) + 2 i + t % 2).
// Warp w takes the k-steps (4 rows) w, w + 4, ... of every slab and keeps the
// full M x M accumulator of each of its GB blocks; the four warps' sums are
// combined in fixed order at the end.
// ---------------------------------------------------------------------------
template <int M, int GB, int R, int NS>
struct GramWide {
    static constexpr int SLAB = R * M;
    static constexpr int STAGE = (GB + 1) * SLAB;
    static constexpr int RED = 4 * GB * M * M;
    static constexpr size_t SMEM = sizeof(double) * (STAGE * NS > RED ? STAGE * NS : RED);
    static_assert(R % 16 == 0, "4 warps x 4-row k-steps");
    static_assert(M % 16 == 0, "pairs of interleaved 8-wide tiles");
};

// ---------------------------------------------------------------------------
// W^T W for one 32-column block (the Pre-CholQR Gram, aortho.py:105) on the
// same ring: the block is streamed once and read as both operands, and only
// the 10 of 16 8 x 8 tiles on and above the diagonal are formed -- a tile
// below it is the transpose of its mirror (same products, same order, same
// bits), so each tile is stored twice.  Out of line, so the general kernel's
// registers and schedule stay as they are.
// ---------------------------------------------------------------------------
template <int R, int NS>
__device__ __noinline__ void gram32_self(const double* __restrict__ Y, long long r0, long long r1, int nsteps,
                                         double* sm, unsigned long long* full, unsigned long long* empty,
                                         double* __restrict__ out) {
    constexpr int M = 32, T = 4, H = 2, SLAB = R * M;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 4) {  // producer: one slab per stage
        if (lane == 0) {
            for (int j = 0; j < nsteps; ++j) {
                const int slot = j % NS;
                if (j >= NS) {
                    mbar_wait(&empty[slot], ((j / NS) - 1) & 1);
                    fence_proxy_async_smem();
                }
                const long long rb = r0 + (long long)j * R;
                const unsigned bytes = (unsigned)(min((long long)R, r1 - rb) * M * sizeof(double));
                mbar_expect_tx(&full[slot], bytes);
                bulk_load(sm + slot * SLAB, Y + rb * M, bytes, &full[slot]);
            }
        }
        return;
    }
    const int lr = lane & 3, lc = lane >> 2;
    double acc[T][T][2];
#pragma unroll
    for (int a = 0; a < T; ++a)
#pragma unroll
        for (int b = 0; b < T; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
    for (int j = 0; j < nsteps; ++j) {
        const int slot = j % NS;
        mbar_wait(&full[slot], (j / NS) & 1);
        const double* st = sm + slot * SLAB;
        const int rr = (int)min((long long)R, r1 - (r0 + (long long)j * R));
#pragma unroll
        for (int q = 0; q < R / 16; ++q) {
            const int row = (q * 4 + warp) * 4 + lr;
            const bool ok = row < rr;
            double f[T];
#pragma unroll
            for (int h = 0; h < H; ++h) {
                const double2 v = ok ? *reinterpret_cast<const double2*>(st + row * M + 16 * h + 2 * lc) : make_double2(0.0, 0.0);
                f[2 * h] = v.x;
                f[2 * h + 1] = v.y;
            }
#pragma unroll
            for (int a = 0; a < T; ++a)
#pragma unroll
                for (int b = a; b < T; ++b) dmma_8x8x4(acc[a][b], f[a], f[b]);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
    }
    // fixed-order reduction of the four consumer warps' accumulators (as in the general kernel)
    named_sync(1, 128);
    double* red = sm;
#pragma unroll
    for (int ta = 0; ta < T; ++ta)
#pragma unroll
        for (int tb = ta; tb < T; ++tb)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int a = 16 * (ta / 2) + 2 * lc + (ta % 2);
                const int b = 16 * (tb / 2) + 2 * (2 * lr + e) + (tb % 2);
                red[(warp * M + a) * M + b] = acc[ta][tb][e];
                if (tb > ta) red[(warp * M + b) * M + a] = acc[ta][tb][e];
            }
    named_sync(1, 128);
    for (int o = threadIdx.x; o < M * M; o += 128) {
        double v = red[o];
#pragma unroll
        for (int w = 1; w < 4; ++w) v += red[w * M * M + o];
        out[o] = v;
    }
}

template <int M, int GB, int R, int NS>
__global__ void __launch_bounds__(160)
gram_wide_stream_kernel(const double* const* __restrict__ Xs, int d, const double* __restrict__ Y, long long n,
                        long long rows_chunk, double* __restrict__ partials, const int* __restrict__ live) {
    EKCG_GATE(live);
    using P = GramWide<M, GB, R, NS>;
    constexpr int T = M / 8, H = T / 2;
    extern __shared__ __align__(128) double sm[];
    __shared__ __align__(8) unsigned long long full[NS], empty[NS];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int i0 = blockIdx.y * GB;
    const int nb = min(GB, d - i0);
    const long long r0 = blockIdx.x * rows_chunk;
    const long long r1 = min(n, r0 + rows_chunk);
    const int nsteps = r1 > r0 ? (int)((r1 - r0 + R - 1) / R) : 0;
    if (threadIdx.x == 0) {
#pragma unroll
        for (int s = 0; s < NS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 4);
        }
        mbar_fence_init();
    }
    __syncthreads();

    if (M == 32 && GB == 1 && d == 1 && Xs[0] == Y) {  // W^T W: tiles on and above the diagonal, one stream
        gram32_self<R, NS>(Y, r0, r1, nsteps, sm, full, empty, partials + (long long)blockIdx.x * (M * M));
        return;
    }
    if (warp == 4) {  // producer
        if (lane == 0) {
            const double* X[GB];
#pragma unroll
            for (int g = 0; g < GB; ++g) X[g] = Xs[min(i0 + g, d - 1)];
            for (int j = 0; j < nsteps; ++j) {
                const int slot = j % NS;
                if (j >= NS) {
                    mbar_wait(&empty[slot], ((j / NS) - 1) & 1);
                    fence_proxy_async_smem();  // the consumers' generic reads of the slot before the TMA write
                }
                const long long rb = r0 + (long long)j * R;
                const unsigned bytes = (unsigned)(min((long long)R, r1 - rb) * M * sizeof(double));
                mbar_expect_tx(&full[slot], bytes * (unsigned)(nb + 1));
                double* st = sm + slot * P::STAGE;
                bulk_load(st, Y + rb * M, bytes, &full[slot]);
#pragma unroll
                for (int g = 0; g < GB; ++g)
                    if (g < nb) bulk_load(st + (g + 1) * P::SLAB, X[g] + rb * M, bytes, &full[slot]);
            }
        }
        return;
    }

    const int lr = lane & 3, lc = lane >> 2;
    double acc[GB][T][T][2];
#pragma unroll
    for (int g = 0; g < GB; ++g)
#pragma unroll
        for (int a = 0; a < T; ++a)
#pragma unroll
            for (int b = 0; b < T; ++b) acc[g][a][b][0] = acc[g][a][b][1] = 0.0;

    for (int j = 0; j < nsteps; ++j) {
        const int slot = j % NS;
        mbar_wait(&full[slot], (j / NS) & 1);
        const double* st = sm + slot * P::STAGE;
        const int rr = (int)min((long long)R, r1 - (r0 + (long long)j * R));
#pragma unroll
        for (int q = 0; q < R / 16; ++q) {
            const int row = (q * 4 + warp) * 4 + lr;
            const bool ok = row < rr;
            double2 b[H];
#pragma unroll
            for (int h = 0; h < H; ++h)
                b[h] = ok ? *reinterpret_cast<const double2*>(st + row * M + 16 * h + 2 * lc) : make_double2(0.0, 0.0);
#pragma unroll
            for (int g = 0; g < GB; ++g) {
                double2 a[H];
#pragma unroll
                for (int h = 0; h < H; ++h)
                    a[h] = (ok && g < nb)
                               ? *reinterpret_cast<const double2*>(st + (g + 1) * P::SLAB + row * M + 16 * h + 2 * lc)
                               : make_double2(0.0, 0.0);
#pragma unroll
                for (int ha = 0; ha < H; ++ha)
#pragma unroll
                    for (int hb = 0; hb < H; ++hb) {
                        dmma_8x8x4(acc[g][2 * ha][2 * hb], a[ha].x, b[hb].x);
                        dmma_8x8x4(acc[g][2 * ha][2 * hb + 1], a[ha].x, b[hb].y);
                        dmma_8x8x4(acc[g][2 * ha + 1][2 * hb], a[ha].y, b[hb].x);
                        dmma_8x8x4(acc[g][2 * ha + 1][2 * hb + 1], a[ha].y, b[hb].y);
                    }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
    }

    // fixed-order reduction of the four consumer warps' accumulators
    named_sync(1, 128);
    double* red = sm;
#pragma unroll
    for (int g = 0; g < GB; ++g)
#pragma unroll
        for (int ta = 0; ta < T; ++ta)
#pragma unroll
            for (int tb = 0; tb < T; ++tb)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int a = 16 * (ta / 2) + 2 * lc + (ta % 2);
                    const int b = 16 * (tb / 2) + 2 * (2 * lr + e) + (tb % 2);
                    red[((warp * GB + g) * M + a) * M + b] = acc[g][ta][tb][e];
                }
    named_sync(1, 128);
    for (int o = threadIdx.x; o < nb * M * M; o += 128) {
        const int g = o / (M * M), e = o % (M * M);
        double s = red[g * M * M + e];
#pragma unroll
        for (int w = 1; w < 4; ++w) s += red[(w * GB + g) * M * M + e];
        partials[((long long)blockIdx.x * d + i0 + g) * (M * M) + e] = s;
    }
}

// ---------------------------------------------------------------------------
// Update: the producer streams, per R-row slab (grid-stride over slabs),
// Q_0 .. Q_{d-1} row slabs through the ring; every C_i sits in shared memory
// for the whole launch (rows padded to M + 4 doubles: the four k-rows of a B
// fragment fall 8 banks apart).  Warp w owns slab rows 8 MR w .. 8 MR w +
// 8 MR - 1 (MR 8-row DMMA tiles).  A fragments come from the slab
// "diagonally": for each octet h of k-steps (32 columns), load j of lane
// (row i, k) reads column 32 h + 4 ((j + i) mod 8) + k, so the rows of a load
// hit distinct bank groups; k-step kk of the octet takes load (kk - i) mod 8
// (a three-level barrel rotation of registers).  Win is read and Wout
// written with 16-B accesses in the epilogue (in place allowed).
// ---------------------------------------------------------------------------
template <int M, int MR, int NS, int CW = 4>
struct UpdWide {
    static constexpr int R = 8 * CW * MR;  // CW consumer warps x MR 8-row tiles
    static constexpr int SLAB = R * M;
    static constexpr int LDC = M + 4;
    static size_t smem(int d) { return sizeof(double) * ((size_t)NS * SLAB + (size_t)d * M * LDC); }
    static_assert(M % 32 == 0, "octets of k-steps");
};

template <int M, int MR, int NS, int CW, bool INIT>
__global__ void __launch_bounds__(32 * (CW + 1))
update_wide_stream_kernel(const double* const* __restrict__ Qs, int d, const double* __restrict__ C, const double* Win,
                          int ldwi, double* Wout, int ldwo, double beta, double sign, long long n,
                          const int* __restrict__ live) {
    EKCG_GATE(live);
    using P = UpdWide<M, MR, NS, CW>;
    constexpr int R = P::R, NT = M / 8, LDC = P::LDC;
    extern __shared__ __align__(128) double sm[];
    __shared__ __align__(8) unsigned long long full[NS], empty[NS];
    double* cs = sm + NS * P::SLAB;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long slabs = (n + R - 1) / R;
    for (int e = threadIdx.x; e < d * M * M; e += blockDim.x) {  // INIT: sign * C, exact for sign = +-1
        const int i = e / (M * M), rem = e % (M * M);
        cs[(i * M + rem / M) * LDC + rem % M] = INIT ? sign * C[e] : C[e];
    }
    if (threadIdx.x == 0) {
#pragma unroll
        for (int s = 0; s < NS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], CW);
        }
        mbar_fence_init();
    }
    __syncthreads();

    if (warp == CW) {  // producer: items (slab, block) in consumption order
        if (lane == 0) {
            long long t = 0;
            for (long long sl = blockIdx.x; sl < slabs; sl += gridDim.x) {
                const long long rb = sl * R;
                const unsigned bytes = (unsigned)(min((long long)R, n - rb) * M * sizeof(double));
                for (int i = 0; i < d; ++i, ++t) {
                    const int slot = (int)(t % NS);
                    if (t >= NS) {
                        mbar_wait(&empty[slot], (unsigned)(((t / NS) - 1) & 1));
                        fence_proxy_async_smem();  // the consumers' generic reads of the slot before the TMA write
                    }
                    mbar_expect_tx(&full[slot], bytes);
                    bulk_load(sm + slot * P::SLAB, Qs[i] + rb * M, bytes, &full[slot]);
                }
            }
        }
        return;
    }

    const int lr = lane & 3, lc = lane >> 2;
    const bool s4 = lc & 4, s2 = lc & 2, s1 = lc & 1;
    long long t = 0;
    for (long long sl = blockIdx.x; sl < slabs; sl += gridDim.x) {
        const long long rb = sl * R;
        const int rr = (int)min((long long)R, n - rb);
        // the accumulators start from beta * Win (loads issued before the first ring wait), so the tile
        // is stored straight from them after the K loop
        double acc[MR][NT][2];
#pragma unroll
        for (int mr = 0; mr < MR; ++mr) {
            const long long r = rb + warp * 8 * MR + 8 * mr + lc;
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
                double2 w = make_double2(0.0, 0.0);
                if (INIT && beta != 0.0 && r < n) {
                    w = *reinterpret_cast<const double2*>(Win + r * ldwi + 8 * nt + 2 * lr);
                    w.x = beta * w.x;
                    w.y = beta * w.y;
                }
                acc[mr][nt][0] = w.x;
                acc[mr][nt][1] = w.y;
            }
        }
        for (int i = 0; i < d; ++i, ++t) {
            const int slot = (int)(t % NS);
            mbar_wait(&full[slot], (unsigned)((t / NS) & 1));
            const double* st = sm + slot * P::SLAB;
            const double* Ci = cs + i * M * LDC;
#pragma unroll
            for (int h = 0; h < M / 32; ++h) {
                double u[MR][8];
#pragma unroll
                for (int mr = 0; mr < MR; ++mr) {
                    const int row = warp * 8 * MR + 8 * mr + lc;
                    const bool ok = row < rr;
                    double v[8];
#pragma unroll
                    for (int j = 0; j < 8; ++j) v[j] = ok ? st[row * M + 32 * h + 4 * ((j + lc) & 7) + lr] : 0.0;
                    // u[kk] = v[(kk - lc) mod 8]: rotate by 4, 2, 1 as the bits of lc say
                    double w4[8], w2[8];
#pragma unroll
                    for (int k = 0; k < 8; ++k) w4[k] = s4 ? v[(k + 4) & 7] : v[k];
#pragma unroll
                    for (int k = 0; k < 8; ++k) w2[k] = s2 ? w4[(k + 6) & 7] : w4[k];
#pragma unroll
                    for (int k = 0; k < 8; ++k) u[mr][k] = s1 ? w2[(k + 7) & 7] : w2[k];
                }
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    double bfr[NT];
#pragma unroll
                    for (int nt = 0; nt < NT; ++nt) bfr[nt] = Ci[(32 * h + 4 * kk + lr) * LDC + 8 * nt + lc];
#pragma unroll
                    for (int mr = 0; mr < MR; ++mr)
#pragma unroll
                        for (int nt = 0; nt < NT; ++nt) dmma_8x8x4(acc[mr][nt], u[mr][kk], bfr[nt]);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[slot]);
        }
#pragma unroll
        for (int mr = 0; mr < MR; ++mr) {
            const long long r = rb + warp * 8 * MR + 8 * mr + lc;
            if (r >= n) continue;
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
                const int b = 8 * nt + 2 * lr;
                double2 o = make_double2(acc[mr][nt][0], acc[mr][nt][1]);
                if (!INIT) {  // long sums: sign * sum_i Q_i C_i first, beta * Win added once
                    o = make_double2(sign * o.x, sign * o.y);
                    if (beta != 0.0) {
                        const double2 wi = *reinterpret_cast<const double2*>(Win + r * ldwi + b);
                        o.x = beta * wi.x + o.x;
                        o.y = beta * wi.y + o.y;
                    }
                }
                *reinterpret_cast<double2*>(Wout + r * ldwo + b) = o;
            }
        }
    }
}

// Resident CTAs per SM for a kernel at a dynamic smem size (0 when it does not fit).
template <typename K>
int resident_ctas(K fn, size_t smem, int threads = 160) {
    if (smem > 227 * 1024) return 0;
    if (cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, smem) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return occ;
}

template <int M, int MR, int NS, int CW>
int launch_update_wide(const double* const* Qs, int d, const double* C, const double* Win, int ldwi, double* Wout,
                       int ldwo, double beta, double sign, long long n, const int* live, cudaStream_t st) {
    using P = UpdWide<M, MR, NS, CW>;
    // short sums (d M <= 256) start the accumulators from beta * Win (see update_smem_kernel, dense.cu)
    auto fn = d * M <= 256 ? update_wide_stream_kernel<M, MR, NS, CW, true> : update_wide_stream_kernel<M, MR, NS, CW, false>;
    const size_t smem = P::smem(d);
    if (smem > 227 * 1024) return EKCG_EINVAL;
    const int occ = resident_ctas(fn, smem, 32 * (CW + 1));
    if (occ < 1) return EKCG_EINVAL;
    const long long slabs = (n + P::R - 1) / P::R;
    const long long slots = (long long)occ * device_sms();
    const int g = (int)(slabs < slots ? slabs : slots);
    launch_k(fn, g, 32 * (CW + 1), smem, st, Qs, d, C, Win, ldwi, Wout, ldwo, beta, sign, n, live);
    return EKCG_OK;
}

}  // namespace

// Rows per Gram step (R) and resident CTAs of the m = 32 streamed Gram.
constexpr int kGram32R = 32, kGram32NS = 4;

int gram_wide_slots(int gb) {
    size_t smem = gb == 2 ? GramWide<32, 2, kGram32R, kGram32NS>::SMEM : GramWide<32, 1, kGram32R, kGram32NS>::SMEM;
    int occ = gb == 2 ? resident_ctas(gram_wide_stream_kernel<32, 2, kGram32R, kGram32NS>, smem)
                      : resident_ctas(gram_wide_stream_kernel<32, 1, kGram32R, kGram32NS>, smem);
    return (occ < 1 ? 1 : occ) * device_sms();
}

// Streamed Gram for 32 contiguous columns (aligned); EKCG_EINVAL otherwise.
int launch_gram_wide(const double* const* Xs, int ldx, int d, int m1, const double* Y, int ldy, int m2, long long n,
                     int chunks, long long rows_chunk, int gb, double* partials, const int* live, cudaStream_t st) {
    if (m1 != 32 || m2 != 32 || ldx != 32 || ldy != 32 || (reinterpret_cast<uintptr_t>(Y) & 15) ||
        rows_chunk % 16 != 0 || (gb != 1 && gb != 2))
        return EKCG_EINVAL;
    dim3 grid(chunks, (d + gb - 1) / gb);
    if (gb == 2) {
        using P = GramWide<32, 2, kGram32R, kGram32NS>;
        auto fn = gram_wide_stream_kernel<32, 2, kGram32R, kGram32NS>;
        if (resident_ctas(fn, P::SMEM) < 1) return EKCG_EINVAL;
        launch_k(fn, grid, 160, P::SMEM, st, Xs, d, Y, n, rows_chunk, partials, live);
    } else {
        using P = GramWide<32, 1, kGram32R, kGram32NS>;
        auto fn = gram_wide_stream_kernel<32, 1, kGram32R, kGram32NS>;
        if (resident_ctas(fn, P::SMEM) < 1) return EKCG_EINVAL;
        launch_k(fn, grid, 160, P::SMEM, st, Xs, d, Y, n, rows_chunk, partials, live);
    }
    return EKCG_OK;
}

// Streamed update for 32 contiguous columns (aligned rows); EKCG_EINVAL
// when it does not apply or C_i do not fit in shared memory.
int launch_update_wide_any(const double* const* Qs, int ldq, int d, int m1, const double* C, const double* Win, int ldwi,
                           double* Wout, int ldwo, int m2, double beta, double sign, long long n, const int* live,
                           cudaStream_t st) {
    if (m1 != 32 || m2 != 32 || ldq != 32 || ldwo % 2 != 0 || (beta != 0.0 && ldwi % 2 != 0) ||
        ((reinterpret_cast<uintptr_t>(Wout) | reinterpret_cast<uintptr_t>(beta != 0.0 ? Win : Wout)) & 15))
        return EKCG_EINVAL;
    // m = 32: 8 consumer warps x 1 tile over a 4-stage Q-slab ring (tools/kernel_times.py --wide).  At m = 64 the
    // register-direct smem-C kernel (dense.cu) is faster (29.8 vs 24.1 TFLOP/s at d = 3): the 64 x 64 C_i leave
    // room for too few ring slots and warps, so the streamed m = 64 variants were dropped.
    return launch_update_wide<32, 1, 4, 8>(Qs, d, C, Win, ldwi, Wout, ldwo, beta, sign, n, live, st);
}
