// Streamed DMMA Gram for 16-column blocks: C_i = X_i^T Y over a row chunk.
//
// A producer warp moves row slabs of Y and of GB blocks X_i into an NS-stage
// shared-memory ring with 1-D bulk copies (TMA engine, mbarrier completion);
// four consumer warps take alternate k-steps (4 rows) of each slab and run
// the fp64 DMMA m8n8k4 on fragments read with 16-B shared loads -- lane
// (i, k) reads columns 2i, 2i+1 of row k, which feed two interleaved 8-wide
// tiles (tile t, element i = column 2i + t), so a warp load is four whole
// 128-B rows, free of bank conflicts.  The loads in flight are bounded by the
// ring, not by registers, and no consumer instruction computes addresses in
// global memory.  Partials per (chunk, block) as in the register-direct Gram
// (dense.cu), reduced by the same fixed-order kernel.
#include "common.cuh"
#include "ekcg_b200.h"
#include "tma.cuh"

namespace {

template <int GB, int R, int NS>
struct Gram16Stream {
    static constexpr int M = 16;
    static constexpr int SLAB = R * M;             // doubles per block slab
    static constexpr int STAGE = (GB + 1) * SLAB;  // Y + GB blocks
    static constexpr int RED = 4 * GB * M * M;     // cross-warp reduction buffer
    static constexpr size_t SMEM = sizeof(double) * (STAGE * NS > RED ? STAGE * NS : RED);
    static_assert(R % 16 == 0, "4 warps x 4-row k-steps");
};

template <int GB, int R, int NS>
__global__ void __launch_bounds__(160)
gram16_stream_kernel(const double* const* __restrict__ Xs, int d, const double* __restrict__ Y, long long n,
                     long long rows_chunk, double* __restrict__ partials, const int* __restrict__ live) {
    EKCG_GATE(live);
    using P = Gram16Stream<GB, R, NS>;
    constexpr int M = 16;
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

    // a block with itself (the Pre-CholQR Gram W^T W): stream it once, read it as both operands
    const bool self_gram = GB == 1 && d == 1 && Xs[0] == Y;
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
                mbar_expect_tx(&full[slot], bytes * (unsigned)(self_gram ? 1 : nb + 1));
                double* st = sm + slot * P::STAGE;
                bulk_load(st, Y + rb * M, bytes, &full[slot]);
                if (!self_gram) {
#pragma unroll
                    for (int g = 0; g < GB; ++g)
                        if (g < nb) bulk_load(st + (g + 1) * P::SLAB, X[g] + rb * M, bytes, &full[slot]);
                }
            }
        }
        return;
    }
    const int xoff = self_gram ? 0 : P::SLAB;  // X_g slab: (g + 1) * SLAB, or the Y slab itself

    const int lr = lane & 3, lc = lane >> 2;
    double acc[GB][2][2][2];
#pragma unroll
    for (int g = 0; g < GB; ++g)
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
            for (int b = 0; b < 2; ++b) acc[g][a][b][0] = acc[g][a][b][1] = 0.0;

    for (int j = 0; j < nsteps; ++j) {
        const int slot = j % NS;
        mbar_wait(&full[slot], (j / NS) & 1);
        const double* st = sm + slot * P::STAGE;
        const int rr = (int)min((long long)R, r1 - (r0 + (long long)j * R));
#pragma unroll
        for (int q = 0; q < R / 16; ++q) {
            const int row = (q * 4 + warp) * 4 + lr;
            const bool ok = row < rr;
            const double2 b = ok ? *reinterpret_cast<const double2*>(st + row * M + 2 * lc) : make_double2(0.0, 0.0);
#pragma unroll
            for (int g = 0; g < GB; ++g) {
                const double2 a = (ok && g < nb)
                                      ? *reinterpret_cast<const double2*>(st + g * P::SLAB + xoff + row * M + 2 * lc)
                                      : make_double2(0.0, 0.0);
                dmma_8x8x4(acc[g][0][0], a.x, b.x);
                dmma_8x8x4(acc[g][0][1], a.x, b.y);
                dmma_8x8x4(acc[g][1][0], a.y, b.x);
                dmma_8x8x4(acc[g][1][1], a.y, b.y);
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
        for (int ta = 0; ta < 2; ++ta)
#pragma unroll
            for (int tb = 0; tb < 2; ++tb)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int a = 2 * lc + ta, b = 2 * (2 * lr + e) + tb;
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

template <int GB, int R, int NS>
int gram16_stream_occupancy() {
    static int cache[kEkcgMaxDevices];
    return kernel_occupancy(gram16_stream_kernel<GB, R, NS>, 160, Gram16Stream<GB, R, NS>::SMEM, cache);
}

template <int GB, int R, int NS>
int launch_gram16_stream(const double* const* Xs, int d, const double* Y, long long n, int chunks,
                         long long rows_chunk, double* partials, const int* live, cudaStream_t st) {
    using P = Gram16Stream<GB, R, NS>;
    if (gram16_stream_occupancy<GB, R, NS>() < 1) return EKCG_EINVAL;
    dim3 grid(chunks, (d + GB - 1) / GB);
    launch_k(gram16_stream_kernel<GB, R, NS>, grid, 160, P::SMEM, st, Xs, d, Y, n, rows_chunk, partials, live);
    return EKCG_OK;
}

// ---------------------------------------------------------------------------
template <int R, int NS, bool INIT>
__global__ void __launch_bounds__(160)
update16_stream_kernel(const double* const* __restrict__ Qs, int d, const double* __restrict__ C, const double* Win,
                       double* Wout, double beta, double sign, long long n, const int* __restrict__ live) {
    EKCG_GATE(live);
    constexpr int M = 16, SLAB = R * M, MR = R / 32;  // 4 consumer warps x MR 8-row tiles
    constexpr int SLOT = SLAB + M * M;                // Q_i row slab + C_i
    static_assert(R % 32 == 0, "R multiple of 32");
    extern __shared__ __align__(128) double sm[];
    __shared__ __align__(8) unsigned long long full[NS], empty[NS];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long slabs = (n + R - 1) / R;
    if (threadIdx.x == 0) {
#pragma unroll
        for (int s = 0; s < NS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 4);
        }
        mbar_fence_init();
    }
    __syncthreads();

    if (warp == 4) {  // producer: items (slab, block) in consumption order
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
                    mbar_expect_tx(&full[slot], bytes + (unsigned)(M * M * sizeof(double)));
                    bulk_load(sm + slot * SLOT, Qs[i] + rb * M, bytes, &full[slot]);
                    bulk_load(sm + slot * SLOT + SLAB, C + (long long)i * M * M, M * M * sizeof(double), &full[slot]);
                }
            }
        }
        return;
    }

    const int lr = lane & 3, lc = lane >> 2, sh = lc & 3;
    long long t = 0;
    for (long long sl = blockIdx.x; sl < slabs; sl += gridDim.x) {
        const long long rb = sl * R;
        const int rr = (int)min((long long)R, n - rb);
        // the accumulators start from beta * Win (loads issued before the first ring wait) and the B
        // fragments carry the sign (exact for +-1), so the tile is stored straight from them
        double acc[MR][2][2];
#pragma unroll
        for (int mr = 0; mr < MR; ++mr) {
            const long long r = rb + warp * 8 * MR + 8 * mr + lc;
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) {
                double2 w = make_double2(0.0, 0.0);
                if (INIT && beta != 0.0 && r < n) {
                    w = *reinterpret_cast<const double2*>(Win + r * M + 8 * nt + 2 * lr);
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
            const double* st = sm + slot * SLOT;
            const double* Ci = st + SLAB;
            double bfr[4][2];
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
#pragma unroll
                for (int nt = 0; nt < 2; ++nt) bfr[kk][nt] = INIT ? sign * Ci[(4 * kk + lr) * M + 8 * nt + lc]
                                                                  : Ci[(4 * kk + lr) * M + 8 * nt + lc];
#pragma unroll
            for (int mr = 0; mr < MR; ++mr) {
                const int row = warp * 8 * MR + 8 * mr + lc;
                const bool ok = row < rr;
                double v[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) v[j] = ok ? st[row * M + 4 * ((j + lc) & 3) + lr] : 0.0;
                // k-step kk is load (kk - sh) mod 4: rotate by 2 then by 1 (branch-free selects)
                const bool b2 = sh & 2, b1 = sh & 1;
                const double t0 = b2 ? v[2] : v[0], t1 = b2 ? v[3] : v[1];
                const double t2 = b2 ? v[0] : v[2], t3 = b2 ? v[1] : v[3];
                const double u[4] = {b1 ? t3 : t0, b1 ? t0 : t1, b1 ? t1 : t2, b1 ? t2 : t3};
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
#pragma unroll
                    for (int nt = 0; nt < 2; ++nt) dmma_8x8x4(acc[mr][nt], u[kk], bfr[kk][nt]);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[slot]);
        }
#pragma unroll
        for (int mr = 0; mr < MR; ++mr) {
            const long long r = rb + warp * 8 * MR + 8 * mr + lc;
            if (r >= n) continue;
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) {
                const int b = 8 * nt + 2 * lr;
                double2 o = make_double2(acc[mr][nt][0], acc[mr][nt][1]);
                if (!INIT) {  // long sums: sign * sum_i Q_i C_i first, beta * Win added once
                    o = make_double2(sign * o.x, sign * o.y);
                    if (beta != 0.0) {
                        const double2 wi = *reinterpret_cast<const double2*>(Win + r * M + b);
                        o.x = beta * wi.x + o.x;
                        o.y = beta * wi.y + o.y;
                    }
                }
                *reinterpret_cast<double2*>(Wout + r * M + b) = o;
            }
        }
    }
}

template <int R, int NS>
int launch_update16_stream(const double* const* Qs, int d, const double* C, const double* Win, double* Wout,
                           double beta, double sign, long long n, const int* live, cudaStream_t st) {
    // short sums (d M <= 256) start the accumulators from beta * Win (see update_smem_kernel, dense.cu)
    auto fn = d * 16 <= 256 ? update16_stream_kernel<R, NS, true> : update16_stream_kernel<R, NS, false>;
    constexpr size_t smem = sizeof(double) * (R * 16 + 256) * NS;
    static int cache[2][kEkcgMaxDevices];
    const int occ = kernel_occupancy(fn, 160, smem, cache[d * 16 <= 256 ? 1 : 0]);
    if (occ < 1) return EKCG_EINVAL;
    const long long grid = (long long)occ * device_sms();
    const long long slabs = (n + R - 1) / R;
    const int g = (int)(slabs < grid ? slabs : grid);
    launch_k(fn, g, 160, smem, st, Qs, d, C, Win, Wout, beta, sign, n, live);
    return EKCG_OK;
}

// The ring shapes (measured on B200, tools/tune_gram.py, tools/dsweep.py): d = 1 Grams take one block per
// CTA with 64-row slabs in 4 stages (3 CTAs per SM); longer histories 4 blocks per CTA sharing 48-row Y
// slabs in 3 stages (2 CTAs per SM); updates 64-row Q slabs in 6 stages (3 CTAs per SM).
constexpr int kGramD1GB = 1, kGramD1R = 64, kGramD1NS = 4;
constexpr int kGramGB = 4, kGramR = 48, kGramNS = 3;
constexpr int kUpdR = 64, kUpdNS = 6;

}  // namespace

// Co-resident CTAs of the streamed m = 16 Gram that ekcg_gram launches for d blocks (the chunking fills whole
// waves of exactly this kernel instance; 0 when it cannot launch here).
int gram16_stream_slots(int d) {
    const int occ = d == 1 ? gram16_stream_occupancy<kGramD1GB, kGramD1R, kGramD1NS>()
                           : gram16_stream_occupancy<kGramGB, kGramR, kGramNS>();
    return occ * device_sms();
}

// Streamed Gram when it applies (16 contiguous columns, aligned); EKCG_EINVAL otherwise.
int launch_gram_stream(const double* const* Xs, int ldx, int d, int m1, const double* Y, int ldy, int m2, long long n,
                       int chunks, long long rows_chunk, double* partials, const int* live, cudaStream_t st) {
    if (m1 != 16 || m2 != 16 || ldx != 16 || ldy != 16 || (reinterpret_cast<uintptr_t>(Y) & 15) ||
        rows_chunk % 16 != 0)
        return EKCG_EINVAL;
    if (d == 1)
        return launch_gram16_stream<kGramD1GB, kGramD1R, kGramD1NS>(Xs, d, Y, n, chunks, rows_chunk, partials, live,
                                                                    st);
    return launch_gram16_stream<kGramGB, kGramR, kGramNS>(Xs, d, Y, n, chunks, rows_chunk, partials, live, st);
}

int launch_update_stream(const double* const* Qs, int ldq, int d, int m1, const double* C, const double* Win, int ldwi,
                         double* Wout, int ldwo, int m2, double beta, double sign, long long n, const int* live,
                         cudaStream_t st) {
    if (m1 != 16 || m2 != 16 || ldq != 16 || ldwo != 16 || (beta != 0.0 && ldwi != 16) ||
        ((reinterpret_cast<uintptr_t>(Wout) | reinterpret_cast<uintptr_t>(beta != 0.0 ? Win : Wout)) & 15))
        return EKCG_EINVAL;
    return launch_update16_stream<kUpdR, kUpdNS>(Qs, d, C, Win, Wout, beta, sign, n, live, st);
}
