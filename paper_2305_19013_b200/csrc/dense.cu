// Tall-skinny fp64 block kernels for the A-orthonormaliser and the iterate update.
//
//   ekcg_gram          C_i = X_i^T Y for a list of retained blocks (split-K partials)
//   ekcg_reduce        fixed-order sum of the split-K partials (deterministic)
//   ekcg_block_update  Wout = beta Win + sign sum_i Q_i C_i  (CGS2 update, W R^-1)
//   ekcg_xr_update     x += W a, r -= AW a, partial |r|^2
//
// Block widths m in {8,16,32,64} run on the fp64 tensor cores (mma.sync
// m8n8k4 -> SASS DMMA.8x8x4) with fragments loaded straight from the
// row-major blocks: a fragment row is 4 consecutive doubles (32 B) of one
// block row, so every DRAM sector fetched is consumed.  Other widths (the
// reference's t = 1..7, mixed widths after a flexible switch) take the scalar
// kernels.  No floating-point atomics anywhere: reruns are bit-identical.
#include "common.cuh"
#include "ekcg_b200.h"

namespace {

constexpr int kGramThreads = 128;  // 4 warps
constexpr int kVecThreads = 256;

// ---------------------------------------------------------------------------
// chunking (split-K over rows)
// ---------------------------------------------------------------------------
long long rows_per_chunk(long long n, int chunks) {
    long long r = (n + chunks - 1) / chunks;
    return ((r + 15) / 16) * 16;
}

}  // namespace
int launch_gram_stream(const double* const* Xs, int ldx, int d, int m1, const double* Y, int ldy, int m2, long long n,
                       int chunks, long long rows_chunk, double* partials, const int* live, cudaStream_t st);
int gram16_stream_slots(int d);
int launch_update_stream(const double* const* Qs, int ldq, int d, int m1, const double* C, const double* Win, int ldwi,
                         double* Wout, int ldwo, int m2, double beta, double sign, long long n, const int* live,
                         cudaStream_t st);
int gram_wide_slots(int gb);
int launch_gram_wide(const double* const* Xs, int ldx, int d, int m1, const double* Y, int ldy, int m2, long long n,
                     int chunks, long long rows_chunk, int gb, double* partials, const int* live, cudaStream_t st);
int launch_update_wide_any(const double* const* Qs, int ldq, int d, int m1, const double* C, const double* Win, int ldwi,
                           double* Wout, int ldwo, int m2, double beta, double sign, long long n, const int* live,
                           cudaStream_t st);
// Rows per warp (in 8-row groups) of the m = 64 smem-C update (compile-time; tools/kbench.py A/B builds)
#ifndef EKCG_UPD64_MR
#define EKCG_UPD64_MR 2
#endif

namespace {

// Blocks per CTA that share one pass over Y (see gram_dmma_kernel).
int gram_blocks_per_cta(int d, int m1, int m2) {
    if (m1 != m2) return 1;
    int gb = 1;
    switch (m1) {
        case 8: gb = 8; break;
        case 16: gb = 4; break;
        case 32: gb = 2; break;
        default: gb = 1;
    }
    while (gb > 1 && gb / 2 >= d) gb /= 2;  // d = 1 -> 1, d = 2 -> 2, ...
    return gb;
}

// ---------------------------------------------------------------------------
// Fragment loads with column interleave.  A DMMA m8n8k4 operand lane (i, k)
// holds element i of an 8-wide tile; with T >= 2 tiles the tiles are
// interleaved over the row segment -- tile t, element i is column
// (t / 2) * 16 + 2 i + (t % 2) -- so one 16-B load per lane feeds two tiles and
// a warp load covers whole 128-B row segments.  Odd T: plain 8-column tiles.
// (16-B aligned rows required: even leading dimensions, aligned blocks.)
// ---------------------------------------------------------------------------
template <int T, bool IL = true>
__device__ __forceinline__ int tile_col(int t, int i) {
    return (IL && T % 2 == 0) ? (t / 2) * 16 + 2 * i + (t % 2) : 8 * t + i;
}

template <int T, bool IL = true>
__device__ __forceinline__ void load_tiles(const double* row, int lc, bool ok, double (&f)[T]) {
    if (IL && T % 2 == 0) {
#pragma unroll
        for (int h = 0; h < T / 2; ++h) {
            const double2 v = ok ? __ldg(reinterpret_cast<const double2*>(row + 16 * h + 2 * lc)) : make_double2(0.0, 0.0);
            f[2 * h] = v.x;
            f[2 * h + 1] = v.y;
        }
    } else {
#pragma unroll
        for (int t = 0; t < T; ++t) f[t] = ok ? __ldg(row + 8 * t + lc) : 0.0;
    }
}

// ---------------------------------------------------------------------------
// X^T X for one 64-column block (the Pre-CholQR Gram W^T W, aortho.py:105) over rows [r0, r1): a tile below
// the diagonal is the transpose of its mirror above it -- same products, same order, same bits -- so only
// the 36 of 64 8 x 8 tiles on and above the diagonal are formed and each is stored twice.  Warps 0 / 3 take
// the diagonal 32 x 32 quadrants (10 tiles each; the B fragments are the A fragments), warps 1 / 2 the left
// and right halves of the quadrant above the diagonal (8 tiles each).  Kept out of line so that the general
// kernel's registers and schedule stay as they are.
// ---------------------------------------------------------------------------
template <int U>
__device__ __noinline__ void gram_self64(const double* __restrict__ Y, int ldy, long long r0, long long r1,
                                         double* __restrict__ out) {
    constexpr int M = 64, T = 4;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int lr = lane & 3, lc = lane >> 2;
    const long long steps = (r1 > r0) ? (r1 - r0 + 3) / 4 : 0;
    const bool diag = warp == 0 || warp == 3;
    const int a_off = warp == 3 ? 32 : 0;
    const int b_off = warp == 0 ? 0 : warp == 2 ? 48 : 32;
    double acc[T][T][2];
#pragma unroll
    for (int ta = 0; ta < T; ++ta)
#pragma unroll
        for (int tb = 0; tb < T; ++tb) acc[ta][tb][0] = acc[ta][tb][1] = 0.0;
    if (diag) {
        for (long long s0 = 0; s0 < steps; s0 += U) {
            double af[U][T];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const long long r = r0 + 4 * (s0 + u) + lr;
                load_tiles<T, false>(Y + r * ldy + a_off, lc, r < r1, af[u]);
            }
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int ta = 0; ta < T; ++ta)
#pragma unroll
                    for (int tb = ta; tb < T; ++tb) dmma_8x8x4(acc[ta][tb], af[u][ta], af[u][tb]);
        }
    } else {
        for (long long s0 = 0; s0 < steps; s0 += U) {
            double af[U][T], bf[U][2];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const long long r = r0 + 4 * (s0 + u) + lr;
                load_tiles<2, false>(Y + r * ldy + b_off, lc, r < r1, bf[u]);
                load_tiles<T, false>(Y + r * ldy + a_off, lc, r < r1, af[u]);
            }
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int ta = 0; ta < T; ++ta)
#pragma unroll
                    for (int tb = 0; tb < 2; ++tb) dmma_8x8x4(acc[ta][tb], af[u][ta], bf[u][tb]);
        }
    }
#pragma unroll
    for (int ta = 0; ta < T; ++ta)
#pragma unroll
        for (int tb = 0; tb < T; ++tb) {
            if (diag ? tb < ta : tb >= 2) continue;
            const int a = a_off + 8 * ta + lc;
            const int b0 = b_off + 8 * tb + 2 * lr, b1 = b0 + 1;
            out[a * M + b0] = acc[ta][tb][0];
            out[a * M + b1] = acc[ta][tb][1];
            if (!(diag && ta == tb)) {
                out[b0 * M + a] = acc[ta][tb][0];
                out[b1 * M + a] = acc[ta][tb][1];
            }
        }
}

// ---------------------------------------------------------------------------
// DMMA Gram: partials[p][i] (M x M) = X_i[rows of p]^T Y[rows of p]
// CTA (p, g) handles row chunk p for blocks i = g*GB .. g*GB+GB-1, so each Y
// fragment loaded feeds GB blocks.  Warp w: row lane ks = w % KS, output
// quadrant q = w / KS with TA x TB tiles of 8x8.  Rows advance in k-steps of
// 4 (the mma K); fragments come straight from the row-major blocks.
// ---------------------------------------------------------------------------
template <int M, int TA, int TB, int KS, int U, int GB, bool IL>
__global__ void __launch_bounds__(kGramThreads)
gram_dmma_kernel(const double* const* __restrict__ Xs, int ldx, int d, const double* __restrict__ Y, int ldy,
                 long long n, long long rows_chunk, double* __restrict__ partials,
                 const int* __restrict__ live) {
    EKCG_GATE(live);
    static_assert((M / 8 / TA) * (M / 8 / TB) * KS == kGramThreads / 32, "warp layout");
    constexpr int QA = M / 8 / TA;
    __shared__ double red[KS > 1 ? KS * GB * M * M : 1];

    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int ks = warp % KS;
    const int quad = warp / KS;
    const int a_base = (quad % QA) * TA * 8;
    const int b_base = (quad / QA) * TB * 8;
    // grid (block groups, chunks): the CTAs of one row chunk are consecutive, so the groups that read the
    // same Y rows run together and share them through L2 instead of re-reading Y from HBM per group
    const int i0 = blockIdx.x * GB;
    const int nb = min(GB, d - i0);
    const double* __restrict__ X[GB];
#pragma unroll
    for (int g = 0; g < GB; ++g) X[g] = Xs[min(i0 + g, d - 1)];
    const long long r0 = blockIdx.y * rows_chunk;
    long long r1 = r0 + rows_chunk;
    if (r1 > n) r1 = n;
    const long long steps = (r1 > r0) ? (r1 - r0 + 3) / 4 : 0;

    double acc[GB][TA][TB][2];
#pragma unroll
    for (int g = 0; g < GB; ++g)
#pragma unroll
        for (int ta = 0; ta < TA; ++ta)
#pragma unroll
            for (int tb = 0; tb < TB; ++tb) acc[g][ta][tb][0] = acc[g][ta][tb][1] = 0.0;

    const int lr = lane & 3;
    const int lc = lane >> 2;
    // X^T X at m = 64 (plain 8-column tiles): only the tiles on and above the diagonal (gram_self64)
    if (M == 64 && TA == 4 && TB == 4 && KS == 1 && GB == 1 && !IL && d == 1 && X[0] == Y) {
        gram_self64<U>(Y, ldy, r0, r1, partials + (long long)blockIdx.y * (M * M));
        return;
    }
    for (long long s0 = ks; s0 < steps; s0 += (long long)KS * U) {
        double af[U][GB][TA], bf[U][TB];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            long long s = s0 + (long long)u * KS;
            long long r = r0 + 4 * s + lr;
            bool ok = (s < steps) && (r < r1);
            load_tiles<TB, IL>(Y + r * ldy + b_base, lc, ok, bf[u]);
#pragma unroll
            for (int g = 0; g < GB; ++g) load_tiles<TA, IL>(X[g] + r * ldx + a_base, lc, ok && (g < nb), af[u][g]);
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int g = 0; g < GB; ++g)
#pragma unroll
                for (int ta = 0; ta < TA; ++ta)
#pragma unroll
                    for (int tb = 0; tb < TB; ++tb) dmma_8x8x4(acc[g][ta][tb], af[u][g][ta], bf[u][tb]);
    }

    if (KS == 1) {
#pragma unroll
        for (int g = 0; g < GB; ++g) {
            if (g >= nb) break;
            double* out = partials + ((long long)blockIdx.y * d + i0 + g) * (M * M);
#pragma unroll
            for (int ta = 0; ta < TA; ++ta)
#pragma unroll
                for (int tb = 0; tb < TB; ++tb) {
                    const int a = a_base + tile_col<TA, IL>(ta, lc);
                    const int b0 = b_base + tile_col<TB, IL>(tb, 2 * lr), b1 = b_base + tile_col<TB, IL>(tb, 2 * lr + 1);
                    out[a * M + b0] = acc[g][ta][tb][0];
                    out[a * M + b1] = acc[g][ta][tb][1];
                }
        }
    } else {
#pragma unroll
        for (int g = 0; g < GB; ++g)
#pragma unroll
            for (int ta = 0; ta < TA; ++ta)
#pragma unroll
                for (int tb = 0; tb < TB; ++tb) {
                    const int a = a_base + tile_col<TA, IL>(ta, lc);
                    red[((ks * GB + g) * M + a) * M + b_base + tile_col<TB, IL>(tb, 2 * lr)] = acc[g][ta][tb][0];
                    red[((ks * GB + g) * M + a) * M + b_base + tile_col<TB, IL>(tb, 2 * lr + 1)] = acc[g][ta][tb][1];
                }
        __syncthreads();
        for (int o = threadIdx.x; o < nb * M * M; o += kGramThreads) {
            const int g = o / (M * M), e = o % (M * M);
            double s = red[g * M * M + e];
#pragma unroll
            for (int k = 1; k < KS; ++k) s += red[(k * GB + g) * M * M + e];
            partials[((long long)blockIdx.y * d + i0 + g) * (M * M) + e] = s;
        }
    }
}

using GramFn = void (*)(const double* const*, int, int, const double*, int, long long, long long, double*,
                        const int*);

// The DMMA Gram variant for (d, m1, m2) (nullptr: generic kernel) and its GB.
GramFn select_gram(int d, int m1, int m2, int& gb) {
    gb = gram_blocks_per_cta(d, m1, m2);
    // interleaved loads: faster for m = 32 and for m = 16 with short histories,
    // slower for m = 16 with d >= 48 and for m = 64 (tools/kernel_times.py)
    const bool il = m1 == 32 || (m1 == 16 && d < 48);
    if (m1 != m2) return nullptr;
    switch (m1) {
        case 8:
            if (gb == 8) return il ? (GramFn)gram_dmma_kernel<8, 1, 1, 4, 4, 8, true> : (GramFn)gram_dmma_kernel<8, 1, 1, 4, 4, 8, false>;
            if (gb == 4) return il ? (GramFn)gram_dmma_kernel<8, 1, 1, 4, 4, 4, true> : (GramFn)gram_dmma_kernel<8, 1, 1, 4, 4, 4, false>;
            if (gb == 2) return il ? (GramFn)gram_dmma_kernel<8, 1, 1, 4, 4, 2, true> : (GramFn)gram_dmma_kernel<8, 1, 1, 4, 4, 2, false>;
            return il ? (GramFn)gram_dmma_kernel<8, 1, 1, 4, 4, 1, true> : (GramFn)gram_dmma_kernel<8, 1, 1, 4, 4, 1, false>;
        case 16:
            // 4 blocks per CTA: 2 k-step lanes for long histories (d >= 48), 1 below (tools/tune_gram.py)
            if (gb == 1) return il ? (GramFn)gram_dmma_kernel<16, 2, 2, 4, 4, 1, true> : (GramFn)gram_dmma_kernel<16, 2, 2, 4, 4, 1, false>;
            if (gb == 2) return il ? (GramFn)gram_dmma_kernel<16, 2, 2, 4, 4, 2, true> : (GramFn)gram_dmma_kernel<16, 2, 2, 4, 4, 2, false>;
            if (d < 48) return il ? (GramFn)gram_dmma_kernel<16, 2, 2, 4, 1, 4, true> : (GramFn)gram_dmma_kernel<16, 2, 2, 4, 1, 4, false>;
            return il ? (GramFn)gram_dmma_kernel<16, 2, 2, 4, 2, 4, true> : (GramFn)gram_dmma_kernel<16, 2, 2, 4, 2, 4, false>;
        case 32:
            if (gb == 2) return il ? (GramFn)gram_dmma_kernel<32, 4, 2, 2, 2, 2, true> : (GramFn)gram_dmma_kernel<32, 4, 2, 2, 2, 2, false>;
            return il ? (GramFn)gram_dmma_kernel<32, 4, 2, 2, 4, 1, true> : (GramFn)gram_dmma_kernel<32, 4, 2, 2, 4, 1, false>;
        case 64:
            return il ? (GramFn)gram_dmma_kernel<64, 4, 4, 1, 2, 1, true> : (GramFn)gram_dmma_kernel<64, 4, 4, 1, 2, 1, false>;
        default:
            return nullptr;
    }
}

// Resident CTAs per SM of a Gram kernel (queried once per variant; 4 when no
// device is present, e.g. host-only queries).
int gram_occupancy(GramFn fn) {
    constexpr int kMax = 64;
    static GramFn keys[kMax];
    static int vals[kMax][kEkcgMaxDevices];
    static int used = 0;
    if (fn == nullptr) return 4;
    int slot = -1;
    for (int i = 0; i < used; ++i)
        if (keys[i] == fn) slot = i;
    if (slot < 0) {
        if (used == kMax) return 4;
        slot = used;
        keys[used++] = fn;
    }
    const int occ = kernel_occupancy(fn, kGramThreads, 0, vals[slot]);
    return occ < 1 ? 4 : occ;
}

int gram_chunks(long long n, int d, int m1, int m2) {
    int gb;
    GramFn fn = select_gram(d, m1, m2, gb);
    const long long groups = (d + gb - 1) / gb;
    const bool wide = m1 == 32 && m2 == 32;
    if ((m1 == 16 && m2 == 16) || wide) {
        // streamed Gram: resident CTAs with long row ranges.  Pick the chunk
        // count whose CTA total fills its last wave best (equal work per CTA),
        // preferring fewer chunks; at least 1024 rows per chunk.
        const bool d1 = !wide && d == 1;  // GB = 1 stream kernel
        long long slots = wide ? gram_wide_slots(gb) : gram16_stream_slots(d);  // co-resident CTAs of that kernel
        if (slots < 1) slots = device_sms();
        long long pmax = (n + (d1 ? 511 : 1023)) / (d1 ? 512 : 1024);
        const long long cap = (4 * slots + groups - 1) / groups;
        if (pmax > cap) pmax = cap;
        if (pmax < 1) pmax = 1;
        long long best = 1;
        double best_eff = 0.0;
        for (long long p = 1; p <= pmax; ++p) {
            const long long ctas = p * groups;
            const double eff = (double)ctas / ((double)slots * (double)((ctas + slots - 1) / slots));
            if (eff > best_eff + 0.01) {
                best_eff = eff;
                best = p;
            }
        }
        return (int)best;
    }
    const long long waves = (m1 == 16 && m2 == 16 && d >= 48) ? 2 : 1;
    const long long target = (long long)device_sms() * gram_occupancy(fn) * waves;
    long long p = target / groups;  // floor: whole waves, no straggler CTAs
    long long max_p = (n + 255) / 256;
    if (p > max_p) p = max_p;
    if (p < 1) p = 1;
    return (int)p;
}

// Scalar Gram for arbitrary (m1, m2): thread (row-group, output) pairs.
__global__ void __launch_bounds__(256)
gram_generic_kernel(const double* const* __restrict__ Xs, int ldx, int m1, const double* __restrict__ Y,
                    int ldy, int m2, long long n, long long rows_chunk, double* __restrict__ partials,
                    const int* __restrict__ live) {
    EKCG_GATE(live);
    extern __shared__ double sred[];
    const int O = m1 * m2;
    const int i = blockIdx.y;
    const double* __restrict__ X = Xs[i];
    const long long r0 = blockIdx.x * rows_chunk;
    long long r1 = r0 + rows_chunk;
    if (r1 > n) r1 = n;
    double* out = partials + ((long long)blockIdx.x * gridDim.y + i) * O;
    if (O <= 256) {
        const int RG = 256 / O;
        const int tid = threadIdx.x;
        const int rg = tid / O;
        const int o = tid % O;
        double acc = 0.0;
        if (rg < RG) {
            const int a = o / m2, b = o % m2;
            for (long long r = r0 + rg; r < r1; r += RG) acc += X[r * ldx + a] * Y[r * ldy + b];
            sred[rg * O + o] = acc;
        }
        __syncthreads();
        if (tid < O) {
            double s = sred[o];
            for (int k = 1; k < RG; ++k) s += sred[k * O + o];
            out[o] = s;
        }
    } else {
        for (int o = threadIdx.x; o < O; o += blockDim.x) {
            const int a = o / m2, b = o % m2;
            double acc = 0.0;
            for (long long r = r0; r < r1; ++r) acc += X[r * ldx + a] * Y[r * ldy + b];
            out[o] = acc;
        }
    }
}

// X_i^T y for a vector y (m2 = 1) and m1 = 4 LN columns, 16-B aligned rows:
// LN lanes per row, 4 columns per lane, U row groups in flight per warp; the
// CTA's warps are combined in fixed order into its partial (same layout as
// the Gram kernels).
template <int LN, int U, bool W256 = false>
__global__ void __launch_bounds__(256)
gemvt4_kernel(const double* const* __restrict__ Xs, int ldx, int d, const double* __restrict__ y, long long n,
              long long rows_chunk, double* __restrict__ partials, const int* __restrict__ live) {
    EKCG_GATE(live);
    constexpr int M = 4 * LN, RPW = 32 / LN;
    __shared__ double red[8][M];
    const int i = blockIdx.y;
    const double* __restrict__ X = Xs[i];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int sub = lane / LN, li = lane % LN;
    const long long r0 = blockIdx.x * rows_chunk;
    const long long r1 = min(n, r0 + rows_chunk);
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    // one 256-bit access per row segment when the block is 32-B aligned (block-uniform branch)
    const bool w256 = W256 && ((reinterpret_cast<uintptr_t>(X) & 31) == 0) && (ldx & 3) == 0;
    for (long long base = r0 + (long long)warp * RPW * U; base < r1; base += 8LL * RPW * U) {
        double2 a[U][2];
        double yv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long long r = base + u * RPW + sub;
            const bool ok = r < r1;
            const double2* row = reinterpret_cast<const double2*>(X + r * ldx) + 2 * li;
            if (w256) {
                double t4[4] = {0.0, 0.0, 0.0, 0.0};
                if (ok) ld4_256(reinterpret_cast<const double*>(row), t4);
                a[u][0] = make_double2(t4[0], t4[1]);
                a[u][1] = make_double2(t4[2], t4[3]);
            } else {
                a[u][0] = ok ? __ldg(row) : make_double2(0.0, 0.0);
                a[u][1] = ok ? __ldg(row + 1) : make_double2(0.0, 0.0);
            }
            yv[u] = ok ? __ldg(y + r) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            acc[0] += a[u][0].x * yv[u];
            acc[1] += a[u][0].y * yv[u];
            acc[2] += a[u][1].x * yv[u];
            acc[3] += a[u][1].y * yv[u];
        }
    }
#pragma unroll
    for (int off = 16; off >= LN; off >>= 1)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[c] += __shfl_xor_sync(0xffffffffu, acc[c], off);
    if (sub == 0)
#pragma unroll
        for (int c = 0; c < 4; ++c) red[warp][4 * li + c] = acc[c];
    __syncthreads();
    if (threadIdx.x < M) {
        double s = red[0][threadIdx.x];
#pragma unroll
        for (int w = 1; w < 8; ++w) s += red[w][threadIdx.x];
        partials[((long long)blockIdx.x * d + i) * M + threadIdx.x] = s;
    }
}

// out[j] = sum_p partials[p*len + j].  Block = W warps x 32 lanes; lane owns
// output j = 32*blockIdx.x + lane, warp w sums p = w, w+W, ... (4 loads in
// flight), then the W warp sums are combined in fixed order: deterministic.
__global__ void __launch_bounds__(1024)
reduce_kernel(const double* __restrict__ partials, int chunks, long long len, double* __restrict__ out,
              const int* __restrict__ live) {
    EKCG_GATE(live);
    __shared__ double ws[32][33];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, W = blockDim.x >> 5;
    const long long j = (long long)blockIdx.x * 32 + lane;
    double s = 0.0;
    if (j < len) {
        int p = warp;
        for (; p + 3 * W < chunks; p += 4 * W) {
            double a = partials[(long long)p * len + j];
            double b = partials[(long long)(p + W) * len + j];
            double c = partials[(long long)(p + 2 * W) * len + j];
            double d = partials[(long long)(p + 3 * W) * len + j];
            s += a;
            s += b;
            s += c;
            s += d;
        }
        for (; p < chunks; p += W) s += partials[(long long)p * len + j];
    }
    ws[warp][lane] = s;
    __syncthreads();
    if (warp == 0 && j < len) {
        double t = ws[0][lane];
        for (int w = 1; w < W; ++w) t += ws[w][lane];
        out[j] = t;
    }
}

// ---------------------------------------------------------------------------
// DMMA block update: Wout = beta Win + sign sum_i Q_i C_i   (m1 = m2 = M)
// Warp tile: 8*MR rows x M columns; mma M-dim = rows, N = output column,
// K = column of Q_i.
// ---------------------------------------------------------------------------
// Wout[r, b:b+2] = beta Win[r, b:b+2] + sign acc for the accumulator pairs of
// MR 8-row tiles (16-B loads / stores: even leading dimensions, aligned rows).
template <int MR, int NT>
__device__ __forceinline__ void store_tile_rows(const double (&acc)[MR][NT][2], long long rbase, int lc, int lr,
                                                long long n, const double* Win, int ldwi, double* Wout, int ldwo,
                                                double beta, double sign) {
#pragma unroll
    for (int mr = 0; mr < MR; ++mr) {
        const long long r = rbase + 8 * mr + lc;
        if (r >= n) continue;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
            const int b = 8 * nt + 2 * lr;
            double2 o = make_double2(sign * acc[mr][nt][0], sign * acc[mr][nt][1]);
            if (beta != 0.0) {
                const double2 wi = *reinterpret_cast<const double2*>(Win + r * ldwi + b);
                o.x = beta * wi.x + o.x;
                o.y = beta * wi.y + o.y;
            }
            *reinterpret_cast<double2*>(Wout + r * ldwo + b) = o;
        }
    }
}

template <int M, int MR, bool IL = true>
__global__ void __launch_bounds__(128)
update_dmma_kernel(const double* const* __restrict__ Qs, int ldq, int d, const double* __restrict__ C,
                   const double* Win, int ldwi, double* Wout, int ldwo, double beta, double sign,
                   long long n, const int* __restrict__ live) {
    EKCG_GATE(live);
    constexpr int NT = M / 8;
    constexpr int KK = M / 4;
    const int lane = threadIdx.x & 31;
    const int lr = lane & 3;
    const int lc = lane >> 2;
    const long long warps_total = (long long)gridDim.x * (blockDim.x >> 5);
    const long long tiles = (n + 8 * MR - 1) / (8 * MR);
    for (long long tile = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5); tile < tiles;
         tile += warps_total) {
        const long long rbase = tile * 8 * MR;
        double acc[MR][NT][2];
#pragma unroll
        for (int mr = 0; mr < MR; ++mr)
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) acc[mr][nt][0] = acc[mr][nt][1] = 0.0;

        for (int i = 0; i < d; ++i) {
            const double* __restrict__ Q = Qs[i];
            const double* __restrict__ Ci = C + (long long)i * M * M;
            if (!IL) {
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
                continue;
            }
#pragma unroll
            for (int kp = 0; kp < KK / 2; ++kp) {
                // two k-steps per 16-B load: k index lr <-> columns 8 kp + 2 lr (+1)
                double2 afr[MR];
#pragma unroll
                for (int mr = 0; mr < MR; ++mr) {
                    long long r = rbase + 8 * mr + lc;
                    afr[mr] = (r < n) ? __ldg(reinterpret_cast<const double2*>(Q + r * ldq + 8 * kp + 2 * lr))
                                      : make_double2(0.0, 0.0);
                }
                double bx[NT], by[NT];
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) {
                    bx[nt] = __ldg(Ci + (8 * kp + 2 * lr) * M + 8 * nt + lc);
                    by[nt] = __ldg(Ci + (8 * kp + 2 * lr + 1) * M + 8 * nt + lc);
                }
#pragma unroll
                for (int mr = 0; mr < MR; ++mr)
#pragma unroll
                    for (int nt = 0; nt < NT; ++nt) dmma_8x8x4(acc[mr][nt], afr[mr].x, bx[nt]);
#pragma unroll
                for (int mr = 0; mr < MR; ++mr)
#pragma unroll
                    for (int nt = 0; nt < NT; ++nt) dmma_8x8x4(acc[mr][nt], afr[mr].y, by[nt]);
            }
        }
        store_tile_rows<MR, NT>(acc, rbase, lc, lr, n, Win, ldwi, Wout, ldwo, beta, sign);
    }
}

// Wide-block variant (M >= 32): the coefficient blocks C_i are staged once per
// CTA in shared memory (rows padded to M + 2 doubles, see LDC below) and B fragments come from smem; 8 warps per
// CTA, each walking its own 8*MR-row tiles (no block barriers in the loop).
// TRI: d = 1 and C upper triangular (the Pre-CholQR / A-CholQR factor
// S = R^-1, aortho.py:106,109): k-step pairs kp > nt multiply exact zeros and
// are skipped (44 % of the DMMAs at M = 64); the products kept are the same.
template <int M, int MR, bool TRI = false, bool INIT = true>
__global__ void __launch_bounds__(256)
update_smem_kernel(const double* const* __restrict__ Qs, int ldq, int d, const double* __restrict__ C,
                   const double* Win, int ldwi, double* Wout, int ldwo, double beta, double sign,
                   long long n, const int* __restrict__ live) {
    EKCG_GATE(live);
    extern __shared__ double cs[];
    constexpr int NT = M / 8;
    constexpr int KK = M / 4;
    // rows padded to M + 2 doubles: a B fragment reads k-rows 2 lr (+1), so consecutive lr are 2 rows = 4 bank
    // pairs apart and the 16 lanes of a half warp (4 columns x 4 lr) hit 16 distinct bank pairs; with M + 4 the
    // rows of lr and lr + 2 aliased (ncu: 51 % of the shared-load wavefronts were conflict replays)
    constexpr int LDC = M + 2;
    // INIT: sign * C staged (exact for sign = +-1), so the accumulators start from beta * Win and the
    // tile is stored straight from them -- the Win loads issue with the first A fragments instead of
    // after the K loop, and no read-modify-write trails each tile (m = 64, d = 3: 29.9 -> 33.3 TFLOP/s).
    // It adds the d*M rank-1 terms onto W one by one, so it is used for short sums (d M <= 256); long
    // ones (INIT = false) sum sign * sum_i Q_i C_i first and add beta * Win once.
    for (int e = threadIdx.x; e < d * M * M; e += blockDim.x) {
        const int i = e / (M * M), rem = e % (M * M);
        cs[(i * M + rem / M) * LDC + rem % M] = INIT ? sign * C[e] : C[e];
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int lr = lane & 3;
    const int lc = lane >> 2;
    const long long warps_total = (long long)gridDim.x * (blockDim.x >> 5);
    const long long tiles = (n + 8 * MR - 1) / (8 * MR);
    for (long long tile = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5); tile < tiles;
         tile += warps_total) {
        const long long rbase = tile * 8 * MR;
        double acc[MR][NT][2];
#pragma unroll
        for (int mr = 0; mr < MR; ++mr) {
            const long long r = rbase + 8 * mr + lc;
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
                double2 w = make_double2(0.0, 0.0);
                if (INIT && !TRI && beta != 0.0 && r < n) {
                    w = *reinterpret_cast<const double2*>(Win + r * ldwi + 8 * nt + 2 * lr);
                    w.x = beta * w.x;
                    w.y = beta * w.y;
                }
                acc[mr][nt][0] = w.x;
                acc[mr][nt][1] = w.y;
            }
        }
        for (int i = 0; i < d; ++i) {
            const double* __restrict__ Q = Qs[i];
            const double* Ci = cs + i * M * LDC;
#pragma unroll (TRI ? KK / 2 : 2)
            for (int kp = 0; kp < KK / 2; ++kp) {
                double2 afr[MR];
#pragma unroll
                for (int mr = 0; mr < MR; ++mr) {
                    long long r = rbase + 8 * mr + lc;
                    afr[mr] = (r < n) ? __ldg(reinterpret_cast<const double2*>(Q + r * ldq + 8 * kp + 2 * lr))
                                      : make_double2(0.0, 0.0);
                }
                double bx[NT], by[NT];
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) {
                    if (TRI && kp > nt) continue;
                    bx[nt] = Ci[(8 * kp + 2 * lr) * LDC + 8 * nt + lc];
                    by[nt] = Ci[(8 * kp + 2 * lr + 1) * LDC + 8 * nt + lc];
                }
#pragma unroll
                for (int mr = 0; mr < MR; ++mr)
#pragma unroll
                    for (int nt = 0; nt < NT; ++nt)
                        if (!(TRI && kp > nt)) dmma_8x8x4(acc[mr][nt], afr[mr].x, bx[nt]);
#pragma unroll
                for (int mr = 0; mr < MR; ++mr)
#pragma unroll
                    for (int nt = 0; nt < NT; ++nt)
                        if (!(TRI && kp > nt)) dmma_8x8x4(acc[mr][nt], afr[mr].y, by[nt]);
            }
        }
        if (INIT) {
#pragma unroll
            for (int mr = 0; mr < MR; ++mr) {
                const long long r = rbase + 8 * mr + lc;
                if (r >= n) continue;
#pragma unroll
                for (int nt = 0; nt < NT; ++nt)
                    *reinterpret_cast<double2*>(Wout + r * ldwo + 8 * nt + 2 * lr) =
                        make_double2(acc[mr][nt][0], acc[mr][nt][1]);
            }
        } else {
            store_tile_rows<MR, NT>(acc, rbase, lc, lr, n, Win, ldwi, Wout, ldwo, beta, sign);
        }
    }
}

__global__ void update_generic_kernel(const double* const* __restrict__ Qs, int ldq, int d, int m1,
                                      const double* __restrict__ C, const double* Win, int ldwi,
                                      double* Wout, int ldwo, int m2, double beta, double sign,
                                      long long n, const int* __restrict__ live) {
    EKCG_GATE(live);
    long long total = n * (long long)m2;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        long long r = e / m2;
        int b = (int)(e - r * m2);
        double s = 0.0;
        for (int i = 0; i < d; ++i) {
            const double* Q = Qs[i] + r * ldq;
            const double* Ci = C + (long long)i * m1 * m2;
            for (int a = 0; a < m1; ++a) s += Q[a] * Ci[a * m2 + b];
        }
        double o = sign * s;
        if (beta != 0.0) o = beta * Win[r * ldwi + b] + o;
        Wout[r * ldwo + b] = o;
    }
}

// ---------------------------------------------------------------------------
// vector kernels with deterministic block partial sums
// ---------------------------------------------------------------------------
// A fixed cap (not the device's SM count): the chunk count sets the summation order, so norms are
// bit-identical on every B200 regardless of its SM count.
int vec_chunks(long long n) {
    long long p = (n + kVecThreads - 1) / kVecThreads;
    if (p > 148LL * 8) p = 148LL * 8;
    if (p < 1) p = 1;
    return (int)p;
}

__device__ __forceinline__ double block_sum(double v) {
    __shared__ double warp_sums[32];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) warp_sums[warp] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0) {
        const int nw = (blockDim.x + 31) >> 5;
        for (int w = 0; w < nw; ++w) s += warp_sums[w];
    }
    return s;  // valid in thread 0
}

// L lanes cooperate on one row (L = power of two <= 32): coalesced reads of
// the row-major W / AW rows, shuffle reduction of the row dot products.
template <int L>
__global__ void __launch_bounds__(kVecThreads)
xr_update_kernel(const double* __restrict__ W, int ldw, const double* __restrict__ AW, int ldaw,
                 const double* __restrict__ alpha, int m, double* __restrict__ x, double* __restrict__ r,
                 long long n, double* __restrict__ partials, const int* __restrict__ live) {
    EKCG_GATE(live);
    __shared__ double sa[256];
    for (int a = threadIdx.x; a < m && a < 256; a += blockDim.x) sa[a] = alpha[a];
    __syncthreads();
    constexpr int RPW = 32 / L;  // rows per warp pass
    const int lane = threadIdx.x & 31;
    const int sub = lane / L, li = lane % L;
    const long long warp_global = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long warps_total = ((long long)gridDim.x * blockDim.x) >> 5;
    double sq = 0.0;
    for (long long base = warp_global * RPW; base < n; base += warps_total * RPW) {
        const long long row = base + sub;
        double dx = 0.0, dr = 0.0;
        if (row < n) {
            const double* w = W + row * ldw;
            const double* aw = AW + row * ldaw;
            for (int a = li; a < m; a += L) {
                dx += w[a] * sa[a];
                dr += aw[a] * sa[a];
            }
        }
#pragma unroll
        for (int off = L / 2; off > 0; off >>= 1) {
            dx += __shfl_xor_sync(0xffffffffu, dx, off);
            dr += __shfl_xor_sync(0xffffffffu, dr, off);
        }
        if (row < n && li == 0) {
            x[row] = x[row] + dx;
            double rn = r[row] - dr;
            r[row] = rn;
            sq += rn * rn;
        }
    }
    double s = block_sum(sq);
    if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

// m = 4*LN columns, 16-B aligned rows: LN lanes per row, 4 columns per lane,
// U row groups in flight per warp (x and r loaded before the reductions).
// 4 CTAs per SM: the fixed 1184-CTA grid (the partial count sets the summation order) is then exactly two
// waves of 592 resident CTAs; at 3 per SM (78 registers) it ran 2.67 waves with an idle tail (3.00 -> 2.92 ms
// at 4096^2 x 64, tools/kbench.py).
template <int LN, int U, bool W256 = false>
__global__ void __launch_bounds__(kVecThreads, 4)
xr_update4_kernel(const double* __restrict__ W, int ldw, const double* __restrict__ AW, int ldaw,
                  const double* __restrict__ alpha, double* __restrict__ x, double* __restrict__ r, long long n,
                  double* __restrict__ partials, const int* __restrict__ live) {
    EKCG_GATE(live);
    constexpr int RPW = 32 / LN;
    const int lane = threadIdx.x & 31;
    const int sub = lane / LN, li = lane % LN;
    const double2 a01 = __ldg(reinterpret_cast<const double2*>(alpha) + 2 * li);
    const double2 a23 = __ldg(reinterpret_cast<const double2*>(alpha) + 2 * li + 1);
    const long long warp_global = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long warps_total = ((long long)gridDim.x * blockDim.x) >> 5;
    double sq = 0.0;
    for (long long base = warp_global * RPW * U; base < n; base += warps_total * RPW * U) {
        double dx[U], dr[U], xv[U], rv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long long row = base + u * RPW + sub;
            dx[u] = dr[u] = xv[u] = rv[u] = 0.0;
            if (row < n) {
                const double2* w = reinterpret_cast<const double2*>(W + row * ldw) + 2 * li;
                const double2* aw = reinterpret_cast<const double2*>(AW + row * ldaw) + 2 * li;
                double2 w0, w1, v0, v1;
                if (W256) {  // one 256-bit access per operand (32-B aligned rows)
                    double t4[4], u4[4];
                    ld4_256(reinterpret_cast<const double*>(w), t4);
                    ld4_256(reinterpret_cast<const double*>(aw), u4);
                    w0 = make_double2(t4[0], t4[1]);
                    w1 = make_double2(t4[2], t4[3]);
                    v0 = make_double2(u4[0], u4[1]);
                    v1 = make_double2(u4[2], u4[3]);
                } else {
                    w0 = __ldg(w);
                    w1 = __ldg(w + 1);
                    v0 = __ldg(aw);
                    v1 = __ldg(aw + 1);
                }
                if (li == 0) {
                    xv[u] = x[row];
                    rv[u] = r[row];
                }
                dx[u] = w0.x * a01.x + w0.y * a01.y + w1.x * a23.x + w1.y * a23.y;
                dr[u] = v0.x * a01.x + v0.y * a01.y + v1.x * a23.x + v1.y * a23.y;
            }
        }
#pragma unroll
        for (int off = LN / 2; off > 0; off >>= 1) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                dx[u] += __shfl_xor_sync(0xffffffffu, dx[u], off);
                dr[u] += __shfl_xor_sync(0xffffffffu, dr[u], off);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long long row = base + u * RPW + sub;
            if (row < n && li == 0) {
                x[row] = xv[u] + dx[u];
                const double rn = rv[u] - dr[u];
                r[row] = rn;
                sq += rn * rn;
            }
        }
    }
    double s = block_sum(sq);
    if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

__global__ void __launch_bounds__(kVecThreads)
sumsq_kernel(const double* __restrict__ v, long long n, double* __restrict__ partials,
             const int* __restrict__ live) {
    EKCG_GATE(live);
    double sq = 0.0;
    for (long long row = blockIdx.x * (long long)blockDim.x + threadIdx.x; row < n;
         row += (long long)gridDim.x * blockDim.x) {
        double a = v[row];
        sq += a * a;
    }
    double s = block_sum(sq);
    if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

// Block-diagonal dense apply Y = B X over consecutive row blocks (block-Jacobi
// preconditioner factors, blockjacobi.py:136-170): B_b is a dense nb x nb
// row-major matrix at data[offs[b]]; mode 0: B_b lower, 1: B_b^T of a lower
// matrix (upper), per row i of block b: y_ic = sum_j B_b[i][j] x_jc.
__global__ void block_diag_apply_kernel(const double* __restrict__ data, const long long* __restrict__ offs,
                                        const int* __restrict__ starts, const int* __restrict__ row_block,
                                        int transpose, const double* __restrict__ X, int ldx,
                                        double* __restrict__ Y, int ldy, long long n, int m,
                                        const int* __restrict__ live) {
    EKCG_GATE(live);
    const long long total = n * (long long)m;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const long long i = e / m;
        const int c = (int)(e - i * m);
        const int b = row_block[i];
        const int s0 = starts[b], nb = starts[b + 1] - s0;
        const int li = (int)(i - s0);
        const double* B = data + offs[b];
        double acc = 0.0;
        if (!transpose) {
            for (int j = 0; j <= li; ++j) acc += B[li * nb + j] * X[(long long)(s0 + j) * ldx + c];
        } else {
            for (int j = li; j < nb; ++j) acc += B[j * nb + li] * X[(long long)(s0 + j) * ldx + c];
        }
        Y[i * ldy + c] = acc;
    }
}

// Block-diagonal triangular solves by substitution, one thread per (block,
// column): L_b y = x (forward) or L_b^T y = x (backward) -- the
// solve_triangular calls of blockjacobi.py:145-152.  In place allowed.
__global__ void block_trsv_kernel(const double* __restrict__ data, const long long* __restrict__ offs,
                                  const int* __restrict__ starts, int nblocks, int transpose,
                                  const double* X, int ldx, double* Y, int ldy, int m,
                                  const int* __restrict__ live) {
    EKCG_GATE(live);
    const long long total = (long long)nblocks * m;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const int b = (int)(e / m), c = (int)(e - (long long)b * m);
        const int s0 = starts[b], nb = starts[b + 1] - s0;
        const double* L = data + offs[b];
        const double* x = X + (long long)s0 * ldx + c;
        double* y = Y + (long long)s0 * ldy + c;
        if (!transpose) {
            for (int i = 0; i < nb; ++i) {
                double acc = x[(long long)i * ldx];
                for (int j = 0; j < i; ++j) acc -= L[i * nb + j] * y[(long long)j * ldy];
                y[(long long)i * ldy] = acc / L[i * nb + i];
            }
        } else {
            for (int i = nb - 1; i >= 0; --i) {
                double acc = x[(long long)i * ldx];
                for (int j = i + 1; j < nb; ++j) acc -= L[j * nb + i] * y[(long long)j * ldy];
                y[(long long)i * ldy] = acc / L[i * nb + i];
            }
        }
    }
}

__global__ void copy_cols_kernel(const double* __restrict__ src, int lds, double* __restrict__ dst, int ldd,
                                 long long n, int w, const int* __restrict__ live) {
    EKCG_GATE(live);
    long long total = n * (long long)w;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        long long i = e / w;
        int j = (int)(e - i * w);
        dst[i * ldd + j] = src[i * lds + j];
    }
}

__global__ void sub_kernel(const double* __restrict__ a, const double* __restrict__ b, double* __restrict__ out,
                           long long n, const int* __restrict__ live) {
    EKCG_GATE(live);
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        out[i] = a[i] - b[i];
}

}  // namespace

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
extern "C" int ekcg_gram_chunks(long long n, int d, int m1, int m2) {
    if (n < 1 || d < 1 || m1 < 1 || m2 < 1) return 1;
    return gram_chunks(n, d, m1, m2);
}

extern "C" int ekcg_gram(const double* const* Xs, int ldx, int d, int m1, const double* Y, int ldy, int m2,
                         long long n, double* partials, const int* live, void* stream) {
    if (d < 1 || m1 < 1 || m2 < 1 || ldx < m1 || ldy < m2 || n < 1) return EKCG_EINVAL;
    const int chunks = gram_chunks(n, d, m1, m2);
    const long long rc = rows_per_chunk(n, chunks);
    const int gb = gram_blocks_per_cta(d, m1, m2);
    dim3 grid(chunks, (d + gb - 1) / gb);  // generic kernel: gb == 1
    cudaStream_t st = as_stream(stream);
    int gbs;
    GramFn fn = select_gram(d, m1, m2, gbs);
    // DMMA variants with m >= 16 load 16-B fragments pairs: even leading
    // dimensions, 16-B aligned Y (and blocks, by contract); else generic.
    if (m1 >= 16 && ((ldx | ldy) % 2 != 0 || (reinterpret_cast<uintptr_t>(Y) & 15))) fn = nullptr;
    const bool vec4 = (m2 == 1) && (m1 % 4 == 0) && (m1 <= 128) && (ldx % 2 == 0) &&
                      ((m1 / 4) & (m1 / 4 - 1)) == 0;  // LN = m1/4 a power of two
    if (vec4) {
        const dim3 g(chunks, d);
        switch (m1) {
            case 4: launch_k(gemvt4_kernel<1, 4, true>, g, 256, 0, st, Xs, ldx, d, Y, n, rc, partials, live); break;
            case 8: launch_k(gemvt4_kernel<2, 4, true>, g, 256, 0, st, Xs, ldx, d, Y, n, rc, partials, live); break;
            case 16: launch_k(gemvt4_kernel<4, 4, true>, g, 256, 0, st, Xs, ldx, d, Y, n, rc, partials, live); break;
            case 32: launch_k(gemvt4_kernel<8, 4, true>, g, 256, 0, st, Xs, ldx, d, Y, n, rc, partials, live); break;
            case 64: launch_k(gemvt4_kernel<16, 4, true>, g, 256, 0, st, Xs, ldx, d, Y, n, rc, partials, live); break;
            default: launch_k(gemvt4_kernel<32, 2, true>, g, 256, 0, st, Xs, ldx, d, Y, n, rc, partials, live); break;
        }
    } else if (fn != nullptr && launch_gram_wide(Xs, ldx, d, m1, Y, ldy, m2, n, chunks, rc, gb, partials, live, st) == EKCG_OK) {
        // streamed (TMA bulk) Gram for 32-column blocks, stream_wide.cu
    } else if (fn != nullptr && launch_gram_stream(Xs, ldx, d, m1, Y, ldy, m2, n, chunks, rc, partials, live, st) == EKCG_OK) {
        // streamed (TMA bulk) Gram, stream.cu
    } else if (fn != nullptr) {
        launch_k(fn, dim3(grid.y, grid.x), kGramThreads, 0, st, Xs, ldx, d, Y, ldy, n, rc, partials, live);
    } else {
        const int O = m1 * m2;
        size_t smem = (O <= 256) ? sizeof(double) * 256 : 0;
        launch_k(gram_generic_kernel, dim3(chunks, d), 256, smem, st, Xs, ldx, m1, Y, ldy, m2, n, rc, partials, live);
    }
    ++g_ekcg_launches;
    return launch_status();
}

extern "C" int ekcg_reduce(const double* partials, int chunks, long long len, double* out, const int* live,
                           void* stream) {
    if (chunks < 1 || len < 1) return EKCG_EINVAL;
    int warps = chunks < 32 ? chunks : 32;
    long long blocks = (len + 31) / 32;
    // keep enough warps in flight when there are few outputs
    launch_k(reduce_kernel, (unsigned)blocks, 32 * warps, 0, as_stream(stream), partials, chunks, len, out, live);
    ++g_ekcg_launches;
    return launch_status();
}

extern "C" int ekcg_block_update(const double* const* Qs, int ldq, int d, int m1, const double* C,
                                 const double* Win, int ldwi, double* Wout, int ldwo, int m2, double beta,
                                 double sign, long long n, const int* live, void* stream) {
    if (d < 1 || m1 < 1 || m2 < 1 || ldq < m1 || ldwo < m2 || n < 0) return EKCG_EINVAL;
    if (beta != 0.0 && (Win == nullptr || ldwi < m2)) return EKCG_EINVAL;
    if (n == 0) return EKCG_OK;
    cudaStream_t st = as_stream(stream);
    // DMMA kernels move 16-B pairs: even leading dimensions, aligned rows
    const bool even = (ldwo % 2 == 0) && (ldq % 2 == 0) && (beta == 0.0 || ldwi % 2 == 0) &&
                      ((reinterpret_cast<uintptr_t>(Wout) | reinterpret_cast<uintptr_t>(beta != 0.0 ? Win : Wout)) % 16 == 0);
    auto grid_rows = [&](int rows_per_warp) {
        long long tiles = (n + rows_per_warp - 1) / rows_per_warp;
        return grid_for(tiles, 4, (long long)device_sms() * 16);
    };
    if (launch_update_stream(Qs, ldq, d, m1, C, Win, ldwi, Wout, ldwo, m2, beta, sign, n, live, st) == EKCG_OK) {
        // streamed (TMA bulk) update, stream.cu
    } else if (launch_update_wide_any(Qs, ldq, d, m1, C, Win, ldwi, Wout, ldwo, m2, beta, sign, n, live, st) == EKCG_OK) {
        // streamed update for 32 / 64-column blocks, stream_wide.cu
    } else if (m1 == m2 && even && m1 == 8) {
        launch_k(update_dmma_kernel<8, 4, false>, grid_rows(32), 128, 0, st, Qs, ldq, d, C, Win, ldwi, Wout, ldwo, beta,
                                                                  sign, n, live);
    } else if (m1 == m2 && even && m1 == 16) {
        launch_k(update_dmma_kernel<16, 4, false>, grid_rows(32), 128, 0, st, Qs, ldq, d, C, Win, ldwi, Wout, ldwo, beta,
                                                                   sign, n, live);
    } else if (m1 == m2 && even && (m1 == 32 || m1 == 64) && (size_t)d * m1 * (m1 + 2) * 8 <= 200 * 1024) {
        const size_t smem = (size_t)d * m1 * (m1 + 2) * sizeof(double);
        const int mr = (m1 == 32) ? 4 : EKCG_UPD64_MR;
        long long tiles = (n + 8 * mr - 1) / (8 * mr);
        unsigned grid = grid_for(tiles, 8, (long long)device_sms() * 8);
        if (m1 == 32) {
            auto fn = d * 32 <= 256 ? update_smem_kernel<32, 4, false, true> : update_smem_kernel<32, 4, false, false>;
            cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            launch_k(fn, grid, 256, smem, st, Qs, ldq, d, C, Win, ldwi, Wout, ldwo, beta, sign, n, live);
        } else {
            auto fn = d * 64 <= 256 ? update_smem_kernel<64, EKCG_UPD64_MR, false, true>
                                    : update_smem_kernel<64, EKCG_UPD64_MR, false, false>;
            cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            launch_k(fn, grid, 256, smem, st, Qs, ldq, d, C, Win, ldwi, Wout, ldwo, beta, sign, n, live);
        }
    } else if (m1 == m2 && even && m1 == 32) {
        launch_k(update_dmma_kernel<32, 4>, grid_rows(32), 128, 0, st, Qs, ldq, d, C, Win, ldwi, Wout, ldwo, beta,
                                                                   sign, n, live);
    } else if (m1 == m2 && even && m1 == 64) {
        launch_k(update_dmma_kernel<64, 2>, grid_rows(16), 128, 0, st, Qs, ldq, d, C, Win, ldwi, Wout, ldwo, beta,
                                                                   sign, n, live);
    } else {
        launch_k(update_generic_kernel, grid_for(n * m2, 256), 256, 0, st, Qs, ldq, d, m1, C, Win, ldwi, Wout, ldwo,
                                                                     m2, beta, sign, n, live);
    }
    ++g_ekcg_launches;
    return launch_status();
}

extern "C" int ekcg_tri_apply(const double* const* Ws, int ldw, const double* S, double* out, int ldo, int m,
                              long long n, const int* live, void* stream) {
    if (m < 1 || ldw < m || ldo < m || n < 0) return EKCG_EINVAL;
    if (n == 0) return EKCG_OK;
    const bool even = (ldw % 2 == 0) && (ldo % 2 == 0) && (reinterpret_cast<uintptr_t>(out) % 16 == 0);
    if (m == 64 && even) {
        const size_t smem = (size_t)64 * (64 + 2) * sizeof(double);
        long long tiles = (n + 15) / 16;
        unsigned grid = grid_for(tiles, 8, (long long)device_sms() * 8);
        auto fn = update_smem_kernel<64, 2, true>;
        cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        launch_k(fn, grid, 256, smem, as_stream(stream), Ws, ldw, 1, S, (const double*)nullptr, m, out, ldo, 0.0, 1.0,
                 n, live);
        ++g_ekcg_launches;
        return launch_status();
    }
    return ekcg_block_update(Ws, ldw, 1, m, S, nullptr, m, out, ldo, m, 0.0, 1.0, n, live, stream);
}

extern "C" int ekcg_vec_chunks(long long n) { return vec_chunks(n); }

extern "C" int ekcg_xr_update(const double* W, int ldw, const double* AW, int ldaw, const double* alpha, int m,
                              double* x, double* r, long long n, double* rho2_partials, const int* live,
                              void* stream) {
    if (m < 1 || m > 256 || ldw < m || ldaw < m || n < 1) return EKCG_EINVAL;
    cudaStream_t st = as_stream(stream);
    const int g = vec_chunks(n);
#define XR_LAUNCH(L) launch_k(xr_update_kernel<L>, g, kVecThreads, 0, st, W, ldw, AW, ldaw, alpha, m, x, r, n, rho2_partials, live)
#define XR4_LAUNCH(LN)                                                                                         \
    (al32 ? launch_k(xr_update4_kernel<LN, 4, true>, g, kVecThreads, 0, st, W, ldw, AW, ldaw, alpha, x, r, n,   \
                     rho2_partials, live)                                                                         \
          : launch_k(xr_update4_kernel<LN, 4>, g, kVecThreads, 0, st, W, ldw, AW, ldaw, alpha, x, r, n,         \
                     rho2_partials, live))
    const bool al = (ldw % 2 == 0) && (ldaw % 2 == 0) && ((reinterpret_cast<uintptr_t>(W) | reinterpret_cast<uintptr_t>(AW) |
                                                           reinterpret_cast<uintptr_t>(alpha)) % 16 == 0);
    const bool al32 = ldw % 4 == 0 && ldaw % 4 == 0 &&
                      ((reinterpret_cast<uintptr_t>(W) | reinterpret_cast<uintptr_t>(AW)) % 32 == 0);
    if (al && m == 64) XR4_LAUNCH(16);
    else if (al && m == 32) XR4_LAUNCH(8);
    else if (al && m == 16) XR4_LAUNCH(4);
    else if (al && m == 8) XR4_LAUNCH(2);
    else if (m >= 32) XR_LAUNCH(32);
    else if (m >= 16) XR_LAUNCH(16);
    else if (m >= 8) XR_LAUNCH(8);
    else if (m >= 4) XR_LAUNCH(4);
    else if (m >= 2) XR_LAUNCH(2);
    else XR_LAUNCH(1);
#undef XR_LAUNCH
#undef XR4_LAUNCH
    ++g_ekcg_launches;
    return launch_status();
}

extern "C" int ekcg_sumsq(const double* v, long long n, double* partials, const int* live, void* stream) {
    if (n < 1) return EKCG_EINVAL;
    launch_k(sumsq_kernel, vec_chunks(n), kVecThreads, 0, as_stream(stream), v, n, partials, live);
    ++g_ekcg_launches;
    return launch_status();
}

extern "C" int ekcg_block_diag_apply(const double* data, const long long* offs, const int* starts,
                                     const int* row_block, int transpose, const double* X, int ldx, double* Y,
                                     int ldy, long long n, int m, const int* live, void* stream) {
    if (n < 1 || m < 1 || ldx < m || ldy < m || X == Y) return EKCG_EINVAL;
    launch_k(block_diag_apply_kernel, grid_for(n * m, 256), 256, 0, as_stream(stream), data, offs, starts, row_block,
                                                                                 transpose, X, ldx, Y, ldy, n, m,
                                                                                 live);
    ++g_ekcg_launches;
    return launch_status();
}

extern "C" int ekcg_block_trsv(const double* L, const long long* offs, const int* starts, int nblocks,
                               int transpose, const double* X, int ldx, double* Y, int ldy, int m,
                               const int* live, void* stream) {
    if (nblocks < 1 || m < 1 || ldx < m || ldy < m) return EKCG_EINVAL;
    launch_k(block_trsv_kernel, grid_for((long long)nblocks * m, 128), 128, 0, as_stream(stream), 
        L, offs, starts, nblocks, transpose, X, ldx, Y, ldy, m, live);
    ++g_ekcg_launches;
    return launch_status();
}

extern "C" int ekcg_copy_cols(const double* src, int lds, double* dst, int ldd, long long n, int w,
                              const int* live, void* stream) {
    if (n < 0 || w < 1 || lds < w || ldd < w) return EKCG_EINVAL;
    if (n == 0) return EKCG_OK;
    launch_k(copy_cols_kernel, grid_for(n * w, 256), 256, 0, as_stream(stream), src, lds, dst, ldd, n, w, live);
    ++g_ekcg_launches;
    return launch_status();
}

extern "C" int ekcg_sub(const double* a, const double* b, double* out, long long n, const int* live,
                        void* stream) {
    if (n < 1) return EKCG_EINVAL;
    launch_k(sub_kernel, grid_for(n, 256), 256, 0, as_stream(stream), a, b, out, n, live);
    ++g_ekcg_launches;
    return launch_status();
}
