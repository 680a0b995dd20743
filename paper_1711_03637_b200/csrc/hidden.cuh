// Inference hot path on sm_100a: input table, window compaction, the fused
// stencil + hidden-LIF kernel, and the event-driven output layer.
//
// Reference behaviour (relative to /root/reference/pkg/src/spikedigits):
//   _input_tables          network.py:224-245  -> k_input_table
//   hidden_current_series  network.py:254-264  -> stencil inside k_hidden
//   run_presentation       network.py:267-326  -> k_hidden + k_output
//   lif_step / kernel_step neurons.py:83-171   -> snn_common.cuh helpers
//
// Work decomposition:
//   k_prep       a window (3x3 pixel patch, 676 per image) is ACTIVE when any
//                of its pixels is non-zero.  Inactive windows receive exactly
//                zero current for the whole trial and never leave rest, so
//                skipping them is exact.  Active windows are compacted in
//                ascending order into tiles of 32 (tile_pos), n_tiles per image.
//   k_tile_scan  exclusive prefix of n_tiles -> tile_base: one compact list of
//                all tiles of the batch, so no warp idles.
//   k_hidden     persistent CTAs of 4 warps; a warp owns one tile, a lane one
//                window and its 12 feature neurons (v, refractory horizon in
//                registers for the whole trial).  The input-trace table is
//                streamed through a 2-stage shared-memory ring by TMA bulk
//                copies.  The stencil is the k-ordered FMA chain OpenBLAS uses
//                for np.tensordot, so currents are bit-identical.  Output: one
//                12-bit spike mask per lane and step (the raster).
//   k_output     one warp per image.  c_hidden @ W is event-driven: every
//                hidden kernel trace is a linear recursion in its own spikes,
//                so sum_k c_k(n) W[k,l] = A_l(n) - B_l(n) with
//                A_l(n) = A_l(n-1) e^{-dt/t1} + G_l(n), G_l(n) = sum of the W
//                rows of the neurons spiking at n.  The warp gathers those W
//                rows with cp.async (a whole batch in flight), sums them in
//                ascending neuron order and runs the 10-neuron output layer.
// Every reduction has a fixed order: results are deterministic run to run.
#pragma once
#include "snn_common.cuh"

namespace snn {

constexpr int kWPC = 4;          // warps (tiles) per k_hidden CTA
constexpr int kThreads = kWPC * 32;
constexpr int kChunk = 8;        // table steps per ring stage
constexpr int kStages = 2;       // table ring depth
constexpr int kOutWarps = 4;     // images per k_output CTA (one warp each)

constexpr int kHalf = kNF / 2;   // features per k_hidden work item

// Raster layout (bytes): image i owns the block starting at tile_base[i]*N*64,
// laid out [step][tile][half][lane]; each byte is the 6-bit spike mask of
// features half*6 .. half*6+5 of the lane's window.
__host__ __device__ inline size_t raster_at(int64_t tile_base_img, int N, int ntiles, int s, int t) {
    return ((size_t)tile_base_img * N + (size_t)s * ntiles + t) * (2 * kTile);
}

struct BatchArgs {
    snn_consts_t c;
    const uint8_t *images;   // [n][784]
    int64_t n_images;
    const double *w;         // [8112][10]
    const double *ctab;      // [N][256]
    uint16_t *tile_pos;      // [n][22][32] window of each lane, 0xFFFF = none
    int32_t *n_tiles;        // [n]
    int32_t *tile_base;      // [n+1] exclusive prefix of n_tiles
    uint8_t *raster;         // sum(n_tiles) * N * 64 spike-mask bytes (see raster_at)
    double *partial;         // [items][N][10] per-item G partials (inference)
    int32_t items_per_tile;  // 1 (default bank) or 2 (generic bank)
    snn_infer_out_t out;     // counts / out_raster / ff / v_out / v_hid
};

__device__ __forceinline__ uint64_t warp_excl_scan_u64(uint64_t x, uint64_t *total) {
    const int lane = threadIdx.x & 31;
    uint64_t inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t y = __shfl_up_sync(kFull, inc, o);
        if (lane >= o) inc += y;
    }
    *total = __shfl_sync(kFull, inc, 31);
    return inc - x;
}

// ---------------------------------------------------------------------------
// k_input_table: the 256 input neurons under constant drive (network.py:233-242)
__global__ void __launch_bounds__(256) k_input_table(snn_consts_t c, double *ctab, uint8_t *spk) {
    const int lv = threadIdx.x;
    const double drive = __dadd_rn(c.i0, __dmul_rn((double)lv, c.ip));
    double v = c.lif_in.el, a = 0.0, b = 0.0;
    int live_from = 0;
    for (int s = 0; s < c.n_steps; ++s) {
        const double cand = lif_candidate(v, drive, c.lif_in);
        const bool live = s >= live_from;
        const bool fired = live && cand >= c.lif_in.vt;
        if (live) v = fired ? c.lif_in.el : cand;
        if (fired) live_from = next_live_step(s, c.lif_in.refr);
        const double bump = fired ? 1.0 : 0.0;
        a = __dadd_rn(__dmul_rn(a, c.decay_slow), bump);
        b = __dadd_rn(__dmul_rn(b, c.decay_fast), bump);
        ctab[(size_t)s * 256 + lv] = __dsub_rn(a, b);
        if (spk) spk[(size_t)s * 256 + lv] = fired ? 1 : 0;
    }
}

// ---------------------------------------------------------------------------
// k_prep: ordered compaction of the active windows, one image per CTA.
__global__ void __launch_bounds__(kThreads) k_prep(const BatchArgs A) {
    __shared__ __align__(16) uint8_t s_img[kSide * kSide];
    __shared__ int s_cnt[8 * kWPC];
    constexpr int kIters = (kNPos + kThreads - 1) / kThreads;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t img = blockIdx.x;
    const uint8_t *gimg = A.images + img * (kSide * kSide);
    if (tid < 49) reinterpret_cast<uint4 *>(s_img)[tid] = __ldg(reinterpret_cast<const uint4 *>(gimg) + tid);
    __syncthreads();
    unsigned bal[kIters];
#pragma unroll
    for (int it = 0; it < kIters; ++it) {
        const int p = it * kThreads + tid;
        bool on = false;
        if (p < kNPos) {
            const int r = p / kFmap, col = p % kFmap;
#pragma unroll
            for (int a = 0; a < 3; ++a)
#pragma unroll
                for (int b = 0; b < 3; ++b) on |= s_img[(r + a) * kSide + col + b] != 0;
        }
        bal[it] = __ballot_sync(kFull, on);
        if (lane == 0) s_cnt[it * kWPC + warp] = __popc(bal[it]);
    }
    __syncthreads();
    int run = 0, off[kIters];
#pragma unroll
    for (int it = 0; it < kIters; ++it)
#pragma unroll
        for (int w = 0; w < kWPC; ++w) {
            if (w == warp) off[it] = run;
            run += s_cnt[it * kWPC + w];
        }
    uint16_t *tp = A.tile_pos + img * (kMaxTiles * kTile);
    for (int k = run + tid; k < kMaxTiles * kTile; k += kThreads) tp[k] = 0xFFFF;
#pragma unroll
    for (int it = 0; it < kIters; ++it)
        if ((bal[it] >> lane) & 1u)
            tp[off[it] + __popc(bal[it] & ((1u << lane) - 1u))] = (uint16_t)(it * kThreads + tid);
    if (tid == 0) A.n_tiles[img] = (run + kTile - 1) / kTile;
}

// k_tile_scan: tile_base = exclusive prefix of n_tiles; one CTA, any n.
__global__ void __launch_bounds__(1024) k_tile_scan(const BatchArgs A) {
    __shared__ int s_w[32];
    __shared__ int s_tot, s_carry;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_carry = 0;
    __syncthreads();
    for (int64_t base = 0; base < A.n_images; base += 1024) {
        const int64_t i = base + tid;
        const int x = i < A.n_images ? A.n_tiles[i] : 0;
        int tot;
        const int ex = warp_excl_scan_int(x, &tot);
        if (lane == 0) s_w[warp] = tot;
        __syncthreads();
        if (warp == 0) {
            int t2;
            const int e2 = warp_excl_scan_int(s_w[lane], &t2);
            s_w[lane] = e2;
            if (lane == 0) s_tot = t2;
        }
        __syncthreads();
        if (i < A.n_images) A.tile_base[i] = s_carry + s_w[warp] + ex;
        __syncthreads();
        if (tid == 0) s_carry += s_tot;
        __syncthreads();
    }
    if (tid == 0) A.tile_base[A.n_images] = s_carry;
}

// ---------------------------------------------------------------------------
// The default filter bank (filters.py:22-31, :63-88) as compile-time taps:
// kernels * (15 nA / positive sum), evaluated in IEEE double exactly like
// numpy does on the host.  The library uses the specialised kernel only when
// the caller's taps are bitwise identical to these.
constexpr double kG1 = 15e-9 / 4.0;   // Sobel gain
constexpr double kG2 = 15e-9 / 20.0;  // corner gain
// integer kernel coefficients (filters.py:22-31, negations, corners)
__host__ __device__ constexpr int def_coef(int f, int k) {
    constexpr int c[kNF][9] = {
        {1, 2, 1, 0, 0, 0, -1, -2, -1},    {1, 0, -1, 2, 0, -2, 1, 0, -1},
        {2, 1, 0, 1, 0, -1, 0, -1, -2},    {0, 1, 2, -1, 0, 1, -2, -1, 0},
        {-1, -2, -1, 0, 0, 0, 1, 2, 1},    {-1, 0, 1, -2, 0, 2, -1, 0, 1},
        {-2, -1, 0, -1, 0, 1, 0, 1, 2},    {0, -1, -2, 1, 0, -1, 2, 1, 0},
        {5, 5, -4, 5, 5, -4, -4, -4, -4},  {-4, 5, 5, -4, 5, 5, -4, -4, -4},
        {-4, -4, -4, 5, 5, -4, 5, 5, -4},  {-4, -4, -4, -4, 5, 5, -4, 5, 5},
    };
    return c[f][k];
}

// FilterBank.weighted = kernels * gains[:, None, None] (float64 product)
__host__ __device__ constexpr double def_tap(int f, int k) {
    return (double)def_coef(f, k) * (f < 8 ? kG1 : kG2);
}

// dgemm's k-ordered FMA chain for a compile-time tap row.  A zero tap adds
// x*0 = +0 (inputs are >= 0), which leaves the sum unchanged up to the sign
// of a zero, so skipping it is exact for everything downstream.
template <int F>
__device__ __forceinline__ double def_current(const double (&x)[9]) {
    double I = 0.0;
    bool first = true;
#pragma unroll
    for (int k = 0; k < 9; ++k) {
        if (def_coef(F, k) != 0) {
            I = first ? __dmul_rn(x[k], def_tap(F, k)) : __fma_rn(x[k], def_tap(F, k), I);
            first = false;
        }
    }
    return I;
}

// One hidden LIF step (neurons.py:113-126).  Two exact identities keep it
// short: a neuron that is not live has v == E_L (it was reset at its spike and
// has been frozen since), so v' = (!live || fired || vn < E_L) ? E_L : vn; and
// since threshold > rest (LifParams validation, neurons.py:39-47),
// max(vn, E_L) >= V_T <=> vn >= V_T.  With SGN (E_L < 0 < V_T, the defaults)
// both comparisons run on the integer pipe on the IEEE bit patterns, which
// order like the values for these signs: vn >= V_T <=> (int64)bits(vn) >=
// bits(V_T); vn < E_L <=> (uint64)bits(vn) > bits(E_L).  That leaves the FP64
// pipe (this kernel's bound) with the five arithmetic ops only.
struct LifK {
    double g, el, beta, vt;
    long long el_bits, vt_bits;
};

__device__ __forceinline__ LifK lif_k(const snn_lif_t &p) {
    return LifK{p.g, p.el, p.beta, p.vt, __double_as_longlong(p.el), __double_as_longlong(p.vt)};
}

template <bool SGN>
__device__ __forceinline__ void lif_update(double I, double &v, int &live_from, int s, int relive, const LifK &ph,
                                           unsigned &m, int bit) {
    double t = __dsub_rn(v, ph.el);
    t = __dmul_rn(ph.g, t);
    t = __dsub_rn(I, t);
    t = __dmul_rn(ph.beta, t);
    const double vn = __dadd_rn(v, t);
    // pr: refractory (s < live_from); pf: fired = live && vn >= V_T;
    // pz: frozen || fired || vn < E_L  ->  v = E_L, else v = vn.
    if (SGN) {  // the threshold test on the integer pipe, the clamp test on the FP64 pipe
        asm("{\n\t.reg .pred pr, pf, pa, pz;\n\t"
            "setp.lt.s32 pr, %3, %1;\n\t"
            "setp.ge.and.s64 pf, %5, %6, !pr;\n\t"
            "or.pred pa, pr, pf;\n\t"
            "setp.lt.or.f64 pz, %4, %7, pa;\n\t"
            "selp.f64 %0, %7, %4, pz;\n\t"
            "@pf mov.b32 %1, %8;\n\t"
            "@pf or.b32 %2, %2, %9;\n\t}"
            : "=d"(v), "+r"(live_from), "+r"(m)
            : "r"(s), "d"(vn), "l"(__double_as_longlong(vn)), "l"(ph.vt_bits), "d"(ph.el), "r"(relive),
              "r"(1u << bit));
    } else {
        asm("{\n\t.reg .pred pr, pf, pa, pz;\n\t"
            "setp.lt.s32 pr, %3, %1;\n\t"
            "setp.ge.and.f64 pf, %4, %5, !pr;\n\t"
            "or.pred pa, pr, pf;\n\t"
            "setp.lt.or.f64 pz, %4, %6, pa;\n\t"
            "selp.f64 %0, %6, %4, pz;\n\t"
            "@pf mov.b32 %1, %7;\n\t"
            "@pf or.b32 %2, %2, %8;\n\t}"
            : "=d"(v), "+r"(live_from), "+r"(m)
            : "r"(s), "d"(vn), "d"(ph.vt), "d"(ph.el), "r"(relive), "r"(1u << bit));
    }
}

// All 12 features of one lane with the default bank: 4 Sobel currents, their
// exact negations (fma(x,-w,-a) == -fma(x,w,a) under round-to-nearest-even),
// and 4 corner currents -- 60 FMAs instead of 108.
template <bool SGN>
__device__ __forceinline__ unsigned hidden_step_def(const LifK &ph, const double (&x)[9],
                                                    double (&v)[kNF], int (&live_from)[kNF], int s,
                                                    int relive) {
    unsigned m = 0;
    const double e0 = def_current<0>(x), e1 = def_current<1>(x), e2 = def_current<2>(x), e3 = def_current<3>(x);
    lif_update<SGN>(e0, v[0], live_from[0], s, relive, ph, m, 0);
    lif_update<SGN>(e1, v[1], live_from[1], s, relive, ph, m, 1);
    lif_update<SGN>(e2, v[2], live_from[2], s, relive, ph, m, 2);
    lif_update<SGN>(e3, v[3], live_from[3], s, relive, ph, m, 3);
    lif_update<SGN>(-e0, v[4], live_from[4], s, relive, ph, m, 4);
    lif_update<SGN>(-e1, v[5], live_from[5], s, relive, ph, m, 5);
    lif_update<SGN>(-e2, v[6], live_from[6], s, relive, ph, m, 6);
    lif_update<SGN>(-e3, v[7], live_from[7], s, relive, ph, m, 7);
    lif_update<SGN>(def_current<8>(x), v[8], live_from[8], s, relive, ph, m, 8);
    lif_update<SGN>(def_current<9>(x), v[9], live_from[9], s, relive, ph, m, 9);
    lif_update<SGN>(def_current<10>(x), v[10], live_from[10], s, relive, ph, m, 10);
    lif_update<SGN>(def_current<11>(x), v[11], live_from[11], s, relive, ph, m, 11);
    return m;
}

// Generic bank: one lane's 6 feature neurons (features H*6 .. H*6+5).
template <int H, bool SGN>
__device__ __forceinline__ unsigned hidden_step(const BatchArgs &A, const LifK &ph, const double (&x)[9],
                                                double (&v)[kNF], int (&live_from)[kNF], int s, int relive) {
    double I[kHalf];
#pragma unroll
    for (int f = 0; f < kHalf; ++f) I[f] = __dmul_rn(x[0], A.c.taps[H * kHalf + f][0]);
#pragma unroll
    for (int k = 1; k < 9; ++k)
#pragma unroll
        for (int f = 0; f < kHalf; ++f) I[f] = __fma_rn(x[k], A.c.taps[H * kHalf + f][k], I[f]);
    unsigned m = 0;
#pragma unroll
    for (int f = 0; f < kHalf; ++f) lif_update<SGN>(I[f], v[f], live_from[f], s, relive, ph, m, f);
    return m;
}

// k_hidden: persistent CTAs walk groups of kWPC consecutive work items.  With
// the default bank (DEF) an item is a tile: a warp owns 32 windows x 12
// features.  With a generic bank an item is (tile, half): 32 windows x 6
// features, which keeps the 54 runtime taps of a warp within the register
// budget.  The table chunks form one continuous stream across groups, so the
// TMA ring never drains between groups.
// Per-item partial of G for the steps of one chunk: G_item(s, l) = sum of
// W[k, l] over the item's neurons k spiking at s, in (lane, feature) order.
// One packed warp scan lists the ids of all 8 steps; then lane (j, q) sums
// step j's rows for outputs q, q+4, q+8 sequentially in list order (fixed
// order: deterministic).  Done at the chunk end so the W loads of 8 steps
// overlap other warps' FP64 work; an item's ~46 spiking neurons keep their W
// rows in L1.
constexpr int kPIds = 256;  // ids per chunk staged in shared memory

__device__ __forceinline__ void chunk_partials(const BatchArgs &A, uint16_t *ids, int item, int s0, int nrows,
                                               uint64_t mlo, uint64_t mhi, int id0) {
    const int lane = threadIdx.x & 31;
    const int N = A.c.n_steps;
    double *P = A.partial + (size_t)item * N * kNO;
    uint64_t cA = 0, cB = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        cA |= (uint64_t)__popc((unsigned)(mlo >> (16 * q)) & 0xFFFFu) << (16 * q);
        cB |= (uint64_t)__popc((unsigned)(mhi >> (16 * q)) & 0xFFFFu) << (16 * q);
    }
    uint64_t tA, tB;
    const uint64_t eA = warp_excl_scan_u64(cA, &tA), eB = warp_excl_scan_u64(cB, &tB);
    int base[kChunk + 1];
    base[0] = 0;
#pragma unroll
    for (int j = 0; j < kChunk; ++j)
        base[j + 1] = base[j] + (int)(((j < 4 ? tA : tB) >> (16 * (j & 3))) & 0xFFFF);
    const int total = base[kChunk];
    const int jj = lane >> 2, q = lane & 3;  // lane -> (step jj, outputs q, q+4, q+8)
    if (total <= kPIds) {
        if (total) {
#pragma unroll
            for (int j = 0; j < kChunk; ++j) {
                unsigned mm = (unsigned)((j < 4 ? mlo : mhi) >> (16 * (j & 3))) & 0xFFFFu;
                int k = base[j] + (int)(((j < 4 ? eA : eB) >> (16 * (j & 3))) & 0xFFFF);
                while (mm) {
                    const int f = __ffs(mm) - 1;
                    mm &= mm - 1;
                    ids[k++] = (uint16_t)(id0 + f);
                }
            }
        }
        __syncwarp();
        if (jj < nrows) {
            int lo = 0, hi = 0;
#pragma unroll
            for (int j = 0; j < kChunk; ++j)
                if (j == jj) {
                    lo = base[j];
                    hi = base[j + 1];
                }
            double g0 = 0.0, g1 = 0.0, g2 = 0.0;
            for (int e = lo; e < hi; ++e) {
                const double *row = A.w + (size_t)ids[e] * kNO;
                g0 = __dadd_rn(g0, __ldg(row + q));
                g1 = __dadd_rn(g1, __ldg(row + q + 4));
                if (q < 2) g2 = __dadd_rn(g2, __ldg(row + q + 8));
            }
            double *dst = P + (size_t)(s0 + jj) * kNO;
            dst[q] = g0;
            dst[q + 4] = g1;
            if (q < 2) dst[q + 8] = g2;
        }
        __syncwarp();
        return;
    }
    // rare: more than kPIds spikes in one chunk of one item -- one step at a time, in windows
    for (int j = 0; j < nrows; ++j) {
        const unsigned m = (unsigned)((j < 4 ? mlo : mhi) >> (16 * (j & 3))) & 0xFFFFu;
        int tot;
        const int off = warp_excl_scan_int(__popc(m), &tot);
        double g[3] = {0.0, 0.0, 0.0};
        for (int w0 = 0; w0 < tot; w0 += kPIds) {
            const int wn = min(kPIds, tot - w0);
            int k = off - w0;
            unsigned mm = m;
            while (mm) {
                const int f = __ffs(mm) - 1;
                mm &= mm - 1;
                if (k >= 0 && k < wn) ids[k] = (uint16_t)(id0 + f);
                ++k;
            }
            __syncwarp();
            if (lane < kNO)
                for (int e = 0; e < wn; ++e) g[0] = __dadd_rn(g[0], __ldg(A.w + (size_t)ids[e] * kNO + lane));
            __syncwarp();
        }
        if (lane < kNO) P[(size_t)(s0 + j) * kNO + lane] = g[0];
    }
}

template <bool TRACE, bool DEF, bool RASTER, bool GSUM, bool SGN>
__global__ void __launch_bounds__(kThreads, 5) k_hidden(const BatchArgs A) {
    __shared__ __align__(128) double s_tab[kStages][kChunk * 256];
    __shared__ uint64_t s_full[kStages];
    __shared__ uint16_t s_ids[kWPC][kPIds];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int N = A.c.n_steps;
    const int nchunks = (N + kChunk - 1) / kChunk;
    const int64_t n = A.n_images;
    constexpr int kItemsPerTile = DEF ? 1 : 2;
    const int total = kItemsPerTile * A.tile_base[n];
    const int ngroups = (total + kWPC - 1) / kWPC;
    if ((int)blockIdx.x >= ngroups) return;
    const int my_groups = (ngroups - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
    const int64_t stream_len = (int64_t)my_groups * nchunks;

    auto issue = [&](int64_t q) {
        const int ch = (int)(q % nchunks), b = (int)(q % kStages);
        const int rows = min(kChunk, N - ch * kChunk);
        mbar_expect_tx(&s_full[b], rows * 256 * 8);
        bulk_g2s(s_tab[b], A.ctab + (size_t)ch * kChunk * 256, rows * 256 * 8, &s_full[b]);
    };
    if (tid == 0) {
        for (int b = 0; b < kStages; ++b) mbar_init(&s_full[b], 1);
        fence_mbar_init();
        for (int64_t q = 0; q < kStages && q < stream_len; ++q) issue(q);
    }
    __syncthreads();

    const double el = A.c.lif_hid.el, refr = A.c.lif_hid.refr;
    const LifK ph = lif_k(A.c.lif_hid);
    int64_t q = 0;
    for (int gi = 0; gi < my_groups; ++gi) {
        const int item = ((int)blockIdx.x + gi * (int)gridDim.x) * kWPC + warp;
        const bool live = item < total;  // warp-uniform
        const int gt = DEF ? item : item >> 1, half = DEF ? 0 : item & 1;
        int64_t img = 0;
        int tile = 0, pos = 0, nt = 0;
        if (live) {
            int64_t lo = 0, hi = n - 1;  // last image with tile_base <= gt
            while (lo < hi) {
                const int64_t mid = (lo + hi + 1) >> 1;
                if (A.tile_base[mid] <= gt) lo = mid;
                else hi = mid - 1;
            }
            img = lo;
            tile = gt - A.tile_base[img];
            nt = A.n_tiles[img];
            pos = A.tile_pos[img * (kMaxTiles * kTile) + tile * kTile + lane];
        }
        const bool on = live && pos != 0xFFFF;
        uint32_t lvp[3];  // the 9 pixel levels of this lane's window, 4 per word
        {
            const int p = on ? pos : 0;
            const int r = p / kFmap, col = p % kFmap;
            const uint8_t *im = A.images + img * (kSide * kSide);
            lvp[0] = lvp[1] = lvp[2] = 0;
#pragma unroll
            for (int a = 0; a < 3; ++a)
#pragma unroll
                for (int b = 0; b < 3; ++b) {
                    const int k = a * 3 + b;
                    const uint32_t lev = on ? __ldg(im + (r + a) * kSide + col + b) : 0u;
                    lvp[k >> 2] |= lev << (8 * (k & 3));
                }
        }
        double v[kNF];
        int live_from[kNF];
#pragma unroll
        for (int f = 0; f < kNF; ++f) {
            v[f] = el;
            live_from[f] = 0;
        }
        uint8_t *rout = (RASTER && live) ? A.raster + raster_at(A.tile_base[img], N, nt, 0, tile) + half * kTile + lane
                                         : nullptr;
        const size_t rstride = (size_t)nt * 2 * kTile;
        const int id0 = pos * kNF + half * kHalf;

        for (int ch = 0; ch < nchunks; ++ch, ++q) {
            const int b = (int)(q % kStages);
            const int s0 = ch * kChunk;
            const int nrows = min(kChunk, N - s0);
            if (live) {
                mbar_wait(&s_full[b], (uint32_t)((q / kStages) & 1));
                uint64_t mlo = 0, mhi = 0;  // the chunk's spike masks (16 bits per step)
#pragma unroll 1
                for (int j = 0; j < nrows; ++j) {
                    const int s = s0 + j;
                    const double *T = s_tab[b] + j * 256;
                    double x[9];
#pragma unroll
                    for (int k = 0; k < 9; ++k) x[k] = T[(lvp[k >> 2] >> (8 * (k & 3))) & 0xFFu];
                    const int relive = next_live_step(s, refr);
                    unsigned m;
                    if (DEF) m = hidden_step_def<SGN>(ph, x, v, live_from, s, relive);
                    else m = half ? hidden_step<1, SGN>(A, ph, x, v, live_from, s, relive)
                                  : hidden_step<0, SGN>(A, ph, x, v, live_from, s, relive);
                    if (TRACE && on && A.out.v_hid) {
                        double *dst = A.out.v_hid + ((size_t)img * N + s) * kNH + pos * kNF + half * kHalf;
#pragma unroll
                        for (int f = 0; f < (DEF ? kNF : kHalf); ++f) dst[f] = v[f];
                    }
                    if (RASTER) {
                        rout[(size_t)s * rstride] = (uint8_t)(m & 0x3Fu);
                        if (DEF) rout[(size_t)s * rstride + kTile] = (uint8_t)(m >> kHalf);
                    }
                    if (GSUM) {
                        const unsigned mo = on ? m : 0u;
                        if (j < 4) mlo |= (uint64_t)mo << (16 * j);
                        else mhi |= (uint64_t)mo << (16 * (j - 4));
                    }
                }
                if (GSUM) chunk_partials(A, s_ids[warp], item, s0, nrows, mlo, mhi, id0);
            }
            __syncthreads();  // every warp is done with stage b
            if (tid == 0 && q + kStages < stream_len) issue(q + kStages);
        }
    }
}

// ---------------------------------------------------------------------------
// Output layer state and one step of it (network.py:308-314), lanes 0..9 of
// one warp = the 10 output neurons (lanes 10..31 shadow lane 9, harmlessly).
// Every lane keeps all ten lateral-inhibition traces and advances them from
// the previous step's spike ballot, so the inhibition sum needs no shuffles
// on the serial path (same operations as the reference, so bit-identical).
struct OutState {
    double Af, Bf;           // event-driven feed-forward recursions (slow, fast)
    double ao[kNO], bo[kNO]; // lateral-inhibition kernels of all output neurons
    double v;
    int live_from, cnt;
    unsigned prev;           // output spikes of the previous step (10-bit)
};

__device__ __forceinline__ void out_init(OutState &st, const snn_consts_t &c) {
    st.Af = st.Bf = 0.0;
#pragma unroll
    for (int k = 0; k < kNO; ++k) st.ao[k] = st.bo[k] = 0.0;
    st.v = c.lif_out.el;
    st.live_from = 0;
    st.cnt = 0;
    st.prev = 0u;
}

// Advances one step given G (sum of W rows of hidden neurons spiking now).
// Returns whether this lane's output neuron l fired; *ff_out = c_hidden @ W.
__device__ __forceinline__ bool out_step(OutState &st, const snn_consts_t &c, double G, int s, int l,
                                         double *ff_out) {
    st.Af = __dadd_rn(__dmul_rn(st.Af, c.decay_slow), G);
    st.Bf = __dadd_rn(__dmul_rn(st.Bf, c.decay_fast), G);
    const double ff = __dsub_rn(st.Af, st.Bf);
    double cc[kNO], co = 0.0;
#pragma unroll
    for (int k = 0; k < kNO; ++k) {  // inhibition sees last step's spikes
        const double bump = ((st.prev >> k) & 1u) ? 1.0 : 0.0;
        st.ao[k] = __dadd_rn(__dmul_rn(st.ao[k], c.decay_slow), bump);
        st.bo[k] = __dadd_rn(__dmul_rn(st.bo[k], c.decay_fast), bump);
        cc[k] = __dsub_rn(st.ao[k], st.bo[k]);
        co = k == l ? cc[k] : co;
    }
    const double S = pairwise10(cc);
    const double drive = __dadd_rn(ff, __dmul_rn(c.inhibition, __dsub_rn(S, co)));
    const double cand = lif_candidate(st.v, drive, c.lif_out);
    const bool live = s >= st.live_from;
    const bool fired = live && cand >= c.lif_out.vt;
    if (live) st.v = fired ? c.lif_out.el : cand;
    if (fired) st.live_from = next_live_step(s, c.lif_out.refr);
    st.prev = __ballot_sync(kFull, fired) & 0x3FFu;
    st.cnt += fired ? 1 : 0;
    *ff_out = ff;
    return fired;
}

// ---------------------------------------------------------------------------
// k_output: one warp per image -- G(s) = sum of the image's item partials in
// item order, then the output layer.  For up to kOSteps steps at a time, lane
// i computes G for steps i, i+32, ... (all 10 outputs, 80-byte partial rows
// as double2 loads, all independent) into shared memory; then lanes 0..9 run
// the sequential output layer from shared memory.
constexpr int kOItems = 2 * kMaxTiles;
constexpr int kOSteps = 96;

struct OutSmem {
    double2 G[kOSteps * 5];
};

__global__ void __launch_bounds__(kOutWarps * 32) k_output(const BatchArgs A) {
    extern __shared__ __align__(16) uint8_t osmem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    OutSmem &S = reinterpret_cast<OutSmem *>(osmem)[warp];
    const int64_t img = (int64_t)blockIdx.x * kOutWarps + warp;
    if (img >= A.n_images) return;
    const int N = A.c.n_steps;
    const int ni = A.n_tiles[img] * A.items_per_tile;
    const int l = lane < kNO ? lane : kNO - 1;
    const double2 *P = reinterpret_cast<const double2 *>(A.partial + (size_t)A.tile_base[img] * A.items_per_tile * N * kNO);
    const size_t istride = (size_t)N * 5;  // double2 per item
    const double *Gd = reinterpret_cast<const double *>(S.G);
    OutState st;
    out_init(st, A.c);
    for (int s0 = 0; s0 < N; s0 += kOSteps) {
        const int ns = min(kOSteps, N - s0);
        for (int j = lane; j < ns; j += 32) {
            double2 g[5];
#pragma unroll
            for (int p = 0; p < 5; ++p) g[p] = make_double2(0.0, 0.0);
            const double2 *src = P + (size_t)(s0 + j) * 5;
            for (int i = 0; i < ni; ++i) {
#pragma unroll
                for (int p = 0; p < 5; ++p) {
                    const double2 a = __ldcg(src + i * istride + p);
                    g[p].x = __dadd_rn(g[p].x, a.x);
                    g[p].y = __dadd_rn(g[p].y, a.y);
                }
            }
#pragma unroll
            for (int p = 0; p < 5; ++p) S.G[j * 5 + p] = g[p];
        }
        __syncwarp();
        for (int j = 0; j < ns; ++j) {
            const int s = s0 + j;
            double ff;
            out_step(st, A.c, Gd[j * kNO + l], s, l, &ff);
            if (A.out.out_raster && lane == 0) A.out.out_raster[(size_t)img * N + s] = (uint16_t)st.prev;
            if (lane < kNO) {
                if (A.out.ff) A.out.ff[((size_t)img * N + s) * kNO + lane] = ff;
                if (A.out.v_out) A.out.v_out[((size_t)img * N + s) * kNO + lane] = st.v;
            }
        }
        __syncwarp();
    }
    if (lane < kNO) A.out.counts[(size_t)img * kNO + lane] = st.cnt;
}

constexpr size_t kOutSmemBytes = sizeof(OutSmem) * kOutWarps;

}  // namespace snn
