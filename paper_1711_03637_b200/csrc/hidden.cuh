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

__device__ __forceinline__ void lif_update(double I, double &v, int &live_from, int s, int relive,
                                           const snn_lif_t &ph, unsigned &m, int bit) {
    const double cand = lif_candidate(v, I, ph);
    const bool ok = s >= live_from;
    const bool fired = ok && cand >= ph.vt;
    v = ok ? (fired ? ph.el : cand) : v;
    live_from = fired ? relive : live_from;
    m |= (fired ? 1u : 0u) << bit;
}

// All 12 features of one lane with the default bank: 4 Sobel currents, their
// exact negations (fma(x,-w,-a) == -fma(x,w,a) under round-to-nearest-even),
// and 4 corner currents -- 60 FMAs instead of 108.
__device__ __forceinline__ unsigned hidden_step_def(const snn_lif_t &ph, const double (&x)[9],
                                                    double (&v)[kNF], int (&live_from)[kNF], int s,
                                                    int relive) {
    unsigned m = 0;
    const double e0 = def_current<0>(x), e1 = def_current<1>(x), e2 = def_current<2>(x), e3 = def_current<3>(x);
    lif_update(e0, v[0], live_from[0], s, relive, ph, m, 0);
    lif_update(e1, v[1], live_from[1], s, relive, ph, m, 1);
    lif_update(e2, v[2], live_from[2], s, relive, ph, m, 2);
    lif_update(e3, v[3], live_from[3], s, relive, ph, m, 3);
    lif_update(-e0, v[4], live_from[4], s, relive, ph, m, 4);
    lif_update(-e1, v[5], live_from[5], s, relive, ph, m, 5);
    lif_update(-e2, v[6], live_from[6], s, relive, ph, m, 6);
    lif_update(-e3, v[7], live_from[7], s, relive, ph, m, 7);
    lif_update(def_current<8>(x), v[8], live_from[8], s, relive, ph, m, 8);
    lif_update(def_current<9>(x), v[9], live_from[9], s, relive, ph, m, 9);
    lif_update(def_current<10>(x), v[10], live_from[10], s, relive, ph, m, 10);
    lif_update(def_current<11>(x), v[11], live_from[11], s, relive, ph, m, 11);
    return m;
}

// Generic bank: one lane's 6 feature neurons (features H*6 .. H*6+5).
template <int H>
__device__ __forceinline__ unsigned hidden_step(const BatchArgs &A, const double (&x)[9], double (&v)[kNF],
                                                int (&live_from)[kNF], int s, int relive) {
    const snn_lif_t &ph = A.c.lif_hid;
    double I[kHalf];
#pragma unroll
    for (int f = 0; f < kHalf; ++f) I[f] = __dmul_rn(x[0], A.c.taps[H * kHalf + f][0]);
#pragma unroll
    for (int k = 1; k < 9; ++k)
#pragma unroll
        for (int f = 0; f < kHalf; ++f) I[f] = __fma_rn(x[k], A.c.taps[H * kHalf + f][k], I[f]);
    unsigned m = 0;
#pragma unroll
    for (int f = 0; f < kHalf; ++f) lif_update(I[f], v[f], live_from[f], s, relive, ph, m, f);
    return m;
}

// k_hidden: persistent CTAs walk groups of kWPC consecutive work items.  With
// the default bank (DEF) an item is a tile: a warp owns 32 windows x 12
// features.  With a generic bank an item is (tile, half): 32 windows x 6
// features, which keeps the 54 runtime taps of a warp within the register
// budget.  The table chunks form one continuous stream across groups, so the
// TMA ring never drains between groups.
template <bool TRACE, bool DEF>
__global__ void __launch_bounds__(kThreads, 5) k_hidden(const BatchArgs A) {
    __shared__ __align__(128) double s_tab[kStages][kChunk * 256];
    __shared__ uint64_t s_full[kStages];
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
        uint8_t *rout = live ? A.raster + raster_at(A.tile_base[img], N, nt, 0, tile) + half * kTile + lane : nullptr;
        const size_t rstride = (size_t)nt * 2 * kTile;

        for (int ch = 0; ch < nchunks; ++ch, ++q) {
            const int b = (int)(q % kStages);
            const int s0 = ch * kChunk;
            const int nrows = min(kChunk, N - s0);
            if (live) {
                mbar_wait(&s_full[b], (uint32_t)((q / kStages) & 1));
#pragma unroll 1
                for (int j = 0; j < nrows; ++j) {
                    const int s = s0 + j;
                    const double *T = s_tab[b] + j * 256;
                    double x[9];
#pragma unroll
                    for (int k = 0; k < 9; ++k) x[k] = T[(lvp[k >> 2] >> (8 * (k & 3))) & 0xFFu];
                    const int relive = next_live_step(s, refr);
                    unsigned m;
                    if (DEF) m = hidden_step_def(A.c.lif_hid, x, v, live_from, s, relive);
                    else m = half ? hidden_step<1>(A, x, v, live_from, s, relive)
                                  : hidden_step<0>(A, x, v, live_from, s, relive);
                    if (TRACE && on && A.out.v_hid) {
                        double *dst = A.out.v_hid + ((size_t)img * N + s) * kNH + pos * kNF + half * kHalf;
#pragma unroll
                        for (int f = 0; f < (DEF ? kNF : kHalf); ++f) dst[f] = v[f];
                    }
                    rout[(size_t)s * rstride] = (uint8_t)(m & 0x3Fu);
                    if (DEF) rout[(size_t)s * rstride + kTile] = (uint8_t)(m >> kHalf);
                }
            }
            __syncthreads();  // every warp is done with stage b
            if (tid == 0 && q + kStages < stream_len) issue(q + kStages);
        }
    }
}

// ---------------------------------------------------------------------------
// Output layer state and one step of it (network.py:308-314), lanes 0..9 of
// one warp = the 10 output neurons (lanes 10..31 shadow lane 9, harmlessly).
struct OutState {
    double Af, Bf;   // event-driven feed-forward recursions (slow, fast)
    double ao, bo;   // lateral-inhibition kernel of this output neuron
    double v;
    int live_from, cnt;
    bool prev;
};

__device__ __forceinline__ void out_init(OutState &st, const snn_consts_t &c) {
    st.Af = st.Bf = st.ao = st.bo = 0.0;
    st.v = c.lif_out.el;
    st.live_from = 0;
    st.cnt = 0;
    st.prev = false;
}

// Advances one step given G (sum of W rows of hidden neurons spiking now).
// Returns whether this lane's output neuron fired; *ff_out = c_hidden @ W.
__device__ __forceinline__ bool out_step(OutState &st, const snn_consts_t &c, double G, int s,
                                         double *ff_out) {
    st.Af = __dadd_rn(__dmul_rn(st.Af, c.decay_slow), G);
    st.Bf = __dadd_rn(__dmul_rn(st.Bf, c.decay_fast), G);
    const double ff = __dsub_rn(st.Af, st.Bf);
    const double bump = st.prev ? 1.0 : 0.0;  // inhibition sees last step's spikes
    st.ao = __dadd_rn(__dmul_rn(st.ao, c.decay_slow), bump);
    st.bo = __dadd_rn(__dmul_rn(st.bo, c.decay_fast), bump);
    const double co = __dsub_rn(st.ao, st.bo);
    double cc[kNO];
#pragma unroll
    for (int k = 0; k < kNO; ++k) cc[k] = __shfl_sync(kFull, co, k);
    const double S = pairwise10(cc);
    const double drive = __dadd_rn(ff, __dmul_rn(c.inhibition, __dsub_rn(S, co)));
    const double cand = lif_candidate(st.v, drive, c.lif_out);
    const bool live = s >= st.live_from;
    const bool fired = live && cand >= c.lif_out.vt;
    if (live) st.v = fired ? c.lif_out.el : cand;
    if (fired) st.live_from = next_live_step(s, c.lif_out.refr);
    st.prev = fired;
    st.cnt += fired ? 1 : 0;
    *ff_out = ff;
    return fired;
}

// ---------------------------------------------------------------------------
// k_output: one warp per image -- G from the raster and W, then the output
// layer, one step at a time.  A step's raster segment is contiguous (nt x 64
// bytes), so the warp loads it with 16-byte vector loads, lists the spiking
// neurons in raster memory order (tile, half, lane, feature) with one popc +
// one warp scan, and 30 lanes add their W rows: lane q*10+l sums a strided
// third for output l, combined as (g0 + g1) + g2 -- a fixed order, so G is
// deterministic.  W rows are plain L1-cached loads: an image's ~1,000
// spiking neurons fire ~7 times each.  G(s) feeds the output layer directly.
constexpr int kIdCap = 512;  // spike ids per round (a step has ~70 on MNIST-like input)

struct OutSmem {
    uint16_t pos[kMaxTiles * kTile];
    uint16_t ids[kIdCap];
};

__global__ void __launch_bounds__(kOutWarps * 32) k_output(const BatchArgs A) {
    extern __shared__ __align__(16) uint8_t osmem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    OutSmem &S = reinterpret_cast<OutSmem *>(osmem)[warp];
    const int64_t img = (int64_t)blockIdx.x * kOutWarps + warp;
    if (img >= A.n_images) return;
    const int N = A.c.n_steps;
    const int nt = A.n_tiles[img];
    const int64_t tb = A.tile_base[img];
    const int l = lane < kNO ? lane : kNO - 1;
    const int q3 = lane / kNO, lq = lane - q3 * kNO;
    const double *W = A.w;
    for (int k = lane; k < nt * kTile; k += 32) S.pos[k] = A.tile_pos[img * (kMaxTiles * kTile) + k];
    __syncwarp();
    const int nvec = nt * 4;  // uint4 per step segment (64 B per tile)
    constexpr int kMaxVec = (kMaxTiles * 4 + 31) / 32;

    OutState st;
    out_init(st, A.c);
    uint4 cur[kMaxVec], nxt[kMaxVec];
    auto load_step = [&](int s, uint4 (&v)[kMaxVec]) {
        const uint4 *src = reinterpret_cast<const uint4 *>(A.raster + raster_at(tb, N, nt, s, 0));
#pragma unroll
        for (int r = 0; r < kMaxVec; ++r) {
            const int k = lane + 32 * r;
            v[r] = k < nvec ? __ldcg(src + k) : make_uint4(0, 0, 0, 0);
        }
    };
    if (N > 0) load_step(0, cur);
    for (int s = 0; s < N; ++s) {
        if (s + 1 < N) load_step(s + 1, nxt);
        int c = 0;
#pragma unroll
        for (int r = 0; r < kMaxVec; ++r) c += __popc(cur[r].x) + __popc(cur[r].y) + __popc(cur[r].z) + __popc(cur[r].w);
        int tot;
        const int off = warp_excl_scan_int(c, &tot);
        double G = 0.0;
        for (int w0 = 0; w0 < tot; w0 += kIdCap) {  // rounds of kIdCap ids (one round in practice)
            const int wn = min(kIdCap, tot - w0);
            int k = off - w0;
#pragma unroll
            for (int r = 0; r < kMaxVec; ++r) {
                const uint32_t wv[4] = {cur[r].x, cur[r].y, cur[r].z, cur[r].w};
#pragma unroll
                for (int wi = 0; wi < 4; ++wi) {
                    uint32_t bits = wv[wi];
                    while (bits) {
                        const int b = __ffs(bits) - 1;
                        bits &= bits - 1;
                        if (k >= 0 && k < wn) {
                            // byte index in the step segment -> (tile, half, lane), bit -> feature
                            const int by = (lane + 32 * r) * 16 + wi * 4 + (b >> 3);
                            const int t = by >> 6, half = (by >> 5) & 1, ln = by & 31;
                            S.ids[k] = (uint16_t)(S.pos[t * kTile + ln] * kNF + half * kHalf + (b & 7));
                        }
                        ++k;
                    }
                }
            }
            __syncwarp();
            double g = 0.0;
            if (q3 < 3)
                for (int e = q3; e < wn; e += 3) g = __dadd_rn(g, __ldg(W + (size_t)S.ids[e] * kNO + lq));
            const double g1 = __shfl_down_sync(kFull, g, kNO), g2 = __shfl_down_sync(kFull, g, 2 * kNO);
            G = __dadd_rn(G, __dadd_rn(__dadd_rn(g, g1), g2));  // valid on lanes 0..9
            __syncwarp();
        }
        G = __shfl_sync(kFull, G, l);
        double ff;
        const bool fired = out_step(st, A.c, G, s, &ff);
        const unsigned om = __ballot_sync(kFull, fired) & 0x3FFu;
        if (A.out.out_raster && lane == 0) A.out.out_raster[(size_t)img * N + s] = (uint16_t)om;
        if (lane < kNO) {
            if (A.out.ff) A.out.ff[((size_t)img * N + s) * kNO + lane] = ff;
            if (A.out.v_out) A.out.v_out[((size_t)img * N + s) * kNO + lane] = st.v;
        }
#pragma unroll
        for (int r = 0; r < kMaxVec; ++r) cur[r] = nxt[r];
    }
    if (lane < kNO) A.out.counts[(size_t)img * kNO + lane] = st.cnt;
}

constexpr size_t kOutSmemBytes = sizeof(OutSmem) * kOutWarps;

}  // namespace snn
