// Inference hot path: input table, fused stencil + hidden LIF + event-driven
// classifier contraction, and the 10-neuron output layer.  sm_100a.
//
// Reference behaviour (relative to /root/reference/pkg/src/spikedigits):
//   _input_tables          network.py:224-245  -> k_input_table
//   hidden_current_series  network.py:254-264  -> stencil inside k_hidden
//   run_presentation       network.py:267-326  -> k_hidden (+ scan_step)
//   lif_step / kernel_step neurons.py:83-171   -> snn_common.cuh helpers
//
// Work decomposition:
//   * a "tile" is 32 consecutive ACTIVE window positions of one image (a
//     window is active when any of its 9 pixels is non-zero; inactive windows
//     receive exactly zero current and never leave rest, so skipping them is
//     exact).  One warp owns one tile; each lane owns one window position and
//     its 12 feature neurons, keeping v and the refractory horizon in
//     registers for the whole trial.
//   * the per-step input traces come from the 256-level table, staged 8 steps
//     at a time into shared memory; the 3x3 stencil is the k-ordered FMA
//     chain OpenBLAS uses for np.tensordot, so currents are bit-identical.
//   * c_hidden @ W is computed event-driven: every hidden kernel trace is a
//     linear recursion in its own spikes, so sum_k c_k(n) W[k,l] =
//     A_l(n) - B_l(n) with A_l(n) = A_l(n-1)*e^{-dt/t1} + G_l(n), where G_l(n)
//     is the sum of the W rows of the neurons spiking at step n.  Each warp
//     writes its G partial per step; the last warp of an image to finish
//     (atomic arrival counter) reduces the partials in fixed tile order and
//     runs the sequential output layer.  Every reduction has a fixed order, so
//     results are deterministic run to run.
#pragma once
#include "snn_common.cuh"

namespace snn {

constexpr int kWPC = 4;                                // warps (tiles) per CTA
constexpr int kThreads = kWPC * 32;
constexpr int kChunk = 8;                              // table steps per smem stage
constexpr int kGroups = (kMaxTiles + kWPC - 1) / kWPC; // CTAs per image

struct HiddenArgs {
    snn_consts_t c;
    const uint8_t *images;
    int64_t n_images;
    const double *w;
    const double *ctab;
    double *partial;   // [n][22][N][10] per-tile G partials (GSUM)
    int *arrive;       // [n] arrival counters (zero on entry, reset on exit)
    snn_infer_out_t out;
};

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
// Ordered compaction of the active window positions of one image (CTA-wide).
__device__ __forceinline__ int compact_windows(const uint8_t *s_img, uint16_t *s_pos, int *s_cnt) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int kIters = (kNPos + kThreads - 1) / kThreads;
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
#pragma unroll
    for (int it = 0; it < kIters; ++it)
        if ((bal[it] >> lane) & 1u)
            s_pos[off[it] + __popc(bal[it] & ((1u << lane) - 1u))] = (uint16_t)(it * kThreads + tid);
    __syncthreads();
    return run;
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

// Inference output layer: G for 32 steps at a time reduced from the tile
// partials in tile order into s_buf, then scanned.  One full warp.
__device__ void infer_output_layer(const HiddenArgs &A, int64_t img, int ntiles, double *s_buf) {
    const int lane = threadIdx.x & 31;
    const int N = A.c.n_steps;
    const int l = lane < kNO ? lane : kNO - 1;
    const double *P = A.partial + (size_t)img * kMaxTiles * N * kNO;
    OutState st;
    out_init(st, A.c);
    for (int s0 = 0; s0 < N; s0 += 32) {
        const int ns = min(32, N - s0);
        if (lane < ns) {
            double G[kNO];
#pragma unroll
            for (int k = 0; k < kNO; ++k) G[k] = 0.0;
            for (int t = 0; t < ntiles; ++t) {
                const double *src = P + ((size_t)t * N + s0 + lane) * kNO;
#pragma unroll
                for (int k = 0; k < kNO; ++k) G[k] = __dadd_rn(G[k], ldcg(src + k));
            }
#pragma unroll
            for (int k = 0; k < kNO; ++k) s_buf[lane * kNO + k] = G[k];
        }
        __syncwarp();
        for (int j = 0; j < ns; ++j) {
            const int s = s0 + j;
            double ff;
            const bool fired = out_step(st, A.c, s_buf[j * kNO + l], s, &ff);
            const unsigned om = __ballot_sync(kFull, fired) & 0x3FFu;
            if (A.out.out_raster && lane == 0) A.out.out_raster[(size_t)img * N + s] = (uint16_t)om;
            if (lane < kNO) {
                if (A.out.ff) A.out.ff[((size_t)img * N + s) * kNO + lane] = ff;
                if (A.out.v_out) A.out.v_out[((size_t)img * N + s) * kNO + lane] = st.v;
            }
        }
        __syncwarp();
    }
    if (lane < kNO) A.out.counts[(size_t)img * kNO + lane] = st.cnt;
}

// ---------------------------------------------------------------------------
// The fused hidden-layer kernel.  grid = n_images * kGroups CTAs of kWPC warps.
//   GSUM   : per-step G partials + last-arriver output layer (inference)
//   RASTER : per-lane 12-bit spike masks per step (training / forward_pass)
//   TRACE  : hidden membrane after every step (parity tests)
template <bool GSUM, bool RASTER, bool TRACE>
__global__ void __launch_bounds__(kThreads) k_hidden(const HiddenArgs A) {
    __shared__ __align__(16) double s_tab[kChunk * 256];
    __shared__ __align__(16) uint8_t s_img[kSide * kSide];
    __shared__ uint16_t s_pos[kNPos + 4];
    __shared__ int s_cnt[8 * kWPC];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t img = blockIdx.x / kGroups;
    const int grp = blockIdx.x % kGroups;
    const int N = A.c.n_steps;

    // stage the image (784 B = 49 x 16 B)
    const uint8_t *gimg = A.images + img * (kSide * kSide);
    if (tid < 49) reinterpret_cast<uint4 *>(s_img)[tid] = __ldg(reinterpret_cast<const uint4 *>(gimg) + tid);
    __syncthreads();
    const int n_act = compact_windows(s_img, s_pos, s_cnt);
    const int ntiles = (n_act + kTile - 1) / kTile;
    if (RASTER && grp == 0 && tid == 0 && A.out.n_tiles) A.out.n_tiles[img] = ntiles;
    if (ntiles == 0) {
        // blank image: the hidden layer stays at rest and G == 0 every step
        if (GSUM && grp == 0 && warp == 0) infer_output_layer(A, img, 0, s_tab);
        return;
    }
    if (grp * kWPC >= ntiles) return;  // whole CTA beyond the image's tiles

    const int tile = grp * kWPC + warp;
    const bool live = tile < ntiles;  // warp-uniform
    const int slot = tile * kTile + lane;
    const bool on = live && slot < n_act;
    const int pos = on ? s_pos[slot] : 0;
    if (RASTER && live && A.out.tile_pos)
        A.out.tile_pos[((size_t)img * kMaxTiles + tile) * kTile + lane] = on ? (uint16_t)pos : (uint16_t)0xFFFF;

    // the 9 pixel levels of this lane's window = column offsets into a table row
    int lv[9];
    {
        const int r = pos / kFmap, col = pos % kFmap;
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int b = 0; b < 3; ++b) lv[a * 3 + b] = on ? s_img[(r + a) * kSide + col + b] : 0;
    }

    const snn_lif_t &ph = A.c.lif_hid;
    double v[kNF];
    int live_from[kNF];
#pragma unroll
    for (int f = 0; f < kNF; ++f) {
        v[f] = ph.el;
        live_from[f] = 0;
    }
    double *Pt = GSUM ? A.partial + ((size_t)img * kMaxTiles + tile) * N * kNO : nullptr;
    uint16_t *Rt = RASTER ? A.out.raster + ((size_t)img * kMaxTiles + tile) * N * kTile : nullptr;
    const double *wbase = A.w + (lane < kNO ? lane : 0);

    for (int s0 = 0; s0 < N; s0 += kChunk) {
        const int nrows = min(kChunk, N - s0);
        __syncthreads();
        {
            const double2 *src = reinterpret_cast<const double2 *>(A.ctab + (size_t)s0 * 256);
            double2 *dst = reinterpret_cast<double2 *>(s_tab);
            for (int i = tid; i < nrows * 128; i += kThreads) dst[i] = __ldg(src + i);
        }
        __syncthreads();
        if (!live) continue;
        for (int j = 0; j < nrows; ++j) {
            const int s = s0 + j;
            const double *T = s_tab + j * 256;
            double x[9];
#pragma unroll
            for (int k = 0; k < 9; ++k) x[k] = T[lv[k]];
            const int relive = next_live_step(s, ph.refr);
            unsigned m = 0;
#pragma unroll
            for (int f = 0; f < kNF; ++f) {
                // network.py:220 -- dgemm's k-ordered FMA chain over the 9 taps
                double I = __dmul_rn(x[0], A.c.taps[f][0]);
#pragma unroll
                for (int k = 1; k < 9; ++k) I = __fma_rn(x[k], A.c.taps[f][k], I);
                const double cand = lif_candidate(v[f], I, ph);
                const bool ok = s >= live_from[f];
                const bool fired = ok && cand >= ph.vt;
                v[f] = ok ? (fired ? ph.el : cand) : v[f];
                live_from[f] = fired ? relive : live_from[f];
                m |= (fired ? 1u : 0u) << f;
            }
            if (TRACE && on && A.out.v_hid) {
                double *dst = A.out.v_hid + ((size_t)img * N + s) * kNH + pos * kNF;
#pragma unroll
                for (int f = 0; f < kNF; ++f) dst[f] = v[f];
            }
            if (RASTER) Rt[(size_t)s * kTile + lane] = (uint16_t)m;
            if (GSUM) {
                unsigned bal = __ballot_sync(kFull, m != 0);
                double g = 0.0;
                while (bal) {
                    const int src = __ffs(bal) - 1;
                    bal &= bal - 1;
                    unsigned mm = __shfl_sync(kFull, m, src);
                    const int pp = __shfl_sync(kFull, pos, src);
                    const double *wr = wbase + (size_t)pp * (kNF * kNO);
                    while (mm) {
                        const int f = __ffs(mm) - 1;
                        mm &= mm - 1;
                        if (lane < kNO) g = __dadd_rn(g, __ldg(wr + f * kNO));
                    }
                }
                if (lane < kNO) Pt[(size_t)s * kNO + lane] = g;
            }
        }
    }
    if (GSUM) {
        __syncthreads();  // every warp of this CTA is done with s_tab
        if (live) {
            __threadfence();
            int prev = 0;
            if (lane == 0) prev = atomicAdd(A.arrive + img, 1);
            prev = __shfl_sync(kFull, prev, 0);
            if (prev == ntiles - 1) {
                __threadfence();
                infer_output_layer(A, img, ntiles, s_tab);
                if (lane == 0) A.arrive[img] = 0;
            }
        }
    }
}

}  // namespace snn
