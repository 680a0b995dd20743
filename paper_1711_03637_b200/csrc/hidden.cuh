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
//                for np.tensordot, so currents are bit-identical.  Output: the
//                spike raster, 6-bit masks per lane, step and feature half,
//                stored once per 8-step chunk (two 8-byte stores per lane).
//   k_output     one warp per image.  c_hidden @ W is event-driven: every
//                hidden kernel trace is a linear recursion in its own spikes,
//                so sum_k c_k(n) W[k,l] = A_l(n) - B_l(n) with
//                A_l(n) = A_l(n-1) e^{-dt/t1} + G_l(n), G_l(n) = sum of the W
//                rows of the neurons spiking at n.  Per chunk the warp turns
//                the raster into per-step spike lists (ascending neuron id),
//                sums the W rows of each list in that order and runs the
//                10-neuron output layer.
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

// Raster layout (bytes; include/snn_b200.h): image i owns the block starting at
// tile_base[i] * nchunks * 512, laid out [chunk][tile][half][lane][8 steps];
// each byte is the 6-bit spike mask of features half*6 .. half*6+5 of the
// lane's window at step chunk*8 + j (0 past the last step).
constexpr int kRastTC = 2 * kTile * kChunk;  // 512 bytes per (tile, chunk)

__host__ __device__ inline int n_chunks(int N) { return (N + kChunk - 1) / kChunk; }

__host__ __device__ inline size_t raster_tc(int64_t tile_base_img, int nchunks, int ntiles, int ch, int t) {
    return ((size_t)tile_base_img * nchunks + (size_t)ch * ntiles + t) * kRastTC;
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
    int32_t *n_win;          // [n]   active windows per image
    int32_t *win_base;       // [n+1] exclusive prefix of n_win
    uint8_t *raster;         // sum(n_tiles) * nchunks * 512 spike-mask bytes (see raster_tc)
    int32_t items_per_tile;  // 1 (default bank) or 2 (generic bank)
    snn_infer_out_t out;     // counts / out_raster / ff / v_out / v_hid / near_ties
    double *gabs;            // [n][N][10] |W| sums (near_ties only)
    int32_t *fix_count;      // guard-band hidden layer (hidden_gb.cuh): flagged windows
    int32_t *fix_list;       // [n * 676] their indices in the compacted window list
    double *wpad;            // [8112][16] W rows padded to 128 bytes (k_prep -> k_gsum), or null
};

// W row stride of the contraction's gathers: 16 doubles (one 128-byte line per
// row, copied by k_prep) for large batches, the caller's 10 otherwise
constexpr int kWPad = 16;
constexpr int kWPadMinImages = 256;

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
    if (A.wpad)  // the contraction's padded W rows: a few pairs per CTA
        for (int64_t t = img * kThreads + tid; t < kNH * kNO / 2; t += (int64_t)gridDim.x * kThreads) {
            const int row = (int)(t / (kNO / 2)), q = (int)(t - (int64_t)row * (kNO / 2));
            reinterpret_cast<double2 *>(A.wpad + (size_t)row * kWPad)[q] = __ldg(reinterpret_cast<const double2 *>(A.w) + t);
        }
    // Skipping all-zero windows is exact only while pixel level 0 never
    // spikes (its input trace, table column 0, stays +0).  The reference
    // accepts i_0 within rel_tol 1e-9 of the rheobase (network.py:133-136),
    // and just above it level 0 does spike in long trials: then every window
    // is simulated.
    int lv0 = 0;
    for (int s = tid; s < A.c.n_steps; s += kThreads) lv0 |= __ldg(A.ctab + (size_t)s * 256) != 0.0;
    const bool all_on = __syncthreads_or(lv0) != 0;
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
            on |= all_on;
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
    if (tid == 0) {
        A.n_tiles[img] = (run + kTile - 1) / kTile;
        A.n_win[img] = run;
    }
}

// k_tile_scan: tile_base / win_base = exclusive prefixes of n_tiles / n_win;
// one CTA, any n.  Both prefixes in one pass, 8 consecutive images per thread
// per round (8,192 images per round): a 10k-image batch takes two rounds.
__global__ void __launch_bounds__(1024) k_tile_scan(const BatchArgs A) {
    constexpr int kPer = 8;
    __shared__ int s_w[2][32];
    __shared__ int s_carry[2];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t n = A.n_images;
    if (tid < 2) s_carry[tid] = 0;
    if (tid == 0 && A.fix_count) *A.fix_count = 0;  // the guard-band kernel's work list (hidden_gb.cuh)
    __syncthreads();
    for (int64_t base = 0; base < n; base += 1024 * kPer) {
        const int64_t i0 = base + (int64_t)tid * kPer;
        int a[kPer], b[kPer], sa = 0, sb = 0;
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
            const bool in = i0 + k < n;
            a[k] = in ? A.n_tiles[i0 + k] : 0;
            b[k] = in ? A.n_win[i0 + k] : 0;
            const int ta = a[k], tb = b[k];
            a[k] = sa;  // exclusive within the thread
            b[k] = sb;
            sa += ta;
            sb += tb;
        }
        int ta, tb;
        const int ea = warp_excl_scan_int(sa, &ta), eb = warp_excl_scan_int(sb, &tb);
        if (lane == 0) {
            s_w[0][warp] = ta;
            s_w[1][warp] = tb;
        }
        __syncthreads();
        if (warp == 0) {
            int t2, t3;
            const int e2 = warp_excl_scan_int(s_w[0][lane], &t2), e3 = warp_excl_scan_int(s_w[1][lane], &t3);
            s_w[0][lane] = e2 + s_carry[0];
            s_w[1][lane] = e3 + s_carry[1];
            __syncwarp();
            if (lane == 0) {
                s_carry[0] += t2;
                s_carry[1] += t3;
            }
        }
        __syncthreads();
        const int oa = s_w[0][warp] + ea, ob = s_w[1][warp] + eb;
#pragma unroll
        for (int k = 0; k < kPer; ++k)
            if (i0 + k < n) {
                A.tile_base[i0 + k] = oa + a[k];
                A.win_base[i0 + k] = ob + b[k];
            }
        __syncthreads();
    }
    if (tid == 0) {
        A.tile_base[n] = s_carry[0];
        A.win_base[n] = s_carry[1];
    }
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

// The distinct tap magnitudes of the default bank, |coef| * gain in IEEE
// double (2*g1 is an exact doubling, 5*g2 and 4*g2 are numpy's products).
// Read from the constant bank, so every DFMA takes its tap as an operand
// (negative taps as a negated operand) instead of re-materialising 64-bit
// immediates into uniform registers on every step.
__constant__ double c_def_tap[4] = {kG1, 2.0 * kG1, 5.0 * kG2, 4.0 * kG2};

__host__ __device__ constexpr int def_tap_slot(int f, int k) {
    return f < 8 ? (def_coef(f, k) == 1 || def_coef(f, k) == -1 ? 0 : 1) : (def_coef(f, k) == 5 ? 2 : 3);
}

__device__ __forceinline__ double def_tap_c(int f, int k) {
    const double t = c_def_tap[def_tap_slot(f, k)];
    return def_coef(f, k) < 0 ? -t : t;
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
            I = first ? __dmul_rn(x[k], def_tap_c(F, k)) : __fma_rn(x[k], def_tap_c(F, k), I);
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

// The same step when the refractory span is the same at every step (FZ frozen
// steps after a spike, e.g. t_ref/dt = 3 -> 3): a neuron is frozen at step s
// iff it spiked at one of the last FZ steps, so the window keeps its last FZ
// 12-bit spike masks and `frozen` = their OR replaces the per-neuron
// refractory horizon.  Per neuron, pa = frozen || vn >= V_T and v = (pa ||
// vn < E_L) ? E_L : vn; the spikes are the pa bits outside `frozen`, masked
// once per window-step.
// Features whose clamp test (vn < E_L) runs on the FP64 pipe (DSETP) instead
// of the integer pipe (two ISETP on the bit pattern): the loop issues one
// instruction fewer per such feature and the FP64 pipe, no longer the bound,
// absorbs it.  Features 0-5 measured best (k_hidden 2.99 -> 2.94 ms per 10k
// images; other masks 2.98-3.15: the schedule, not the count, decides).
#ifndef SNN_FZ_F64CLAMP
#define SNN_FZ_F64CLAMP 0x3F
#endif
template <bool SGN, bool F64CLAMP>
__device__ __forceinline__ void lif_update_fz(double I, double &v, unsigned frozen, const LifK &ph, unsigned &pm,
                                              int bit) {
    double t = __dsub_rn(v, ph.el);
    t = __dmul_rn(ph.g, t);
    t = __dsub_rn(I, t);
    t = __dmul_rn(ph.beta, t);
    const double vn = __dadd_rn(v, t);
    if (SGN && !F64CLAMP) {
        asm("{\n\t.reg .pred pr, pa, pz;\n\t.reg .b32 q;\n\t"
            "and.b32 q, %2, %5;\n\t"
            "setp.ne.u32 pr, q, 0;\n\t"
            "setp.ge.or.s64 pa, %4, %6, pr;\n\t"
            "setp.gt.or.u64 pz, %4, %8, pa;\n\t"
            "selp.f64 %0, %7, %3, pz;\n\t"
            "@pa or.b32 %1, %1, %5;\n\t}"
            : "=d"(v), "+r"(pm)
            : "r"(frozen), "d"(vn), "l"(__double_as_longlong(vn)), "r"(1u << bit), "l"(ph.vt_bits), "d"(ph.el),
              "l"(ph.el_bits));
    } else if (SGN) {
        asm("{\n\t.reg .pred pr, pa, pz;\n\t.reg .b32 q;\n\t"
            "and.b32 q, %2, %5;\n\t"
            "setp.ne.u32 pr, q, 0;\n\t"
            "setp.ge.or.s64 pa, %4, %6, pr;\n\t"
            "setp.lt.or.f64 pz, %3, %7, pa;\n\t"
            "selp.f64 %0, %7, %3, pz;\n\t"
            "@pa or.b32 %1, %1, %5;\n\t}"
            : "=d"(v), "+r"(pm)
            : "r"(frozen), "d"(vn), "l"(__double_as_longlong(vn)), "r"(1u << bit), "l"(ph.vt_bits), "d"(ph.el));
    } else {
        asm("{\n\t.reg .pred pr, pa, pz;\n\t.reg .b32 q;\n\t"
            "and.b32 q, %2, %4;\n\t"
            "setp.ne.u32 pr, q, 0;\n\t"
            "setp.ge.or.f64 pa, %3, %5, pr;\n\t"
            "setp.lt.or.f64 pz, %3, %6, pa;\n\t"
            "selp.f64 %0, %6, %3, pz;\n\t"
            "@pa or.b32 %1, %1, %4;\n\t}"
            : "=d"(v), "+r"(pm)
            : "r"(frozen), "d"(vn), "r"(1u << bit), "d"(ph.vt), "d"(ph.el));
    }
}

template <bool SGN>
__device__ __forceinline__ unsigned hidden_step_def_fz(const LifK &ph, const double (&x)[9], double (&v)[kNF],
                                                       unsigned frozen) {
    unsigned pm = 0;
    const double e0 = def_current<0>(x), e1 = def_current<1>(x), e2 = def_current<2>(x), e3 = def_current<3>(x);
    lif_update_fz<SGN, ((SNN_FZ_F64CLAMP >> 0) & 1) != 0>(e0, v[0], frozen, ph, pm, 0);
    lif_update_fz<SGN, ((SNN_FZ_F64CLAMP >> 1) & 1) != 0>(e1, v[1], frozen, ph, pm, 1);
    lif_update_fz<SGN, ((SNN_FZ_F64CLAMP >> 2) & 1) != 0>(e2, v[2], frozen, ph, pm, 2);
    lif_update_fz<SGN, ((SNN_FZ_F64CLAMP >> 3) & 1) != 0>(e3, v[3], frozen, ph, pm, 3);
    lif_update_fz<SGN, ((SNN_FZ_F64CLAMP >> 4) & 1) != 0>(-e0, v[4], frozen, ph, pm, 4);
    lif_update_fz<SGN, ((SNN_FZ_F64CLAMP >> 5) & 1) != 0>(-e1, v[5], frozen, ph, pm, 5);
    lif_update_fz<SGN, ((SNN_FZ_F64CLAMP >> 6) & 1) != 0>(-e2, v[6], frozen, ph, pm, 6);
    lif_update_fz<SGN, ((SNN_FZ_F64CLAMP >> 7) & 1) != 0>(-e3, v[7], frozen, ph, pm, 7);
    lif_update_fz<SGN, ((SNN_FZ_F64CLAMP >> 8) & 1) != 0>(def_current<8>(x), v[8], frozen, ph, pm, 8);
    lif_update_fz<SGN, ((SNN_FZ_F64CLAMP >> 9) & 1) != 0>(def_current<9>(x), v[9], frozen, ph, pm, 9);
    lif_update_fz<SGN, ((SNN_FZ_F64CLAMP >> 10) & 1) != 0>(def_current<10>(x), v[10], frozen, ph, pm, 10);
    lif_update_fz<SGN, ((SNN_FZ_F64CLAMP >> 11) & 1) != 0>(def_current<11>(x), v[11], frozen, ph, pm, 11);
    return pm & ~frozen;
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

// k_hidden work items: the active windows of the whole batch, image after
// image, cut into groups of 32 (one per warp; with a generic bank an item is
// a group and one half of the features, which keeps the 54 runtime taps of a
// warp within the register budget).  A group may span two images: every lane
// finds its own image and writes its masks into that image's raster block,
// so no lane idles at image boundaries.
struct ItemState {
    int64_t img;
    int pos, half;
    bool live, on;
    uint32_t lvp[3];  // the 9 pixel levels of this lane's window, 4 per word
    uint8_t *rout;    // this lane's raster bytes of chunk 0
    size_t rstride;   // one chunk of this lane's image
};

__device__ __forceinline__ int hidden_items(const BatchArgs &A, int ipt) {
    return ipt * ((A.win_base[A.n_images] + kTile - 1) / kTile);
}

// One window of the batch (gw: index in the batch's compacted window list,
// image after image): its image, position, pixel levels and raster slot.
// `live` is warp-uniform (the work item exists); lanes past the batch's last
// window get pos = 0xFFFF (on = false).
__device__ __forceinline__ void window_setup(const BatchArgs &A, bool live, int gw, int half, int nchunks,
                                             ItemState &it) {
    const int64_t n = A.n_images;
    it.live = live;
    it.half = half;
    it.img = 0;
    it.pos = 0xFFFF;
    it.rout = nullptr;
    it.rstride = 0;
    if (it.live && gw < A.win_base[n]) {
        int64_t lo = 0, hi = n - 1;  // last image with win_base <= gw
        while (lo < hi) {
            const int64_t mid = (lo + hi + 1) >> 1;
            if (A.win_base[mid] <= gw) lo = mid;
            else hi = mid - 1;
        }
        it.img = lo;
        const int w = gw - A.win_base[lo];
        const int nt = A.n_tiles[lo];
        it.pos = A.tile_pos[lo * (kMaxTiles * kTile) + w];
        it.rout = A.raster + raster_tc(A.tile_base[lo], nchunks, nt, 0, w / kTile) + it.half * (kRastTC / 2) +
                  (w % kTile) * kChunk;
        it.rstride = (size_t)nt * kRastTC;
    }
    it.on = it.pos != 0xFFFF;
    const int p = it.on ? it.pos : 0;
    const int r = p / kFmap, col = p % kFmap;
    const uint8_t *im = A.images + it.img * (kSide * kSide);
    it.lvp[0] = it.lvp[1] = it.lvp[2] = 0;
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) {
            const int k = a * 3 + b;
            const uint32_t lev = it.on ? __ldg(im + (r + a) * kSide + col + b) : 0u;
            it.lvp[k >> 2] |= lev << (8 * (k & 3));
        }
}

template <bool DEF>
__device__ __forceinline__ void item_setup(const BatchArgs &A, int item, int total, int nchunks, ItemState &it) {
    const int lane = threadIdx.x & 31;
    const int grp = DEF ? item : item >> 1;
    window_setup(A, item < total, grp * kTile + lane, DEF ? 0 : item & 1, nchunks, it);
}

// The steps of one chunk for one live item (tab = the chunk's [8][256] table
// rows in shared memory); stores the chunk's raster bytes.
// FZ > 0 (default bank, constant refractory span of FZ steps): live_from[0 ..
// FZ-1] hold the window's last FZ spike masks instead of refractory horizons.
template <bool TRACE, bool DEF, bool SGN, int FZ = 0>
__device__ __forceinline__ void item_chunk(const BatchArgs &A, const LifK &ph, const ItemState &it, const double *tab,
                                           int ch, double (&v)[kNF], int (&live_from)[kNF]) {
    static_assert(FZ == 0 || (DEF && !TRACE && FZ <= kNF), "FZ: default bank, no traces");
    const int N = A.c.n_steps;
    const double refr = A.c.lif_hid.refr;
    const int s0 = ch * kChunk;
    const int nrows = min(kChunk, N - s0);
    uint64_t p0 = 0, p1 = 0;  // the chunk's 6-bit masks, one byte per step
#pragma unroll 1
    for (int j = 0; j < nrows; ++j) {
        const int s = s0 + j;
        const double *T = tab + j * 256;
        double x[9];
#pragma unroll
        for (int k = 0; k < 9; ++k) x[k] = T[(it.lvp[k >> 2] >> (8 * (k & 3))) & 0xFFu];
        unsigned m;
        if (FZ) {
            unsigned frozen = 0;
#pragma unroll
            for (int q = 0; q < FZ; ++q) frozen |= (unsigned)live_from[q];
            m = hidden_step_def_fz<SGN>(ph, x, v, frozen);
#pragma unroll
            for (int q = FZ - 1; q > 0; --q) live_from[q] = live_from[q - 1];
            live_from[0] = (int)m;
        } else if (DEF) m = hidden_step_def<SGN>(ph, x, v, live_from, s, next_live_step(s, refr));
        else m = it.half ? hidden_step<1, SGN>(A, ph, x, v, live_from, s, next_live_step(s, refr))
                         : hidden_step<0, SGN>(A, ph, x, v, live_from, s, next_live_step(s, refr));
        if (TRACE && it.on && A.out.v_hid) {
            double *dst = A.out.v_hid + ((size_t)it.img * N + s) * kNH + it.pos * kNF + it.half * kHalf;
#pragma unroll
            for (int f = 0; f < (DEF ? kNF : kHalf); ++f) dst[f] = v[f];
        }
        p0 |= (uint64_t)(m & 0x3Fu) << (8 * j);
        if (DEF) p1 |= (uint64_t)(m >> kHalf) << (8 * j);
    }
    if (it.on) {
        uint64_t *dst = reinterpret_cast<uint64_t *>(it.rout + (size_t)ch * it.rstride);
        dst[0] = p0;
        if (DEF) dst[kTile] = p1;  // the second half plane, 256 bytes on
    }
}

// Ring variant: the table streams through a 2-stage ring shared by the CTA's
// warps, which therefore step through the chunks together (any N).
template <bool TRACE, bool DEF, bool SGN>
__global__ void __launch_bounds__(kThreads, 5) k_hidden(const BatchArgs A) {
    __shared__ __align__(128) double s_tab[kStages][kChunk * 256];
    __shared__ uint64_t s_full[kStages];
    const int tid = threadIdx.x, warp = tid >> 5;
    const int N = A.c.n_steps;
    const int nchunks = (N + kChunk - 1) / kChunk;
    const int total = hidden_items(A, DEF ? 1 : 2);
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

    const double el = A.c.lif_hid.el;
    const LifK ph = lif_k(A.c.lif_hid);
    int64_t q = 0;
    for (int gi = 0; gi < my_groups; ++gi) {
        const int item = ((int)blockIdx.x + gi * (int)gridDim.x) * kWPC + warp;
        ItemState it;
        item_setup<DEF>(A, item, total, nchunks, it);
        double v[kNF];
        int live_from[kNF];
#pragma unroll
        for (int f = 0; f < kNF; ++f) {
            v[f] = el;
            live_from[f] = 0;
        }
        for (int ch = 0; ch < nchunks; ++ch, ++q) {
            const int b = (int)(q % kStages);
            if (it.live) {
                mbar_wait(&s_full[b], (uint32_t)((q / kStages) & 1));
                item_chunk<TRACE, DEF, SGN>(A, ph, it, s_tab[b], ch, v, live_from);
            }
            __syncthreads();  // every warp is done with stage b
            if (tid == 0 && q + kStages < stream_len) issue(q + kStages);
        }
    }
}

// Resident variant (N <= kResMaxSteps): one CTA of kResWarps warps per SM holds
// the whole [N][256] table in shared memory (one bulk load), so its warps run
// their items independently -- no ring, no per-chunk barrier.
constexpr int kResWarps = 20;
constexpr int kResMaxSteps = 108;  // 108 * 2 KB = 216 KB of table

template <bool TRACE, bool DEF, bool SGN, int FZ = 0>
__global__ void __launch_bounds__(kResWarps * 32, 1) k_hidden_res(const BatchArgs A) {
    extern __shared__ __align__(128) double r_tab[];
    __shared__ uint64_t r_full;
    const int tid = threadIdx.x, warp = tid >> 5;
    const int N = A.c.n_steps;
    const int nchunks = (N + kChunk - 1) / kChunk;
    const int total = hidden_items(A, DEF ? 1 : 2);
    if (tid == 0) {
        mbar_init(&r_full, 1);
        fence_mbar_init();
        mbar_expect_tx(&r_full, (uint32_t)N * 256 * 8);
        for (int ch = 0; ch < nchunks; ++ch) {
            const int rows = min(kChunk, N - ch * kChunk);
            bulk_g2s(r_tab + (size_t)ch * kChunk * 256, A.ctab + (size_t)ch * kChunk * 256, rows * 256 * 8, &r_full);
        }
    }
    __syncthreads();
    mbar_wait(&r_full, 0);
    const double el = A.c.lif_hid.el;
    const LifK ph = lif_k(A.c.lif_hid);
    // items interleaved over the CTAs, so a small batch spreads over many SMs
    const int stride = (int)gridDim.x * kResWarps;
    for (int item = warp * (int)gridDim.x + (int)blockIdx.x; item < total; item += stride) {
        ItemState it;
        item_setup<DEF>(A, item, total, nchunks, it);
        double v[kNF];
        int live_from[kNF];
#pragma unroll
        for (int f = 0; f < kNF; ++f) {
            v[f] = el;
            live_from[f] = 0;
        }
        for (int ch = 0; ch < nchunks; ++ch)
            item_chunk<TRACE, DEF, SGN, FZ>(A, ph, it, r_tab + (size_t)ch * kChunk * 256, ch, v, live_from);
    }
}

// ---------------------------------------------------------------------------
// Output layer state and one step of it (network.py:308-314), lanes 0..9 of
// one warp = the 10 output neurons (lanes 10..31 shadow lane 9, harmlessly).
// Every lane keeps all ten lateral-inhibition traces, so the inhibition sum
// needs no shuffles.  The serial chain is cut short by speculation: the
// traces enter step s as a*e^{-dt/tau} (their values before this step's
// spike input), and the no-spike outcome -- S0 = pairwise sum of the ten
// c = a - b and this lane's own c0 -- is computed one step ahead, off the
// chain.  After a step without output spikes (most steps) the next step
// only needs S0; otherwise the bumps are added and the sum is redone.  Every
// value is the reference's own operation sequence (a*lam + 0 == a*lam
// exactly for a >= 0), so results are bit-identical either way.
struct OutState {
    double Af, Bf;             // event-driven feed-forward recursions (slow, fast)
    double al[kNO], bl[kNO];   // inhibition traces times their decay (before this step's bumps)
    double al_o, bl_o;         // the same for this lane's own neuron
    double S0, c0;             // pairwise sum and own trace if no output spiked last step
    double v;
    int live_from, cnt;
    unsigned prev;             // output spikes of the previous step (10-bit)
};

__device__ __forceinline__ void out_init(OutState &st, const snn_consts_t &c) {
    st.Af = st.Bf = 0.0;
#pragma unroll
    for (int k = 0; k < kNO; ++k) st.al[k] = st.bl[k] = 0.0;
    st.al_o = st.bl_o = 0.0;
    st.S0 = st.c0 = 0.0;  // pairwise10 of ten +0 is +0
    st.v = c.lif_out.el;
    st.live_from = 0;
    st.cnt = 0;
    st.prev = 0u;
}

// Advances one step given G (sum of W rows of hidden neurons spiking now).
// Returns whether this lane's output neuron l fired; *ff_out = c_hidden @ W.
// TieInfo (k_output<TIES> only): the step's candidate potential, drive and
// liveness, for the near-tie bound.
struct TieInfo {
    double vn, drive;
    bool live;
};

__device__ __forceinline__ bool out_step(OutState &st, const snn_consts_t &c, double G, int s, int l,
                                         double *ff_out, TieInfo *ti = nullptr) {
    st.Af = __dadd_rn(__dmul_rn(st.Af, c.decay_slow), G);
    st.Bf = __dadd_rn(__dmul_rn(st.Bf, c.decay_fast), G);
    const double ff = __dsub_rn(st.Af, st.Bf);
    // inhibition traces after this step's bumps (the previous step's output spikes)
    double a[kNO], b[kNO], ao, bo, S, co;
    if (st.prev == 0u) {  // warp-uniform
#pragma unroll
        for (int k = 0; k < kNO; ++k) {
            a[k] = st.al[k];
            b[k] = st.bl[k];
        }
        ao = st.al_o;
        bo = st.bl_o;
        S = st.S0;
        co = st.c0;
    } else {
        double cc[kNO];
#pragma unroll
        for (int k = 0; k < kNO; ++k) {
            const double bump = ((st.prev >> k) & 1u) ? 1.0 : 0.0;
            a[k] = __dadd_rn(st.al[k], bump);
            b[k] = __dadd_rn(st.bl[k], bump);
            cc[k] = __dsub_rn(a[k], b[k]);
        }
        const double bo_ = ((st.prev >> l) & 1u) ? 1.0 : 0.0;
        ao = __dadd_rn(st.al_o, bo_);
        bo = __dadd_rn(st.bl_o, bo_);
        S = pairwise10(cc);
        co = __dsub_rn(ao, bo);
    }
    // the next step's decayed traces and its no-spike outcome: independent of
    // this step's chain, issued before it so the two interleave
    double cc0[kNO];
#pragma unroll
    for (int k = 0; k < kNO; ++k) {
        st.al[k] = __dmul_rn(a[k], c.decay_slow);
        st.bl[k] = __dmul_rn(b[k], c.decay_fast);
        cc0[k] = __dsub_rn(st.al[k], st.bl[k]);
    }
    st.al_o = __dmul_rn(ao, c.decay_slow);
    st.bl_o = __dmul_rn(bo, c.decay_fast);
    st.S0 = pairwise10(cc0);
    st.c0 = __dsub_rn(st.al_o, st.bl_o);
    const double drive = __dadd_rn(ff, __dmul_rn(c.inhibition, __dsub_rn(S, co)));
    // LIF (neurons.py:113-126); a refractory neuron holds v == E_L
    const snn_lif_t &p = c.lif_out;
    double t = __dsub_rn(st.v, p.el);
    t = __dmul_rn(p.g, t);
    t = __dsub_rn(drive, t);
    t = __dmul_rn(p.beta, t);
    const double vn = __dadd_rn(st.v, t);
    const bool live = s >= st.live_from;
    const bool fired = live && vn >= p.vt;
    st.v = (!live || fired || vn < p.el) ? p.el : vn;
    if (fired) st.live_from = next_live_step(s, p.refr);
    st.prev = __ballot_sync(kFull, fired) & 0x3FFu;
    st.cnt += fired ? 1 : 0;
    *ff_out = ff;
    if (ti) {
        ti->vn = vn;
        ti->drive = drive;
        ti->live = live;
    }
    return fired;
}

// out_step for a caller that has the next step's G at hand (the NormAD leader
// scan): the next step's feed-forward term and its whole no-spike drive D0 =
// ff + inh * (S0 - c0) are formed at the end of this step, so after a step
// without output spikes the chain is just the LIF.  Same operations in the
// same order as out_step (bit-identical); 3-4% faster in the cluster kernel.
struct OutD {
    OutState o;
    double D0;  // ff(s) + inh * (S0(s) - c0(s)) for the step about to run
};

__device__ __forceinline__ bool outd_step(OutD &X, const snn_consts_t &c, double Gn, int s, int l) {
    OutState &st = X.o;
    double drive;
    double a[kNO], b[kNO], ao, bo;
    if (st.prev == 0u) {
#pragma unroll
        for (int k = 0; k < kNO; ++k) {
            a[k] = st.al[k];
            b[k] = st.bl[k];
        }
        ao = st.al_o;
        bo = st.bl_o;
        drive = X.D0;
    } else {
        double cc[kNO];
#pragma unroll
        for (int k = 0; k < kNO; ++k) {
            const double bump = ((st.prev >> k) & 1u) ? 1.0 : 0.0;
            a[k] = __dadd_rn(st.al[k], bump);
            b[k] = __dadd_rn(st.bl[k], bump);
            cc[k] = __dsub_rn(a[k], b[k]);
        }
        const double bo_ = ((st.prev >> l) & 1u) ? 1.0 : 0.0;
        ao = __dadd_rn(st.al_o, bo_);
        bo = __dadd_rn(st.bl_o, bo_);
        const double S = pairwise10(cc);
        const double co = __dsub_rn(ao, bo);
        drive = __dadd_rn(__dsub_rn(st.Af, st.Bf), __dmul_rn(c.inhibition, __dsub_rn(S, co)));
    }
    const snn_lif_t &p = c.lif_out;
    double t = __dsub_rn(st.v, p.el);
    t = __dmul_rn(p.g, t);
    t = __dsub_rn(drive, t);
    t = __dmul_rn(p.beta, t);
    const double vn = __dadd_rn(st.v, t);
    const bool live = s >= st.live_from;
    const bool fired = live && vn >= p.vt;
    st.v = (!live || fired || vn < p.el) ? p.el : vn;
    if (fired) st.live_from = next_live_step(s, p.refr);
    st.prev = __ballot_sync(kFull, fired) & 0x3FFu;
    st.cnt += fired ? 1 : 0;
    // the next step: decayed traces, no-spike sum, feed-forward and drive
    double cc0[kNO];
#pragma unroll
    for (int k = 0; k < kNO; ++k) {
        st.al[k] = __dmul_rn(a[k], c.decay_slow);
        st.bl[k] = __dmul_rn(b[k], c.decay_fast);
        cc0[k] = __dsub_rn(st.al[k], st.bl[k]);
    }
    st.al_o = __dmul_rn(ao, c.decay_slow);
    st.bl_o = __dmul_rn(bo, c.decay_fast);
    const double S0 = pairwise10(cc0);
    const double c0 = __dsub_rn(st.al_o, st.bl_o);
    st.Af = __dadd_rn(__dmul_rn(st.Af, c.decay_slow), Gn);
    st.Bf = __dadd_rn(__dmul_rn(st.Bf, c.decay_fast), Gn);
    X.D0 = __dadd_rn(__dsub_rn(st.Af, st.Bf), __dmul_rn(c.inhibition, __dsub_rn(S0, c0)));
    return fired;
}

// ---------------------------------------------------------------------------
// k_gsum: G(s, l) = sum of W[k, l] over the hidden neurons k spiking at step
// s (network.py:311 restated event-driven), summed in a fixed order that
// depends only on the image, so results never depend on the batch it is in.  One warp per
// (image, 8-step chunk); chunks are independent, so a single image spreads
// over ceil(N/8) warps.
//   lists  per tile (in order) the warp is transposed: lane (j, g) takes step j
//          of the tile's windows g, g+4, .., g+28 (interleaved, so spatially
//          clustered spikes spread over the 4 lanes; masks staged in shared
//          memory), counts their spikes, a 4-lane prefix gives its offset in
//          step j's list, and it writes their neuron ids.  The list order
//          (tile, window group, window, feature) depends only on the image.
//   sums   lane (j, p) walks step j's list for outputs 2p, 2p+1 (16-byte W
//          loads, 8 in flight).  A step with more than kStepCap spikes is
//          summed afterwards tile by tile in ascending neuron id.
#ifndef SNN_GSUM_CAP
#define SNN_GSUM_CAP 192
#endif
constexpr int kStepCap = SNN_GSUM_CAP;
constexpr int kGWarps = 4;

__device__ __forceinline__ uint32_t byte_popc(uint32_t x) {  // popcount of each byte
    x = x - ((x >> 1) & 0x55555555u);
    x = (x & 0x33333333u) + ((x >> 2) & 0x33333333u);
    return (x + (x >> 4)) & 0x0F0F0F0Fu;
}

// 12-bit mask of chunk step j from the two 6-bit planes
__device__ __forceinline__ unsigned chunk_mask(uint64_t p0, uint64_t p1, int j) {
    return (unsigned)((p0 >> (8 * j)) & 0x3Fu) | ((unsigned)((p1 >> (8 * j)) & 0x3Fu) << kHalf);
}

__device__ __forceinline__ uint64_t warp_incl_scan_u64(uint64_t x) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t y = __shfl_up_sync(kFull, x, o);
        if (lane >= o) x += y;
    }
    return x;
}

// A step list's row stride: CAP + 8 ids (16 bytes) shifts consecutive rows by
// four banks, so the 8 list writers (one per step) and the 6 readers of a sums
// round hit distinct banks; rows stay 16-byte aligned for the 8-id loads.
template <int CAP>
constexpr int ids_stride() { return CAP + 8; }
static_assert(kNO % 2 == 0 && kNH * (kWPad / 2) <= 0xFFFF, "list entries: W row offsets in double2 units fit 16 bits");

template <int CAP>
struct GsumSmem {
    alignas(16) uint16_t ids[kChunk * ids_stride<CAP>()];  // the chunk's step lists
    uint16_t pos[kMaxTiles * kTile];  // window position of each (tile, lane)
};

// One (image, chunk) task of one warp: lists, then sums, into G's chunk rows.
// ABS (near-tie accounting only, snn_infer_out_t.near_ties): also Gabs(s, l) =
// sum of |W[k, l]| over the same spikes, the magnitude the rounding bound of
// k_output<TIES> needs.
template <int CAP, bool ABS = false, int WS = kNO>
__device__ __forceinline__ void gsum_task(const BatchArgs &A, double *G, double *Gabs, int64_t img, int ch,
                                          GsumSmem<CAP> &S) {
    const int kStepCap = CAP;
    const int lane = threadIdx.x & 31;
    const int N = A.c.n_steps, nch = n_chunks(N);
    const int s0 = ch * kChunk, ns = min(kChunk, N - s0);
    __syncwarp();  // a warp running several tasks: the previous one is done with S
    const int nt = A.n_tiles[img];
    for (int k = lane; k < nt * kTile; k += 32) S.pos[k] = A.tile_pos[img * (kMaxTiles * kTile) + k];
    const uint16_t *PP = S.pos;
    const uint8_t *R = A.raster + raster_tc(A.tile_base[img], nch, nt, ch, 0) + lane * kChunk;
    const double *W = WS == kNO ? A.w : A.wpad;  // row stride WS doubles
    // ---- lists: lane (jl, g) = (step, window group of 8)
    const int jl = lane >> 2, g = lane & 3;
    uint32_t runl = 0;  // step jl's list length so far
    uint64_t n0 = 0, n1 = 0;  // the next tile's planes, loaded ahead
    if (nt > 0) {
        n0 = __ldcs(reinterpret_cast<const unsigned long long *>(R));
        n1 = __ldcs(reinterpret_cast<const unsigned long long *>(R + kRastTC / 2));
    }
    // 8x8 byte transpose among lanes g, g+4, .., g+28 (three butterfly
    // stages, shuffles xor 16 / 8 / 4): lane (jl, g) then holds byte jl (step
    // jl) of the planes of windows g + 4i in byte i.  Per-lane byte selectors:
    const int ti = lane >> 2;
    const uint32_t s2s = (ti & 2) ? 0x5410u : 0x7632u, s2l = (ti & 2) ? 0x3254u : 0x5410u,
                   s2h = (ti & 2) ? 0x3276u : 0x7610u;
    const uint32_t s3s = (ti & 1) ? 0x6420u : 0x7531u, s3l = (ti & 1) ? 0x3514u : 0x5240u,
                   s3h = (ti & 1) ? 0x3716u : 0x7260u;
    auto transpose = [&](uint64_t v, uint32_t &lo, uint32_t &hi) {
        lo = (uint32_t)v;
        hi = (uint32_t)(v >> 32);
        const uint32_t r1 = __shfl_xor_sync(kFull, (ti & 4) ? lo : hi, 16);
        if (ti & 4) lo = r1;
        else hi = r1;
        const uint32_t r2 = __shfl_xor_sync(kFull, __byte_perm(lo, hi, s2s), 8);
        lo = __byte_perm(lo, r2, s2l);
        hi = __byte_perm(hi, r2, s2h);
        const uint32_t r3 = __shfl_xor_sync(kFull, __byte_perm(lo, hi, s3s), 4);
        lo = __byte_perm(lo, r3, s3l);
        hi = __byte_perm(hi, r3, s3h);
    };
    for (int t = 0; t < nt; ++t) {
        if (PP[t * kTile + lane] == 0xFFFF) n0 = n1 = 0ull;  // raster bytes exist only for windows
        const bool any = __any_sync(kFull, (n0 | n1) != 0ull);
        uint32_t p0l, p0h, p1l, p1h;
        if (any) {
            transpose(n0, p0l, p0h);
            transpose(n1, p1l, p1h);
        }
        if (t + 1 < nt) {
            const uint8_t *nxt = R + (size_t)(t + 1) * kRastTC;
            n0 = __ldcs(reinterpret_cast<const unsigned long long *>(nxt));
            n1 = __ldcs(reinterpret_cast<const unsigned long long *>(nxt + kRastTC / 2));
        }
        if (!any) continue;  // warp-uniform: no spike in this tile-chunk
        // word q: windows g + 8q (bytes 0, 2: features 0-5, 6-11) and g + 8q + 4
        // (bytes 1, 3); interleaved windows spread spatially clustered spikes
        // over the 4 lanes of a step
        const uint32_t wq[4] = {__byte_perm(p0l, p1l, 0x5410u), __byte_perm(p0l, p1l, 0x7632u),
                                __byte_perm(p0h, p1h, 0x5410u), __byte_perm(p0h, p1h, 0x7632u)};
        const unsigned cnt = __popc(wq[0]) + __popc(wq[1]) + __popc(wq[2]) + __popc(wq[3]);
        // prefix over the 4 window groups of step jl
        unsigned inc = cnt;
        unsigned y = __shfl_up_sync(kFull, inc, 1);
        if (g >= 1) inc += y;
        y = __shfl_up_sync(kFull, inc, 2);
        if (g >= 2) inc += y;
        const unsigned tot = __shfl_sync(kFull, inc, lane | 3);
        uint16_t *dst = S.ids + jl * ids_stride<CAP>();
        // shared-window byte addresses of this lane's next list slot and of the cap slot
        const uint32_t scap = (uint32_t)__cvta_generic_to_shared(dst + kStepCap);
        uint32_t sk = (uint32_t)__cvta_generic_to_shared(dst) + 2u * (runl + inc - cnt);
        const uint16_t *tp = PP + t * kTile + g;
        // spikes taken highest bit first (a fixed order per image), one FLO
        // and one clear per spike; bit b: window byte (b >> 3) & 1, feature
        // (b & 7) + 6 (b >> 4)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            uint32_t w = wq[q];
            if (w) {
                // list entries are W row offsets in double2 units: neuron id * kNO / 2
                constexpr int kR = WS / 2;
                // b = 16 plane + 8 window + feature-in-plane t:
                // id * kR = r_window + kR t + kHalf kR plane = kR b + r'_window - (16 - kHalf) kR plane
                const int r0 = (int)tp[8 * q] * (kNF * kR), r1 = (int)tp[8 * q + 4] * (kNF * kR) - 8 * kR;
                do {
                    int b;
                    asm("bfind.u32 %0, %1;" : "=r"(b) : "r"(w));  // highest set bit
                    w &= ~(1u << b);
                    const int e = kR * b + ((b & 8) ? r1 : r0) - (16 - kHalf) * kR * (b >> 4);
                    // past the cap: the row's padding slot (never read)
                    asm volatile("st.shared.u16 [%0], %1;" ::"r"(min(sk, scap)), "h"((unsigned short)e));
                    sk += 2;
                } while (w);
            }
        }
        runl += tot;
    }
    __syncwarp();
    // steps whose list overflowed kStepCap (bit j), warp-uniform
    const unsigned ovf = __ballot_sync(kFull, g == 0 && runl > (uint32_t)kStepCap) ;
    double *Gi = G + ((size_t)img * N + s0) * kNO;
    // ---- sums: lane (j, p) -> G[j][2p], G[j][2p+1]; rounds of 6 steps
#pragma unroll 1
    for (int j0 = 0; j0 < ns; j0 += 6) {
        const int j = j0 + lane / 5, p = lane % 5;
        const unsigned cnt = __shfl_sync(kFull, runl, (j & 7) * 4);
        if (lane < 30 && j < ns && cnt <= kStepCap) {
            const uint16_t *lst = S.ids + j * ids_stride<CAP>();
            const double2 *W2 = reinterpret_cast<const double2 *>(W) + p;
            double g0 = 0.0, g1 = 0.0, a0 = 0.0, a1 = 0.0;
            unsigned e = 0;
            for (; e + 8 <= cnt; e += 8) {
                const uint4 q = *reinterpret_cast<const uint4 *>(lst + e);  // 8 ids in one load
                const uint32_t qw[4] = {q.x, q.y, q.z, q.w};
                double2 v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) v[u] = __ldg(W2 + ((qw[u >> 1] >> (16 * (u & 1))) & 0xFFFFu));
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    g0 = __dadd_rn(g0, v[u].x);
                    g1 = __dadd_rn(g1, v[u].y);
                    if (ABS) {
                        a0 += fabs(v[u].x);
                        a1 += fabs(v[u].y);
                    }
                }
            }
            for (; e < cnt; ++e) {
                const double2 v = __ldg(W2 + lst[e]);
                g0 = __dadd_rn(g0, v.x);
                g1 = __dadd_rn(g1, v.y);
                if (ABS) {
                    a0 += fabs(v.x);
                    a1 += fabs(v.y);
                }
            }
            reinterpret_cast<double2 *>(Gi + (size_t)j * kNO)[p] = make_double2(g0, g1);
            if (ABS) reinterpret_cast<double2 *>(Gabs + ((size_t)img * N + s0 + j) * kNO)[p] = make_double2(a0, a1);
        }
    }
    // rare: a step with more than kStepCap spikes -- tile by tile, ascending id
    for (unsigned ov = ovf; ov; ov &= ov - 1u) {
        const int j = (__ffs(ov) - 1) >> 2;
        __syncwarp();
        double g = 0.0, ga = 0.0;
        for (int t = 0; t < nt; ++t) {
            const uint8_t *src = R + (size_t)t * kRastTC;
            unsigned m = PP[t * kTile + lane] == 0xFFFF
                             ? 0u
                             : chunk_mask(__ldcs(reinterpret_cast<const unsigned long long *>(src)),
                                          __ldcs(reinterpret_cast<const unsigned long long *>(src + kRastTC / 2)), j);
            int tt;
            int k = warp_excl_scan_int(__popc(m), &tt);
            const int id0 = (int)PP[t * kTile + lane] * kNF;
            while (m) {
                const int f = __ffs(m) - 1;
                m &= m - 1u;
                S.ids[k++] = (uint16_t)(id0 + f);
            }
            __syncwarp();
            if (lane < kNO)
                for (int e = 0; e < tt; ++e) {
                    const double wv = __ldg(W + (size_t)S.ids[e] * WS + lane);
                    g = __dadd_rn(g, wv);
                    if (ABS) ga += fabs(wv);
                }
            __syncwarp();
        }
        if (lane < kNO) {
            Gi[(size_t)j * kNO + lane] = g;
            if (ABS) Gabs[((size_t)img * N + s0 + j) * kNO + lane] = ga;
        }
    }
}

#ifndef SNN_GSUM_MINB
#define SNN_GSUM_MINB 10
#endif
template <bool ABS, int WS = kNO>
__global__ void __launch_bounds__(kGWarps * 32, SNN_GSUM_MINB) k_gsum(const BatchArgs A, double *G, double *Gabs) {
    __shared__ __align__(16) GsumSmem<kStepCap> smem[kGWarps];
    const int warp = threadIdx.x >> 5;
    const int nch = n_chunks(A.c.n_steps);
    const int64_t task = (int64_t)blockIdx.x * kGWarps + warp;
    if (task >= A.n_images * nch) return;
    const int64_t img = task / nch;
    gsum_task<kStepCap, ABS, WS>(A, G, Gabs, img, (int)(task - img * nch), smem[warp]);
}

// ---------------------------------------------------------------------------
// k_output: the 10-neuron output layer (network.py:308-314), one warp per
// image over its G rows (staged in shared memory kOSteps steps at a time).
//
// TIES: near-tie accounting (snn_infer_out_t.near_ties).  The
// reference forms ff = c_hidden @ W by dgemv over per-neuron traces; this
// library by the event-driven A - B recursions over G.  Both are within
// u * (8114 S_A + 2 S_B ... ) of the exact value, where (u = 2^-53)
//   Gabs(s) = sum of |W[k, l]| over the neurons spiking at s,
//   Abar(s) = Abar(s-1) e^{-dt/t1} + Gabs(s)   (= sum_k a_k(s) |W[k, l]|),
//   S_A(s)  = S_A(s-1) e^{-dt/t1} + Abar(s)    (same with e^{-dt/t2}: Bbar, S_B),
// so |ff_ref - ff_here| <= dff = 2^-38 (S_A + S_B + |ff|) (the event sum:
// per step at most 8112 terms plus two roundings of the recursion, summed
// with its decay; the reference: two roundings per neuron recursion, the
// dgemv's gamma_8112 and the trace difference; 2^-38 > 16229 u with slack).
// While the output spikes agree, the inhibition terms agree and the membrane
// difference obeys |dv(s)| <= Ev(s) = Ev(s-1) |1 - beta g| + beta dff(s) + 8u
// (magnitudes of the LIF's operands), reset to 0 whenever v is E_L in both
// (spike or refractory).  A step of a live neuron with |vn - V_T| <= Ev is a
// near tie: only there can the reference's threshold decision differ.
#ifndef SNN_OSTEPS
#define SNN_OSTEPS 96
#endif
constexpr int kOSteps = SNN_OSTEPS;  // G rows staged per round (one round for N <= kOSteps)
constexpr int kOutWarps2 = 4;

template <bool TIES, bool OUTS = true>
__global__ void __launch_bounds__(kOutWarps2 * 32) k_output(const BatchArgs A, const double *G, const double *Gabs) {
    __shared__ __align__(16) double s_g[kOutWarps2][kOSteps * kNO];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t img = (int64_t)blockIdx.x * kOutWarps2 + warp;
    if (img >= A.n_images) return;
    const int N = A.c.n_steps;
    const int l = lane < kNO ? lane : kNO - 1;
    const double *Gi = G + (size_t)img * N * kNO;
    double *sg = s_g[warp];
    // register copies of the step's constants (through a shuffle, so ptxas
    // cannot re-read them from the constant bank inside the loop)
    snn_consts_t kc;
    kc.lif_out = A.c.lif_out;
    kc.decay_slow = A.c.decay_slow;
    kc.decay_fast = A.c.decay_fast;
    kc.inhibition = A.c.inhibition;
    {
        double *v[8] = {&kc.lif_out.g, &kc.lif_out.el, &kc.lif_out.vt, &kc.lif_out.beta,
                        &kc.lif_out.refr, &kc.decay_slow, &kc.decay_fast, &kc.inhibition};
#pragma unroll
        for (int q = 0; q < 8; ++q) *v[q] = __shfl_sync(kFull, *v[q], 0);
    }
    OutState st;
    out_init(st, kc);
    const snn_lif_t &p = A.c.lif_out;
    constexpr double kU = 0x1p-53, kTieK = 0x1p-38;
    const double damp = fabs(1.0 - p.beta * p.g);
    double Ab = 0.0, Bb = 0.0, SA = 0.0, SB = 0.0, Ev = 0.0;
    int ties = 0;
    for (int s0 = 0; s0 < N; s0 += kOSteps) {
        const int ns = min(kOSteps, N - s0);
        for (int k = lane; k < ns * kNO; k += 32) sg[k] = __ldcs(Gi + (size_t)s0 * kNO + k);
        __syncwarp();
        for (int j = 0; j < ns; ++j) {
            const int s = s0 + j;
            double ff;
            if (TIES) {
                TieInfo ti;
                const double vprev = st.v;
                const bool fired = out_step(st, kc, sg[j * kNO + l], s, l, &ff, &ti);
                const double ga = __ldcs(Gabs + ((size_t)img * N + s) * kNO + l);
                Ab = Ab * A.c.decay_slow + ga;
                Bb = Bb * A.c.decay_fast + ga;
                SA = SA * A.c.decay_slow + Ab;
                SB = SB * A.c.decay_fast + Bb;
                const double dff = kTieK * (SA + SB + fabs(ff));
                const double mag = fabs(ti.vn) + fabs(vprev) + fabs(p.el) +
                                   p.beta * (2.0 * fabs(ff) + fabs(ti.drive) + p.g * (fabs(vprev) + fabs(p.el)));
                Ev = Ev * damp + p.beta * dff + 8.0 * kU * mag;
                if (lane < kNO && ti.live && fabs(ti.vn - p.vt) <= Ev) ++ties;
                if (!ti.live || fired) Ev = 0.0;  // v == E_L exactly in both
            } else {
                out_step(st, kc, sg[j * kNO + l], s, l, &ff);
            }
            if (OUTS) {
                if (A.out.out_raster && lane == 0) A.out.out_raster[(size_t)img * N + s] = (uint16_t)st.prev;
                if (lane < kNO) {
                    if (A.out.ff) A.out.ff[((size_t)img * N + s) * kNO + lane] = ff;
                    if (A.out.v_out) A.out.v_out[((size_t)img * N + s) * kNO + lane] = st.v;
                }
            }
        }
        __syncwarp();
    }
    if (lane < kNO) A.out.counts[(size_t)img * kNO + lane] = st.cnt;
    if (TIES) {
        for (int o = 16; o > 0; o >>= 1) ties += __shfl_xor_sync(kFull, ties, o);
        if (lane == 0) A.out.near_ties[img] = ties;
    }
}


// ---------------------------------------------------------------------------
// k_output_dist: the same output layer with the lane-distributed step
// (dist_step): lane q < 10 owns inhibition trace q and the warp speculates the
// next step's inhibition sums through 512 B of shared memory per warp -- the
// reference's operation sequences, bit-identical to out_step, with ~28 FP64
// instructions per lane-step instead of ~64.  On the serial chain of ONE warp
// it is slower than out_step (263 vs 232 cycles per step,
// scripts/scan_micro.py), but k_output over a large batch is bound by the
// FP64 pipe (73% busy), so batches of >= 256 images take this kernel.
// Each lane owns one trace; candidates are exchanged through shared memory:
constexpr int kDistSpecHalf = 256;  // 15 x 16 B used; 512-aligned pair of buffers
constexpr int kDistSpecBytes = 2 * kDistSpecHalf;

struct DistState {
    double Af, Bf;      // event-driven feed-forward recursions (slow, fast)
    double al, bl;      // trace q times its decay, entering the next step
    double ap, bp;      // al + 1, bl + 1
    double c0, c1;      // own c for the next step: neuron q did not / did fire
    double T;           // this lane's speculative inhibition sum for the next step
    double v;
    int live_from, cnt;
    unsigned prev;      // output spikes of the previous step (10-bit)
    unsigned cur;       // shared address of the buffer holding this step's candidates
    unsigned rd[5];     // byte offsets of this lane's five pair loads
    unsigned w0a, w0b, w1;  // byte offsets of the owner's c0 (twice) and c1 stores
};

__device__ __forceinline__ void sts64(unsigned a, double v) {
    asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}
__device__ __forceinline__ double lds64(unsigned a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ double2 lds128(unsigned a) {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a) : "memory");
    return v;
}

__device__ __forceinline__ void dist_init(DistState &st, const snn_consts_t &c, char *spec, int lane) {
    st.Af = st.Bf = 0.0;
    st.al = st.bl = 0.0;
    st.ap = st.bp = 1.0;
    st.c0 = st.c1 = 0.0;  // (0 + 1) - (0 + 1) == +0
    st.T = 0.0;           // pairwise10 of ten +0 is +0
    st.v = c.lif_out.el;
    st.live_from = 0;
    st.cnt = 0;
    st.prev = 0u;
    st.cur = (unsigned)__cvta_generic_to_shared(spec);
    const int sub = (lane >= kNO && lane < 2 * kNO) ? lane - kNO : -1;
#pragma unroll
    for (int m = 0; m < 5; ++m)
        st.rd[m] = 48u * m + ((sub >= 0 && (sub >> 1) == m) ? 16u * (1u + (sub & 1)) : 0u);
    const unsigned q = lane < kNO ? lane : kNO - 1, m = q >> 1, odd = q & 1u;
    st.w0a = lane < kNO ? 48u * m + 8u * odd : 240u;  // 240..255: scratch slot
    st.w0b = lane < kNO ? 48u * m + (odd ? 16u : 32u) + 8u * odd : 240u;
    st.w1 = lane < kNO ? 48u * m + (odd ? 32u : 16u) + 8u * odd : 240u;
}

// The output layer's constants, held in registers across the scan.
struct DistK {
    double lam1, lam2, inh, el, vt, g, beta, refr;
};

__device__ __forceinline__ DistK dist_k(const snn_consts_t &c) {
    return DistK{c.decay_slow, c.decay_fast, c.inhibition, c.lif_out.el, c.lif_out.vt,
                c.lif_out.g, c.lif_out.beta, c.lif_out.refr};
}

// Advances one step given G (sum of W rows of hidden neurons spiking now).
// Returns whether this lane's output neuron l fired; *ff_out = c_hidden @ W.
// MARGIN (the speculative NormAD scan, normad_spec.cuh): *margin = the
// candidate potential's distance to the threshold when the neuron is live,
// +inf otherwise.
template <bool MARGIN = false>
__device__ __forceinline__ bool dist_step(DistState &st, const DistK &k, double G, int s, int l, int lane,
                                         double *ff_out, double *margin = nullptr) {
    st.Af = __dadd_rn(__dmul_rn(st.Af, k.lam1), G);
    st.Bf = __dadd_rn(__dmul_rn(st.Bf, k.lam2), G);
    const double ff = __dsub_rn(st.Af, st.Bf);
    const unsigned pv = st.prev;  // warp-uniform
    const bool mine = (pv >> l) & 1u;
    const double a = mine ? st.ap : st.al;
    const double b = mine ? st.bp : st.bl;
    const double co = mine ? st.c1 : st.c0;
    // this step's inhibition sum
    double S = st.T;
    if (pv != 0u) {
        if ((pv & (pv - 1u)) == 0u) {
            S = __shfl_sync(kFull, st.T, 9 + __ffs((int)pv));
        } else {
            double x[kNO];
#pragma unroll
            for (int q = 0; q < kNO; ++q) {
                const unsigned m = q >> 1, bit = (pv >> q) & 1u;
                const unsigned off = (q & 1) ? (bit ? 48u * m + 40u : 48u * m + 8u) : (bit ? 48u * m + 16u : 48u * m);
                x[q] = lds64(st.cur + off);
            }
            S = pairwise10(x);
        }
    }
    // candidates for the next step: traces, stores, loads (consumed below)
    st.al = __dmul_rn(a, k.lam1);
    st.bl = __dmul_rn(b, k.lam2);
    st.c0 = __dsub_rn(st.al, st.bl);
    st.ap = __dadd_rn(st.al, 1.0);
    st.bp = __dadd_rn(st.bl, 1.0);
    st.c1 = __dsub_rn(st.ap, st.bp);
    // the two buffers are kDistSpecHalf apart: flip to the other one
    const unsigned nxt = (st.cur & 256u) ? st.cur - 256u : st.cur + 256u;
    st.cur = nxt;
    sts64(nxt + st.w0a, st.c0);  // lanes >= 10 write a scratch slot
    sts64(nxt + st.w0b, st.c0);
    sts64(nxt + st.w1, st.c1);
    __syncwarp();
    double x[kNO];
#pragma unroll
    for (int m = 0; m < 5; ++m) {
        const double2 p = lds128(nxt + st.rd[m]);
        x[2 * m] = p.x;
        x[2 * m + 1] = p.y;
    }
    // this step's drive and LIF (neurons.py:113-126); a refractory neuron holds v == E_L
    const double drive = __dadd_rn(ff, __dmul_rn(k.inh, __dsub_rn(S, co)));
    double t = __dsub_rn(st.v, k.el);
    t = __dmul_rn(k.g, t);
    t = __dsub_rn(drive, t);
    t = __dmul_rn(k.beta, t);
    const double vn = __dadd_rn(st.v, t);
    const bool live = s >= st.live_from;
    const bool fired = live && vn >= k.vt;
    if (MARGIN) *margin = live ? fabs(vn - k.vt) : __longlong_as_double(0x7ff0000000000000LL);
    st.v = (!live || fired || vn < k.el) ? k.el : vn;
    if (fired) st.live_from = next_live_step(s, k.refr);
    st.prev = __ballot_sync(kFull, fired) & 0x3FFu;
    st.cnt += fired ? 1 : 0;
    // the next step's speculative sum
    st.T = pairwise10(x);
    *ff_out = ff;
    return fired;
}



constexpr int kOutDistMinImages = 256;
// OUTS: the optional per-step outputs (out_raster, ff, v_out) are requested;
// without them the step loop carries no per-step branches or stores.
template <bool OUTS>
__global__ void __launch_bounds__(kOutWarps2 * 32) k_output_dist(const BatchArgs A, const double *G) {
    __shared__ __align__(16) double s_g[kOutWarps2][kOSteps * kNO];
    __shared__ __align__(512) char spec[kOutWarps2][kDistSpecBytes];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t img = (int64_t)blockIdx.x * kOutWarps2 + warp;
    if (img >= A.n_images) return;
    const int N = A.c.n_steps;
    const int l = lane < kNO ? lane : kNO - 1;
    const double *Gi = G + (size_t)img * N * kNO;
    double *sg = s_g[warp];
    DistState st;
    dist_init(st, A.c, spec[warp], lane);
    DistK k = dist_k(A.c);
    {  // register copies (through a shuffle, so ptxas cannot re-read them from the constant bank in the loop)
        double *v[8] = {&k.lam1, &k.lam2, &k.inh, &k.el, &k.vt, &k.g, &k.beta, &k.refr};
#pragma unroll
        for (int q = 0; q < 8; ++q) *v[q] = __shfl_sync(kFull, *v[q], 0);
    }
    for (int s0 = 0; s0 < N; s0 += kOSteps) {
        const int ns = min(kOSteps, N - s0);
        for (int q = lane; q < ns * kNO; q += 32) sg[q] = __ldcs(Gi + (size_t)s0 * kNO + q);
        __syncwarp();
        for (int j = 0; j < ns; ++j) {
            const int s = s0 + j;
            double ff;
            dist_step(st, k, sg[j * kNO + l], s, l, lane, &ff);
            if (OUTS) {
                if (A.out.out_raster && lane == 0) A.out.out_raster[(size_t)img * N + s] = (uint16_t)st.prev;
                if (lane < kNO) {
                    if (A.out.ff) A.out.ff[((size_t)img * N + s) * kNO + lane] = ff;
                    if (A.out.v_out) A.out.v_out[((size_t)img * N + s) * kNO + lane] = st.v;
                }
            }
        }
        __syncwarp();
    }
    if (lane < kNO) A.out.counts[(size_t)img * kNO + lane] = st.cnt;
}

}  // namespace snn
