// Guard-band hidden layer: packed-FP32 simulation with an exact FP64 fallback
// (default filter bank, constant refractory span FZ, N <= kGbMaxSteps).
//
// The reference simulates the 8,112 hidden LIF neurons in float64
// (network.py:261-326, neurons.py:83-126).  k_hidden_res reproduces that bit
// for bit on the FP64 pipe.  This kernel runs the same dynamics in float32,
// two windows per lane packed into float2 registers (FFMA2/FADD2: half the
// instructions and twice the pipe rate of FP64), and proves per window that
// its spikes are the FP64 kernel's:
//
//   state  w = v - E_L >= 0 (so the LIF step is ONE fused multiply-add:
//          w' = w D + beta I, D = 1 - beta g, with beta folded into the taps);
//          reset / clamp / refractory as in the FP64 kernel (w = 0 <=> v = E_L);
//   bound  while the two runs take the same spike decisions, the float32 and
//          float64 trajectories differ by at most e(s) <= D e(s-1) + eps, eps =
//          24 u beta S_w + 2.1 u (1.01 theta D + beta S_w) + 2^-50 (...),
//          u = 2^-24, theta = V_T - E_L and S_w = max over features of
//          sum_k |tap_{f,k}| max_s |c(s, level_k)| for THIS window (the table
//          rounding, the 9-term float32 stencil, the constants' rounding and
//          the one FFMA; the float64 side's own rounding in the 2^-50 term),
//          so |e| <= e_max = eps / (1 - D);
//   band   a live neuron with theta - delta <= w' < theta + delta, delta =
//          2 e_max + 4 u theta, could take a different decision: the window
//          is flagged.  Outside the band both runs decide alike, so by
//          induction an unflagged window's spike raster IS the FP64 raster;
//   redo   flagged windows (a few per cent) are re-simulated by k_hidden_fix
//          with the FP64 step of k_hidden_res, overwriting their raster.
//
// The result is the bit-identical hidden raster of the FP64 kernel (tests:
// test_hidden_kernel_variants_identical, the per-neuron counts of 1,000
// reference images).
#pragma once
#include "hidden.cuh"

namespace snn {

constexpr int kGbWarps = 20;  // 5 per scheduler: 1.93 ms vs 2.03 (16), 2.03 (19), 2.13 (18), 2.15 (24) per 10k images
constexpr int kGbWarpsSmall = 16;  // k_hidden_gb's other CTA size (the host picks the one with fewer wave-cycles)
constexpr int kGbMaxSteps = 200;  // fp32 table [N][256] + [256] level maxima in <= 201 KB
// Below this batch size the float64 kernel is faster (scripts/small_n.py: one
// image 34 vs 64 us, 148 images 59 vs 87 us, crossover ~250): the guard band's
// setup and its float64 redo launch (a 100-step serial chain) are fixed costs.
constexpr int kGbMinImages = 256;

__host__ __device__ inline size_t gb_smem_bytes(int N) { return ((size_t)N + 1) * 256 * sizeof(float); }

// Work list of flagged windows (indices in the batch's compacted window list).
__device__ __forceinline__ void gb_flag(const BatchArgs &A, bool flag, int gw) {
    const unsigned b = __ballot_sync(kFull, flag);
    if (!b) return;
    const int lane = threadIdx.x & 31;
    int base = 0;
    if (lane == __ffs(b) - 1) base = atomicAdd(A.fix_count, __popc(b));
    base = __shfl_sync(kFull, base, __ffs(b) - 1);
    if (flag) A.fix_list[base + __popc(b & ((1u << lane) - 1u))] = gw;
}

// Stencil sums of the default bank for two windows at once (x: the 9 input
// traces of window A in .x, of window B in .y): chain k-ordered like the FP64
// kernel, zero taps skipped, taps pre-scaled by beta.
template <int F>
__device__ __forceinline__ float2 gb_current(const float2 (&x)[9], const float (&tau)[4]) {
    float2 I = make_float2(0.f, 0.f);
    bool first = true;
#pragma unroll
    for (int k = 0; k < 9; ++k) {
        if (def_coef(F, k) != 0) {
            const float t = def_coef(F, k) < 0 ? -tau[def_tap_slot(F, k)] : tau[def_tap_slot(F, k)];
            const float2 tt = make_float2(t, t);
            I = first ? __fmul2_rn(x[k], tt) : __ffma2_rn(x[k], tt, I);
            first = false;
        }
    }
    return I;
}

// Per-window float64 error bound -> the flag band, as float32 bit patterns
// [blo, blo + bw): theta - delta and the band width 2 delta.
struct GbBand {
    float lo;    // theta - delta
    uint32_t bw; // bits of 2 delta (q = w' - lo: near <=> 0 <= q < 2 delta <=> (uint)bits(q) < bw)
};

__device__ __forceinline__ GbBand gb_band(const ItemState &it, const float *cmax, const snn_lif_t &p) {
    double lv[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) lv[k] = (double)cmax[(it.lvp[k >> 2] >> (8 * (k & 3))) & 0xFFu];
    double S = 0.0;
#pragma unroll
    for (int f = 0; f < kNF; ++f) {
        if (f >= 4 && f < 8) continue;  // negations of 0-3: the same sums
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < 9; ++k) s += fabs(def_tap(f, k)) * lv[k];
        S = fmax(S, s);
    }
    S *= 1.0 + 0x1p-40;
    const double u = 0x1p-24;
    const double beta = p.beta, D = 1.0 - beta * p.g, theta = p.vt - p.el;
    const double bS = beta * S;
    const double eps = 24.0 * u * bS + 2.1 * u * (1.01 * theta * D + bS) +
                       0x1p-50 * (fabs(p.el) + fabs(p.vt) + bS + 1.01 * theta);
    const double emax = eps / (1.0 - D);
    const double delta = 2.0 * emax + 4.0 * u * theta;
    GbBand b;
    b.lo = (float)(theta - delta);
    b.bw = __float_as_uint((float)(2.0 * delta));
    return b;
}

// The decisions of feature f for both windows (inline PTX: ptxas otherwise
// materialises the frozen bits through predicate spills).  q = w' - (theta -
// delta), qh = w' - (theta + delta); the sign bits of q and qh are shifted
// into nf / nh ("not fired" below / above the band, feature f at bit f after
// the 12 features are done, highest first).  w' is kept (clamped at 0) iff
// the neuron is live (frozen bit f clear) and 0 <= w' < theta - delta, one
// unsigned compare of the bit pattern against ul = bits(theta - delta).
__device__ __forceinline__ void gb_decide(float2 wn, float2 q, float2 qh, unsigned Fa, unsigned Fb, unsigned bit,
                                          uint32_t ula, uint32_t ulb, unsigned &nfa, unsigned &nfb, unsigned &nha,
                                          unsigned &nhb, float2 &w) {
    float wa, wb;
    asm("{\n\t.reg .pred pa, pb, ka, kb;\n\t.reg .b32 ta, tb;\n\t"
        "and.b32 ta, %6, %8;\n\t"
        "and.b32 tb, %7, %8;\n\t"
        "setp.ne.u32 pa, ta, 0;\n\t"
        "setp.ne.u32 pb, tb, 0;\n\t"
        "setp.lt.and.u32 ka, %9, %11, !pa;\n\t"
        "setp.lt.and.u32 kb, %10, %12, !pb;\n\t"
        "selp.b32 %0, %9, 0, ka;\n\t"
        "selp.b32 %1, %10, 0, kb;\n\t"
        "shf.l.clamp.b32 %2, %13, %2, 1;\n\t"
        "shf.l.clamp.b32 %3, %14, %3, 1;\n\t"
        "shf.l.clamp.b32 %4, %15, %4, 1;\n\t"
        "shf.l.clamp.b32 %5, %16, %5, 1;\n\t}"
        : "=r"(*reinterpret_cast<uint32_t *>(&wa)), "=r"(*reinterpret_cast<uint32_t *>(&wb)), "+r"(nfa), "+r"(nfb),
          "+r"(nha), "+r"(nhb)
        : "r"(Fa), "r"(Fb), "r"(bit), "r"(__float_as_uint(wn.x)), "r"(__float_as_uint(wn.y)), "r"(ula), "r"(ulb),
          "r"(__float_as_uint(q.x)), "r"(__float_as_uint(q.y)), "r"(__float_as_uint(qh.x)),
          "r"(__float_as_uint(qh.y)));
    w = make_float2(wa, wb);
}

template <int FZ>
__global__ void __launch_bounds__(kGbWarps * 32, 1) k_hidden_gb1(const BatchArgs A) {
    extern __shared__ __align__(16) float gtab[];  // [N][256] fp32 input traces, then [256] max |c| per level
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int N = A.c.n_steps;
    const int nchunks = n_chunks(N);
    float *cmax = gtab + (size_t)N * 256;
    for (int i = tid; i < N * 256; i += kGbWarps * 32) gtab[i] = (float)__ldg(A.ctab + i);
    if (tid < 256) {
        double m = 0.0;
        for (int s = 0; s < N; ++s) m = fmax(m, fabs(__ldg(A.ctab + (size_t)s * 256 + tid)));
        cmax[tid] = (float)(m * (1.0 + 0x1p-20));  // rounded up
    }
    __syncthreads();
    const snn_lif_t &p = A.c.lif_hid;
    const float D = (float)(1.0 - p.beta * p.g);
    const float2 D2 = make_float2(D, D);
    float tau[4];
#pragma unroll
    for (int m = 0; m < 4; ++m) tau[m] = (float)(p.beta * c_def_tap[m]);
    const int groups = hidden_items(A, 1);          // groups of 32 windows
    const int items = (groups + 1) >> 1;            // a lane takes window gw and gw + 32
    const int stride = (int)gridDim.x * kGbWarps;
    for (int item = warp * (int)gridDim.x + (int)blockIdx.x; item < items; item += stride) {
        ItemState ia, ib;
        window_setup(A, true, (2 * item) * kTile + lane, 0, nchunks, ia);
        window_setup(A, 2 * item + 1 < groups, (2 * item + 1) * kTile + lane, 0, nchunks, ib);
        const GbBand ba = gb_band(ia, cmax, p), bb = gb_band(ib, cmax, p);
        const float2 lo2 = make_float2(-ba.lo, -bb.lo);
        const float2 hi2 = make_float2(-(ba.lo + __uint_as_float(ba.bw)), -(bb.lo + __uint_as_float(bb.bw)));
        const uint32_t ula = __float_as_uint(ba.lo), ulb = __float_as_uint(bb.lo);
        uint32_t offa[9], offb[9];  // byte offsets of the 9 levels in a table row
#pragma unroll
        for (int k = 0; k < 9; ++k) {
            offa[k] = ((ia.lvp[k >> 2] >> (8 * (k & 3))) & 0xFFu) * 4u;
            offb[k] = ((ib.lvp[k >> 2] >> (8 * (k & 3))) & 0xFFu) * 4u;
        }
        float2 w[kNF];
#pragma unroll
        for (int f = 0; f < kNF; ++f) w[f] = make_float2(0.f, 0.f);
        unsigned fza[FZ], fzb[FZ];
#pragma unroll
        for (int q = 0; q < FZ; ++q) fza[q] = fzb[q] = 0u;
        bool near_a = false, near_b = false;
        for (int ch = 0; ch < nchunks; ++ch) {
            const int s0 = ch * kChunk;
            const int nrows = min(kChunk, N - s0);
            uint64_t pa0 = 0, pa1 = 0, pb0 = 0, pb1 = 0;
#pragma unroll 1
            for (int j = 0; j < nrows; ++j) {
                const char *T = reinterpret_cast<const char *>(gtab + (size_t)(s0 + j) * 256);
                float2 x[9];
#pragma unroll
                for (int k = 0; k < 9; ++k)
                    x[k] = make_float2(*reinterpret_cast<const float *>(T + offa[k]),
                                       *reinterpret_cast<const float *>(T + offb[k]));
                unsigned Fa = 0, Fb = 0;
#pragma unroll
                for (int q = 0; q < FZ; ++q) {
                    Fa |= fza[q];
                    Fb |= fzb[q];
                }
                float2 I[kNF];
                I[0] = gb_current<0>(x, tau);
                I[1] = gb_current<1>(x, tau);
                I[2] = gb_current<2>(x, tau);
                I[3] = gb_current<3>(x, tau);
#pragma unroll
                for (int f = 4; f < 8; ++f) I[f] = make_float2(-I[f - 4].x, -I[f - 4].y);
                I[8] = gb_current<8>(x, tau);
                I[9] = gb_current<9>(x, tau);
                I[10] = gb_current<10>(x, tau);
                I[11] = gb_current<11>(x, tau);
                unsigned nfa = 0, nfb = 0, nha = 0, nhb = 0;  // sign bits below / above the band
#pragma unroll
                for (int f = kNF - 1; f >= 0; --f) {
                    const float2 wn = __ffma2_rn(w[f], D2, I[f]);
                    gb_decide(wn, __fadd2_rn(wn, lo2), __fadd2_rn(wn, hi2), Fa, Fb, 1u << f, ula, ulb, nfa, nfb, nha,
                              nhb, w[f]);
                }
                // near the threshold: at or above theta - delta, below theta + delta, live
                near_a |= (~nfa & nha & ~Fa & 0xFFFu) != 0u;
                near_b |= (~nfb & nhb & ~Fb & 0xFFFu) != 0u;
                const unsigned ma = ~nfa & ~Fa & 0xFFFu, mb = ~nfb & ~Fb & 0xFFFu;
#pragma unroll
                for (int q = FZ - 1; q > 0; --q) {
                    fza[q] = fza[q - 1];
                    fzb[q] = fzb[q - 1];
                }
                fza[0] = ma;
                fzb[0] = mb;
                pa0 |= (uint64_t)(ma & 0x3Fu) << (8 * j);
                pa1 |= (uint64_t)(ma >> kHalf) << (8 * j);
                pb0 |= (uint64_t)(mb & 0x3Fu) << (8 * j);
                pb1 |= (uint64_t)(mb >> kHalf) << (8 * j);
            }
            if (ia.on) {
                uint64_t *dst = reinterpret_cast<uint64_t *>(ia.rout + (size_t)ch * ia.rstride);
                dst[0] = pa0;
                dst[kTile] = pa1;
            }
            if (ib.on) {
                uint64_t *dst = reinterpret_cast<uint64_t *>(ib.rout + (size_t)ch * ib.rstride);
                dst[0] = pb0;
                dst[kTile] = pb1;
            }
        }
        gb_flag(A, near_a && ia.on, (2 * item) * kTile + lane);
        gb_flag(A, near_b && ib.on, (2 * item + 1) * kTile + lane);
    }
}

// ---------------------------------------------------------------------------
// k_hidden_gb (v2): the same guard band with a cheaper step.
//
//   scaled state   Sobel features (0-7) carry w / (beta g1), corners (8-11)
//                  w / (beta g2) (g1, g2: the bank's two gains), so the stencil
//                  sums integer-coefficient combinations of the input traces
//                  and the LIF step stays one FFMA2: w' = w D + I.
//   stencil        any summation order is admissible here (the band covers the
//                  rounding of THIS order, gb_band2), so it shares subexpressions:
//                  each Sobel is 5 ops; the corners are 9 Q - 4 T with Q the
//                  sum of the corner's 2x2 block and T the window sum -- 39
//                  packed ops for the 12 features instead of 56 multiply-adds.
//   decision       q = w' - lo (one FADD2): its sign is the spike decision
//                  (FMUL.SAT q * 2^100 -> 0 / 1, accumulated into the 12-bit
//                  mask by one FFMA2 on the float pipe); near <=> 0 <= q < bw,
//                  one unsigned compare of the bit pattern; keep <=> live and
//                  0 <= w' < lo, one unsigned compare; w = keep ? w' : 0.
//                  A refractory neuron (w = 0, w' = I) may test near: that only
//                  adds a (rare) redo, never a wrong raster.
constexpr float kGbBig = 0x1p100f;

struct GbBand2 {
    float lo1, lo2;     // band lower edges, Sobel / corner units (rounded down)
    uint32_t bw1, bw2;  // bit patterns of the band widths (rounded up)
};

// Rigorous per-window bound of |float32 trajectory - float64 trajectory| (volts)
// for the v2 step, from the window's per-level trace maxima m[k] (cmax, rounded
// up): every FP32 op of the stencil rounds its result by at most u |bound of the
// result| (the intermediate bounds below follow the op tree of gb2_currents),
// the table entries by u m[k] per use (weighted by |coefficient|); then the
// FFMA and the rounding of D, the float64 side (2^-50 terms), and e <= D e + eps
// -> e_max = eps / (1 - D).  delta = 2 e_max + 8 u theta.
__device__ __forceinline__ GbBand2 gb_band2(const ItemState &it, const float *cmax, const snn_lif_t &p,
                                            double s1, double s2, double D) {
    double m[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) m[k] = (double)cmax[(it.lvp[k >> 2] >> (8 * (k & 3))) & 0xFFu];
    // Sobel H / V: (xa + xb) + 2 xc - ((xd + xe) + 2 xf); ops p1, h1, p2, h2, h1 - h2; table h1 + h2
    auto sob = [&](int a, int b, int c, int d, int e, int f, double &mag) {
        const double p1 = m[a] + m[b], h1 = p1 + 2.0 * m[c], p2 = m[d] + m[e], h2 = p2 + 2.0 * m[f];
        mag = h1 + h2;
        return (p1 + h1) + (p2 + h2) + 2.0 * (h1 + h2);
    };
    double g1 = 0.0, S1 = 0.0;
    double mH, mV;
    const double eH = sob(0, 2, 1, 6, 8, 7, mH), eV = sob(0, 6, 3, 2, 8, 5, mV);
    g1 = fmax(eH, eV);
    S1 = fmax(mH, mV);
    // D = 0.5 (H + V) + (x0 - x8), AD = 0.5 (H - V) + (x2 - x6) (gb2_currents): half of
    // H's and V's errors, the rounding of H +- V (bounded by |H| + |V|), the difference
    // (its rounding and its two table entries: 2 (m_a + m_b)) and the FMA's rounding
    const double mD = 2.0 * (m[0] + m[8]) + m[1] + m[3] + m[5] + m[7];
    const double mAD = 2.0 * (m[2] + m[6]) + m[1] + m[5] + m[3] + m[7];
    g1 = fmax(g1, 0.5 * (eH + eV + mH + mV) + 2.0 * (m[0] + m[8]) + mD);
    g1 = fmax(g1, 0.5 * (eH + eV + mH + mV) + 2.0 * (m[2] + m[6]) + mAD);
    S1 = fmax(S1, fmax(mD, mAD));
    // corners: pair sums, Q = sA + sB (error 2 Q), T = (Q_tl + Q_br) + ((x2 + x6) - x4),
    // C = fma(Q, 9, -4 T)
    const double all = m[0] + m[1] + m[2] + m[3] + m[4] + m[5] + m[6] + m[7] + m[8];
    const double Q[4] = {m[0] + m[1] + m[3] + m[4], m[1] + m[2] + m[4] + m[5], m[3] + m[4] + m[6] + m[7],
                         m[4] + m[5] + m[7] + m[8]};
    const double t1 = Q[0] + Q[3], a26 = m[2] + m[6], t3 = a26 + m[4], TB = t1 + t3;
    const double eT = 3.0 * t1 + a26 + t3 + TB;
    double g2 = 0.0, S2 = 0.0;
#pragma unroll
    for (int f = 0; f < 4; ++f) {
        const double tab = 5.0 * Q[f] + 4.0 * (all - Q[f]);
        g2 = fmax(g2, 18.0 * Q[f] + 4.0 * eT + 9.0 * Q[f] + 4.0 * TB + tab);
        S2 = fmax(S2, tab);
    }
    const double u = 0x1p-24;
    const double es = u * fmax(s1 * g1, s2 * g2) * (1.0 + 0x1p-20);
    const double bS = fmax(s1 * S1, s2 * S2) * (1.0 + 0x1p-20);
    const double theta = p.vt - p.el;
    const double eps = es + u * (2.02 * theta * D + 1.01 * bS) +
                       0x1p-50 * (fabs(p.el) + fabs(p.vt) + bS + 1.01 * theta);
    const double emax = eps / (1.0 - D);
    const double delta = 2.0 * emax + 8.0 * u * theta;
    GbBand2 b;
    if (theta - delta <= 0.0) {  // degenerate band: every decision is near
        b.lo1 = b.lo2 = 0.f;
        b.bw1 = b.bw2 = 0x7F800000u;
        return b;
    }
    b.lo1 = __double2float_rd((theta - delta) / s1);
    b.lo2 = __double2float_rd((theta - delta) / s2);
    b.bw1 = __float_as_uint(__double2float_ru(((theta + delta) / s1 - (double)b.lo1) * (1.0 + 0x1p-20)));
    b.bw2 = __float_as_uint(__double2float_ru(((theta + delta) / s2 - (double)b.lo2) * (1.0 + 0x1p-20)));
    return b;
}

// a - b on packed float2 (sub.rn.f32x2; there is no CUDA intrinsic for it)
__device__ __forceinline__ float2 gb_fsub2(float2 a, float2 b) {
    unsigned long long r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(*reinterpret_cast<unsigned long long *>(&a)),
        "l"(*reinterpret_cast<unsigned long long *>(&b)));
    return *reinterpret_cast<float2 *>(&r);
}

// The 12 scaled currents of two windows (the op tree gb_band2 bounds); the
// negated Sobels (features 4-7) are formed by the caller.
__device__ __forceinline__ void gb2_currents(const float2 (&x)[9], float2 (&I)[kNF]) {
    const float2 two = make_float2(2.f, 2.f), nine = make_float2(9.f, 9.f), m4 = make_float2(-4.f, -4.f);
    // Sobel H, V
    I[0] = gb_fsub2(__ffma2_rn(x[1], two, __fadd2_rn(x[0], x[2])), __ffma2_rn(x[7], two, __fadd2_rn(x[6], x[8])));
    I[1] = gb_fsub2(__ffma2_rn(x[3], two, __fadd2_rn(x[0], x[6])), __ffma2_rn(x[5], two, __fadd2_rn(x[2], x[8])));
    // Sobel D, AD
    // Sobel D, AD from H and V: D = 0.5 (H + V) + (x0 - x8), AD = 0.5 (H - V) + (x2 - x6)
    const float2 half = make_float2(0.5f, 0.5f);
    I[2] = __ffma2_rn(__fadd2_rn(I[0], I[1]), half, gb_fsub2(x[0], x[8]));
    I[3] = __ffma2_rn(gb_fsub2(I[0], I[1]), half, gb_fsub2(x[2], x[6]));
    // corners
    const float2 s01 = __fadd2_rn(x[0], x[1]), s34 = __fadd2_rn(x[3], x[4]), s12 = __fadd2_rn(x[1], x[2]);
    const float2 s45 = __fadd2_rn(x[4], x[5]), s67 = __fadd2_rn(x[6], x[7]), s78 = __fadd2_rn(x[7], x[8]);
    const float2 q0 = __fadd2_rn(s01, s34), q1 = __fadd2_rn(s12, s45), q2 = __fadd2_rn(s34, s67),
                 q3 = __fadd2_rn(s45, s78);
    const float2 T = __fadd2_rn(__fadd2_rn(q0, q3), gb_fsub2(__fadd2_rn(x[2], x[6]), x[4]));
    const float2 T4 = __fmul2_rn(T, m4);
    I[8] = __ffma2_rn(q0, nine, T4);
    I[9] = __ffma2_rn(q1, nine, T4);
    I[10] = __ffma2_rn(q2, nine, T4);
    I[11] = __ffma2_rn(q3, nine, T4);
}

// w' if the neuron is live (bit clear in the frozen mask F) and 0 <= w' < lo
// (one unsigned compare of the bit pattern), else 0: LOP3 -> predicate,
// ISETP.AND, SEL (inline PTX: the compiler otherwise splits it into two selects).
__device__ __forceinline__ float gb2_keep(float wn, unsigned F, unsigned bit, uint32_t ul) {
    uint32_t r;
    asm("{\n\t.reg .pred pf, pk;\n\t.reg .b32 t;\n\t"
        "and.b32 t, %1, %2;\n\t"
        "setp.ne.u32 pf, t, 0;\n\t"
        "setp.lt.and.u32 pk, %3, %4, !pf;\n\t"
        "selp.b32 %0, %3, 0, pk;\n\t}"
        : "=r"(r)
        : "r"(F), "r"(bit), "r"(__float_as_uint(wn)), "r"(ul));
    return __uint_as_float(r);
}

template <int FZ, int WARPS = kGbWarps>
__global__ void __launch_bounds__(WARPS * 32, 1) k_hidden_gb(const BatchArgs A) {
    extern __shared__ __align__(16) float gtab[];  // [N][256] fp32 input traces, then [256] max |c| per level
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int N = A.c.n_steps;
    const int nchunks = n_chunks(N);
    float *cmax = gtab + (size_t)N * 256;
    for (int i = tid; i < N * 256; i += WARPS * 32) gtab[i] = (float)__ldg(A.ctab + i);
    __syncthreads();
    if (tid < 256) {  // from the float table in shared memory (|float(c)| >= |c| (1 - 2^-24)), rounded up
        float m = 0.f;
        for (int s = 0; s < N; ++s) m = fmaxf(m, fabsf(gtab[s * 256 + tid]));
        cmax[tid] = (float)((double)m * (1.0 + 0x1p-20));
    }
    __syncthreads();
    const snn_lif_t &p = A.c.lif_hid;
    const double Dd = 1.0 - p.beta * p.g, s1 = p.beta * c_def_tap[0], s2 = p.beta * (c_def_tap[3] * 0.25);
    const float2 D2 = make_float2((float)Dd, (float)Dd);
    const int groups = hidden_items(A, 1);          // groups of 32 windows
    const int items = (groups + 1) >> 1;            // a lane takes window gw and gw + 32
    const int stride = (int)gridDim.x * WARPS;
    for (int item = warp * (int)gridDim.x + (int)blockIdx.x; item < items; item += stride) {
        ItemState ia, ib;
        window_setup(A, true, (2 * item) * kTile + lane, 0, nchunks, ia);
        window_setup(A, 2 * item + 1 < groups, (2 * item + 1) * kTile + lane, 0, nchunks, ib);
        const GbBand2 ba = gb_band2(ia, cmax, p, s1, s2, Dd), bb = gb_band2(ib, cmax, p, s1, s2, Dd);
        const float2 nlo1 = make_float2(-ba.lo1, -bb.lo1), nlo2 = make_float2(-ba.lo2, -bb.lo2);
        const uint32_t ula1 = __float_as_uint(ba.lo1), ulb1 = __float_as_uint(bb.lo1);
        const uint32_t ula2 = __float_as_uint(ba.lo2), ulb2 = __float_as_uint(bb.lo2);
        uint32_t offa[9], offb[9];  // byte offsets of the 9 levels in a table row
#pragma unroll
        for (int k = 0; k < 9; ++k) {
            offa[k] = ((ia.lvp[k >> 2] >> (8 * (k & 3))) & 0xFFu) * 4u;
            offb[k] = ((ib.lvp[k >> 2] >> (8 * (k & 3))) & 0xFFu) * 4u;
        }
        float2 w[kNF];
#pragma unroll
        for (int f = 0; f < kNF; ++f) w[f] = make_float2(0.f, 0.f);
        unsigned fza[FZ], fzb[FZ];
#pragma unroll
        for (int q = 0; q < FZ; ++q) fza[q] = fzb[q] = 0u;
        // smallest q bit pattern per window and feature class: near <=> min < bw
        // (one unsigned min per neuron-step; negative q never counts)
        uint32_t qa1 = 0xFFFFFFFFu, qa2 = 0xFFFFFFFFu, qb1 = 0xFFFFFFFFu, qb2 = 0xFFFFFFFFu;
        for (int ch = 0; ch < nchunks; ++ch) {
            const int s0 = ch * kChunk;
            const int nrows = min(kChunk, N - s0);
            uint64_t pa0 = 0, pa1 = 0, pb0 = 0, pb1 = 0;
#pragma unroll 1
            for (int j = 0; j < nrows; ++j) {
                const char *T = reinterpret_cast<const char *>(gtab + (size_t)(s0 + j) * 256);
                float2 x[9];
#pragma unroll
                for (int k = 0; k < 9; ++k)
                    x[k] = make_float2(*reinterpret_cast<const float *>(T + offa[k]),
                                       *reinterpret_cast<const float *>(T + offb[k]));
                unsigned Fa = 0, Fb = 0;
#pragma unroll
                for (int q = 0; q < FZ; ++q) {
                    Fa |= fza[q];
                    Fb |= fzb[q];
                }
                float2 I[kNF];
                gb2_currents(x, I);
                float2 acc = make_float2(0x1p23f, 0x1p23f);  // 2^23 + sum of fired bits: the mask is the low mantissa
#pragma unroll
                for (int f = 0; f < kNF; ++f) {
                    const float2 Ic = f >= 4 && f < 8 ? make_float2(-I[f - 4].x, -I[f - 4].y) : I[f];
                    const float2 wn = __ffma2_rn(w[f], D2, Ic);
                    const float2 q = __fadd2_rn(wn, f < 8 ? nlo1 : nlo2);
                    const float fa = __saturatef(q.x * kGbBig), fb = __saturatef(q.y * kGbBig);
                    acc = __ffma2_rn(make_float2(fa, fb), make_float2((float)(1 << f), (float)(1 << f)), acc);
                    if (f < 8) {
                        qa1 = min(qa1, __float_as_uint(q.x));
                        qb1 = min(qb1, __float_as_uint(q.y));
                    } else {
                        qa2 = min(qa2, __float_as_uint(q.x));
                        qb2 = min(qb2, __float_as_uint(q.y));
                    }
                    w[f] = make_float2(gb2_keep(wn.x, Fa, 1u << f, f < 8 ? ula1 : ula2),
                                       gb2_keep(wn.y, Fb, 1u << f, f < 8 ? ulb1 : ulb2));
                }
                const unsigned ma = __float_as_uint(acc.x) & ~Fa & 0xFFFu, mb = __float_as_uint(acc.y) & ~Fb & 0xFFFu;
#pragma unroll
                for (int q = FZ - 1; q > 0; --q) {
                    fza[q] = fza[q - 1];
                    fzb[q] = fzb[q - 1];
                }
                fza[0] = ma;
                fzb[0] = mb;
                pa0 |= (uint64_t)(ma & 0x3Fu) << (8 * j);
                pa1 |= (uint64_t)(ma >> kHalf) << (8 * j);
                pb0 |= (uint64_t)(mb & 0x3Fu) << (8 * j);
                pb1 |= (uint64_t)(mb >> kHalf) << (8 * j);
            }
            if (ia.on) {
                uint64_t *dst = reinterpret_cast<uint64_t *>(ia.rout + (size_t)ch * ia.rstride);
                dst[0] = pa0;
                dst[kTile] = pa1;
            }
            if (ib.on) {
                uint64_t *dst = reinterpret_cast<uint64_t *>(ib.rout + (size_t)ch * ib.rstride);
                dst[0] = pb0;
                dst[kTile] = pb1;
            }
        }
        const bool near_a = qa1 < ba.bw1 || qa2 < ba.bw2, near_b = qb1 < bb.bw1 || qb2 < bb.bw2;
        gb_flag(A, near_a && ia.on, (2 * item) * kTile + lane);
        gb_flag(A, near_b && ib.on, (2 * item + 1) * kTile + lane);
    }
}

// Taps of the default bank per feature (def_tap), for k_hidden_fix's lanes.
__constant__ double c_fix_tap[kNF][9] = {
#define SNN_TAPROW(f) {def_tap(f, 0), def_tap(f, 1), def_tap(f, 2), def_tap(f, 3), def_tap(f, 4), def_tap(f, 5), \
                       def_tap(f, 6), def_tap(f, 7), def_tap(f, 8)}
    SNN_TAPROW(0), SNN_TAPROW(1), SNN_TAPROW(2), SNN_TAPROW(3), SNN_TAPROW(4), SNN_TAPROW(5),
    SNN_TAPROW(6), SNN_TAPROW(7), SNN_TAPROW(8), SNN_TAPROW(9), SNN_TAPROW(10), SNN_TAPROW(11)
#undef SNN_TAPROW
};

// One LIF step of a hidden neuron with the frozen-history refractory rule of
// lif_update_fz (hidden.cuh): returns whether it spiked.
template <bool SGN, int FZ>
__device__ __forceinline__ bool fix_lif(double I, double &v, unsigned &hist, const LifK &ph) {
    double t = __dsub_rn(v, ph.el);
    t = __dmul_rn(ph.g, t);
    t = __dsub_rn(I, t);
    t = __dmul_rn(ph.beta, t);
    const double vn = __dadd_rn(v, t);
    const bool frozen = hist != 0u;
    const bool pa = frozen || (SGN ? __double_as_longlong(vn) >= ph.vt_bits : vn >= ph.vt);
    v = (pa || vn < ph.el) ? ph.el : vn;
    const bool fired = pa && !frozen;
    hist = ((hist << 1) | (fired ? 1u : 0u)) & ((1u << FZ) - 1u);
    return fired;
}

// FP64 re-simulation of the flagged windows with the exact step of
// k_hidden_res<.., FZ> (hidden_step_def_fz).  A window's 12 neurons are
// independent given its input traces, so four lanes share a window: lane g
// runs Sobel g, its negation g + 4 and corner g + 8 (the full 9-tap dgemm
// chain: a zero tap adds x * 0 exactly and fma(x, t, 0) = x * t, so the
// currents equal def_current's up to the sign of a zero, which the LIF update
// cannot see since v != 0); two shuffles OR the lanes' bits into the step's
// 12-bit mask.  A CTA's 32 windows advance in lockstep, so the table rows of
// the next 8-step chunk are copied into shared memory (cp.async, double
// buffered) while the current chunk computes: a step costs one stencil + one
// LIF, not an L2 round trip.
constexpr int kFixThreads = 128;
template <bool SGN, int FZ>
__global__ void __launch_bounds__(kFixThreads) k_hidden_fix(const BatchArgs A) {
    __shared__ __align__(16) double ftab[2][kChunk * 256];
    const int N = A.c.n_steps;
    const int nchunks = n_chunks(N);
    const int count = *A.fix_count;
    const LifK ph = lif_k(A.c.lif_hid);
    const int g = threadIdx.x & 3;
    double ts[9], tc[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) {
        ts[k] = c_fix_tap[g][k];
        tc[k] = c_fix_tap[8 + g][k];
    }
    // copy table rows [ch * 8, ch * 8 + 8) into buffer b (16-byte cp.async)
    auto fetch = [&](int ch, int b) {
        const int rows = min(kChunk, N - ch * kChunk);
        const double *src = A.ctab + (size_t)ch * kChunk * 256;
        for (int i = threadIdx.x; i < rows * 128; i += kFixThreads) {
            const uint32_t dst = (uint32_t)__cvta_generic_to_shared(&ftab[b][2 * i]);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src + 2 * i));
        }
        asm volatile("cp.async.commit_group;");
    };
    const int nthr = (int)(gridDim.x * kFixThreads);
    for (int tb = (int)(blockIdx.x * kFixThreads); tb < 4 * count; tb += nthr) {  // CTA-uniform
        const int t = (tb + (int)threadIdx.x) >> 2;  // this quad's window
        const bool have = t < count;
        ItemState it;
        window_setup(A, have, have ? A.fix_list[t] : 0, 0, nchunks, it);
        uint32_t off[9];
#pragma unroll
        for (int k = 0; k < 9; ++k) off[k] = (it.lvp[k >> 2] >> (8 * (k & 3))) & 0xFFu;
        double v0 = A.c.lif_hid.el, v1 = v0, v2 = v0;
        unsigned h0 = 0, h1 = 0, h2 = 0;
        __syncthreads();  // the previous pass is done with both buffers
        fetch(0, 0);
        for (int ch = 0; ch < nchunks; ++ch) {
            if (ch + 1 < nchunks) {
                fetch(ch + 1, (ch + 1) & 1);
                asm volatile("cp.async.wait_group 1;");
            } else {
                asm volatile("cp.async.wait_group 0;");
            }
            __syncthreads();  // chunk ch is in buffer ch & 1
            const double *T = ftab[ch & 1];
            const int nrows = min(kChunk, N - ch * kChunk);
            uint64_t p0 = 0, p1 = 0;
            for (int j = 0; j < nrows; ++j) {
                double x[9];
#pragma unroll
                for (int k = 0; k < 9; ++k) x[k] = T[j * 256 + off[k]];
                double Is = __dmul_rn(x[0], ts[0]), Ic = __dmul_rn(x[0], tc[0]);
#pragma unroll
                for (int k = 1; k < 9; ++k) {
                    Is = __fma_rn(x[k], ts[k], Is);
                    Ic = __fma_rn(x[k], tc[k], Ic);
                }
                unsigned m = fix_lif<SGN, FZ>(Is, v0, h0, ph) ? 1u << g : 0u;
                m |= fix_lif<SGN, FZ>(-Is, v1, h1, ph) ? 1u << (g + 4) : 0u;
                m |= fix_lif<SGN, FZ>(Ic, v2, h2, ph) ? 1u << (g + 8) : 0u;
                m |= __shfl_xor_sync(kFull, m, 1);
                m |= __shfl_xor_sync(kFull, m, 2);
                p0 |= (uint64_t)(m & 0x3Fu) << (8 * j);
                p1 |= (uint64_t)(m >> kHalf) << (8 * j);
            }
            if (g == 0 && have && it.on) {
                uint64_t *dst = reinterpret_cast<uint64_t *>(it.rout + (size_t)ch * it.rstride);
                dst[0] = p0;
                dst[kTile] = p1;
            }
            __syncthreads();  // everyone is done with buffer ch & 1 before it is refilled
        }
    }
}

// The same redo with the whole [N][256] table resident in shared memory (one
// cooperative load per CTA, N <= kResMaxSteps): no per-chunk copies or
// barriers, so a window's 4 lanes run their N steps back to back.  512
// threads per CTA, one CTA per SM, windows dealt round-robin over the CTAs
// (the redo list of a small batch still spreads over every SM); a CTA with no
// flagged window returns before loading the table.
constexpr int kFixResThreads = 512;
template <bool SGN, int FZ>
__global__ void __launch_bounds__(kFixResThreads, 1) k_hidden_fix_res(const BatchArgs A) {
    extern __shared__ __align__(16) double rtab[];  // [N][256]
    const int N = A.c.n_steps;
    const int count = *A.fix_count;
    if ((int)blockIdx.x >= count) return;  // CTA-uniform: no flagged window for this CTA
    {
        const uint4 *src = reinterpret_cast<const uint4 *>(A.ctab);
        uint4 *dst = reinterpret_cast<uint4 *>(rtab);
        for (int i = threadIdx.x; i < N * 128; i += kFixResThreads) dst[i] = __ldg(src + i);
    }
    __syncthreads();
    const int nchunks = n_chunks(N);
    const LifK ph = lif_k(A.c.lif_hid);
    const int g = threadIdx.x & 3;
    double ts[9], tc[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) {
        ts[k] = c_fix_tap[g][k];
        tc[k] = c_fix_tap[8 + g][k];
    }
    // windows dealt round-robin over the CTAs (quad q of CTA b takes windows
    // q * G + b, + 128 G, ...), so a short list still spreads over every SM;
    // a warp whose 8 windows are all past the list skips the pass
    const int G = (int)gridDim.x, quad = (int)threadIdx.x >> 2, warp = (int)threadIdx.x >> 5;
    for (int base = 0; base < count; base += (kFixResThreads / 4) * G) {
        if (base + warp * 8 * G + (int)blockIdx.x >= count) break;  // warp-uniform
        const int t = base + quad * G + (int)blockIdx.x;  // this quad's window
        const bool have = t < count;
        ItemState it;
        window_setup(A, have, have ? A.fix_list[t] : 0, 0, nchunks, it);
        uint32_t off[9];
#pragma unroll
        for (int k = 0; k < 9; ++k) off[k] = (it.lvp[k >> 2] >> (8 * (k & 3))) & 0xFFu;
        double v0 = A.c.lif_hid.el, v1 = v0, v2 = v0;
        unsigned h0 = 0, h1 = 0, h2 = 0;
        for (int ch = 0; ch < nchunks; ++ch) {
            const double *T = rtab + (size_t)ch * kChunk * 256;
            const int nrows = min(kChunk, N - ch * kChunk);
#ifdef SNN_FIX_PIPE
            // the chunk's currents first (16 independent 9-tap chains), then the
            // lane's three membrane chains step by step
            double Is[kChunk], Ic[kChunk];
#pragma unroll
            for (int j = 0; j < kChunk; ++j) {
                const double *R = T + (j < nrows ? j : 0) * 256;
                double x[9];
#pragma unroll
                for (int k = 0; k < 9; ++k) x[k] = R[off[k]];
                Is[j] = __dmul_rn(x[0], ts[0]);
                Ic[j] = __dmul_rn(x[0], tc[0]);
#pragma unroll
                for (int k = 1; k < 9; ++k) {
                    Is[j] = __fma_rn(x[k], ts[k], Is[j]);
                    Ic[j] = __fma_rn(x[k], tc[k], Ic[j]);
                }
            }
            // this lane's bits of the chunk's planes: feature g (plane 0), g + 4
            // (plane 0 for g < 2, else plane 1 bit g - 2), g + 8 (plane 1 bit g + 2)
            uint64_t p0 = 0, p1 = 0;
#pragma unroll
            for (int j = 0; j < kChunk; ++j) {
                if (j < nrows) {
                    const uint64_t b0 = fix_lif<SGN, FZ>(Is[j], v0, h0, ph) ? 1u : 0u;
                    const uint64_t b1 = fix_lif<SGN, FZ>(-Is[j], v1, h1, ph) ? 1u : 0u;
                    const uint64_t b2 = fix_lif<SGN, FZ>(Ic[j], v2, h2, ph) ? 1u : 0u;
                    p0 |= b0 << (8 * j + g);
                    if (g < 2) p0 |= b1 << (8 * j + g + 4);
                    else p1 |= b1 << (8 * j + g - 2);
                    p1 |= b2 << (8 * j + g + 2);
                }
            }
            p0 |= __shfl_xor_sync(kFull, p0, 1);
            p1 |= __shfl_xor_sync(kFull, p1, 1);
            p0 |= __shfl_xor_sync(kFull, p0, 2);
            p1 |= __shfl_xor_sync(kFull, p1, 2);
#else
            uint64_t p0 = 0, p1 = 0;
            for (int j = 0; j < nrows; ++j) {
                double x[9];
#pragma unroll
                for (int k = 0; k < 9; ++k) x[k] = T[j * 256 + off[k]];
                double Is = __dmul_rn(x[0], ts[0]), Ic = __dmul_rn(x[0], tc[0]);
#pragma unroll
                for (int k = 1; k < 9; ++k) {
                    Is = __fma_rn(x[k], ts[k], Is);
                    Ic = __fma_rn(x[k], tc[k], Ic);
                }
                unsigned m = fix_lif<SGN, FZ>(Is, v0, h0, ph) ? 1u << g : 0u;
                m |= fix_lif<SGN, FZ>(-Is, v1, h1, ph) ? 1u << (g + 4) : 0u;
                m |= fix_lif<SGN, FZ>(Ic, v2, h2, ph) ? 1u << (g + 8) : 0u;
                m |= __shfl_xor_sync(kFull, m, 1);
                m |= __shfl_xor_sync(kFull, m, 2);
                p0 |= (uint64_t)(m & 0x3Fu) << (8 * j);
                p1 |= (uint64_t)(m >> kHalf) << (8 * j);
            }
#endif
            if (g == 0 && have && it.on) {
                uint64_t *dst = reinterpret_cast<uint64_t *>(it.rout + (size_t)ch * it.rstride);
                dst[0] = p0;
                dst[kTile] = p1;
            }
        }
    }
}

}  // namespace snn
