// Microbenchmark of the serial output-layer scan (out_step) and of the FP64
// dependent-issue latency, one warp, clock64 timing.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        --expt-relaxed-constexpr -Xcompiler -fPIC -shared -I include \
//        -o scripts/libscan_micro.so scripts/scan_micro.cu
#include "../paper_1711_03637_b200/csrc/hidden.cuh"

using namespace snn;
namespace {

// A lane-distributed alternative to the product out_step (hidden.cuh), kept
// here as a measured experiment: each lane owns one trace and the warp
// speculates the inhibition sums through shared memory.  Bit-identical, fewer
// instructions, but slower on the serial chain (scripts/scan_micro.py).
// ---------------------------------------------------------------------------
// Output layer (network.py:308-314): lanes 0..9 of one warp are the 10 output
// neurons (lanes 10..31 shadow lane 9 and are masked out of the ballot), and
// lane q < 10 also owns the lateral-inhibition trace of neuron q.
//
// The step is serial, so its chain is cut short by speculating one step
// ahead.  While step s runs, each trace owner forms both candidates of its
// c = a - b for step s+1: c0 if neuron q does not fire at s (a*lam + 0 ==
// a*lam exactly, a >= 0) and c1 = (a*lam + 1) - (b*lam + 1) if it does.  The
// warp then evaluates numpy's pairwise sum of the ten c's for the outcomes
// that cover >99% of steps: lanes 0..9 and 20..31 the no-spike sum S0, lane
// 10+q the sum with only neuron q's c1 substituted.  Step s+1 picks its sum
// with no arithmetic (no output spike at s) or one shuffle (one spike); two
// or more simultaneous spikes redo the sum from the staged candidates.  The
// candidates are exchanged through kDistSpecBytes of shared memory per warp
// (two step-parity buffers of 5 pairs x 3 variants (c0,c0) (c1,c0) (c0,c1),
// 16 B each), so every lane loads its own ten inputs with five 16-byte
// loads.  Every value is the reference's own operation sequence, so results
// are bit-identical whichever path a step takes.
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
__device__ __forceinline__ bool dist_step(DistState &st, const DistK &k, double G, int s, int l, int lane,
                                         double *ff_out) {
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
    st.v = (!live || fired || vn < k.el) ? k.el : vn;
    if (fired) st.live_from = next_live_step(s, k.refr);
    st.prev = __ballot_sync(kFull, fired) & 0x3FFu;
    st.cnt += fired ? 1 : 0;
    // the next step's speculative sum
    st.T = pairwise10(x);
    *ff_out = ff;
    return fired;
}


__global__ void k_lat(double *out, long long *cyc, int iters, double x0) {
    double a = x0, b = x0 * 0.5, m = 1.0000001;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        a = __dadd_rn(a, b);
        a = __dmul_rn(a, m);
    }
    long long t1 = clock64();
    out[threadIdx.x] = a;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

// A compact output step (measured, not used: 292 vs 232 cycles per step --
// fewer FP64 instructions but more branch and predicate latency on the chain)
// Compact form of the same step while at most two output neurons have ever
// spiked in this trial (>90% of images): the traces of a neuron that never
// spiked are exactly +0, and the pairwise sum of ten values of which at most
// two are non-zero (all >= +0) is exactly their plain sum -- so only the two
// occupied trace slots are carried (22 FP64 ops per step instead of ~57).
// outc_step returns false, before touching the state, when a third neuron
// spikes; the caller then converts to OutState (outc_to_full) and continues
// with out_step from that step.  Bit-identical to out_step throughout.
struct OutC {
    double Af, Bf;
    double al0, bl0, al1, bl1;  // slot traces times their decay (before this step's bumps)
    double S0, c0;              // no-spike sum and own c for this step
    double v;
    int q0, q1;                 // output neuron of each slot, -1 = free (warp-uniform)
    int live_from, cnt;
    unsigned prev;
};

__device__ __forceinline__ void outc_init(OutC &st, const snn_consts_t &c) {
    st.Af = st.Bf = 0.0;
    st.al0 = st.bl0 = st.al1 = st.bl1 = 0.0;
    st.S0 = st.c0 = 0.0;
    st.v = c.lif_out.el;
    st.q0 = st.q1 = -1;
    st.live_from = 0;
    st.cnt = 0;
    st.prev = 0u;
}

__device__ __forceinline__ void outc_to_full(const OutC &sc, OutState &st, int l) {
    st.Af = sc.Af;
    st.Bf = sc.Bf;
#pragma unroll
    for (int k = 0; k < kNO; ++k) {
        st.al[k] = k == sc.q0 ? sc.al0 : k == sc.q1 ? sc.al1 : 0.0;
        st.bl[k] = k == sc.q0 ? sc.bl0 : k == sc.q1 ? sc.bl1 : 0.0;
    }
    st.al_o = l == sc.q0 ? sc.al0 : l == sc.q1 ? sc.al1 : 0.0;
    st.bl_o = l == sc.q0 ? sc.bl0 : l == sc.q1 ? sc.bl1 : 0.0;
    st.S0 = sc.S0;
    st.c0 = sc.c0;
    st.v = sc.v;
    st.live_from = sc.live_from;
    st.cnt = sc.cnt;
    st.prev = sc.prev;
}

__device__ __forceinline__ bool outc_step(OutC &st, const snn_consts_t &c, double G, int s, int l, double *ff_out) {
    const unsigned pv = st.prev;  // warp-uniform
    int q0 = st.q0, q1 = st.q1;
    if (pv != 0u) {
        const unsigned slots = (q0 >= 0 ? 1u << q0 : 0u) | (q1 >= 0 ? 1u << q1 : 0u);
        unsigned nw = pv & ~slots;
        if (nw) {  // first spikes of new neurons take the free slots, in ascending order
            const int free = (q0 < 0) + (q1 < 0);
            if (__popc(nw) > free) return false;
            if (q0 < 0) {
                q0 = __ffs(nw) - 1;
                nw &= nw - 1u;
            }
            if (nw) q1 = __ffs(nw) - 1;
        }
    }
    st.q0 = q0;
    st.q1 = q1;
    st.Af = __dadd_rn(__dmul_rn(st.Af, c.decay_slow), G);
    st.Bf = __dadd_rn(__dmul_rn(st.Bf, c.decay_fast), G);
    const double ff = __dsub_rn(st.Af, st.Bf);
    double a0 = st.al0, b0 = st.bl0, a1 = st.al1, b1 = st.bl1, S, co;
    if (pv == 0u) {
        S = st.S0;
        co = st.c0;
    } else {
        const double u0 = (q0 >= 0 && ((pv >> q0) & 1u)) ? 1.0 : 0.0;
        const double u1 = (q1 >= 0 && ((pv >> q1) & 1u)) ? 1.0 : 0.0;
        a0 = __dadd_rn(a0, u0);
        b0 = __dadd_rn(b0, u0);
        a1 = __dadd_rn(a1, u1);
        b1 = __dadd_rn(b1, u1);
        const double c0 = __dsub_rn(a0, b0), c1 = __dsub_rn(a1, b1);
        S = q1 >= 0 ? __dadd_rn(c0, c1) : c0;
        co = l == q0 ? c0 : l == q1 ? c1 : 0.0;
    }
    st.al0 = __dmul_rn(a0, c.decay_slow);
    st.bl0 = __dmul_rn(b0, c.decay_fast);
    st.al1 = __dmul_rn(a1, c.decay_slow);
    st.bl1 = __dmul_rn(b1, c.decay_fast);
    const double n0 = __dsub_rn(st.al0, st.bl0), n1 = __dsub_rn(st.al1, st.bl1);
    st.S0 = q1 >= 0 ? __dadd_rn(n0, n1) : n0;
    st.c0 = l == q0 ? n0 : l == q1 ? n1 : 0.0;
    const double drive = __dadd_rn(ff, __dmul_rn(c.inhibition, __dsub_rn(S, co)));
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
    return true;
}


// experimental step variants (same state as OutState; extra fields below)
struct XState {
    DistState o;
    double gv;   // g * (v - E_L) of the current v
    double D0;   // drive if no output spiked at the previous step
};

// V 2: drive chain first in program order; V 3: + precomputed g*(v-EL) and
// no-spike drive D0
template <int V>
__device__ __forceinline__ bool x_step(XState &X, const DistK &k, double G, double Gn, int s, int l, int lane) {
    DistState &st = X.o;
    const unsigned pv = st.prev;
    const bool mine = (pv >> l) & 1u;
    const double a = mine ? st.ap : st.al;
    const double b = mine ? st.bp : st.bl;
    const double co = mine ? st.c1 : st.c0;
    double drive;
    double ff;
    if (V == 3) {
        ff = 0.0;
        if (pv == 0u) {
            drive = X.D0;
        } else {
            double S;
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
            const double f = __dsub_rn(st.Af, st.Bf);
            drive = __dadd_rn(f, __dmul_rn(k.inh, __dsub_rn(S, co)));
        }
    } else {
        st.Af = __dadd_rn(__dmul_rn(st.Af, k.lam1), G);
        st.Bf = __dadd_rn(__dmul_rn(st.Bf, k.lam2), G);
        ff = __dsub_rn(st.Af, st.Bf);
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
        drive = __dadd_rn(ff, __dmul_rn(k.inh, __dsub_rn(S, co)));
    }
    double t;
    if (V == 3) t = X.gv;
    else t = __dmul_rn(k.g, __dsub_rn(st.v, k.el));
    t = __dsub_rn(drive, t);
    t = __dmul_rn(k.beta, t);
    const double vn = __dadd_rn(st.v, t);
    const bool live = s >= st.live_from;
    const bool fired = live && vn >= k.vt;
    st.v = (!live || fired || vn < k.el) ? k.el : vn;
    if (fired) st.live_from = next_live_step(s, k.refr);
    st.prev = __ballot_sync(kFull, fired) & 0x3FFu;
    st.cnt += fired ? 1 : 0;
    // candidates for the next step
    st.al = __dmul_rn(a, k.lam1);
    st.bl = __dmul_rn(b, k.lam2);
    st.c0 = __dsub_rn(st.al, st.bl);
    st.ap = __dadd_rn(st.al, 1.0);
    st.bp = __dadd_rn(st.bl, 1.0);
    st.c1 = __dsub_rn(st.ap, st.bp);
    const unsigned nxt = (st.cur & 256u) ? st.cur - 256u : st.cur + 256u;
    st.cur = nxt;
    sts64(nxt + st.w0a, st.c0);
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
    st.T = pairwise10(x);
    if (V == 3) {
        X.gv = __dmul_rn(k.g, __dsub_rn(st.v, k.el));
        // next step's feed-forward and no-spike drive
        st.Af = __dadd_rn(__dmul_rn(st.Af, k.lam1), Gn);
        st.Bf = __dadd_rn(__dmul_rn(st.Bf, k.lam2), Gn);
        const double f = __dsub_rn(st.Af, st.Bf);
        X.D0 = __dadd_rn(f, __dmul_rn(k.inh, __dsub_rn(st.T, st.c0)));
    }
    return fired;
}

// G: [N][10] per image in global; one warp scans n_img images back to back
// with G staged in shared memory, as the cluster leader does.  variant 0 =
// product out_step (replicated traces), 1 = lane-distributed dist_step.  Output masks per
// step go to om_out [n_img][N] and final v to v_out [n_img][10].
template <int V>
__global__ void k_scan(snn_consts_t c, const double *G, int n_img, int32_t *counts, long long *cyc,
                       uint16_t *om_out, double *v_out) {
    extern __shared__ double sG[];
    __shared__ __align__(512) char spec[kDistSpecBytes];
    const int N = c.n_steps;
    const int lane = threadIdx.x & 31;
    long long tot = 0;
    for (int i = 0; i < n_img; ++i) {
        for (int t = threadIdx.x; t < N * kNO; t += blockDim.x) sG[t] = G[(size_t)i * N * kNO + t];
        __syncthreads();
        if (threadIdx.x < 32) {
            const int l = lane < kNO ? lane : kNO - 1;
            const double *gp = sG + l;
            uint16_t *om = om_out + (size_t)i * N;
            long long t0, t1;
            double v;
            int cnt;
            if (V == 0) {
                OutState st;
                out_init(st, c);
                t0 = clock64();
                for (int s = 0; s < N; ++s) {
                    double ff;
                    out_step(st, c, gp[s * kNO], s, l, &ff);
                    if (lane == 0) om[s] = (uint16_t)st.prev;
                }
                t1 = clock64();
                v = st.v; cnt = st.cnt;
            } else if (V == 7) {
                OutD X;
                out_init(X.o, c);
                // step 0's feed-forward and drive (no spikes before it: S0 = c0 = +0)
                X.o.Af = __dadd_rn(__dmul_rn(0.0, c.decay_slow), gp[0]);
                X.o.Bf = __dadd_rn(__dmul_rn(0.0, c.decay_fast), gp[0]);
                X.D0 = __dadd_rn(__dsub_rn(X.o.Af, X.o.Bf), __dmul_rn(c.inhibition, __dsub_rn(0.0, 0.0)));
                t0 = clock64();
                for (int s = 0; s < N; ++s) {
                    outd_step(X, c, gp[(s + 1 < N ? s + 1 : s) * kNO], s, l);
                    if (lane == 0) om[s] = (uint16_t)X.o.prev;
                }
                t1 = clock64();
                v = X.o.v; cnt = X.o.cnt;
            } else if (V == 6) {
                OutC sc;
                outc_init(sc, c);
                t0 = clock64();
                int s = 0;
                double ff;
                for (; s < N; ++s) {
                    if (!outc_step(sc, c, gp[s * kNO], s, l, &ff)) break;
                    if (lane == 0) om[s] = (uint16_t)sc.prev;
                }
                if (s < N) {
                    OutState st;
                    outc_to_full(sc, st, l);
                    for (; s < N; ++s) {
                        out_step(st, c, gp[s * kNO], s, l, &ff);
                        if (lane == 0) om[s] = (uint16_t)st.prev;
                    }
                    v = st.v; cnt = st.cnt;
                } else {
                    v = sc.v; cnt = sc.cnt;
                }
                t1 = clock64();
            } else if (V >= 2) {
                XState X;
                dist_init(X.o, c, spec, lane);
                const DistK ok = dist_k(c);
                constexpr int VV = V % 10;
                if (VV == 3) {
                    X.gv = __dmul_rn(ok.g, __dsub_rn(X.o.v, ok.el));
                    X.o.Af = gp[0];
                    X.o.Bf = gp[0];
                    X.D0 = __dadd_rn(__dsub_rn(X.o.Af, X.o.Bf), __dmul_rn(ok.inh, __dsub_rn(X.o.T, X.o.c0)));
                }
                t0 = clock64();
                if (V >= 10) {
#pragma unroll 2
                    for (int s = 0; s < N; ++s) {
                        x_step<VV>(X, ok, gp[s * kNO], gp[(s + 1 < N ? s + 1 : s) * kNO], s, l, lane);
                        if (lane == 0) om[s] = (uint16_t)X.o.prev;
                    }
                } else {
#pragma unroll 1
                    for (int s = 0; s < N; ++s) {
                        x_step<VV>(X, ok, gp[s * kNO], gp[(s + 1 < N ? s + 1 : s) * kNO], s, l, lane);
                        if (lane == 0) om[s] = (uint16_t)X.o.prev;
                    }
                }
                t1 = clock64();
                v = X.o.v; cnt = X.o.cnt;
            } else {
                DistState st;
                dist_init(st, c, spec, lane);
                const DistK ok = dist_k(c);
                t0 = clock64();
                for (int s = 0; s < N; ++s) {
                    double ff;
                    dist_step(st, ok, gp[s * kNO], s, l, lane, &ff);
                    if (lane == 0) om[s] = (uint16_t)st.prev;
                }
                t1 = clock64();
                v = st.v; cnt = st.cnt;
            }
            tot += t1 - t0;
            if (lane < kNO) {
                counts[i * kNO + lane] = cnt;
                v_out[i * kNO + lane] = v;
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) cyc[1] = tot;
}


// latency probes (one warp): 0 = LDS.64 pointer chase, 1 = STS -> syncwarp
// -> LDS round trip, 2 = DSETP -> VOTE -> select chain, 3 = SHFL.IDX chain
// of a double, 4 = DADD chain
__global__ void k_probe(int mode, int iters, long long *cyc, double *out) {
    __shared__ __align__(16) double buf[64];
    const int lane = threadIdx.x;
    buf[lane] = (double)((lane + 1) & 31);
    buf[32 + lane] = 0.0;
    __syncwarp();
    const unsigned base = (unsigned)__cvta_generic_to_shared(buf);
    double x = (double)lane;
    int idx = lane;
    long long t0 = clock64();
    if (mode == 0) {
        for (int i = 0; i < iters; ++i) idx = (int)lds64(base + 8u * idx);
    } else if (mode == 1) {
        for (int i = 0; i < iters; ++i) {
            sts64(base + 256u + 8u * ((lane + 1) & 31), x);
            __syncwarp();
            x = lds64(base + 256u + 8u * lane) + 0.0;
        }
    } else if (mode == 2) {
        for (int i = 0; i < iters; ++i) {
            const unsigned b = __ballot_sync(0xffffffffu, x >= 3.0);
            x = (b & 1u) ? x : x + 1.0;
        }
    } else if (mode == 3) {
        for (int i = 0; i < iters; ++i) x = __shfl_sync(0xffffffffu, x, (lane + 1) & 31);
    } else {
        for (int i = 0; i < iters; ++i) x = __dadd_rn(x, 1.0);
    }
    long long t1 = clock64();
    out[lane] = x + idx;
    if (lane == 0) cyc[0] = t1 - t0;
}
// ---- two-warp scan: warp 0 (driver) runs the output LIF chain, warp 1
// (speculator) turns the spikes of step s-1 into the inhibition sums of step
// s+1 for the no-spike case (S0) and every single-spike case (S1[q]).  The
// two talk through shared memory: each value slot is written once and read
// by polling (a NaN sentinel marks "not yet").
constexpr int kS2Max = 128;
constexpr unsigned long long kSent = 0x7FF8DEAD0000BEEFull;
struct Scan2Smem {
    double sum[kS2Max + 1][11];
    double cc[2][2][kNO];  // driver: each trace's c0 / c1 candidates, by step parity (multi-spike steps)
    unsigned pm[kS2Max + 1];
};

__device__ __forceinline__ double poll_f64(const double *p) {
    const volatile long long *q = reinterpret_cast<const volatile long long *>(p);
    long long x;
    do {
        x = *q;
    } while (x == (long long)kSent);
    return __longlong_as_double(x);
}
__device__ __forceinline__ unsigned poll_u32(const unsigned *p) {
    const volatile unsigned *q = p;
    unsigned x;
    do {
        x = *q;
    } while (x == 0xFFFFFFFFu);
    return x;
}
__device__ __forceinline__ void post_f64(double *p, double v) { *reinterpret_cast<volatile double *>(p) = v; }
__device__ __forceinline__ void post_u32(unsigned *p, unsigned v) { *reinterpret_cast<volatile unsigned *>(p) = v; }

// driver: lane l = output neuron l (lanes >= 10 shadow neuron 9)
__device__ __forceinline__ int scan2_driver(const snn_consts_t &c, const double *gp, int N, Scan2Smem &X,
                                            uint16_t *om, double *v_out) {
    const int lane = threadIdx.x & 31, l = lane < kNO ? lane : kNO - 1;
    const double lam1 = c.decay_slow, lam2 = c.decay_fast, inh = c.inhibition;
    const double el = c.lif_out.el, vt = c.lif_out.vt, g = c.lif_out.g, beta = c.lif_out.beta, refr = c.lif_out.refr;
    double Af = 0.0, Bf = 0.0, v = el, al = 0.0, bl = 0.0, ap = 1.0, bp = 1.0, c0 = 0.0, c1 = 0.0;
    int live_from = 0, cnt = 0;
    unsigned prev = 0u;
    for (int s = 0; s < N; ++s) {
        const double G = gp[s * kNO];
        Af = __dadd_rn(__dmul_rn(Af, lam1), G);
        Bf = __dadd_rn(__dmul_rn(Bf, lam2), G);
        const double ff = __dsub_rn(Af, Bf);
        const unsigned pv = prev;
        const bool mine = (pv >> l) & 1u;
        const double c0c = c0, c1c = c1;  // this step's own candidates
        const double co = mine ? c1c : c0c;
        // own trace into the next step
        const double a = mine ? ap : al, b = mine ? bp : bl;
        al = __dmul_rn(a, lam1);
        bl = __dmul_rn(b, lam2);
        c0 = __dsub_rn(al, bl);
        ap = __dadd_rn(al, 1.0);
        bp = __dadd_rn(bl, 1.0);
        c1 = __dsub_rn(ap, bp);
        double S;
        if (s == 0) {
            S = 0.0;
        } else if (pv == 0u) {
            S = poll_f64(&X.sum[s][0]);
        } else if ((pv & (pv - 1u)) == 0u) {
            S = poll_f64(&X.sum[s][__ffs((int)pv)]);
        } else {  // two or more spikes: the sum with their bumps
            __syncwarp();
            const double *cc = &X.cc[s & 1][0][0];
            double x[kNO];
#pragma unroll
            for (int k = 0; k < kNO; ++k) x[k] = cc[(((pv >> k) & 1u) ? kNO : 0) + k];
            S = pairwise10(x);
        }
        if (lane < kNO) {  // the next step's candidates, for a multi-spike step
            X.cc[(s + 1) & 1][0][lane] = c0;
            X.cc[(s + 1) & 1][1][lane] = c1;
        }
        const double drive = __dadd_rn(ff, __dmul_rn(inh, __dsub_rn(S, co)));
        double t = __dsub_rn(v, el);
        t = __dmul_rn(g, t);
        t = __dsub_rn(drive, t);
        t = __dmul_rn(beta, t);
        const double vn = __dadd_rn(v, t);
        const bool live = s >= live_from;
        const bool fired = live && vn >= vt;
        v = (!live || fired || vn < el) ? el : vn;
        if (fired) live_from = next_live_step(s, refr);
        prev = __ballot_sync(kFull, fired) & 0x3FFu;
        cnt += fired ? 1 : 0;
        if (lane == 0) {
            post_u32(&X.pm[s + 1], prev);
            om[s] = (uint16_t)prev;
        }
    }
    if (lane < kNO) v_out[lane] = v;
    return cnt;
}

// speculator: lane q < 10 owns trace q; lanes 10 + q form the single-spike sums
__device__ __forceinline__ void scan2_spec(const snn_consts_t &c, int N, Scan2Smem &X, char *xbuf) {
    const int lane = threadIdx.x & 31;
    const double lam1 = c.decay_slow, lam2 = c.decay_fast;
    DistState st;
    dist_init(st, c, xbuf, lane);
    const int q = lane < kNO ? lane : kNO - 1;
    for (int s = 0; s + 1 < N; ++s) {
        const unsigned pv = poll_u32(&X.pm[s]);
        const bool mine = (pv >> q) & 1u;
        const double a = mine ? st.ap : st.al, b = mine ? st.bp : st.bl;
        st.al = __dmul_rn(a, lam1);
        st.bl = __dmul_rn(b, lam2);
        st.c0 = __dsub_rn(st.al, st.bl);
        st.ap = __dadd_rn(st.al, 1.0);
        st.bp = __dadd_rn(st.bl, 1.0);
        st.c1 = __dsub_rn(st.ap, st.bp);
        const unsigned nxt = (st.cur & 256u) ? st.cur - 256u : st.cur + 256u;
        st.cur = nxt;
        sts64(nxt + st.w0a, st.c0);
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
        const double T = pairwise10(x);
        if (lane == 0) post_f64(&X.sum[s + 1][0], T);
        else if (lane >= kNO && lane < 2 * kNO) post_f64(&X.sum[s + 1][1 + lane - kNO], T);
    }
}

__global__ void __launch_bounds__(128) k_scan2(snn_consts_t c, const double *G, int n_img, int32_t *counts, long long *cyc,
                        uint16_t *om_out, double *v_out) {
    extern __shared__ double sG[];
    __shared__ Scan2Smem X;
    __shared__ __align__(512) char xbuf[kDistSpecBytes];
    const int N = c.n_steps;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    long long tot = 0;
    for (int i = 0; i < n_img; ++i) {
        for (int t = threadIdx.x; t < N * kNO; t += blockDim.x) sG[t] = G[(size_t)i * N * kNO + t];
        for (int t = threadIdx.x; t < (N + 1) * 11; t += blockDim.x)
            (&X.sum[0][0])[t] = __longlong_as_double((long long)kSent);
        for (int t = threadIdx.x; t <= N; t += blockDim.x) X.pm[t] = t == 0 ? 0u : 0xFFFFFFFFu;
        for (int t = threadIdx.x; t < 2 * 2 * kNO; t += blockDim.x) (&X.cc[0][0][0])[t] = 0.0;
        __syncthreads();
        if (warp == 0) {
            const long long t0 = clock64();
            const int l = lane < kNO ? lane : kNO - 1;
            const int cnt = scan2_driver(c, sG + l, N, X, om_out + (size_t)i * N, v_out + i * kNO);
            tot += clock64() - t0;
            if (lane < kNO) counts[i * kNO + lane] = cnt;
        } else if (warp == 1) {
#ifndef NO_SPEC
            scan2_spec(c, N, X, xbuf);
#endif
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) cyc[1] = tot;
}

// cross-warp ping-pong through shared memory (volatile store -> polling load)
__global__ void k_pingpong(int iters, long long *cyc) {
    __shared__ unsigned flag[2];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x < 2) flag[threadIdx.x] = 0xFFFFFFFFu;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        if (warp == 0) {
            if (lane == 0) post_u32(&flag[0], (unsigned)i);
            unsigned x;
            do { x = *reinterpret_cast<volatile unsigned *>(&flag[1]); } while (x != (unsigned)i);
        } else if (warp == 1) {
            unsigned x;
            do { x = *reinterpret_cast<volatile unsigned *>(&flag[0]); } while (x != (unsigned)i);
            if (lane == 0) post_u32(&flag[1], (unsigned)i);
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

// cross-warp ping-pong through named barriers (producer bar.arrive, consumer bar.sync)
__global__ void k_pingbar(int iters, long long *cyc, unsigned *sink) {
    __shared__ unsigned box[2];
    const int warp = threadIdx.x >> 5;
    unsigned acc = 0;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        if (warp == 0) {
            box[0] = i + acc;
            asm volatile("bar.arrive 1, 64;" ::: "memory");
            asm volatile("bar.sync 2, 64;" ::: "memory");
            acc += box[1];
        } else if (warp == 1) {
            asm volatile("bar.sync 1, 64;" ::: "memory");
            const unsigned x = box[0];
            box[1] = x + 1;
            asm volatile("bar.arrive 2, 64;" ::: "memory");
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; sink[0] = acc; }
}

}  // namespace

extern "C" int micro_lat(double *out, long long *cyc, int iters) {
    k_lat<<<1, 32>>>(out, cyc, iters, 1.0);
    return (int)cudaDeviceSynchronize();
}

extern "C" int micro_scan(const snn_consts_t *c, const double *G, int n_img, int32_t *counts, long long *cyc,
                          int threads, int variant, uint16_t *om, double *v) {
    const size_t sm = c->n_steps * kNO * 8;
    switch (variant) {
    case 0: k_scan<0><<<1, threads, sm>>>(*c, G, n_img, counts, cyc, om, v); break;
    case 1: k_scan<1><<<1, threads, sm>>>(*c, G, n_img, counts, cyc, om, v); break;
    case 2: k_scan<2><<<1, threads, sm>>>(*c, G, n_img, counts, cyc, om, v); break;
    case 3: k_scan<3><<<1, threads, sm>>>(*c, G, n_img, counts, cyc, om, v); break;
    case 12: k_scan<12><<<1, threads, sm>>>(*c, G, n_img, counts, cyc, om, v); break;
    case 13: k_scan<13><<<1, threads, sm>>>(*c, G, n_img, counts, cyc, om, v); break;
    case 7: k_scan<7><<<1, threads, sm>>>(*c, G, n_img, counts, cyc, om, v); break;
    case 6: k_scan<6><<<1, threads, sm>>>(*c, G, n_img, counts, cyc, om, v); break;
    case 4: k_scan2<<<1, threads < 64 ? 64 : threads, sm>>>(*c, G, n_img, counts, cyc, om, v); break;
    default: return -1;
    }
    return (int)cudaDeviceSynchronize();
}

extern "C" int micro_probe(int mode, int iters, long long *cyc, double *out) {
    k_probe<<<1, 32>>>(mode, iters, cyc, out);
    return (int)cudaDeviceSynchronize();
}

extern "C" int micro_pingpong(int iters, long long *cyc) {
    k_pingpong<<<1, 64>>>(iters, cyc);
    return (int)cudaDeviceSynchronize();
}

extern "C" int micro_pingbar(int iters, long long *cyc, unsigned *sink) {
    k_pingbar<<<1, 64>>>(iters, cyc, sink);
    return (int)cudaDeviceSynchronize();
}
