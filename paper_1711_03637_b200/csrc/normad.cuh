// NormAD online training (normad.py:141-207) on sm_100a.
//
// The reference runs, per image, the whole network step by step and calls a
// hook that filters the hidden kernel traces into d_hat, compares output and
// target spikes and accumulates the normalised update (normad.py:156-159).
// Only the 10-neuron output layer couples to the weights, so the trial splits
// into a weight-independent part that runs ahead for a whole chunk of images
// in parallel, and a short weight-dependent part that must run image after
// image (W_{i+1} = W_i + r * dW_i):
//
//   K1 k_hidden           (parallel)  hidden spike raster per image
//   K2 k_compact          (parallel)  active-neuron list, per-neuron spike
//                                     lists, per-step spike lists (CSR), and
//                                     the d_hat norm of every step
//   K3 k_normad           (sequential, one CTA, loops over the images)
//        G(s,l)  = sum of W rows of hidden neurons spiking at s
//        scan    = output layer + error signal + gate; sigma(s,l) = e*dt/|d_hat|
//        R(u,l)  = sum_{s>=u} sigma(s,l) H(s-u), H = d_hat response of one spike
//        dW[k,l] = sum over spikes u of neuron k of R(u,l);  W += r*dW
//
// d_hat_k(s) = sum_{u<=s} H(s-u) over k's spikes (both trace recursions are
// linear), hence dW[k,l] = sum_s d_hat_k(s) sigma(s,l) = sum_u R(u,l): the
// event-driven form touches only the ~7k spikes of an image instead of the
// dense 8112 x N trace.  All sums run in a fixed order (deterministic).
#pragma once
#include "hidden.cuh"

namespace snn {

constexpr int kCThreads = kMaxTiles * 32;  // 704: one thread per (tile, lane) slot
constexpr int kTThreads = 512;             // sequential NormAD CTA (128 regs/thread)

struct TrainWS {
    uint8_t *raster;    // sum(n_tiles) x nchunks x 512 bytes (raster_tc layout)
    uint16_t *tile_pos; // [n][22][32]
    int32_t *n_tiles;   // [n]
    int32_t *tile_base; // [n+1]
    int32_t *n_win;     // [n]   active windows per image
    int32_t *win_base;  // [n+1]
    int32_t *n_act;     // [n]
    uint16_t *act_k;    // [n][8112]  active neuron ids, ascending
    int32_t *act_off;   // [n][8113]  per active neuron: start in nsp
    uint16_t *nsp;      // [n][evcap] spike steps per active neuron
    int32_t *step_off;  // [n][N+1]   per step: start in step_k
    uint16_t *step_k;   // [n][evcap] per step: active-list index of each spiking neuron, ascending
    double *norm;       // [n][N]     |d_hat(s)|
    double *wp;         // [n][22][N] per-warp partial sums of d_hat^2
    int32_t *fix;       // [1 + n * 676] guard-band hidden layer: count, flagged windows
    int64_t evcap;
};

struct TrainArgs {
    snn_consts_t c;
    TrainWS ws;
    const uint8_t *labels;  // chunk-relative
    double *w;
    int32_t *counts;        // chunk-relative [n][10]
    int32_t *status;        // [4]
    int64_t n;              // images in this chunk
    int64_t first;          // absolute index of the chunk's first image
};

__device__ __forceinline__ uint64_t warp_incl_scan(uint64_t x) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t y = __shfl_up_sync(kFull, x, o);
        if (lane >= o) x += y;
    }
    return x;
}

// Exclusive block scan of uint64 (callers alternate two 32-entry buffers).
__device__ __forceinline__ uint64_t block_excl_scan(uint64_t x, uint64_t *buf, uint64_t *total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const uint64_t inc = warp_incl_scan(x);
    if (lane == 31) buf[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        uint64_t t = lane < nw ? buf[lane] : 0;
        t = warp_incl_scan(t);
        if (lane < nw) buf[lane] = t;
    }
    __syncthreads();
    *total = buf[nw - 1];
    return (warp ? buf[warp - 1] : 0) + inc - x;
}

__device__ __forceinline__ double warp_sum_fixed(double x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x = __dadd_rn(x, __shfl_xor_sync(kFull, x, o));
    return x;
}

// ---------------------------------------------------------------------------
// K2: per image, lists + d_hat norms.  grid = n, block = 704.
__global__ void __launch_bounds__(kCThreads) k_compact(const TrainArgs T) {
    __shared__ uint64_t s_buf[2][32];
    const int tid = threadIdx.x, lane = tid & 31, tile = tid >> 5;
    const int64_t img = blockIdx.x;
    const int N = T.c.n_steps;
    const TrainWS &W = T.ws;
    const int ntiles = W.n_tiles[img];
    int pos = 0xFFFF;
    if (tile < ntiles) pos = W.tile_pos[((size_t)img * kMaxTiles + tile) * kTile + lane];
    const bool valid = pos != 0xFFFF;
    const size_t rstride = (size_t)ntiles * kRastTC;  // raster chunk stride of this image
    const uint8_t *R =
        W.raster + (tile < ntiles ? raster_tc(W.tile_base[img], n_chunks(N), ntiles, 0, tile) : 0) + lane * kChunk;
    auto mask12 = [&](int s) {
        const uint8_t *p = R + (size_t)(s / kChunk) * rstride + (s % kChunk);
        return (unsigned)p[0] | ((unsigned)p[kRastTC / 2] << kHalf);
    };

    // pass 1: which of my 12 neurons ever fire, and how often
    unsigned ever = 0;
    int cnt[kNF];
#pragma unroll
    for (int f = 0; f < kNF; ++f) cnt[f] = 0;
    if (valid)
        for (int s = 0; s < N; ++s) {
            const unsigned m = mask12(s);
            ever |= m;
#pragma unroll
            for (int f = 0; f < kNF; ++f) cnt[f] += (m >> f) & 1u;
        }
    int ev = 0;
#pragma unroll
    for (int f = 0; f < kNF; ++f) ev += cnt[f];
    constexpr uint64_t kLow = (1ull << 40) - 1;
    uint64_t tot;
    const uint64_t ex = block_excl_scan(((uint64_t)__popc(ever) << 40) | (uint64_t)ev, s_buf[0], &tot);
    const int n_act = (int)(tot >> 40);
    const int64_t n_ev = (int64_t)(tot & kLow);
    uint16_t *act_k = W.act_k + (size_t)img * kNH;
    int32_t *act_off = W.act_off + (size_t)img * (kNH + 1);
    uint16_t *nsp = W.nsp + (size_t)img * W.evcap;
    uint16_t *step_k = W.step_k + (size_t)img * W.evcap;
    int32_t *step_off = W.step_off + (size_t)img * (N + 1);
    if (n_ev > W.evcap) {  // cannot happen with the worst-case capacity; fail loudly
        if (tid == 0) atomicCAS(T.status, 0, SNN_ENOMEM);
        return;
    }
    if (tid == 0) {
        W.n_act[img] = n_act;
        act_off[n_act] = (int32_t)n_ev;
    }
    int cursor[kNF];
    const int act_base = (int)(ex >> 40);
    {
        int r = act_base, e = (int)(ex & kLow);
#pragma unroll
        for (int f = 0; f < kNF; ++f) {
            cursor[f] = e;
            if ((ever >> f) & 1u) {
                act_k[r] = (uint16_t)(pos * kNF + f);
                act_off[r] = e;
                ++r;
                e += cnt[f];
            }
        }
    }

    // pass 2: per-step CSR (4 steps per packed scan) and per-neuron spike steps
    int step_base = 0, parity = 1;
    for (int s0 = 0; s0 < N; s0 += 4) {
        unsigned ms[4];
        uint64_t pk = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int s = s0 + q;
            ms[q] = (valid && s < N) ? mask12(s) : 0u;
            pk |= (uint64_t)__popc(ms[q]) << (16 * q);
        }
        uint64_t t4;
        const uint64_t ex4 = block_excl_scan(pk, s_buf[parity], &t4);
        parity ^= 1;
        int before = step_base;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int s = s0 + q;
            if (s < N) {
                if (tid == 0) step_off[s] = before;
                int o = before + (int)((ex4 >> (16 * q)) & 0xFFFF);
                const unsigned m = ms[q];
#pragma unroll
                for (int f = 0; f < kNF; ++f)
                    if ((m >> f) & 1u) {
                        step_k[o++] = (uint16_t)(act_base + __popc(ever & ((1u << f) - 1u)));
                        nsp[cursor[f]++] = (uint16_t)s;
                    }
            }
            before += (int)((t4 >> (16 * q)) & 0xFFFF);
        }
        step_base = before;
    }
    if (tid == 0) step_off[N] = step_base;
    __syncthreads();

    // pass 3: |d_hat(s)|^2 = sum_k d_hat_k(s)^2 over the active neurons, replaying
    // each neuron's kernel and d_hat recursions exactly as normad.py:82-83 /
    // neurons.py:169-171 do.  Fixed reduction order: per-warp butterfly, then
    // warps in index order.
    double *wp = W.wp + (size_t)img * kMaxTiles * N;
    const double lam1 = T.c.decay_slow, lam2 = T.c.decay_fast, lamL = T.c.decay_learn, kap = T.c.dhat_scale;
    for (int base = 0; base < n_act || base == 0; base += kCThreads) {
        const int j = base + tid;
        const bool ok = j < n_act;
        int e0 = ok ? act_off[j] : 0;
        const int e1 = ok ? act_off[j + 1] : 0;
        int nxt = e0 < e1 ? (int)nsp[e0] : 0x7fffffff;
        double a = 0.0, b = 0.0, d = 0.0;
        for (int s = 0; s < N; ++s) {
            const bool sp = s == nxt;
            if (sp) {
                ++e0;
                nxt = e0 < e1 ? (int)nsp[e0] : 0x7fffffff;
            }
            const double bump = sp ? 1.0 : 0.0;
            a = __dadd_rn(__dmul_rn(a, lam1), bump);
            b = __dadd_rn(__dmul_rn(b, lam2), bump);
            const double c = __dsub_rn(a, b);
            d = __dadd_rn(__dmul_rn(d, lamL), __dmul_rn(c, kap));
            const double x = warp_sum_fixed(ok ? __dmul_rn(d, d) : 0.0);
            if (lane == 0) wp[(size_t)tile * N + s] = base == 0 ? x : __dadd_rn(wp[(size_t)tile * N + s], x);
        }
        if (base + kCThreads >= n_act) break;
    }
    __syncthreads();
    double *nrm = W.norm + (size_t)img * N;
    for (int s = tid; s < N; s += kCThreads) {
        double q = 0.0;
        for (int w = 0; w < kMaxTiles; ++w) q = __dadd_rn(q, wp[(size_t)w * N + s]);
        nrm[s] = __dsqrt_rn(q);
    }
}

// ---------------------------------------------------------------------------
// K3: the sequential part, one CTA walking the chunk's images in order.
//
// Per image everything the weight-dependent chain touches is staged in shared
// memory first (step lists, spike lists, |d_hat|, and the W rows of the
// image's active neurons, ~80 KB), so the chain itself runs out of smem:
//   G -> output scan (one warp; the only serial part) -> R (adjoint, O(N))
//   -> dW / W update of the active rows (all-or-nothing, normad.py:122-124).
// Images whose lists do not fit the smem caps take the same path reading the
// lists and W from global memory instead.
struct NormadCaps {
    int acap;   // active neurons whose W rows / lists fit in smem
    int ecap;   // spike events whose lists fit in smem
};

__host__ __device__ inline size_t normad_smem_bytes(int N, NormadCaps cap) {
    size_t b = 0;
    b += (size_t)N * kNO * 8 * 2;            // GR, SIG
    b += (size_t)N * 8 * 2;                  // H, NRM
    b += (size_t)cap.acap * kNO * 8;         // WACT
    b += ((size_t)N + 1) * 4;                // SOFF
    b += (size_t)N * 2;                      // OMASK
    b += ((size_t)cap.acap + 1) * 4;         // AOFF
    b += (size_t)cap.acap * 2;               // AK
    b += (size_t)cap.ecap * 2 * 2;           // EV, NSP
    return b + 64;
}

__global__ void __launch_bounds__(kTThreads) k_normad(const TrainArgs T, const NormadCaps cap) {
    extern __shared__ __align__(16) double smem[];
    const int N = T.c.n_steps;
    double *GR = smem;                             // G(s,l), then R(u,l)
    double *SIG = GR + (size_t)N * kNO;            // sigma(s,l)
    double *H = SIG + (size_t)N * kNO;
    double *NRM = H + N;
    double *WACT = NRM + N;                        // [acap][10] W rows of active neurons
    int *SOFF = reinterpret_cast<int *>(WACT + (size_t)cap.acap * kNO);
    int *AOFF = SOFF + N + 1;
    uint16_t *AK = reinterpret_cast<uint16_t *>(AOFF + cap.acap + 1);
    uint16_t *EV = AK + cap.acap;
    uint16_t *NSP = EV + cap.ecap;
    uint16_t *OMASK = NSP + cap.ecap;              // output spikes of each step (10-bit)

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const snn_consts_t &c = T.c;
    const TrainWS &W = T.ws;

    if (T.status[0] != 0) return;  // an earlier chunk failed
    if (tid == 0) {
        // d_hat response to one hidden spike at lag m (kernel then d_hat filter)
        double a = 0.0, b = 0.0, d = 0.0;
        for (int m = 0; m < N; ++m) {
            const double bump = m == 0 ? 1.0 : 0.0;
            a = __dadd_rn(__dmul_rn(a, c.decay_slow), bump);
            b = __dadd_rn(__dmul_rn(b, c.decay_fast), bump);
            d = __dadd_rn(__dmul_rn(d, c.decay_learn), __dmul_rn(__dsub_rn(a, b), c.dhat_scale));
            H[m] = d;
        }
    }

    for (int64_t i = 0; i < T.n; ++i) {
        const int n_act = W.n_act[i];
        const int32_t *g_aoff = W.act_off + (size_t)i * (kNH + 1);
        const uint16_t *g_ak = W.act_k + (size_t)i * kNH;
        const uint16_t *g_ev = W.step_k + (size_t)i * W.evcap;
        const uint16_t *g_nsp = W.nsp + (size_t)i * W.evcap;
        const int32_t *g_soff = W.step_off + (size_t)i * (N + 1);
        const int n_ev = g_aoff[n_act];
        const bool fast = n_act <= cap.acap && n_ev <= cap.ecap;

        // ---- stage (coalesced, all threads)
        for (int s = tid; s <= N; s += kTThreads) SOFF[s] = g_soff[s];
        for (int s = tid; s < N; s += kTThreads) NRM[s] = W.norm[(size_t)i * N + s];
        if (fast) {
            for (int e = tid; e < n_ev; e += kTThreads) {
                EV[e] = g_ev[e];
                NSP[e] = g_nsp[e];
            }
            for (int j = tid; j <= n_act; j += kTThreads) AOFF[j] = g_aoff[j];
            for (int j = tid; j < n_act; j += kTThreads) AK[j] = g_ak[j];
            for (int t = tid; t < n_act * kNO; t += kTThreads) {
                const int j = t / kNO, l = t - j * kNO;
                WACT[t] = __ldcg(T.w + (size_t)g_ak[j] * kNO + l);
            }
        }
        __syncthreads();
        const uint16_t *ev = fast ? EV : g_ev;
        const uint16_t *nsp = fast ? NSP : g_nsp;
        const int *aoff = fast ? AOFF : g_aoff;
        const uint16_t *ak = fast ? AK : g_ak;

        // ---- (1) G(s,l): sum of W rows over the step's spiking neurons, ascending id
        for (int t = tid; t < N * kNO; t += kTThreads) {
            const int s = t / kNO, l = t - s * kNO;
            double g = 0.0;
            const int e1 = SOFF[s + 1];
            if (fast)
                for (int e = SOFF[s]; e < e1; ++e) g = __dadd_rn(g, WACT[ev[e] * kNO + l]);
            else
                for (int e = SOFF[s]; e < e1; ++e) g = __dadd_rn(g, __ldcg(T.w + (size_t)ak[ev[e]] * kNO + l));
            GR[t] = g;
        }
        __syncthreads();

        // ---- (2) output layer (network.py:308-314): the only serial chain.  The
        // error signal and gate are evaluated afterwards in parallel.
        if (warp == 0) {
            const int l = lane < kNO ? lane : kNO - 1;
            OutState st;
            out_init(st, c);
            for (int s = 0; s < N; ++s) {
                double ff;
                out_step(st, c, GR[s * kNO + l], s, l, &ff);
                if (lane == 0) OMASK[s] = (uint16_t)st.prev;
            }
            if (lane < kNO) T.counts[(size_t)i * kNO + lane] = st.cnt;
        }
        __syncthreads();
        // error signal, gate and normalised step (normad.py:156-159, :87-91, :104-113):
        // e = desired - observed; a step counts if any e != 0 and |d_hat| > eps;
        // sigma(s,l) = (e_l * dt) / |d_hat(s)|
        {
            const int label = T.labels[i];
            const int per = c.desired_period;
            for (int t = tid; t < N * kNO; t += kTThreads) {
                const int s = t / kNO, l = t - s * kNO;
                const bool want_step = per > 0 && s >= per - 1 && (s - (per - 1)) % per == 0;
                const unsigned wmask = want_step ? (1u << label) : 0u;
                const unsigned om = OMASK[s];
                const int e = (int)((wmask >> l) & 1u) - (int)((om >> l) & 1u);
                const double nv = NRM[s];
                double sg = 0.0;
                if (om != wmask && nv > c.norm_eps && e != 0) sg = __ddiv_rn(__dmul_rn((double)e, c.dt), nv);
                SIG[t] = sg;
            }
        }
        __syncthreads();

        // ---- (3) R(u,l) = sum_{s>=u} sigma(s,l) H(s-u), via the adjoint of the
        // kernel -> d_hat recursions (backward, O(N) per output)
        if (warp == 0 && lane < kNO) {
            double pd = 0.0, pa = 0.0, pb = 0.0;
            for (int u = N - 1; u >= 0; --u) {
                pd = __dadd_rn(__dmul_rn(pd, c.decay_learn), SIG[u * kNO + lane]);
                const double q = __dmul_rn(pd, c.dhat_scale);
                pa = __dadd_rn(__dmul_rn(pa, c.decay_slow), q);
                pb = __dadd_rn(__dmul_rn(pb, c.decay_fast), q);
                // (a spike adds 1 to a and b alike, so its lag-0 trace is 0)
                GR[u * kNO + lane] = __dsub_rn(pa, pb);
            }
        }
        __syncthreads();

        // ---- (4) dW per active neuron (spikes ascending) and W + r*dW, all-or-nothing
        bool bad = false;
        for (int j = tid; j < n_act; j += kTThreads) {
            double acc[kNO];
#pragma unroll
            for (int l = 0; l < kNO; ++l) acc[l] = 0.0;
            const int e1 = aoff[j + 1];
            for (int e = aoff[j]; e < e1; ++e) {
                const double *r = GR + (int)nsp[e] * kNO;
#pragma unroll
                for (int l = 0; l < kNO; ++l) acc[l] = __dadd_rn(acc[l], r[l]);
            }
            const double *wrow = fast ? WACT + (size_t)j * kNO : T.w + (size_t)ak[j] * kNO;
#pragma unroll
            for (int l = 0; l < kNO; ++l) {
                const double wn = __dadd_rn(fast ? wrow[l] : __ldcg(wrow + l), __dmul_rn(c.learning_rate, acc[l]));
                bad |= !isfinite(wn);
                if (fast) WACT[(size_t)j * kNO + l] = wn;
            }
        }
        if (__syncthreads_or(bad)) {
            if (tid == 0) {
                T.status[0] = SNN_ENONFINITE;
                T.status[1] = (int32_t)(T.first + i);
            }
            return;
        }
        if (fast) {
            for (int t = tid; t < n_act * kNO; t += kTThreads) {
                const int j = t / kNO, l = t - j * kNO;
                T.w[(size_t)AK[j] * kNO + l] = WACT[t];
            }
        } else {
            for (int j = tid; j < n_act; j += kTThreads) {
                double acc[kNO];
#pragma unroll
                for (int l = 0; l < kNO; ++l) acc[l] = 0.0;
                const int e1 = aoff[j + 1];
                for (int e = aoff[j]; e < e1; ++e) {
                    const double *r = GR + (int)nsp[e] * kNO;
#pragma unroll
                    for (int l = 0; l < kNO; ++l) acc[l] = __dadd_rn(acc[l], r[l]);
                }
                double *wrow = T.w + (size_t)ak[j] * kNO;
#pragma unroll
                for (int l = 0; l < kNO; ++l) wrow[l] = __dadd_rn(__ldcg(wrow + l), __dmul_rn(c.learning_rate, acc[l]));
            }
        }
        __syncthreads();
        if (tid == 0) T.status[2] = (int32_t)(T.first + i + 1);
    }
}

}  // namespace snn
