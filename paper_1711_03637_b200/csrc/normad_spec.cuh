// Sequential NormAD chain with a speculative output scan (sm_100a cluster).
//
// k_normad_cl (normad_cl.cuh) runs, per image i, G_i (W_i) -> output scan ->
// sigma, R -> dW_i -> W_{i+1}: the one-warp output scan (~half of the time)
// and the update alternate on the critical path.  Here the scan of image i+1
// runs WHILE image i's update is computed, on G'_{i+1} = the sums of W_i rows
// (the weights before image i's update), and is then proven equal to the scan
// on the exact G_{i+1} (W_{i+1} rows) or redone:
//
//   * the output layer's spikes depend on G only through the feed-forward
//     recursions A, B (linear, decays lambda_s, lambda_f; ff = A - B) and the
//     LIF (slope D = |1 - beta g| < 1 between resets); with identical spikes
//     the inhibition terms are bitwise identical, so the candidate potentials
//     of the two scans differ by at most E(s) = D E(s-1) + beta |dff(s)| +
//     rounding, dff = the signed response of A - B to d = G - G' (so a step
//     change of G, which enters A and B alike, costs nothing at lag 0), plus
//     2^-40 times the magnitudes of every operand of the step (>> the
//     roundings of the two runs);
//   * the speculative scan records |vn - V_T| for every live (step, output);
//     if each exceeds E there, every threshold decision -- hence the spike
//     raster, the counts, sigma, R and dW -- is exactly what the scan on
//     G_{i+1} gives; otherwise that scan is run.
//
// The weight trajectory is therefore bitwise identical to k_normad_cl's (same
// partial sums in the same order, same scan, same update), which the GPU tests
// check.  Per image the leader's scan warp runs [speculative scan | check |
// broadcast], everything else (sigma, R, dW, the partials of G_{i+1} and
// G'_{i+2}, their gathers and E*) runs on the other 15 warps of the 8 CTAs
// underneath it.
#pragma once
#include "normad_cl.cuh"

namespace snn {

#ifndef SNN_SP_THREADS
#define SNN_SP_THREADS 384
#endif
constexpr int kSpThreads = SNN_SP_THREADS;  // CTA size of the speculative kernel
constexpr int kSpBufs = 4;  // staged list buffers: images i, i+1, i+2 in use, i+3 being staged

__host__ __device__ inline size_t normad_spec_smem_bytes(int N) {
    const size_t g = (size_t)N * kNO * 8;
    return (size_t)kClRows * kNO * 8           // W shard
           + 3 * g                             // P (G_{i+1} partial), Pn (G'_{i+2} partial), SR (sigma -> R)
           + 2 * (size_t)((N + 1) & ~1) * 8    // Q double buffer (image parity)
           + 2 * (size_t)((N + 7) & ~7) * 2    // OMASK double buffer
           + 64 + 16                           // flags
           + kSpBufs * ((cl_buf_bytes(N) + 15) & ~(size_t)15)
           + 5 * g;                            // leader: G' being scanned, next G', exact G, margins, E
}

// outd_step (hidden.cuh) that also returns the candidate potential's distance
// to the threshold when the neuron is live (+inf otherwise).
__device__ __forceinline__ bool outd_step_m(OutD &X, const snn_consts_t &c, double Gn, int s, int l,
                                            double &margin) {
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
    margin = live ? fabs(vn - p.vt) : __longlong_as_double(0x7ff0000000000000LL);
    st.v = (!live || fired || vn < p.el) ? p.el : vn;
    if (fired) st.live_from = next_live_step(s, p.refr);
    st.prev = __ballot_sync(kFull, fired) & 0x3FFu;
    st.cnt += fired ? 1 : 0;
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

// The output scan of one image over G (one warp; lanes 0..9 = outputs): the
// exact sequence of k_normad_cl's leader scan.  Writes the per-step spike
// masks to om; returns this lane's count and (MARGIN) its smallest live
// distance to the threshold.
#ifdef SNN_SPEC_SCAN_NOINLINE
#define SNN_SCAN_INLINE __noinline__
#else
#define SNN_SCAN_INLINE __forceinline__
#endif
#ifdef SNN_SPEC_SCAN_DIST
// Lane-distributed step (measured slower: 268 against 228 cycles per step,
// the candidate store -> load -> pairwise sum latency is on the chain;
// DESIGN.md 9): dist_step (hidden.cuh: each lane owns one output's
// inhibition traces; the ten candidates of the next step's sum go through a
// 512-byte shared buffer), the same float64 operations as outd_step, so the
// same bits, with half the FP64 instructions per lane of the replicated
// step below.  dspec: 512-byte aligned.
template <bool MARGIN>
__device__ SNN_SCAN_INLINE int spec_scan(const snn_consts_t &c, const double *G, uint16_t *om, int N,
                                         double *M, char *dspec, long long *stp = nullptr) {
    const int lane = threadIdx.x & 31;
    const int l = lane < kNO ? lane : kNO - 1;
    DistState st;
    dist_init(st, c, dspec, lane);
    // register copies of the constants, passed through a shuffle so ptxas
    // cannot re-read them from the constant bank inside the loop (under this
    // kernel's uniform-register pressure it otherwise reloads them on the
    // step's dependency chain)
    DistK k = dist_k(c);
    {
        double *v[8] = {&k.lam1, &k.lam2, &k.inh, &k.el, &k.vt, &k.g, &k.beta, &k.refr};
#pragma unroll
        for (int q = 0; q < 8; ++q) *v[q] = __shfl_sync(kFull, *v[q], 0);
    }
    const double *gp = G + l;
    for (int s = 0; s < N; ++s) {
#ifdef SNN_SCAN_STAMPS
        if (stp && lane == 0) stp[s] = clock64();
#endif
        double ff, m;
        dist_step<MARGIN>(st, k, gp[s * kNO], s, l, lane, &ff, &m);
        // unconditional stores (lanes >= kNO repeat lane kNO - 1's values; om[s]
        // is the same ballot in every lane): no branch inside the step
        if (MARGIN) M[s * kNO + l] = m;
        om[s] = (uint16_t)st.prev;
    }
#ifdef SNN_SCAN_STAMPS
    if (stp && lane == 0) stp[N] = clock64();
#endif
    return st.cnt;
}
#elif defined(SNN_SPEC_SCAN_GATHER)
// Lane-owned traces with the ten values of each pairwise sum gathered by
// shuffles (no shared-memory round trip): the same float64 operations, in the
// same order, as outd_step_m, so the same bits; 12 instead of ~39 FP64
// instructions per lane for the sums.
__device__ __forceinline__ double pairwise10_lanes(double x) {
    double v[kNO];
#pragma unroll
    for (int j = 0; j < kNO; ++j) v[j] = __shfl_sync(kFull, x, j);
    return pairwise10(v);
}

template <bool MARGIN>
__device__ SNN_SCAN_INLINE int spec_scan(const snn_consts_t &c, const double *G, uint16_t *om, int N,
                                         double *M, char *, long long *stp = nullptr) {
    const int lane = threadIdx.x & 31;
    const int l = lane < kNO ? lane : kNO - 1;
    double lam1 = c.decay_slow, lam2 = c.decay_fast, inh = c.inhibition, el = c.lif_out.el, vt = c.lif_out.vt,
           gl = c.lif_out.g, beta = c.lif_out.beta, refr = c.lif_out.refr;
    {
        double *v[8] = {&lam1, &lam2, &inh, &el, &vt, &gl, &beta, &refr};
#pragma unroll
        for (int q = 0; q < 8; ++q) *v[q] = __shfl_sync(kFull, *v[q], 0);  // opaque to ptxas
    }
    const double *gp = G + l;
    double al = 0.0, bl = 0.0;  // this lane's output traces times their decay
    double Af = __dadd_rn(__dmul_rn(0.0, lam1), gp[0]), Bf = __dadd_rn(__dmul_rn(0.0, lam2), gp[0]);
    double D0 = __dadd_rn(__dsub_rn(Af, Bf), __dmul_rn(inh, __dsub_rn(0.0, 0.0)));
    double v = el;
    int live_from = 0, cnt = 0;
    unsigned prev = 0u;
    for (int s = 0; s < N; ++s) {
#ifdef SNN_SCAN_STAMPS
        if (stp && lane == 0) stp[s] = clock64();
#endif
        const double Gn = gp[(s + 1 < N ? s + 1 : s) * kNO];
        double a = al, b = bl, drive = D0;
        if (prev != 0u) {
            const double bump = ((prev >> l) & 1u) ? 1.0 : 0.0;
            a = __dadd_rn(al, bump);
            b = __dadd_rn(bl, bump);
            const double cc = __dsub_rn(a, b);
            const double S = pairwise10_lanes(cc);
            drive = __dadd_rn(__dsub_rn(Af, Bf), __dmul_rn(inh, __dsub_rn(S, cc)));
        }
        double t = __dsub_rn(v, el);
        t = __dmul_rn(gl, t);
        t = __dsub_rn(drive, t);
        t = __dmul_rn(beta, t);
        const double vn = __dadd_rn(v, t);
        const bool live = s >= live_from;
        const bool fired = live && vn >= vt;
        if (MARGIN) M[s * kNO + l] = live ? fabs(vn - vt) : __longlong_as_double(0x7ff0000000000000LL);
        v = (!live || fired || vn < el) ? el : vn;
        if (fired) live_from = next_live_step(s, refr);
        prev = __ballot_sync(kFull, fired) & 0x3FFu;
        cnt += fired ? 1 : 0;
        al = __dmul_rn(a, lam1);
        bl = __dmul_rn(b, lam2);
        const double c0 = __dsub_rn(al, bl);
        const double S0 = pairwise10_lanes(c0);
        Af = __dadd_rn(__dmul_rn(Af, lam1), Gn);
        Bf = __dadd_rn(__dmul_rn(Bf, lam2), Gn);
        D0 = __dadd_rn(__dsub_rn(Af, Bf), __dmul_rn(inh, __dsub_rn(S0, c0)));
        om[s] = (uint16_t)prev;
    }
#ifdef SNN_SCAN_STAMPS
    if (stp && lane == 0) stp[N] = clock64();
#endif
    return cnt;
}
#else
template <bool MARGIN>
__device__ SNN_SCAN_INLINE int spec_scan(const snn_consts_t &c, const double *G, uint16_t *om, int N,
                                         double *M, char *, long long *stp = nullptr) {
    const int lane = threadIdx.x & 31;
    const int l = lane < kNO ? lane : kNO - 1;
    // Register copies of the constants a step reads, passed through a shuffle
    // so ptxas cannot re-read them from the constant bank: under this
    // kernel's uniform-register pressure it otherwise reloads them (LDCU)
    // inside the loop, on the step's dependency chain (358 against 233
    // cycles per step, scripts/scan_stamps.py).
    snn_consts_t k;
    k.lif_out = c.lif_out;
    k.decay_slow = c.decay_slow;
    k.decay_fast = c.decay_fast;
    k.inhibition = c.inhibition;
    {
        double *v[8] = {&k.lif_out.g, &k.lif_out.el, &k.lif_out.vt, &k.lif_out.beta,
                        &k.lif_out.refr, &k.decay_slow, &k.decay_fast, &k.inhibition};
#pragma unroll
        for (int q = 0; q < 8; ++q) {
#ifndef SNN_SPEC_NOLAUNDER
            *v[q] = __shfl_sync(kFull, *v[q], 0);  // opaque to ptxas
#endif
        }
    }
    OutD X;
    out_init(X.o, k);
    const double *gp = G + l;
    X.o.Af = __dadd_rn(__dmul_rn(0.0, c.decay_slow), gp[0]);
    X.o.Bf = __dadd_rn(__dmul_rn(0.0, c.decay_fast), gp[0]);
    X.D0 = __dadd_rn(__dsub_rn(X.o.Af, X.o.Bf), __dmul_rn(c.inhibition, __dsub_rn(0.0, 0.0)));
    for (int s = 0; s < N; ++s) {
#ifdef SNN_SCAN_STAMPS
        if (stp && lane == 0) stp[s] = clock64();
#endif
        const double Gn = gp[(s + 1 < N ? s + 1 : s) * kNO];
        // unconditional stores (lanes >= kNO repeat lane kNO - 1's values, and
        // om[s] is the same ballot in every lane): a branch around them would
        // keep ptxas from overlapping the next step's feed-forward sums with
        // this step's membrane chain
        if (MARGIN) {
            double m;
            outd_step_m(X, k, Gn, s, l, m);
            M[s * kNO + l] = m;
        } else {
            outd_step(X, k, Gn, s, l);
        }
        om[s] = (uint16_t)X.o.prev;
    }
#ifdef SNN_SCAN_STAMPS
    if (stp && lane == 0) stp[N] = clock64();
#endif
    return X.o.cnt;
}

#endif

__device__ __forceinline__ void cl_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ void cl_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
// Workers: the warps of scheduler partitions 1..3 (warp % 4 != 0), so the scan
// warp (warp 0) has its partition's issue slots to itself while they run.
constexpr int kSpWorkers = kSpThreads / 4 * 3;
__device__ __forceinline__ void workers_sync() { asm volatile("bar.sync 1, %0;" ::"n"(kSpWorkers) : "memory"); }
// CTA-wide syncs of this kernel on their own named barriers (ids 2..8), so a
// sync point can never pair with another one's phase
template <int ID>
__device__ __forceinline__ void cta_sync() { asm volatile("bar.sync %0, %1;" ::"n"(ID), "n"(kSpThreads) : "memory"); }
template <int ID>
__device__ __forceinline__ int cta_sync_or(int x) {
    int r;
    asm volatile("{\n\t.reg .pred p, q;\n\tsetp.ne.s32 p, %1, 0;\n\tbar.red.or.pred q, %2, %3, p;\n\t"
                 "selp.s32 %0, 1, 0, q;\n\t}"
                 : "=r"(r) : "r"(x), "n"(ID), "n"(kSpThreads) : "memory");
    return r;
}

__global__ void __cluster_dims__(kCl, 1, 1) __launch_bounds__(kSpThreads, 1)
    k_normad_spec(const TrainArgs T, const ShardWS SW) {
    extern __shared__ __align__(16) double csm[];
    cg::cluster_group cluster = cg::this_cluster();
    const int r = (int)cluster.block_rank();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool worker = (warp & 3) != 0;
    const int wt = (warp - (warp >> 2) - 1) * 32 + lane;  // dense index of a worker thread
    const int N = T.c.n_steps;
    const snn_consts_t &c = T.c;
    const TrainWS &W = T.ws;
    const size_t g = (size_t)N * kNO;
    double *Wsh = csm;                               // [kClRows][10]
    double *P = Wsh + (size_t)kClRows * kNO;         // [N][10] this shard's partial of G_{i+1} (W_{i+1})
    double *Pn = P + g;                              // [N][10] this shard's partial of G'_{i+2} (W_{i+1})
    double *SR = Pn + g;                             // [N][10] sigma -> R
    const int QN = (N + 1) & ~1;
    double *Qb = SR + g;                             // [2][QN] dt / |d_hat|, by image parity
    uint16_t *OM = reinterpret_cast<uint16_t *>(Qb + 2 * QN);  // [2][N8] output spikes, by image parity
    const int N8 = (N + 7) & ~7;
    int *flags = reinterpret_cast<int *>(OM + 2 * N8);  // leader: per-CTA non-finite flags
    uint8_t *bufmem = reinterpret_cast<uint8_t *>(flags + 16);
    const size_t bstride = (cl_buf_bytes(N) + 15) & ~(size_t)15;
    // leader: two G' buffers (the one being scanned alternates with the image
    // parity; selected by offset from the shared base, never by swapping
    // pointers, so every access stays a shared-space load), then the exact G
    double *const Gb = reinterpret_cast<double *>(bufmem + kSpBufs * bstride);
    double *Gx = Gb + 2 * g;
    double *Mg = Gx + g;                                                   // leader: |vn - V_T| of the scan
    double *Eb = Mg + g;                                                   // leader: the bound E
    __shared__ ClBuf s_buf[kSpBufs];
    __shared__ __align__(512) char s_dspec[kDistSpecBytes];  // the scan warp's dist_step buffers
    __shared__ int s_abort, s_bad, s_lab[2];

    const int rows = cl_rows(r);
    if (T.status[0] != 0) return;  // an earlier chunk failed (uniform over the cluster)
    const int64_t n = T.n;
    double *undo = SW.undo + (size_t)r * kClRows * kNO;
    for (int t = tid; t < rows * kNO; t += kSpThreads)
        Wsh[t] = __ldcg(T.w + (size_t)cl_id(r, t / kNO) * kNO + t % kNO);
    if (tid < kCl) flags[tid] = 0;
    int *flags_lead = cluster.map_shared_rank(flags, 0);

    // stage image j's lists of this shard into buffer b (thread t of nt)
    auto stage = [&](int64_t j, int b, int t, int nt) {
        uint8_t *m = bufmem + b * bstride;
        int32_t *soff = reinterpret_cast<int32_t *>(m);
        int32_t *aoff = soff + (N + 1);
        uint16_t *sid = reinterpret_cast<uint16_t *>(aoff + (kClACap + 1));
        uint16_t *nsp = sid + kClECap;
        uint16_t *act = nsp + kClECap;
        const int32_t *ab = SW.abase + j * (kCl + 1), *nb = SW.nbase + j * (kCl + 1);
        const int a0 = ab[r], na = ab[r + 1] - a0;
        const int32_t *gaoff = SW.saoff + (size_t)j * (kNH + kCl) + a0 + r;
        const int ne = gaoff[na];
        const uint16_t *gact = SW.sact + (size_t)j * kNH + a0;
        const uint16_t *gnsp = SW.snsp + (size_t)j * W.evcap + nb[r];
        const int32_t *gso = SW.soff + ((size_t)j * kCl + r) * (N + 1);
        const int nid = gso[N];
        const uint16_t *gsid = SW.sid + (size_t)j * W.evcap + SW.ebase[j * (kCl + 1) + r];
        const bool fa = na <= kClACap && ne <= kClECap, fs = nid <= kClECap;
        for (int k = t; k <= N; k += nt) soff[k] = gso[k];
        if (fs)
            for (int k = t; k < nid; k += nt) sid[k] = gsid[k];
        if (fa) {
            for (int k = t; k <= na; k += nt) aoff[k] = gaoff[k];
            for (int k = t; k < na; k += nt) act[k] = gact[k];
            for (int k = t; k < ne; k += nt) nsp[k] = gnsp[k];
        }
        if (t == 0) {
            ClBuf &B = s_buf[b];
            B.soff = soff;
            B.sid = fs ? sid : gsid;
            B.act = fa ? act : gact;
            B.aoff = fa ? aoff : gaoff;
            B.nsp = fa ? nsp : gnsp;
            B.n_act = na;
        }
    };
    // this shard's G partial over buffer B's step lists (ascending id)
    auto partial = [&](const ClBuf &B, double *dst, int t0, int nt) {
        for (int t = t0; t < N * (kNO / 2); t += nt) {
            const int s = t / (kNO / 2), l = 2 * (t - s * (kNO / 2));
            const int e1 = B.soff[s + 1];
            double g0 = 0.0, g1 = 0.0;
            int e = B.soff[s];
            for (; e + 4 <= e1; e += 4) {
                int id[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) id[u] = B.sid[e + u];
                double2 wv[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) wv[u] = *reinterpret_cast<const double2 *>(Wsh + id[u] * kNO + l);
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    g0 = __dadd_rn(g0, wv[u].x);
                    g1 = __dadd_rn(g1, wv[u].y);
                }
            }
            for (; e < e1; ++e) {
                const double2 wv = *reinterpret_cast<const double2 *>(Wsh + (int)B.sid[e] * kNO + l);
                g0 = __dadd_rn(g0, wv.x);
                g1 = __dadd_rn(g1, wv.y);
            }
            *reinterpret_cast<double2 *>(dst + s * kNO + l) = make_double2(g0, g1);
        }
    };
    // leader: G = P_0 + ... + P_7 (rank order, DSMEM reads)
    auto gather = [&](const double *src, double *dst, int t0, int nt) {
        for (int t = t0; t < N * kNO; t += nt) {
            double v[kCl];
#pragma unroll
            for (int q = 0; q < kCl; ++q) v[q] = q ? cluster.map_shared_rank(const_cast<double *>(src), q)[t] : src[t];
            double gs = v[0];
#pragma unroll
            for (int q = 1; q < kCl; ++q) gs = __dadd_rn(gs, v[q]);
            dst[t] = gs;
        }
    };
    // the leader's scan warp: an image's output spikes (one OMASK parity
    // buffer) into the other CTAs' copies, as 32-bit pairs
    // (16-byte remote stores: each DSMEM store is one transaction of the SM's
    // memory pipe, so fewer and wider ones keep it free for the check's loads)
    auto push_om = [&](const uint16_t *om) {
        __syncwarp();  // every lane's om stores are visible to the warp
        const int nw = N8 / 8;
        const uint4 *src = reinterpret_cast<const uint4 *>(om);
        const int base = (int)(om - OM) / 8;
        for (int t = lane; t < (kCl - 1) * nw; t += 32) {
            const int q = 1 + t / nw, w = t - (q - 1) * nw;
            reinterpret_cast<uint4 *>(cluster.map_shared_rank(OM, q))[base + w] = src[w];
        }
    };

    // ---- prologue: lists of images 0..2, G_0 and G'_1 (both with W_0), scan of image 0
    for (int64_t j = 0; j < 3 && j < n; ++j) stage(j, (int)j, tid, kSpThreads);
    cta_sync<5>();
    if (n > 0) partial(s_buf[0], P, tid, kSpThreads);
    if (n > 1) partial(s_buf[1], Pn, tid, kSpThreads);
    cluster.sync();
    if (r == 0 && n > 0) {
        gather(P, Gx, tid, kSpThreads);
        if (n > 1) gather(Pn, Gb, tid, kSpThreads);  // G'_1: buffer 1 & 1 ^ 1 = 0
        cta_sync<6>();
        if (warp == 0) {
            const int cnt = spec_scan<false>(c, Gx, OM, N, nullptr, s_dspec);
            if (lane < kNO) T.counts[lane] = cnt;
        }
        cta_sync<7>();
        for (int t = tid; t < (kCl - 1) * N; t += kSpThreads) {
            const int q = 1 + t / N, s = t - (q - 1) * N;
            cluster.map_shared_rank(OM, q)[s] = OM[s];
        }
    }
    if (n > 0) {
        for (int s = tid; s < N; s += kSpThreads) Qb[s] = SW.q[s];
        if (tid == 0) s_lab[0] = T.labels[0];
    }
    cluster.sync();  // OMASK_0 everywhere; the leader is done reading P, Pn

    const snn_lif_t &po = c.lif_out;
#ifdef SNN_SPEC_PROFILE
    long long *clk = nullptr;
#define SP_STAMP(th, k) \
    if (clk && tid == (th)) clk[k] = clock64();
#else
#define SP_STAMP(th, k)
#endif
    for (int64_t i = 0; i < n; ++i) {
#ifdef SNN_SPEC_PROFILE
        clk = (SW.clk && r == 0 && T.first + i < 64) ? SW.clk + (T.first + i) * 16 : nullptr;
#endif
        SP_STAMP(0, 0)
        const int par = (int)(i & 1);
        const uint16_t *OMi = OM + par * N8;        // image i's output spikes (final)
        uint16_t *OMs = OM + (par ^ 1) * N8;        // image i+1's (speculative, then final)
        const bool spec = i + 1 < n;
        const ClBuf &Bi = s_buf[i % kSpBufs];
        double *const Gs = Gb + (size_t)par * g;          // G'_{i+1} (scanned now)
        double *const Gn = Gb + (size_t)(par ^ 1) * g;    // G'_{i+2} (gathered now)
        int cnt = 0;  // warp 0 of the leader: image i+1's counts
        if (!worker) {
            // warp 0 of the leader: image i+1's output scan on G'_{i+1}; warps 4, 8, 12
            // (and warp 0 elsewhere) leave the scan warp's partition idle
            cl_arrive();
#ifndef SNN_SPEC_NOSPEC
#ifdef SNN_SCAN_STAMPS
            if (r == 0 && spec && warp == 0)
                cnt = spec_scan<true>(c, Gs, OMs, N, Mg, s_dspec, T.first + i + 1 == SNN_SCAN_STAMPS ? g_scan_stamps : nullptr);
#else
            if (r == 0 && spec && warp == 0) cnt = spec_scan<true>(c, Gs, OMs, N, Mg, s_dspec);
#endif
            if (r == 0 && spec && warp == 0) {  // final unless the check below fails
                push_om(OMs);
                if (lane < kNO) T.counts[(size_t)(i + 1) * kNO + lane] = cnt;
            }
#endif
            SP_STAMP(0, 1)
            cl_wait();
        } else {
            // ---- workers: image i's update, then the partials of images i+1 / i+2
            SP_STAMP(32, 14)
            {  // sigma (all workers), then R by the adjoint recursion of k_normad_cl (warp 1)
                const int label = s_lab[par];
                const double *Q = Qb + par * QN;
                const int per = c.desired_period;
                for (int t = wt; t < N * kNO; t += kSpWorkers) {
                    const int s = t / kNO, l = t - s * kNO;
                    const bool want = per > 0 && (s + 1) % per == 0 && l == label;  // network.py:191-193
                    const bool got = (OMi[s] >> l) & 1u;
                    const double q = Q[s];
                    SR[t] = want == got ? 0.0 : (want ? q : -q);
                }
                workers_sync();
                if (warp == 1 && lane < kNO) {
                    double pd = 0.0, pa = 0.0, pb = 0.0;
                    for (int u = N - 1; u >= 0; --u) {
                        pd = __dadd_rn(__dmul_rn(pd, c.decay_learn), SR[u * kNO + lane]);
                        const double q = __dmul_rn(pd, c.dhat_scale);
                        pa = __dadd_rn(__dmul_rn(pa, c.decay_slow), q);
                        pb = __dadd_rn(__dmul_rn(pb, c.decay_fast), q);
                        SR[u * kNO + lane] = __dsub_rn(pa, pb);
                    }
                } else if (warp != 1 && spec) {
                    // while warp 1 runs R: image i+1's gate values and label into the
                    // other parity's buffers (iteration i-1 released them at its end)
                    double *Qn = Qb + (par ^ 1) * QN;
                    for (int s = wt - 32; s < N; s += kSpWorkers - 32) Qn[s] = SW.q[(size_t)(i + 1) * N + s];
                    if (wt == 32) s_lab[par ^ 1] = T.labels[i + 1];
                }
            }
            SP_STAMP(32, 15)
            if (wt == 0) s_bad = 0;
            workers_sync();
            SP_STAMP(32, 2)
            // dW for the shard's active neurons (spikes ascending); commit with an undo log
            bool bad = false;
            for (int t = wt; t < 5 * Bi.n_act; t += kSpWorkers) {
                const int a = t / 5, h = (t - a * 5) * 2;
                const int row = Bi.act[a];
                double acc[2] = {0.0, 0.0};
                const int e1 = Bi.aoff[a + 1];
                for (int e = Bi.aoff[a]; e < e1; ++e) {
                    const double *rr = SR + (int)Bi.nsp[e] * kNO + h;
#pragma unroll
                    for (int l = 0; l < 2; ++l) acc[l] = __dadd_rn(acc[l], rr[l]);
                }
#pragma unroll
                for (int l = 0; l < 2; ++l) {
                    const double old = Wsh[row * kNO + h + l];
                    const double nw = __dadd_rn(old, __dmul_rn(c.learning_rate, acc[l]));
                    bad |= !isfinite(nw);
                    undo[row * kNO + h + l] = old;
                    Wsh[row * kNO + h + l] = nw;
                }
            }
            if (__any_sync(kFull, bad) && lane == 0) atomicOr(&s_bad, 1);
            workers_sync();  // W_{i+1} committed in this shard
            SP_STAMP(32, 3)
            if (wt == 0) flags_lead[r] = s_bad;  // every image: this shard's non-finite flag
            if (spec) partial(s_buf[(i + 1) % kSpBufs], P, wt, kSpWorkers);
            if (i + 2 < n) partial(s_buf[(i + 2) % kSpBufs], Pn, wt, kSpWorkers);
            SP_STAMP(32, 4)
            cl_arrive();
            cl_wait();  // every shard's W_{i+1}, flag and partials are visible
            SP_STAMP(32, 5)
            if (wt == 0) {
                int fb = 0;
#pragma unroll
                for (int q = 0; q < kCl; ++q) fb |= flags_lead[q];
                s_abort = fb;
            }
            workers_sync();
            if (!s_abort && r != 0 && i + 3 < n) stage(i + 3, (int)((i + 3) % kSpBufs), wt, kSpWorkers);
            if (!s_abort && r == 0) {
                if (spec) gather(P, Gx, wt, kSpWorkers);
                if (i + 2 < n) gather(Pn, Gn, wt, kSpWorkers);
                workers_sync();
                SP_STAMP(32, 6)
                // image i+3's lists: the workers that do not form E (worker warps 5..)
                if (wt >= 160 && i + 3 < n) stage(i + 3, (int)((i + 3) % kSpBufs), wt - 160, kSpWorkers - 160);
                if (spec && wt < 160) {
                    // E(s, l): bound on |vn_exact - vn_spec| (header comment): d = G - G',
                    // its signed feed-forward response dA - dB, and the rounding of both
                    // runs bounded per output by constants (2^-40 x magnitudes of G, of
                    // the A / B recursions and of every LIF operand).  Every recurrence
                    // is first-order linear, so it runs as a parallel scan: worker warp
                    // k < 5 takes outputs 2k, 2k+1 (one per half-warp), lane j of a half
                    // a block of K consecutive steps (an affine map carry -> lambda^len
                    // carry + local), composed over the 16 lanes by shuffles.
                    const int l = 2 * (wt >> 5) + (lane >> 4), j = lane & 15;
                    const int K = (N + 15) >> 4, a0 = min(j * K, N), b0 = min(a0 + K, N);
                    const double ls = c.decay_slow, lf = c.decay_fast;
                    const double K2 = 1.0 / (1.0 - ls) + 1.0 / (1.0 - lf);
                    const double D = fabs(1.0 - po.beta * po.g);
                    // pass 1: local dA, dB (carry 0) and the magnitudes
                    double dA = 0.0, dB = 0.0, pA = 1.0, pB = 1.0, gm = 0.0, dmx = 0.0;
                    for (int t = a0; t < b0; ++t) {
                        const double x = Gx[t * kNO + l], y = Gs[t * kNO + l], d = x - y;
                        dA = __fma_rn(dA, ls, d);
                        dB = __fma_rn(dB, lf, d);
                        pA *= ls;
                        pB *= lf;
                        gm = fmax(gm, fmax(fabs(x), fabs(y)));
                        dmx = fmax(dmx, fabs(d));
                    }
#pragma unroll
                    for (int o = 1; o < 16; o <<= 1) {
                        gm = fmax(gm, __shfl_xor_sync(kFull, gm, o));
                        dmx = fmax(dmx, __shfl_xor_sync(kFull, dmx, o));
                    }
                    // forward composition of the blocks' maps (16-lane groups)
                    double cA = dA, cB = dB, qA = pA, qB = pB;
#pragma unroll
                    for (int o = 1; o < 16; o <<= 1) {
                        const double cA2 = __shfl_up_sync(kFull, cA, o, 16), qA2 = __shfl_up_sync(kFull, qA, o, 16);
                        const double cB2 = __shfl_up_sync(kFull, cB, o, 16), qB2 = __shfl_up_sync(kFull, qB, o, 16);
                        if (j >= o) {
                            cA = __fma_rn(qA, cA2, cA);
                            qA *= qA2;
                            cB = __fma_rn(qB, cB2, cB);
                            qB *= qB2;
                        }
                    }
                    double inA = __shfl_up_sync(kFull, cA, 1, 16), inB = __shfl_up_sync(kFull, cB, 1, 16);
                    if (j == 0) inA = inB = 0.0;
                    const double kR = 0x1p-40;
                    const double inh = fabs(c.inhibition) * kNO / (1.0 - ls);
                    const double rA = kR * 2.0 * K2 * gm;
                    const double mag = fabs(po.el) + fabs(po.vt) + po.beta * po.g * (fabs(po.el) + fabs(po.vt)) +
                                       po.beta * (K2 * gm + K2 * dmx + inh) + 1.0;
                    const double cst = po.beta * (rA + kR * 2.0 * K2 * K2 * dmx) + kR * mag;
                    // pass 2: dA, dB from their carries; local E (carry 0)
                    dA = inA;
                    dB = inB;
                    double E = 0.0, pE = 1.0;
                    for (int t = a0; t < b0; ++t) {
                        const double d = Gx[t * kNO + l] - Gs[t * kNO + l];
                        dA = __fma_rn(dA, ls, d);
                        dB = __fma_rn(dB, lf, d);
                        E = __fma_rn(E, D, __fma_rn(po.beta, fabs(dA - dB) * (1.0 + 0x1p-40), cst));
                        pE *= D;
                        Eb[t * kNO + l] = E;
                    }
                    double cE = E, qE = pE;
#pragma unroll
                    for (int o = 1; o < 16; o <<= 1) {
                        const double cE2 = __shfl_up_sync(kFull, cE, o, 16), qE2 = __shfl_up_sync(kFull, qE, o, 16);
                        if (j >= o) {
                            cE = __fma_rn(qE, cE2, cE);
                            qE *= qE2;
                        }
                    }
                    double inE = __shfl_up_sync(kFull, cE, 1, 16);
                    if (j == 0) inE = 0.0;
                    // pass 3: E with its carry (all terms >= 0; rounded up by 2^-20)
                    const double infv = __longlong_as_double(0x7ff0000000000000LL);
                    double pw = 1.0;
                    for (int t = a0; t < b0; ++t) {
                        pw *= D;
                        Eb[t * kNO + l] = D < 1.0 ? __fma_rn(pw, inE, Eb[t * kNO + l]) * (1.0 + 0x1p-20) : infv;
                    }
                }
            }
        }
        SP_STAMP(32, 7)
        SP_STAMP(0, 11)
        cta_sync<2>();  // (1) the scan, E and the flags are done
        SP_STAMP(0, 8)
        if (s_abort) {  // image i produced a non-finite weight: undo it and stop
            for (int t = tid; t < Bi.n_act * kNO; t += kSpThreads) {
                const int row = Bi.act[t / kNO];
                Wsh[row * kNO + t % kNO] = undo[row * kNO + t % kNO];
            }
            if (r == 0 && tid == 0) {
                T.status[0] = SNN_ENONFINITE;
                T.status[1] = (int32_t)(T.first + i);
                T.status[2] = (int32_t)(T.first + i);
            }
            break;
        }
        if (r == 0 && spec) {
            // the speculative spikes are exact iff every live decision clears E
            int fail = 0;
            for (int t = tid; t < N * kNO; t += kSpThreads) fail |= !(Mg[t] > Eb[t]);
#ifdef SNN_SPEC_NOSPEC
            fail = 1;
#endif
            SP_STAMP(0, 12)
            fail = cta_sync_or<3>(fail);
            SP_STAMP(0, 13)
            if (warp == 0 && fail) {  // redo on the exact G_{i+1}; its spikes and counts replace the speculative ones
                cnt = spec_scan<false>(c, Gx, OMs, N, nullptr, s_dspec);
                push_om(OMs);
                if (lane < kNO) T.counts[(size_t)(i + 1) * kNO + lane] = cnt;
                if (lane == 0) atomicAdd(&T.status[3], 1);
            }
            SP_STAMP(0, 9)
        }
        // ---- image i is done; hand over to image i+1 (its gate values and
        // label were prefetched by the workers)
        if (r == 0 && tid == 0) T.status[2] = (int32_t)(T.first + i + 1);
        cluster.sync();  // OMASK_{i+1} everywhere; the leader is done reading P, Pn
        SP_STAMP(0, 10)
    }
#undef SP_STAMP
    cta_sync<8>();
    for (int t = tid; t < rows * kNO; t += kSpThreads) T.w[(size_t)cl_id(r, t / kNO) * kNO + t % kNO] = Wsh[t];
    cluster.sync();  // no CTA leaves while others may still read its shared memory
}

}  // namespace snn
