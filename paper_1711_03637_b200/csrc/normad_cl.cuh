// Sequential NormAD chain on a thread-block cluster (sm_100a, DSMEM).
//
// The weight-dependent part of online NormAD (normad.py:141-162, :179-207)
// must run image after image: W_{i+1} = W_i + r * dW_i.  k_normad (normad.cuh)
// runs it on one CTA and re-stages the W rows of every image from global
// memory.  Here a cluster of kCl CTAs keeps the whole weight matrix resident
// in distributed shared memory for the whole chunk of images -- CTA r owns the
// rows of the windows w = r, r + 8, r + 16, ... (81.6 KB each; interleaving
// the windows balances the spiking neurons over the CTAs).  Per image i:
//
//   G partials  every CTA sums, per step, the W rows of its shard's spiking
//               neurons in ascending id: P_r(s, l)
//   -- cluster barrier B1 --   (also publishes the non-finite flags of i-1)
//   leader      G(s, l) = P_0 + P_1 + ... + P_7 in rank order (DSMEM reads);
//               output-layer scan (network.py:308-314, one warp); error, gate,
//               sigma(s, l) = e * dt / |d_hat(s)| (normad.py:87-113, with
//               dt / |d_hat(s)| precomputed by k_shard); R(u, l) =
//               sum_{s >= u} sigma(s, l) H(s - u) by the adjoint recursion
//               (one warp).  Meanwhile every other warp of the cluster stages
//               image i+1's shard lists in shared memory.
//   -- cluster barrier B2 --
//   dW          every CTA copies R (DSMEM), computes dW[k, l] = sum over k's
//               spikes u of R(u, l) for its shard's active neurons and commits
//               W + lr * dW in place, logging the old rows to global memory;
//               a non-finite value raises its flag on the leader.  The flags
//               are read after the next B1: if any is set, every CTA restores
//               the logged rows and the chunk stops with the weights of before
//               that image (normad.py:122-124).
//
// Two cluster barriers and two one-warp recursions over N steps per image;
// everything else is spread over kCl SMs.  All sums run in a fixed order:
// results are deterministic and independent of the chunking.
#pragma once
#include <cooperative_groups.h>

#include "hidden_gb.cuh"
#include "normad.cuh"

namespace snn {

#ifdef SNN_SCAN_STAMPS
// experiment builds only: clock64() at every step of image SNN_SCAN_STAMPS's output scan
__device__ long long g_scan_stamps[256];
#endif

namespace cg = cooperative_groups;

constexpr int kCl = 8;                          // CTAs per cluster = W shards
constexpr int kClWin = (kNPos + kCl - 1) / kCl;  // 85 windows per shard (w % kCl == r)
constexpr int kClRows = kClWin * kNF;            // 1020 rows per shard

// neuron id <-> (shard, shard-local row)
__host__ __device__ inline int cl_shard(int id) { return (id / kNF) % kCl; }
__host__ __device__ inline int cl_row(int id) { return (id / kNF) / kCl * kNF + id % kNF; }
__host__ __device__ inline int cl_id(int r, int row) { return ((row / kNF) * kCl + r) * kNF + row % kNF; }
__host__ __device__ inline int cl_rows(int r) { return (kNPos - r + kCl - 1) / kCl * kNF; }
constexpr int kClThreads = 512;
constexpr int kClECap = 3072;                   // staged spike events per shard and image
constexpr int kClACap = 512;                    // staged active neurons per shard and image

// Per-image shard data written by k_shard (shard-major blocks, each in
// ascending neuron id).
struct ShardWS {
    long long *clk;   // optional [64][16] leader phase clocks (snn_normad_phase_clocks)
    double *q;        // [n][N]            dt / |d_hat(s)|, 0 where the gate is closed
    int32_t *soff;    // [n][kCl][N + 1]   per shard: start of each step in its id block
    int32_t *ebase;   // [n][kCl + 1]      start of each shard's id block in sid
    uint16_t *sid;    // [n][evcap]        shard-major step lists, shard-local rows
    int32_t *abase;   // [n][kCl + 1]      start of each shard's neurons in sact
    uint16_t *sact;   // [n][kNH]          shard-major active neurons, shard-local rows
    uint16_t *sidx;   // [n][kNH]          ... and their index in the active list
    int32_t *saoff;   // [n][kNH + kCl]    per shard: start of each neuron's spikes in its block (+ end)
    int32_t *nbase;   // [n][kCl + 1]      start of each shard's spike block in snsp
    uint16_t *snsp;   // [n][evcap]        shard-major spike steps of the active neurons
    double *undo;     // [kCl][kClRows][10] old rows of the last committed image
    int push;         // G partials pushed to the leader through DSMEM stores (normad_cl_smem_bytes)
    int alias;        // sigma/R share P's shared memory (long trials; G is dead after the scan)
    int skip;         // profiling only (snn_normad_skip): bit 0 scan, 1 R, 2 dW, 3 G partials, 4 gather
};

// one image's lists of one shard, staged (or pointing into global memory
// when they exceed the caps)
struct ClBuf {
    const int32_t *soff;   // [N + 1] relative to the id block
    const uint16_t *sid;   // shard-local rows
    const uint16_t *act;   // shard-local rows of the shard's active neurons
    const int32_t *aoff;   // [n_act + 1] start of each neuron's spikes in nsp
    const uint16_t *nsp;   // spike steps
    int n_act;
};

__host__ __device__ inline size_t cl_buf_bytes(int N) {
    return (size_t)(N + 1) * 4 + (size_t)(kClACap + 1) * 4 + (size_t)kClECap * 2 * 2 + (size_t)kClACap * 2 + 16;
}

// push: every CTA stores its G partials straight into the leader's shared
// memory, so the leader reads no remote shared memory on the serial path;
// needs kCl partial buffers on the leader.  (R is not transferred: the leader
// sends the output spikes and every CTA derives sigma and R itself.)
__host__ __device__ inline size_t normad_cl_smem_bytes(int N, bool push, bool alias = false) {
    return (size_t)kClRows * kNO * 8          // W shard
           + (size_t)N * kNO * 8 * (alias ? 1 : 2)  // P (G on the leader), sigma -> R
           + (size_t)((N + 1) & ~1) * 8       // q (padded to 16 bytes)
           + (size_t)N * 2 + 64 + 16          // OMASK, flags
           + 2 * ((cl_buf_bytes(N) + 15) & ~(size_t)15)
           + (push ? (size_t)kCl * N * kNO * 8 : 0);  // the partials of every CTA (leader)
}

// k_shard: grid = images.  dt / |d_hat(s)|, and the image's active neurons,
// their spike lists and the step lists regrouped shard by shard (stable, so
// ascending id within every shard), as shard-local rows.
constexpr int kShThreads = 256;

__global__ void __launch_bounds__(kShThreads) k_shard(const TrainArgs T, const ShardWS S) {
    const int64_t i = blockIdx.x;
    const int N = T.c.n_steps;
    const TrainWS &W = T.ws;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    [[maybe_unused]] constexpr int kWarps = kShThreads / 32;
    const int n_act = W.n_act[i];
    const uint16_t *act_k = W.act_k + (size_t)i * kNH;
    const int32_t *aoff = W.act_off + (size_t)i * (kNH + 1);
    const uint16_t *nsp = W.nsp + (size_t)i * W.evcap;
    const int32_t *soff = W.step_off + (size_t)i * (N + 1);
    const uint16_t *sk = W.step_k + (size_t)i * W.evcap;
    __shared__ int s_cnt[kCl], s_abase[kCl + 1], s_nbase[kCl + 1], s_ebase[kCl + 1];
#ifdef SNN_SHARD_STABLE
    __shared__ int s_run[kCl];
    __shared__ int s_wc[kWarps][kCl];
#endif
    extern __shared__ int s_len[];  // [N][kCl] step-list counts, then offsets
    for (int s = tid; s < N; s += kShThreads) {
        const double nv = W.norm[(size_t)i * N + s];
        S.q[(size_t)i * N + s] = nv > T.c.norm_eps ? __ddiv_rn(T.c.dt, nv) : 0.0;
    }
    if (tid < kCl) {
        s_cnt[tid] = 0;
#ifdef SNN_SHARD_STABLE
        s_run[tid] = 0;
#endif
    }
    __syncthreads();
    // ---- active neurons: counts and spike totals per shard, then a stable partition
    for (int a = tid; a < n_act; a += kShThreads) atomicAdd(&s_cnt[cl_shard(act_k[a])], 1);
    __syncthreads();
    if (tid == 0) {
        s_abase[0] = 0;
        for (int r = 0; r < kCl; ++r) s_abase[r + 1] = s_abase[r] + s_cnt[r];
    }
    __syncthreads();
    uint16_t *sact = S.sact + (size_t)i * kNH, *sidx = S.sidx + (size_t)i * kNH;
#ifdef SNN_SHARD_STABLE
    for (int a0 = 0; a0 < n_act; a0 += kShThreads) {
        const int a = a0 + tid;
        const int r = a < n_act ? cl_shard(act_k[a]) : -1;
        int rank = 0;
#pragma unroll
        for (int q = 0; q < kCl; ++q) {
            const unsigned b = __ballot_sync(kFull, r == q);
            if (r == q) rank = __popc(b & ((1u << lane) - 1u));
            if (lane == 0) s_wc[warp][q] = __popc(b);
        }
        __syncthreads();
        if (r >= 0) {
            int pos = s_abase[r] + s_run[r] + rank;
            for (int w = 0; w < warp; ++w) pos += s_wc[w][r];
            sact[pos] = (uint16_t)cl_row(act_k[a]);
            sidx[pos] = (uint16_t)a;
        }
        __syncthreads();
        if (tid < kCl)
            for (int w = 0; w < kWarps; ++w) s_run[tid] += s_wc[w][tid];
        __syncthreads();
    }
#else
    // within a shard, neurons by descending spike count (buckets of 0..31+
    // spikes): the cluster kernel's dW gives thread t row t / 5 in rounds of
    // its 512 threads, so the heaviest rows share the first round instead of
    // lengthening every round.  Each row's update is independent of the
    // order (same weights bit for bit); positions inside a bucket come from
    // shared-memory atomics.
    __shared__ int s_bk[kCl][32];
    for (int k = tid; k < kCl * 32; k += kShThreads) (&s_bk[0][0])[k] = 0;
    __syncthreads();
    for (int a = tid; a < n_act; a += kShThreads)
        atomicAdd(&s_bk[cl_shard(act_k[a])][31 - min(aoff[a + 1] - aoff[a], 31)], 1);
    __syncthreads();
    if (warp < kCl) {  // warp r: exclusive prefix of shard r's 32 buckets -> cursors
        int tot;
        const int ex = warp_excl_scan_int(s_bk[warp][lane], &tot);
        s_bk[warp][lane] = s_abase[warp] + ex;
    }
    __syncthreads();
    for (int a = tid; a < n_act; a += kShThreads) {
        const int r = cl_shard(act_k[a]);
        const int pos = atomicAdd(&s_bk[r][31 - min(aoff[a + 1] - aoff[a], 31)], 1);
        sact[pos] = (uint16_t)cl_row(act_k[a]);
        sidx[pos] = (uint16_t)a;
    }
    __syncthreads();
#endif
    // per-shard spike-block offsets: warp r walks shard r's neurons in order
    int32_t *saoff = S.saoff + (size_t)i * (kNH + kCl);
    if (warp < kCl) {
        const int r = warp, b0 = s_abase[r], b1 = s_abase[r + 1];
        int run = 0;
        for (int k0 = b0; k0 < b1; k0 += 32) {
            const int k = k0 + lane;
            const int a = k < b1 ? sidx[k] : 0;
            const int len = k < b1 ? aoff[a + 1] - aoff[a] : 0;
            int tot;
            const int ex = warp_excl_scan_int(len, &tot);
            if (k < b1) saoff[k + r] = run + ex;
            run += tot;
        }
        if (lane == 0) {
            saoff[b1 + r] = run;
            s_cnt[r] = run;
        }
    }
    __syncthreads();
    if (tid == 0) {
        s_nbase[0] = 0;
        for (int r = 0; r < kCl; ++r) s_nbase[r + 1] = s_nbase[r] + s_cnt[r];
        for (int r = 0; r <= kCl; ++r) {
            S.abase[i * (kCl + 1) + r] = s_abase[r];
            S.nbase[i * (kCl + 1) + r] = s_nbase[r];
        }
    }
    __syncthreads();
    uint16_t *snsp = S.snsp + (size_t)i * W.evcap;
    for (int k = tid; k < n_act; k += kShThreads) {  // shard-major spike blocks
        int r = 0;
        while (k >= s_abase[r + 1]) ++r;
        const int a = sidx[k];
        uint16_t *dst = snsp + s_nbase[r] + saoff[k + r];
        for (int e = aoff[a]; e < aoff[a + 1]; ++e) *dst++ = nsp[e];
    }
    // ---- step lists: counts per (step, shard), offsets, stable scatter
    for (int s = tid; s < N; s += kShThreads) {
        int cnt[kCl];
#pragma unroll
        for (int r = 0; r < kCl; ++r) cnt[r] = 0;
        for (int e = soff[s]; e < soff[s + 1]; ++e) {
            const int r = cl_shard(act_k[sk[e]]);
#pragma unroll
            for (int q = 0; q < kCl; ++q) cnt[q] += q == r;
        }
#pragma unroll
        for (int r = 0; r < kCl; ++r) s_len[s * kCl + r] = cnt[r];
    }
    __syncthreads();
    if (tid < kCl) {  // per-shard prefix over steps
        const int r = tid;
        int run = 0;
        int32_t *so = S.soff + ((size_t)i * kCl + r) * (N + 1);
        for (int s = 0; s < N; ++s) {
            so[s] = run;
            const int len = s_len[s * kCl + r];
            s_len[s * kCl + r] = run;
            run += len;
        }
        so[N] = run;
        s_cnt[r] = run;
    }
    __syncthreads();
    if (tid == 0) {
        s_ebase[0] = 0;
        for (int r = 0; r < kCl; ++r) s_ebase[r + 1] = s_ebase[r] + s_cnt[r];
        for (int r = 0; r <= kCl; ++r) S.ebase[i * (kCl + 1) + r] = s_ebase[r];
    }
    __syncthreads();
    uint16_t *sid = S.sid + (size_t)i * W.evcap;
    for (int s = tid; s < N; s += kShThreads) {
        int pos[kCl];
#pragma unroll
        for (int r = 0; r < kCl; ++r) pos[r] = s_ebase[r] + s_len[s * kCl + r];
        for (int e = soff[s]; e < soff[s + 1]; ++e) {
            const int id = act_k[sk[e]], r = cl_shard(id);
            int p = 0;
#pragma unroll
            for (int q = 0; q < kCl; ++q)
                if (q == r) p = pos[q]++;
            sid[p] = (uint16_t)cl_row(id);
        }
    }
}

__host__ __device__ inline size_t k_shard_smem(int N) { return (size_t)N * kCl * 4; }

__global__ void __cluster_dims__(kCl, 1, 1) __launch_bounds__(kClThreads, 1)
    k_normad_cl(const TrainArgs T, const ShardWS SW) {
    extern __shared__ __align__(16) double csm[];
    cg::cluster_group cluster = cg::this_cluster();
    const int r = (int)cluster.block_rank();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int N = T.c.n_steps;
    const snn_consts_t &c = T.c;
    const TrainWS &W = T.ws;
    double *Wsh = csm;                          // [kClRows][10]
    double *P = Wsh + (size_t)kClRows * kNO;    // [N][10] partial G (leader: G)
    double *SR = SW.alias ? P : P + (size_t)N * kNO;  // [N][10] sigma, then R in place
    double *Q = P + (size_t)N * kNO * (SW.alias ? 1 : 2);  // [N] dt / |d_hat|
    uint16_t *OMASK = reinterpret_cast<uint16_t *>(Q + ((N + 1) & ~1));  // keeps what follows 16-byte aligned
    int *flags = reinterpret_cast<int *>(OMASK + ((N + 7) & ~7));  // leader: per-CTA non-finite flags
    uint8_t *bufmem = reinterpret_cast<uint8_t *>(flags + 16);
    const size_t bstride = (cl_buf_bytes(N) + 15) & ~(size_t)15;
    double *PQ = reinterpret_cast<double *>(bufmem + 2 * bstride);  // leader, push: [kCl][N][10]
    const bool push = SW.push != 0;
    __shared__ ClBuf s_buf[2];
    __shared__ int s_abort, s_label;

    const int rows = cl_rows(r);
    if (T.status[0] != 0) return;  // an earlier chunk failed (uniform over the cluster)
    double *undo = SW.undo + (size_t)r * kClRows * kNO;
#ifdef SNN_W_TMA
    // the W shard by TMA bulk copies: window w = r + 8 j owns 12 consecutive
    // rows (960 B) of W, so one cp.async.bulk per window into the shard's
    // rows 12 j .. 12 j + 11, all on one mbarrier.  Built only with
    // -DSNN_W_TMA: the 82 KB load is once per chunk of ~320 images either
    // way, and this variant moved the serial scan's register allocation
    // (19.27 vs 19.00 us per image)
    __shared__ __align__(8) uint64_t s_wbar;
    if (tid == 0) {
        mbar_init(&s_wbar, 1);
        fence_mbar_init();
        const int nw = rows / kNF;
        mbar_expect_tx(&s_wbar, (uint32_t)(rows * kNO * 8));
        for (int j = 0; j < nw; ++j)
            bulk_g2s(Wsh + (size_t)j * kNF * kNO, T.w + (size_t)((j * kCl + r) * kNF) * kNO, kNF * kNO * 8, &s_wbar);
    }
    __syncthreads();
    mbar_wait(&s_wbar, 0);
#else
    for (int t = tid; t < rows * kNO; t += kClThreads)  // once per chunk (L2-coherent loads)
        Wsh[t] = __ldcg(T.w + (size_t)cl_id(r, t / kNO) * kNO + t % kNO);
#endif
    if (tid < kCl) flags[tid] = 0;
    double *PQ_lead = cluster.map_shared_rank(PQ, 0) + (size_t)r * N * kNO;  // this CTA's partials there
    int *flags_lead = cluster.map_shared_rank(flags, 0);

    // stage image j's lists of this shard into buffer b with threads [t0, t0 + nt)
    auto stage = [&](int64_t j, int b, int t0, int nt) {
        const int t = tid - t0;
        if (t < 0 || t >= nt) return;
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
    // put back the rows image j changed (undo log)
    auto restore = [&](const ClBuf &B) {
        for (int t = tid; t < B.n_act * kNO; t += kClThreads) {
            const int row = B.act[t / kNO];
            Wsh[row * kNO + t % kNO] = undo[row * kNO + t % kNO];
        }
    };

    if (T.n > 0) stage(0, 0, 0, kClThreads);
    cluster.sync();

    bool failed = false;
    // profiling builds only (-DSNN_NORMAD_PROFILE): phase clocks and phase
    // ablation.  The product kernel compiles neither: even dead hooks change
    // the register allocation of the serial output scan.
#ifdef SNN_NORMAD_PROFILE
    const int skip = SW.skip;
    long long *clk = nullptr;
    auto stamp = [&](int ph) {
        if (clk && tid == 0) clk[ph] = clock64();
    };
#else
    constexpr int skip = 0;
    auto stamp = [](int) {};
#endif
    for (int64_t i = 0; i < T.n; ++i) {
#ifdef SNN_NORMAD_PROFILE
        clk = (SW.clk && r == 0 && T.first + i < 64) ? SW.clk + (T.first + i) * 16 : nullptr;
#endif
        stamp(0);
        const ClBuf &B = s_buf[i & 1];
        // ---- G partials of this shard (ascending id within the shard)
        // a thread per (step, output pair): two sums, one 16-byte store
        for (int t = tid; t < ((skip & 8) ? 0 : N * (kNO / 2)); t += kClThreads) {
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
            double2 *dst = reinterpret_cast<double2 *>((push ? PQ_lead : P) + s * kNO + l);
            *dst = make_double2(g0, g1);
        }
        stamp(1);
        cluster.sync();  // B1: partials ready, flags of image i-1 published
        stamp(2);
        if (tid == 0) {
            int bad = 0;
#pragma unroll
            for (int q = 0; q < kCl; ++q) bad |= flags_lead[q];
            s_abort = bad;
        }
        __syncthreads();
        if (s_abort) {  // image i-1 produced a non-finite weight: undo it and stop
            restore(s_buf[(i - 1) & 1]);
            failed = true;
            if (r == 0 && tid == 0) {
                T.status[0] = SNN_ENONFINITE;
                T.status[1] = (int32_t)(T.first + i - 1);
                T.status[2] = (int32_t)(T.first + i - 1);
            }
            break;
        }
        const bool more = i + 1 < T.n;
        if (r == 0) {
            // G = P_0 + P_1 + ... + P_{kCl-1}, in rank order
            for (int t = tid; t < ((skip & 16) ? 0 : N * kNO); t += kClThreads) {
                double v[kCl];
#pragma unroll
                for (int q = 0; q < kCl; ++q)
                    v[q] = push ? PQ[(size_t)q * N * kNO + t] : (q ? cluster.map_shared_rank(P, q)[t] : P[t]);
                double g = v[0];
#pragma unroll
                for (int q = 1; q < kCl; ++q) g = __dadd_rn(g, v[q]);
                P[t] = g;
            }
            __syncthreads();
            stamp(3);
            if (warp == 0) {
                // output layer (network.py:308-314): the serial chain
                const int l = lane < kNO ? lane : kNO - 1;
                OutD X;
                out_init(X.o, c);
                const double *gp = P + l;
                uint16_t *om = OMASK;
                X.o.Af = __dadd_rn(__dmul_rn(0.0, c.decay_slow), gp[0]);
                X.o.Bf = __dadd_rn(__dmul_rn(0.0, c.decay_fast), gp[0]);
                X.D0 = __dadd_rn(__dsub_rn(X.o.Af, X.o.Bf), __dmul_rn(c.inhibition, __dsub_rn(0.0, 0.0)));
                const int ns = (skip & 1) ? 0 : N;
#ifdef SNN_SCAN_STAMPS
                long long *stp = (T.first + i == SNN_SCAN_STAMPS && cluster.block_rank() == 0) ? g_scan_stamps : nullptr;
#endif
                for (int s = 0; s < ns; ++s) {
#ifdef SNN_SCAN_STAMPS
                    if (stp && lane == 0) stp[s] = clock64();
#endif
                    outd_step(X, c, gp[(s + 1 < N ? s + 1 : s) * kNO], s, l);
                    if (lane == 0) om[s] = (uint16_t)X.o.prev;
                }
#ifdef SNN_SCAN_STAMPS
                if (stp && lane == 0) stp[ns] = clock64();
#endif
                if (lane < kNO) T.counts[(size_t)i * kNO + lane] = X.o.cnt;
#ifdef SNN_NORMAD_PROFILE
                if (clk && lane == 0) clk[12] = clock64();
#endif
            } else {
                // this image's gate values and label, off the chain; the next image's lists
                for (int s = tid - 32; s < N; s += kClThreads - 32) Q[s] = SW.q[(size_t)i * N + s];
                if (tid == 32) s_label = T.labels[i];
                if (more) stage(i + 1, (int)((i + 1) & 1), 32, kClThreads - 32);
#ifdef SNN_NORMAD_PROFILE
                if (clk && lane == 0) atomicMax((unsigned long long *)&clk[13], (unsigned long long)clock64());
#endif
            }
            __syncthreads();
            stamp(4);
            // the output spikes to every CTA: each derives sigma and R itself
            for (int t = tid; t < (kCl - 1) * N; t += kClThreads) {
                const int q = 1 + t / N, s = t - (q - 1) * N;
                cluster.map_shared_rank(OMASK, q)[s] = OMASK[s];
            }
        } else {
            for (int s = tid; s < N; s += kClThreads) Q[s] = SW.q[(size_t)i * N + s];
            if (tid == 0) s_label = T.labels[i];
            if (more) stage(i + 1, (int)((i + 1) & 1), 0, kClThreads);
        }
        cluster.sync();  // B2: output spikes everywhere, next lists staged
        stamp(5);
        // error signal and gate (normad.py:156-159, :87-91, :104-113): the step
        // counts when some e != 0 and |d_hat| > eps; sigma = e * dt / |d_hat| =
        // +-(dt / |d_hat|) (IEEE division is sign-symmetric)
        {
            const int label = s_label;
            const int per = c.desired_period;
            for (int t = tid; t < N * kNO; t += kClThreads) {
                const int s = t / kNO, l = t - s * kNO;
                const bool want = per > 0 && (s + 1) % per == 0 && l == label;  // network.py:191-193
                const bool got = (OMASK[s] >> l) & 1u;
                const double q = Q[s];
                SR[t] = want == got ? 0.0 : (want ? q : -q);
            }
        }
        __syncthreads();
        stamp(6);
        // R(u, l) = sum_{s >= u} sigma(s, l) H(s - u): adjoint of kernel -> d_hat,
        // backward; every CTA runs it on its own copy (no R transfer)
        if (warp == 0 && lane < kNO) {
            double pd = 0.0, pa = 0.0, pb = 0.0;
            for (int u = (skip & 2) ? -1 : N - 1; u >= 0; --u) {
                pd = __dadd_rn(__dmul_rn(pd, c.decay_learn), SR[u * kNO + lane]);
                const double q = __dmul_rn(pd, c.dhat_scale);
                pa = __dadd_rn(__dmul_rn(pa, c.decay_slow), q);
                pb = __dadd_rn(__dmul_rn(pb, c.decay_fast), q);
                SR[u * kNO + lane] = __dsub_rn(pa, pb);
            }
        }
        __syncthreads();
        stamp(7);
        const double *Rloc = SR;
        stamp(8);
        // dW for the shard's active neurons (spikes ascending); commit with an undo log
        bool bad = false;
        // five threads per active row, two outputs each
        for (int t = tid; t < ((skip & 4) ? 0 : 5 * B.n_act); t += kClThreads) {
            const int a = t / 5, h = (t - a * 5) * 2;
            const int row = B.act[a];
            double acc[2];
#pragma unroll
            for (int l = 0; l < 2; ++l) acc[l] = 0.0;
            const int e1 = B.aoff[a + 1];
            for (int e = B.aoff[a]; e < e1; ++e) {
                const double *rr = Rloc + (int)B.nsp[e] * kNO + h;
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
        const int any_bad = __syncthreads_or(bad);
        if (tid == 0) flags_lead[r] = any_bad;
        stamp(9);
        if (r == 0 && tid == 0) T.status[2] = (int32_t)(T.first + i + 1);
    }
    if (!failed) {  // the flags of the last image
        cluster.sync();
        if (tid == 0) {
            int bad = 0;
#pragma unroll
            for (int q = 0; q < kCl; ++q) bad |= flags_lead[q];
            s_abort = bad;
        }
        __syncthreads();
        if (s_abort && T.n > 0) {
            restore(s_buf[(T.n - 1) & 1]);
            if (r == 0 && tid == 0) {
                T.status[0] = SNN_ENONFINITE;
                T.status[1] = (int32_t)(T.first + T.n - 1);
                T.status[2] = (int32_t)(T.first + T.n - 1);
            }
        }
    }
    __syncthreads();
    for (int t = tid; t < rows * kNO; t += kClThreads) T.w[(size_t)cl_id(r, t / kNO) * kNO + t % kNO] = Wsh[t];
    cluster.sync();  // no CTA leaves while others may still read its shared memory
}

}  // namespace snn
