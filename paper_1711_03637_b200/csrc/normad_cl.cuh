// Sequential NormAD chain on a thread-block cluster (sm_100a, DSMEM).
//
// The weight-dependent part of online NormAD (normad.py:141-162, :179-207)
// must run image after image: W_{i+1} = W_i + r * dW_i.  k_normad (normad.cuh)
// runs it on one CTA and re-stages the W rows of every image from global
// memory.  Here a cluster of kCl CTAs keeps the whole weight matrix resident
// in distributed shared memory for the whole chunk of images -- CTA r owns
// rows [r * kClRows, (r + 1) * kClRows) (81 KB each).  Per image i:
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

#include "normad.cuh"

namespace snn {

namespace cg = cooperative_groups;

constexpr int kCl = 8;                          // CTAs per cluster = W shards
constexpr int kClRows = (kNH + kCl - 1) / kCl;  // 1014 rows per shard
constexpr int kClThreads = 512;
constexpr int kClECap = 3072;                   // staged spike events per shard and image
constexpr int kClACap = 512;                    // staged active neurons per shard and image

// Per-image shard data written by k_shard.  Lists are in ascending neuron id,
// so every shard's share of the active list and of each step list is one
// contiguous segment.
struct ShardWS {
    long long *clk;   // optional [64][16] leader phase clocks (snn_normad_phase_clocks)
    int32_t *act;     // [n][kCl + 1]     first active index of each shard
    int32_t *soff;    // [n][kCl][N + 1]  per shard: start of each step in its id block
    int32_t *ebase;   // [n][kCl + 1]     start of each shard's id block in sid
    uint16_t *sid;    // [n][evcap]       shard-major step lists, shard-local rows
    double *q;        // [n][N]           dt / |d_hat(s)|, 0 where the gate is closed
    double *undo;     // [kCl][kClRows][10] old rows of the last committed image
};

// one image's lists of one shard, staged (or pointing into global memory
// when they exceed the caps)
struct ClBuf {
    const int32_t *soff;   // [N + 1] relative to the id block
    const uint16_t *sid;   // shard-local rows
    const uint16_t *act;   // global ids of the shard's active neurons
    const int32_t *aoff;   // [n_act + 1] spike-list offsets (minus abias)
    const uint16_t *nsp;   // spike steps
    int n_act, abias;
};

__host__ __device__ inline size_t cl_buf_bytes(int N) {
    return (size_t)(N + 1) * 4 + (size_t)(kClACap + 1) * 4 + (size_t)kClECap * 2 * 2 + (size_t)kClACap * 2 + 16;
}

__host__ __device__ inline size_t normad_cl_smem_bytes(int N) {
    return (size_t)kClRows * kNO * 8          // W shard
           + (size_t)N * kNO * 8 * 3          // P (G on the leader), R copy, sigma / R (leader)
           + (size_t)N * 8                    // q (leader)
           + (size_t)N * 2 + 64 + 16          // OMASK, flags
           + 2 * ((cl_buf_bytes(N) + 15) & ~(size_t)15);
}

__host__ __device__ inline size_t k_shard_smem(int N) { return (size_t)N * kCl * 4; }

// k_shard: grid = images.  Shard boundaries, shard-major step lists with
// shard-local rows, and dt / |d_hat(s)|.
__global__ void __launch_bounds__(256) k_shard(const TrainArgs T, const ShardWS S) {
    const int64_t i = blockIdx.x;
    const int N = T.c.n_steps;
    const TrainWS &W = T.ws;
    const int n_act = W.n_act[i];
    const uint16_t *act_k = W.act_k + (size_t)i * kNH;
    const int32_t *soff = W.step_off + (size_t)i * (N + 1);
    const uint16_t *sk = W.step_k + (size_t)i * W.evcap;
    __shared__ int s_act[kCl + 1];
    __shared__ int s_base[kCl + 1];
    extern __shared__ int s_len[];  // [N][kCl] segment lengths, then their offsets
    if (threadIdx.x <= kCl) {
        const int r = threadIdx.x;
        int lo = 0, hi = n_act;  // first active index with id >= r * kClRows
        const int key = r * kClRows;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if ((int)act_k[mid] < key) lo = mid + 1;
            else hi = mid;
        }
        s_act[r] = r == kCl ? n_act : lo;
        S.act[i * (kCl + 1) + r] = s_act[r];
    }
    const double *nrm = W.norm + (size_t)i * N;
    for (int s = threadIdx.x; s < N; s += blockDim.x) {
        const double nv = nrm[s];
        S.q[(size_t)i * N + s] = nv > T.c.norm_eps ? __ddiv_rn(T.c.dt, nv) : 0.0;
    }
    __syncthreads();
    // segment [lo, hi) of shard r in step s's list
    auto seg = [&](int s, int r, int &lo, int &hi) {
        auto lower = [&](int key) {
            int a = soff[s], b = soff[s + 1];
            while (a < b) {
                const int mid = (a + b) >> 1;
                if ((int)sk[mid] < key) a = mid + 1;
                else b = mid;
            }
            return a;
        };
        lo = lower(s_act[r]);
        hi = r + 1 < kCl ? lower(s_act[r + 1]) : soff[s + 1];
    };
    for (int t = threadIdx.x; t < N * kCl; t += blockDim.x) {
        int lo, hi;
        seg(t / kCl, t % kCl, lo, hi);
        s_len[t] = hi - lo;
    }
    __syncthreads();
    if (threadIdx.x < kCl) {  // per-shard prefix over steps
        const int r = threadIdx.x;
        int run = 0;
        int32_t *so = S.soff + ((size_t)i * kCl + r) * (N + 1);
        for (int s = 0; s < N; ++s) {
            so[s] = run;
            const int len = s_len[s * kCl + r];
            s_len[s * kCl + r] = run;
            run += len;
        }
        so[N] = run;
        s_base[r + 1] = run;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        s_base[0] = 0;
        for (int r = 0; r < kCl; ++r) s_base[r + 1] += s_base[r];
        for (int r = 0; r <= kCl; ++r) S.ebase[i * (kCl + 1) + r] = s_base[r];
    }
    __syncthreads();
    uint16_t *sid = S.sid + (size_t)i * W.evcap;
    for (int t = threadIdx.x; t < N * kCl; t += blockDim.x) {
        const int s = t / kCl, r = t % kCl;
        int lo, hi;
        seg(s, r, lo, hi);
        uint16_t *dst = sid + s_base[r] + s_len[t];
        for (int e = lo; e < hi; ++e) dst[e - lo] = (uint16_t)((int)act_k[sk[e]] - r * kClRows);
    }
}

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
    double *Rl = P + (size_t)N * kNO;           // [N][10] local copy of R
    double *SR = Rl + (size_t)N * kNO;          // [N][10] leader: sigma, then R in place
    double *Q = SR + (size_t)N * kNO;           // [N] leader: dt / |d_hat|
    uint16_t *OMASK = reinterpret_cast<uint16_t *>(Q + N);
    int *flags = reinterpret_cast<int *>(OMASK + ((N + 7) & ~7));  // leader: per-CTA non-finite flags
    uint8_t *bufmem = reinterpret_cast<uint8_t *>(flags + 16);
    const size_t bstride = (cl_buf_bytes(N) + 15) & ~(size_t)15;
    __shared__ ClBuf s_buf[2];
    __shared__ int s_abort;

    const int k_lo = r * kClRows, k_hi = min(k_lo + kClRows, kNH);
    const int rows = k_hi - k_lo;
    if (T.status[0] != 0) return;  // an earlier chunk failed (uniform over the cluster)
    double *undo = SW.undo + (size_t)r * kClRows * kNO;
    for (int t = tid; t < rows * kNO; t += kClThreads) Wsh[t] = __ldcg(T.w + (size_t)k_lo * kNO + t);
    if (tid < kCl) flags[tid] = 0;
    const double *SR_lead = cluster.map_shared_rank(SR, 0);
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
        const int32_t *sa = SW.act + j * (kCl + 1);
        const int a0 = sa[r], a1 = sa[r + 1];
        const int32_t *gaoff = W.act_off + (size_t)j * (kNH + 1);
        const int e0 = gaoff[a0], e1 = gaoff[a1];
        const int32_t *gso = SW.soff + ((size_t)j * kCl + r) * (N + 1);
        const int nid = gso[N];
        const uint16_t *gsid = SW.sid + (size_t)j * W.evcap + SW.ebase[j * (kCl + 1) + r];
        const bool fa = a1 - a0 <= kClACap && e1 - e0 <= kClECap, fs = nid <= kClECap;
        for (int k = t; k <= N; k += nt) soff[k] = gso[k];
        if (fs)
            for (int k = t; k < nid; k += nt) sid[k] = gsid[k];
        if (fa) {
            for (int k = t; k <= a1 - a0; k += nt) aoff[k] = gaoff[a0 + k];
            for (int k = t; k < a1 - a0; k += nt) act[k] = W.act_k[(size_t)j * kNH + a0 + k];
            for (int k = t; k < e1 - e0; k += nt) nsp[k] = W.nsp[(size_t)j * W.evcap + e0 + k];
        }
        if (t == 0) {
            ClBuf &B = s_buf[b];
            B.soff = soff;
            B.sid = fs ? sid : gsid;
            B.act = fa ? act : W.act_k + (size_t)j * kNH + a0;
            B.aoff = fa ? aoff : gaoff + a0;
            B.nsp = fa ? nsp : W.nsp + (size_t)j * W.evcap + e0;
            B.abias = fa ? e0 : 0;
            B.n_act = a1 - a0;
        }
    };
    // put back the rows image j changed (undo log)
    auto restore = [&](const ClBuf &B) {
        for (int t = tid; t < B.n_act * kNO; t += kClThreads) {
            const int row = (int)B.act[t / kNO] - k_lo;
            Wsh[row * kNO + t % kNO] = undo[row * kNO + t % kNO];
        }
    };

    if (T.n > 0) stage(0, 0, 0, kClThreads);
    cluster.sync();

    bool failed = false;
    long long *clk = nullptr;
    auto stamp = [&](int ph) {
        if (clk && tid == 0) clk[ph] = clock64();
    };
    for (int64_t i = 0; i < T.n; ++i) {
        clk = (SW.clk && r == 0 && T.first + i < 64) ? SW.clk + (T.first + i) * 16 : nullptr;
        stamp(0);
        const ClBuf &B = s_buf[i & 1];
        // ---- G partials of this shard (ascending id within the shard)
        for (int t = tid; t < N * kNO; t += kClThreads) {
            const int s = t / kNO, l = t - s * kNO;
            const int e1 = B.soff[s + 1];
            double g = 0.0;
            int e = B.soff[s];
            for (; e + 4 <= e1; e += 4) {
                int id[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) id[u] = B.sid[e + u];
#pragma unroll
                for (int u = 0; u < 4; ++u) g = __dadd_rn(g, Wsh[id[u] * kNO + l]);
            }
            for (; e < e1; ++e) g = __dadd_rn(g, Wsh[(int)B.sid[e] * kNO + l]);
            P[t] = g;
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
            for (int t = tid; t < N * kNO; t += kClThreads) {
                double v[kCl];
#pragma unroll
                for (int q = 1; q < kCl; ++q) v[q] = cluster.map_shared_rank(P, q)[t];
                double g = P[t];
#pragma unroll
                for (int q = 1; q < kCl; ++q) g = __dadd_rn(g, v[q]);
                P[t] = g;
            }
            for (int s = tid; s < N; s += kClThreads) Q[s] = SW.q[(size_t)i * N + s];
            __syncthreads();
            stamp(3);
            if (warp == 0) {
                // output layer (network.py:308-314): the serial chain
                const int l = lane < kNO ? lane : kNO - 1;
                OutState st;
                out_init(st, c);
                for (int s = 0; s < N; ++s) {
                    double ff;
                    out_step(st, c, P[s * kNO + l], s, l, &ff);
                    if (lane == 0) OMASK[s] = (uint16_t)st.prev;
                }
                if (lane < kNO) T.counts[(size_t)i * kNO + lane] = st.cnt;
            } else if (more) {
                stage(i + 1, (int)((i + 1) & 1), 32, kClThreads - 32);
            }
            __syncthreads();
            stamp(4);
            // error signal and gate (normad.py:156-159, :87-91, :104-113): the
            // step counts when some e != 0 and |d_hat| > eps; sigma = e * dt / |d_hat|
            {
                const int label = T.labels[i];
                const int per = c.desired_period;
                for (int t = tid; t < N * kNO; t += kClThreads) {
                    const int s = t / kNO, l = t - s * kNO;
                    const bool want = per > 0 && s >= per - 1 && (s - (per - 1)) % per == 0 && l == label;
                    const bool got = (OMASK[s] >> l) & 1u;
                    const double q = Q[s];
                    SR[t] = want == got ? 0.0 : (want ? q : -q);  // (+-dt) / |d_hat| == +-(dt / |d_hat|)
                }
            }
            __syncthreads();
            stamp(5);
            // R(u, l) = sum_{s >= u} sigma(s, l) H(s - u): adjoint of kernel -> d_hat, backward
            if (warp == 0 && lane < kNO) {
                double pd = 0.0, pa = 0.0, pb = 0.0;
                for (int u = N - 1; u >= 0; --u) {
                    pd = __dadd_rn(__dmul_rn(pd, c.decay_learn), SR[u * kNO + lane]);
                    const double q = __dmul_rn(pd, c.dhat_scale);
                    pa = __dadd_rn(__dmul_rn(pa, c.decay_slow), q);
                    pb = __dadd_rn(__dmul_rn(pb, c.decay_fast), q);
                    SR[u * kNO + lane] = __dsub_rn(pa, pb);
                }
            }
            __syncthreads();
            stamp(6);
        } else if (more) {
            stage(i + 1, (int)((i + 1) & 1), 0, kClThreads);
        }
        cluster.sync();  // B2: R ready on the leader, next lists staged
        stamp(7);
        for (int t = tid; t < N * kNO; t += kClThreads) Rl[t] = SR_lead[t];
        __syncthreads();
        stamp(8);
        // dW for the shard's active neurons (spikes ascending); commit with an undo log
        bool bad = false;
        for (int a = tid; a < B.n_act; a += kClThreads) {
            const int row = (int)B.act[a] - k_lo;
            double acc[kNO];
#pragma unroll
            for (int l = 0; l < kNO; ++l) acc[l] = 0.0;
            const int e1 = B.aoff[a + 1] - B.abias;
            for (int e = B.aoff[a] - B.abias; e < e1; ++e) {
                const double *rr = Rl + (int)B.nsp[e] * kNO;
#pragma unroll
                for (int l = 0; l < kNO; ++l) acc[l] = __dadd_rn(acc[l], rr[l]);
            }
#pragma unroll
            for (int l = 0; l < kNO; ++l) {
                const double old = Wsh[row * kNO + l];
                const double nw = __dadd_rn(old, __dmul_rn(c.learning_rate, acc[l]));
                bad |= !isfinite(nw);
                undo[row * kNO + l] = old;
                Wsh[row * kNO + l] = nw;
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
    for (int t = tid; t < rows * kNO; t += kClThreads) T.w[(size_t)k_lo * kNO + t] = Wsh[t];
    cluster.sync();  // no CTA leaves while others may still read its shared memory
}

}  // namespace snn
