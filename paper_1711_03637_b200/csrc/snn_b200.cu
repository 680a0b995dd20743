// C ABI of the spiking-digit hot path (include/snn_b200.h).  One translation
// unit: the kernels live in hidden.cuh (inference) and normad.cuh (training).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>

#include "normad_cl.cuh"
#include "normad_spec.cuh"
#include "preprocess.cuh"

using namespace snn;

namespace {

thread_local char g_err[512] = "";

int set_error(int code, const char *msg) {
    snprintf(g_err, sizeof(g_err), "%s", msg);
    return code;
}

int cuda_check(const char *where) {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        char buf[512];
        snprintf(buf, sizeof(buf), "%s: %s", where, cudaGetErrorString(e));
        return set_error(SNN_ECUDA, buf);
    }
    return SNN_OK;
}

int validate(const snn_consts_t *c) {
    if (!c) return set_error(SNN_EINVAL, "consts is NULL");
    if (c->n_steps <= 0 || c->n_steps > (1 << 20)) return set_error(SNN_EINVAL, "n_steps out of range");
    if (c->desired_period < 0) return set_error(SNN_EINVAL, "desired_period must be >= 0");
    if (!(c->dt > 0)) return set_error(SNN_EINVAL, "dt must be positive");
    return SNN_OK;
}

size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

constexpr int kMaxSub = 64;  // sub-batches of one pipelined snn_infer call

// The specialised kernel is exact for any bank whose taps EQUAL the default
// ones (+0.0 and -0.0 zero taps are both skipped, see def_current).
bool is_default_bank(const snn_consts_t &c) {
    for (int f = 0; f < kNF; ++f)
        for (int k = 0; k < 9; ++k)
            if (!(c.taps[f][k] == def_tap(f, k))) return false;
    return true;
}

// Hidden-layer comparisons can run on the integer pipe when E_L < 0 < V_T
// (see lif_update); any other sign pattern takes the FP64 compares.
bool signed_lif(const snn_consts_t &c) { return c.lif_hid.el < 0.0 && c.lif_hid.vt > 0.0; }

// upper bound of the compact raster of n images (every image at 22 tiles)
size_t raster_bytes(const snn_consts_t *c, int64_t n) { return (size_t)n * kMaxTiles * n_chunks(c->n_steps) * kRastTC; }

// ---- inference workspace: tile_pos | n_tiles | tile_base | raster (upper bound)
struct InferWS {
    uint16_t *tile_pos;
    int32_t *n_tiles, *tile_base, *n_win, *win_base;
    uint8_t *raster;
    double *g;     // [n][N][10] G rows (k_gsum -> k_output)
    double *gabs;  // [n][N][10] sum of |W| rows (near-tie accounting only)
    int32_t *fix;  // [1 + n * 676] guard-band hidden layer: count, flagged windows
    double *wpad;  // [8112][16] padded W rows for k_gsum (batches of >= kWPadMinImages), else null
};

size_t infer_ws_layout(const snn_consts_t *c, int64_t n, char *base, InferWS *w) {
    size_t off = 0;
    auto take = [&](size_t bytes) {
        char *p = base ? base + off : nullptr;
        off += al(bytes);
        return p;
    };
    InferWS x;
    x.tile_pos = (uint16_t *)take((size_t)n * kMaxTiles * kTile * 2);
    x.n_tiles = (int32_t *)take((size_t)n * 4);
    x.tile_base = (int32_t *)take((size_t)(n + 1 + kMaxSub) * 4);
    x.n_win = (int32_t *)take((size_t)n * 4);
    x.win_base = (int32_t *)take((size_t)(n + 1 + kMaxSub) * 4);
    x.raster = (uint8_t *)take(raster_bytes(c, n));
    x.g = (double *)take((size_t)n * c->n_steps * kNO * 8);
    x.gabs = (double *)take((size_t)n * c->n_steps * kNO * 8);
    x.fix = (int32_t *)take(((size_t)n * kNPos + 1) * 4);
    x.wpad = n >= kWPadMinImages ? (double *)take((size_t)kNH * kWPad * 8) : nullptr;

    if (w) *w = x;
    return off;
}

size_t infer_ws(const snn_consts_t *c, int64_t n) { return infer_ws_layout(c, n, nullptr, nullptr); }

// ---- training workspace (per chunk)
int64_t train_evcap(const snn_consts_t *c) {
    // worst case: every hidden neuron fires as often as its refractory period allows
    const int gap = std::max(1, (int)floor(c->lif_hid.refr));
    const int64_t per_neuron = std::min<int64_t>(c->n_steps, c->n_steps / gap + 1);
    return (int64_t)kNH * per_neuron;
}

size_t train_ws_per_image(const snn_consts_t *c) {
    const size_t N = c->n_steps, cap = train_evcap(c);
    return raster_bytes(c, 1) + kNPos * 4 + kMaxTiles * kTile * 2 + 4 + 4 + 4 + kNH * 2 + (kNH + 1) * 4 + cap * 2 +
           (N + 1) * 4 + cap * 2 + N * 8 + kMaxTiles * N * 8 + 3 * (kCl + 1) * 4 + 8 + kCl * (N + 1) * 4 + 2 * cap * 2 +
           N * 8 + kNH * 2 * 2 + (kNH + kCl) * 4 + (size_t)kCl * kClRows * kNO * 8 / 64;
}

int64_t train_chunk(const snn_consts_t *c, int64_t n) {
    const size_t budget = (size_t)768 << 20;
    int64_t ch = (int64_t)(budget / train_ws_per_image(c));
    ch = std::max<int64_t>(1, std::min<int64_t>(ch, 1024));
    return std::min<int64_t>(ch, std::max<int64_t>(n, 1));
}

size_t train_ws(const snn_consts_t *c, int64_t chunk, TrainWS *out, char *base, ShardWS *sh = nullptr) {
    const size_t N = c->n_steps, cap = train_evcap(c), n = chunk;
    size_t off = 0;
    auto take = [&](size_t bytes) {
        char *p = base ? base + off : nullptr;
        off += al(bytes);
        return p;
    };
    TrainWS w;
    w.raster = (uint8_t *)take(raster_bytes(c, (int64_t)n));
    w.tile_pos = (uint16_t *)take(n * kMaxTiles * kTile * 2);
    w.n_tiles = (int32_t *)take(n * 4);
    w.tile_base = (int32_t *)take((n + 1) * 4);
    w.n_win = (int32_t *)take(n * 4);
    w.win_base = (int32_t *)take((n + 1) * 4);
    w.n_act = (int32_t *)take(n * 4);
    w.act_k = (uint16_t *)take(n * kNH * 2);
    w.act_off = (int32_t *)take(n * (kNH + 1) * 4);
    w.nsp = (uint16_t *)take(n * cap * 2);
    w.step_off = (int32_t *)take(n * (N + 1) * 4);
    w.step_k = (uint16_t *)take(n * cap * 2);
    w.norm = (double *)take(n * N * 8);
    w.wp = (double *)take(n * kMaxTiles * N * 8);
    w.fix = (int32_t *)take((n * kNPos + 1) * 4);
    w.evcap = (int64_t)cap;
    ShardWS x;
    memset(&x, 0, sizeof(x));  // flags (push, alias, skip) are set by the caller
    x.clk = nullptr;
    x.q = (double *)take(n * N * 8);
    x.soff = (int32_t *)take(n * kCl * (N + 1) * 4);
    x.ebase = (int32_t *)take(n * (kCl + 1) * 4);
    x.sid = (uint16_t *)take(n * cap * 2);
    x.abase = (int32_t *)take(n * (kCl + 1) * 4);
    x.sact = (uint16_t *)take(n * kNH * 2);
    x.sidx = (uint16_t *)take(n * kNH * 2);
    x.saoff = (int32_t *)take(n * (kNH + kCl) * 4);
    x.nbase = (int32_t *)take(n * (kCl + 1) * 4);
    x.snsp = (uint16_t *)take(n * cap * 2);
    x.undo = (double *)take((size_t)kCl * kClRows * kNO * 8);
    if (out) *out = w;
    if (sh) *sh = x;
    return off;
}

cudaEvent_t g_ev_before = nullptr, g_ev_after = nullptr;  // snn_profile_events
cudaEvent_t g_stage[7] = {};  // snn_profile_stage_events (6: between the guard-band kernel and its redo)
inline void stage_mark(int k, cudaStream_t st) {
    if (g_stage[k]) cudaEventRecord(g_stage[k], st);
}

// Per-device state: function attributes, occupancy and SM counts are
// properties of a device context, and the tuning knobs (snn_set_*) apply to
// the calling thread's current device, so one process may drive several
// B200s (one Engine per device) with independent settings.
constexpr int kMaxDev = 64;

int cur_dev() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDev) dev = 0;
    return dev;
}

int g_sms[kMaxDev] = {};

int sm_count() {
    const int dev = cur_dev();
    if (!g_sms[dev]) {
        int sms = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        g_sms[dev] = sms > 0 ? sms : 148;
    }
    return g_sms[dev];
}

#ifndef SNN_HID_FZ
#define SNN_HID_FZ 1
#endif
struct Knobs {
    int hid_ctas = 0;                  // k_hidden CTAs per SM (0 = occupancy limit); snn_set_pipeline
    int hid_res = 1;                   // snn_set_hidden_resident
    int hid_gb = 1;                    // guard-band FP32 hidden kernel when it applies (snn_set_hidden_resident)
    int hid_gb_small = 0;              // ... also below kGbMinImages (snn_set_hidden_resident(5), tests)
    int out_dist = 1;                  // k_output_dist for large batches (snn_set_output_dist)
    int hid_fz = SNN_HID_FZ;           // -DSNN_HID_FZ=0: never the frozen-mask variant (A/B builds)
    int normad_cluster = 4;            // snn_set_normad_cluster (4: speculative scan)
    long long *phase_clk = nullptr;    // snn_normad_phase_clocks
    int normad_skip = 0;               // snn_normad_skip (profiling only)
    int64_t pipe_images = 0;           // snn_set_pipeline
};
Knobs g_knobs[kMaxDev];

Knobs &knobs() { return g_knobs[cur_dev()]; }

// Frozen steps after a hidden spike, next_live_step(s) - s - 1 (the same fp64
// expression as the kernels), if it is the same for every step of the trial;
// else -1.
int refr_span(const snn_consts_t &c) {
    int k = -1;
    for (int s = 0; s < c.n_steps; ++s) {
        const int d = (int)std::floor((double)s + c.lif_hid.refr) - s;
        if (s == 0) k = d;
        else if (d != k) return -1;
    }
    return k;
}
// Guard-band FP32 hidden kernel + FP64 redo of the flagged windows
// (hidden_gb.cuh): the same raster as k_hidden_res<.., FZ = 3>.  The band
// analysis needs a contracting step (0 < D = 1 - beta g < 1) and a positive
// threshold distance whose scaled values are normal float32 numbers.
bool gb_applies(const snn_consts_t &c) {
    const snn_lif_t &p = c.lif_hid;
    const double D = 1.0 - p.beta * p.g, theta = p.vt - p.el;
    const double s1 = p.beta * kG1, s2 = p.beta * kG2;
    if (!(D > 0x1p-10 && D < 1.0 - 0x1p-16 && theta > 0.0 && s1 > 0.0 && s2 > 0.0)) return false;
    const double r1 = theta / s1, r2 = theta / s2;
    return r1 > 0x1p-40 && r1 < 0x1p40 && r2 > 0x1p-40 && r2 < 0x1p40 && std::isfinite(D);
}

template <bool SGN>
int launch_hidden_gb(const BatchArgs &A, cudaStream_t st, int variant) {
    static bool attr[kMaxDev][3] = {};
    const int dev = cur_dev();
    const int64_t items = ((int64_t)A.n_images * kMaxTiles + 1) / 2;  // upper bound for the grid
    // CTA size: each warp runs its items in waves over the SMs; with the
    // measured per-item times of the two sizes (16 warps: 84.6 us, 20 warps:
    // 101.6 us per wave at N = 100), take the one with the smaller
    // ceil(items / slots) x wave time -- 20 warps for large batches, 16 when
    // 20 would leave a mostly empty last wave (e.g. 1,250 images: 254 vs 305 us)
    // (the active-window count is only known on the device; 357 per image is
    // the MNIST-like average, and either size gives the same raster)
    const int64_t est = (int64_t)A.n_images * 357 / 64 + 1;
    const int64_t s16 = (int64_t)sm_count() * kGbWarpsSmall, s20 = (int64_t)sm_count() * kGbWarps;
    const bool small = variant != 2 && ((est + s16 - 1) / s16) * 846 < ((est + s20 - 1) / s20) * 1016;
    const int vi = variant == 2 ? 1 : small ? 2 : 0;
    if (!attr[dev][vi]) {
        cudaError_t e = vi == 1 ? cudaFuncSetAttribute(k_hidden_gb1<3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                       (int)gb_smem_bytes(kGbMaxSteps))
                        : vi == 2 ? cudaFuncSetAttribute(k_hidden_gb<3, kGbWarpsSmall>,
                                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                         (int)gb_smem_bytes(kGbMaxSteps))
                                  : cudaFuncSetAttribute(k_hidden_gb<3, kGbWarps>,
                                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                         (int)gb_smem_bytes(kGbMaxSteps));
        if (e != cudaSuccess) return cuda_check("cudaFuncSetAttribute(k_hidden_gb)");
        attr[dev][vi] = true;
    }
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(sm_count(), items));
    const size_t smem = gb_smem_bytes(A.c.n_steps);
    if (vi == 1) k_hidden_gb1<3><<<grid, kGbWarps * 32, smem, st>>>(A);
    else if (vi == 2) k_hidden_gb<3, kGbWarpsSmall><<<grid, kGbWarpsSmall * 32, smem, st>>>(A);
    else k_hidden_gb<3, kGbWarps><<<grid, kGbWarps * 32, smem, st>>>(A);
    int rc = cuda_check("k_hidden_gb");
    if (rc) return rc;
    stage_mark(6, st);
    if (A.c.n_steps <= kResMaxSteps) {  // table resident in shared memory
        const size_t fsm = (size_t)A.c.n_steps * 256 * 8;
        static int attr_set[kMaxDev] = {};
        int &done = attr_set[cur_dev()];
        if (done < (int)fsm) {
            if (cudaFuncSetAttribute(k_hidden_fix_res<SGN, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)fsm) != cudaSuccess)
                return cuda_check("cudaFuncSetAttribute(k_hidden_fix_res)");
            done = (int)fsm;
        }
        k_hidden_fix_res<SGN, 3><<<(unsigned)sm_count(), kFixResThreads, fsm, st>>>(A);
    } else {
        k_hidden_fix<SGN, 3><<<(unsigned)(4 * sm_count()), kFixThreads, 0, st>>>(A);
    }
    if ((rc = cuda_check("k_hidden_fix"))) return rc;
    if (A.out.hidden_redo) cudaMemcpyAsync(A.out.hidden_redo, A.fix_count, 4, cudaMemcpyDeviceToDevice, st);
    return SNN_OK;
}

template <bool TRACE, bool DEF, bool SGN, int FZ>
int launch_hidden_res(const BatchArgs &A, cudaStream_t st) {
    static bool attr[kMaxDev] = {};  // per device context (idempotent if two threads race)
    const size_t smem = (size_t)A.c.n_steps * 256 * 8;
    const int dev = cur_dev();
    if (!attr[dev]) {
        if (cudaFuncSetAttribute(k_hidden_res<TRACE, DEF, SGN, FZ>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)(kResMaxSteps * 256 * 8)) != cudaSuccess)
            return cuda_check("cudaFuncSetAttribute(k_hidden_res)");
        attr[dev] = true;
    }
    const int64_t max_items = (int64_t)A.items_per_tile * A.n_images * kMaxTiles;
    const unsigned grid = (unsigned)std::min<int64_t>(sm_count(), max_items);
    k_hidden_res<TRACE, DEF, SGN, FZ><<<grid, kResWarps * 32, smem, st>>>(A);
    return SNN_OK;
}

// prep -> tile scan -> hidden (persistent): the hidden raster of A's images
template <bool TRACE, bool DEF, bool SGN>
int launch_hidden(const BatchArgs &A, cudaStream_t st) {
    static int hid_blocks_dev[kMaxDev] = {};
    const Knobs &K = knobs();
    int &hid_blocks = hid_blocks_dev[cur_dev()];
    if (!hid_blocks) {
        int b = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_hidden<TRACE, DEF, SGN>, kThreads, 0) !=
                cudaSuccess ||
            b <= 0)
            b = 4;
        hid_blocks = b;
    }
    const int per_sm = K.hid_ctas > 0 ? std::min(K.hid_ctas, hid_blocks) : hid_blocks;
    int rc;
    const unsigned n = (unsigned)A.n_images;
    stage_mark(0, st);
    k_prep<<<n, kThreads, 0, st>>>(A);
    if ((rc = cuda_check("k_prep"))) return rc;
    stage_mark(1, st);
    k_tile_scan<<<1, 1024, 0, st>>>(A);
    if ((rc = cuda_check("k_tile_scan"))) return rc;
    stage_mark(2, st);
    if (g_ev_before) cudaEventRecord(g_ev_before, st);
    bool gb = false;
    if constexpr (DEF && !TRACE)
        gb = K.hid_res && K.hid_gb && K.hid_fz && A.fix_count && A.c.n_steps <= kGbMaxSteps && refr_span(A.c) == 3 &&
             gb_applies(A.c) && (A.n_images >= kGbMinImages || K.hid_gb_small);
    if (gb) {
        if ((rc = launch_hidden_gb<SGN>(A, st, K.hid_gb))) return rc;
    } else if (K.hid_res && A.c.n_steps <= kResMaxSteps) {  // table resident in shared memory
        if constexpr (DEF && !TRACE) {
            if (K.hid_fz && refr_span(A.c) == 3) rc = launch_hidden_res<TRACE, DEF, SGN, 3>(A, st);
            else rc = launch_hidden_res<TRACE, DEF, SGN, 0>(A, st);
        } else {
            rc = launch_hidden_res<TRACE, DEF, SGN, 0>(A, st);
        }
        if (rc) return rc;
    } else {
        const int64_t max_groups = (2 * A.n_images * kMaxTiles + kWPC - 1) / kWPC;
        const unsigned grid = (unsigned)std::min<int64_t>((int64_t)per_sm * sm_count(), max_groups);
        k_hidden<TRACE, DEF, SGN><<<grid, kThreads, 0, st>>>(A);
    }
    if ((rc = cuda_check("k_hidden"))) return rc;
    if (g_ev_after) cudaEventRecord(g_ev_after, st);
    stage_mark(3, st);
    return SNN_OK;
}

// G rows, then the output layer.  With near_ties requested, also the |W|
// sums (second half of the G buffer, see InferWS) and the tie bound.
int launch_contract(const BatchArgs &A, double *g, cudaStream_t st) {
    int rc;
    const int64_t n = A.n_images;
    const int64_t tasks = n * n_chunks(A.c.n_steps);
    const unsigned gg = (unsigned)((tasks + kGWarps - 1) / kGWarps), og = (unsigned)((n + kOutWarps2 - 1) / kOutWarps2);
    double *gabs = A.out.near_ties ? A.gabs : nullptr;
    if (gabs && A.wpad) k_gsum<true, kWPad><<<gg, kGWarps * 32, 0, st>>>(A, g, gabs);
    else if (gabs) k_gsum<true><<<gg, kGWarps * 32, 0, st>>>(A, g, gabs);
    else if (A.wpad) k_gsum<false, kWPad><<<gg, kGWarps * 32, 0, st>>>(A, g, nullptr);
    else k_gsum<false><<<gg, kGWarps * 32, 0, st>>>(A, g, nullptr);
    if ((rc = cuda_check("k_gsum"))) return rc;
    stage_mark(4, st);
    // large batches: the lane-distributed step (fewer FP64 instructions; the
    // kernel is FP64-throughput bound there), small ones: the replicated step
    // (shorter serial chain per image)
    if (gabs) k_output<true><<<og, kOutWarps2 * 32, 0, st>>>(A, g, gabs);
    else if (A.n_images >= kOutDistMinImages && knobs().out_dist) {
        if (A.out.out_raster || A.out.ff || A.out.v_out) k_output_dist<true><<<og, kOutWarps2 * 32, 0, st>>>(A, g);
        else k_output_dist<false><<<og, kOutWarps2 * 32, 0, st>>>(A, g);
    }
    else if (A.out.out_raster || A.out.ff || A.out.v_out) k_output<false, true><<<og, kOutWarps2 * 32, 0, st>>>(A, g, nullptr);
    else k_output<false, false><<<og, kOutWarps2 * 32, 0, st>>>(A, g, nullptr);
    stage_mark(5, st);
    return cuda_check("k_output");
}

template <bool TRACE, bool DEF, bool SGN>
int launch_batch(const BatchArgs &A, double *g, cudaStream_t st) {
    int rc = launch_hidden<TRACE, DEF, SGN>(A, st);
    if (rc || !g) return rc;
    return launch_contract(A, g, st);
}

template <bool DEF>
int launch_hidden_fast(const BatchArgs &A, cudaStream_t st) {
    return signed_lif(A.c) ? launch_hidden<false, DEF, true>(A, st) : launch_hidden<false, DEF, false>(A, st);
}

// Picks the k_hidden instantiation: TRACE variants always use FP64 compares.
template <bool DEF>
int launch_fast(const BatchArgs &A, double *g, cudaStream_t st) {
    return signed_lif(A.c) ? launch_batch<false, DEF, true>(A, g, st) : launch_batch<false, DEF, false>(A, g, st);
}

// Per-device auxiliary stream + events of the pipelined inference path.
struct Pipe {
    cudaStream_t aux = nullptr;
    cudaEvent_t ev[kMaxSub + 1] = {};
};
std::mutex g_pipe_mu;
Pipe g_pipes[64];

// Per-device auxiliary stream + events of snn_train's chunk preparation.
struct TrainPipe {
    cudaStream_t aux = nullptr;
    cudaEvent_t fork = nullptr, pre[2] = {}, done[2] = {};
};
TrainPipe g_tpipes[64];

TrainPipe *train_pipe_for_device() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
    std::lock_guard<std::mutex> lk(g_pipe_mu);
    TrainPipe &p = g_tpipes[dev];
    if (!p.aux) {
        if (cudaStreamCreateWithFlags(&p.aux, cudaStreamNonBlocking) != cudaSuccess) return nullptr;
        for (cudaEvent_t *e : {&p.fork, &p.pre[0], &p.pre[1], &p.done[0], &p.done[1]})
            if (cudaEventCreateWithFlags(e, cudaEventDisableTiming) != cudaSuccess) return nullptr;
    }
    return &p;
}

Pipe *pipe_for_device() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
    Pipe &p = g_pipes[dev];
    if (!p.aux) {
        if (cudaStreamCreateWithFlags(&p.aux, cudaStreamNonBlocking) != cudaSuccess) return nullptr;
        for (auto &e : p.ev)
            if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return nullptr;
    }
    return &p;
}

// Shared-memory caps of k_normad: as many active neurons / events as fit in
// ~200 KB next to the per-step arrays (roughly 1.5k neurons, 8k events at N=100).
NormadCaps normad_caps(const snn_consts_t *c) {
    const size_t budget = 200 * 1024;
    NormadCaps cap{0, 0};
    if (normad_smem_bytes(c->n_steps, cap) > budget) return cap;
    const size_t left = budget - normad_smem_bytes(c->n_steps, cap);
    // split: per active neuron 80+4+2 B, per event 4 B, ~6 events per active neuron
    const size_t unit = 86 + 6 * 4;
    cap.acap = (int)std::min<size_t>(kNH, left / unit);
    cap.ecap = (int)std::min<size_t>(65535, (left - (size_t)cap.acap * 86) / 4);
    return cap;
}

}  // namespace

extern "C" int snn_abi_version(void) { return SNN_ABI_VERSION; }

extern "C" void snn_profile_events(void *before, void *after) {
    g_ev_before = (cudaEvent_t)before;
    g_ev_after = (cudaEvent_t)after;
}
extern "C" void snn_profile_stage_events(void *const *events, int n_events) {
    for (int k = 0; k < 7; ++k) g_stage[k] = (events && k < n_events) ? (cudaEvent_t)events[k] : nullptr;
}

extern "C" const char *snn_last_error(void) { return g_err; }

#ifdef SNN_SCAN_STAMPS
extern "C" int snn_debug_scan_stamps(long long *out, int n) {
    return cudaMemcpyFromSymbol(out, snn::g_scan_stamps, sizeof(long long) * (size_t)std::min(n, 256)) == cudaSuccess ? 0 : 1;
}
#endif

extern "C" int snn_input_table(const snn_consts_t *c, double *d_ctab, uint8_t *d_spk, void *stream) {
    int rc = validate(c);
    if (rc) return rc;
    if (!d_ctab) return set_error(SNN_EINVAL, "d_ctab is NULL");
    k_input_table<<<1, 256, 0, (cudaStream_t)stream>>>(*c, d_ctab, d_spk);
    return cuda_check("k_input_table");
}

extern "C" size_t snn_infer_workspace(const snn_consts_t *c, int64_t n) {
    if (!c || n < 0 || c->n_steps <= 0) return 0;
    return infer_ws(c, n);
}

extern "C" int snn_infer(const snn_consts_t *c, const uint8_t *d_images, int64_t n, const double *d_w,
                         const double *d_ctab, const snn_infer_out_t *out, void *d_ws, size_t ws_bytes,
                         void *stream) {
    int rc = validate(c);
    if (rc) return rc;
    if (n < 0) return set_error(SNN_EINVAL, "n_images < 0");
    if (n == 0) return SNN_OK;
    if (!out || !out->counts) return set_error(SNN_EINVAL, "counts output is required");
    if (!d_images || !d_w || !d_ctab) return set_error(SNN_EINVAL, "NULL input pointer");
    if (((uintptr_t)d_images & 15) != 0) return set_error(SNN_EINVAL, "images must be 16-byte aligned");
    if (n * kMaxTiles > 0x7fffffffLL) return set_error(SNN_EINVAL, "too many images in one call");
    if (out->raster && (!out->tile_pos || !out->n_tiles || !out->tile_base))
        return set_error(SNN_EINVAL, "raster output needs tile_pos, n_tiles and tile_base");
    if (!d_ws || ws_bytes < infer_ws(c, n)) return set_error(SNN_ENOMEM, "workspace too small");
    cudaStream_t s = (cudaStream_t)stream;
    InferWS w;
    infer_ws_layout(c, n, (char *)d_ws, &w);
    BatchArgs A;
    memset(&A, 0, sizeof(A));
    A.c = *c;
    A.images = d_images;
    A.n_images = n;
    A.w = d_w;
    A.ctab = d_ctab;
    A.tile_pos = out->tile_pos ? out->tile_pos : w.tile_pos;
    A.n_tiles = out->n_tiles ? out->n_tiles : w.n_tiles;
    A.tile_base = out->tile_base ? out->tile_base : w.tile_base;
    A.n_win = w.n_win;
    A.win_base = w.win_base;
    A.raster = out->raster ? out->raster : w.raster;
    A.gabs = w.gabs;
    A.fix_count = w.fix;
    A.fix_list = w.fix + 1;
    A.wpad = w.wpad;

    A.out = *out;
    const bool def = is_default_bank(*c);
    A.items_per_tile = def ? 1 : 2;
    if (out->v_hid) return def ? launch_batch<true, true, false>(A, w.g, s) : launch_batch<true, false, false>(A, w.g, s);
    // Pipelined: sub-batches of pipe_images; the hidden layer of sub-batch
    // b+1 (main stream) runs while the contraction + output layer of sub-batch
    // b run on an auxiliary stream, and each sub-batch's raster is still in L2
    // when it is read.  Only when no caller-visible raster is requested (that
    // one is indexed by a single tile_base).
    const bool caller_raster = out->raster || out->tile_pos || out->n_tiles || out->tile_base;
    const int64_t pipe_images = knobs().pipe_images;
    Pipe *pp = (pipe_images > 0 && !caller_raster && n > pipe_images) ? pipe_for_device() : nullptr;
    if (!pp) return def ? launch_fast<true>(A, w.g, s) : launch_fast<false>(A, w.g, s);
    std::lock_guard<std::mutex> lk(g_pipe_mu);
    const int64_t per = std::max<int64_t>(pipe_images, (n + kMaxSub - 1) / kMaxSub);
    const int N = c->n_steps, nch = n_chunks(N);
    int b = 0;
    for (int64_t i0 = 0; i0 < n; i0 += per, ++b) {
        BatchArgs B = A;
        B.images = d_images + i0 * SNN_N_PIXELS;
        B.n_images = std::min(per, n - i0);
        B.tile_pos = w.tile_pos + i0 * kMaxTiles * kTile;
        B.n_tiles = w.n_tiles + i0;
        B.tile_base = w.tile_base + i0 + b;
        B.n_win = w.n_win + i0;
        B.win_base = w.win_base + i0 + b;
        B.raster = w.raster + (size_t)i0 * kMaxTiles * nch * kRastTC;
        B.out.counts = out->counts + i0 * kNO;
        if (out->out_raster) B.out.out_raster = out->out_raster + i0 * N;
        if (out->ff) B.out.ff = out->ff + i0 * N * kNO;
        if (out->v_out) B.out.v_out = out->v_out + i0 * N * kNO;
        if (out->near_ties) B.out.near_ties = out->near_ties + i0;
        B.gabs = w.gabs + (size_t)i0 * N * kNO;
        B.wpad = nullptr;  // sub-batches overlap: each one's k_gsum reads the caller's W
        if ((rc = def ? launch_hidden_fast<true>(B, s) : launch_hidden_fast<false>(B, s))) return rc;
        cudaEventRecord(pp->ev[b], s);
        cudaStreamWaitEvent(pp->aux, pp->ev[b], 0);
        if ((rc = launch_contract(B, w.g + (size_t)i0 * N * kNO, pp->aux))) return rc;
    }
    cudaEventRecord(pp->ev[kMaxSub], pp->aux);
    cudaStreamWaitEvent(s, pp->ev[kMaxSub], 0);
    return cuda_check("snn_infer pipeline");
}

extern "C" void snn_set_normad_cluster(int enable) { knobs().normad_cluster = enable; }
extern "C" void snn_set_output_dist(int enable) { knobs().out_dist = enable; }

extern "C" void snn_set_hidden_resident(int enable) {
    Knobs &K = knobs();
    K.hid_res = enable != 0;  // 4: the first guard-band kernel (k_hidden_gb1), for A/B
    K.hid_fz = enable == 2 ? 0 : SNN_HID_FZ;
    K.hid_gb = enable == 1 || enable == 5 ? 1 : enable == 4 ? 2 : 0;
    K.hid_gb_small = enable == 5;
}

extern "C" void snn_normad_phase_clocks(long long *d_clk) { knobs().phase_clk = d_clk; }

extern "C" void snn_normad_skip(int mask) { knobs().normad_skip = mask; }

extern "C" void snn_set_pipeline(int64_t images_per_subbatch, int hidden_ctas_per_sm) {
    Knobs &K = knobs();
    K.pipe_images = images_per_subbatch;
    K.hid_ctas = hidden_ctas_per_sm;
}

extern "C" int64_t snn_train_chunk(const snn_consts_t *c, int64_t n) {
    if (!c || n <= 0 || c->n_steps <= 0) return 0;
    return train_chunk(c, n);
}

extern "C" size_t snn_train_workspace(const snn_consts_t *c, int64_t n) {
    if (!c || n < 0 || c->n_steps <= 0) return 0;
    const int64_t chunk = train_chunk(c, n);
    const size_t one = train_ws(c, chunk, nullptr, nullptr);
    return n > chunk ? 2 * one : one;  // two chunk buffers: the next chunk is prepared during this one
}

extern "C" int snn_train(const snn_consts_t *c, const uint8_t *d_images, const uint8_t *d_labels, int64_t n,
                         double *d_w, const double *d_ctab, int32_t *d_counts, int32_t *d_status, void *d_ws,
                         size_t ws_bytes, void *stream) {
    int rc = validate(c);
    if (rc) return rc;
    if (n < 0) return set_error(SNN_EINVAL, "n_images < 0");
    if (!d_status) return set_error(SNN_EINVAL, "d_status is NULL");
    cudaStream_t s = (cudaStream_t)stream;
    cudaMemsetAsync(d_status, 0, 4 * sizeof(int32_t), s);
    if (n == 0) return cuda_check("snn_train");
    if (!d_images || !d_labels || !d_w || !d_ctab || !d_counts) return set_error(SNN_EINVAL, "NULL pointer");
    if (((uintptr_t)d_images & 15) != 0) return set_error(SNN_EINVAL, "images must be 16-byte aligned");
    if (c->n_steps > 65535) return set_error(SNN_EINVAL, "training supports n_steps <= 65535");
    // the W-resident cluster kernel when its shared memory fits, else the one-CTA kernel
    const Knobs &K = knobs();
    // mode 4 (default): the speculative-scan cluster kernel (normad_spec.cuh,
    // DESIGN.md 4.1) when its shared memory fits, else mode 1; 1 / 3: the
    // cluster kernel (partials pushed), 2: pulled; 0: one CTA.  1-4 give the
    // same weights bit for bit.
    const size_t sp_smem = normad_spec_smem_bytes(c->n_steps);
    const bool use_spec = K.normad_cluster == 4 && sp_smem <= 227 * 1024;
    const bool cl_push = (K.normad_cluster == 1 || K.normad_cluster == 3 || K.normad_cluster == 4) &&
                         normad_cl_smem_bytes(c->n_steps, true) <= 227 * 1024;
    // long trials: sigma/R reuse the G array, so the cluster kernel fits up to N ~ 1,300
    const bool cl_alias = !cl_push && normad_cl_smem_bytes(c->n_steps, false) > 227 * 1024;
    const size_t cl_smem = normad_cl_smem_bytes(c->n_steps, cl_push, cl_alias);
    const bool use_cl = K.normad_cluster && cl_smem <= 227 * 1024;
    const NormadCaps caps = normad_caps(c);
    const size_t smem = normad_smem_bytes(c->n_steps, caps);
    if (!use_cl && !use_spec && smem > 220 * 1024)
        return set_error(SNN_EINVAL, "n_steps too large for the sequential NormAD CTA");
    const int64_t chunk = train_chunk(c, n);
    TrainArgs T;
    memset(&T, 0, sizeof(T));
    ShardWS SW;
    const size_t need = train_ws(c, chunk, &T.ws, (char *)d_ws, &SW);
    SW.clk = K.phase_clk;
    SW.push = cl_push ? 1 : 0;
    SW.alias = cl_alias ? 1 : 0;
    SW.skip = K.normad_skip;
    if (!d_ws || ws_bytes < need) return set_error(SNN_ENOMEM, "workspace too small");
    if (use_spec) {
        if (cudaFuncSetAttribute(k_normad_spec, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sp_smem) !=
            cudaSuccess)
            return cuda_check("cudaFuncSetAttribute(k_normad_spec)");
    } else if (use_cl) {
        if (cudaFuncSetAttribute(k_normad_cl, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cl_smem) != cudaSuccess)
            return cuda_check("cudaFuncSetAttribute(k_normad_cl)");
    } else if (cudaFuncSetAttribute(k_normad, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
        return cuda_check("cudaFuncSetAttribute(k_normad)");
    }
    T.c = *c;
    T.w = d_w;
    T.status = d_status;
    // Chunk k's preparation (hidden raster, compaction, shard lists) does not
    // depend on the weights, so with more than one chunk it runs on an
    // auxiliary stream into the other buffer set while chunk k-1's NormAD
    // kernel (8 SMs) runs on the caller's stream.
    TrainArgs Tb[2] = {T, T};
    ShardWS Sb[2] = {SW, SW};
    const bool two = n > chunk;
    if (two) {
        const size_t one = train_ws(c, chunk, nullptr, nullptr);
        if (ws_bytes < 2 * one) return set_error(SNN_ENOMEM, "workspace too small");
        train_ws(c, chunk, &Tb[1].ws, (char *)d_ws + one, &Sb[1]);
        Sb[1].clk = SW.clk;
        Sb[1].push = SW.push;
        Sb[1].alias = SW.alias;
        Sb[1].skip = SW.skip;
        Sb[1].skip = SW.skip;
    }
    auto prepare = [&](int64_t i0, int64_t cn, int b, cudaStream_t st) -> int {
        TrainArgs &U = Tb[b];
        BatchArgs A;
        memset(&A, 0, sizeof(A));
        A.c = *c;
        A.images = d_images + i0 * SNN_N_PIXELS;
        A.n_images = cn;
        A.w = d_w;
        A.ctab = d_ctab;
        A.raster = U.ws.raster;
        A.tile_pos = U.ws.tile_pos;
        A.n_tiles = U.ws.n_tiles;
        A.tile_base = U.ws.tile_base;
        A.n_win = U.ws.n_win;
        A.win_base = U.ws.win_base;
        A.items_per_tile = is_default_bank(*c) ? 1 : 2;
        A.fix_count = U.ws.fix;
        A.fix_list = U.ws.fix + 1;
        int r;
        if ((r = is_default_bank(*c) ? launch_fast<true>(A, nullptr, st) : launch_fast<false>(A, nullptr, st)))
            return r;
        U.n = cn;
        U.first = i0;
        U.labels = d_labels + i0;
        U.counts = d_counts + i0 * kNO;
        k_compact<<<(unsigned)cn, kCThreads, 0, st>>>(U);
        if ((r = cuda_check("k_compact"))) return r;
        if (use_cl || use_spec) {
            k_shard<<<(unsigned)cn, kShThreads, k_shard_smem(c->n_steps), st>>>(U, Sb[b]);
            if ((r = cuda_check("k_shard"))) return r;
        }
        return SNN_OK;
    };
    auto normad = [&](int b, cudaStream_t st) -> int {
        if (use_spec) {
            k_normad_spec<<<kCl, kSpThreads, sp_smem, st>>>(Tb[b], Sb[b]);
            return cuda_check("k_normad_spec");
        }
        if (use_cl) {
            k_normad_cl<<<kCl, kClThreads, cl_smem, st>>>(Tb[b], Sb[b]);
            return cuda_check("k_normad_cl");
        }
        k_normad<<<1, kTThreads, smem, st>>>(Tb[b], caps);
        return cuda_check("k_normad");
    };
    if (!two) {
        if ((rc = prepare(0, n, 0, s))) return rc;
        return normad(0, s);
    }
    TrainPipe *tp = train_pipe_for_device();
    if (!tp) return set_error(SNN_ECUDA, "could not create the training streams");
    // one call's enqueue sequence at a time: calls from several host threads
    // share the auxiliary stream and events (each has its own workspace)
    static std::mutex train_mu;
    std::lock_guard<std::mutex> lk(train_mu);
    cudaEventRecord(tp->fork, s);  // inputs written on the caller's stream
    cudaStreamWaitEvent(tp->aux, tp->fork, 0);
    // a short first chunk: only its preparation is exposed
    const int64_t first = std::min<int64_t>(chunk, 64);
    int64_t k = 0;
    if ((rc = prepare(0, first, 0, tp->aux))) return rc;
    cudaEventRecord(tp->pre[0], tp->aux);
    for (int64_t i0 = 0; i0 < n; ++k) {
        const int b = (int)(k & 1);
        cudaStreamWaitEvent(s, tp->pre[b], 0);
        if ((rc = normad(b, s))) return rc;
        cudaEventRecord(tp->done[b], s);
        const int64_t i1 = i0 + (k == 0 ? first : chunk);
        if (i1 < n) {
            const int b1 = b ^ 1;
            if (k >= 1) cudaStreamWaitEvent(tp->aux, tp->done[b1], 0);  // chunk k-1 is done with buffer b1
            if ((rc = prepare(i1, std::min(chunk, n - i1), b1, tp->aux))) return rc;
            cudaEventRecord(tp->pre[b1], tp->aux);
        }
        i0 = i1;
    }
    return SNN_OK;
}

extern "C" int snn_preprocess(const uint8_t *d_pixels, const int64_t *d_offsets, const int32_t *d_shapes,
                              const int32_t *d_thresholds, int64_t n, const double *blur3x3, uint8_t *d_out,
                              int32_t *d_status, void *stream) {
    if (n < 0) return set_error(SNN_EINVAL, "n < 0");
    if (n == 0) return SNN_OK;
    if (!d_pixels || !d_offsets || !d_shapes || !d_thresholds || !blur3x3 || !d_out || !d_status)
        return set_error(SNN_EINVAL, "NULL pointer");
    if (n > 0x7fffffffLL) return set_error(SNN_EINVAL, "too many canvases in one call");
    PreArgs P;
    P.pixels = d_pixels;
    P.offsets = d_offsets;
    P.shapes = d_shapes;
    P.thresholds = d_thresholds;
    P.n = n;
    for (int k = 0; k < 9; ++k) P.blur[k] = blur3x3[k];
    P.out = d_out;
    P.status = d_status;
    k_preprocess<<<(unsigned)n, kPThreads, 0, (cudaStream_t)stream>>>(P);
    return cuda_check("k_preprocess");
}
