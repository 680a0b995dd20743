// C ABI of the spiking-digit hot path (include/snn_b200.h).  One translation
// unit: the kernels live in hidden.cuh (inference) and normad.cuh (training).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>

#include "normad.cuh"

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

// ---- inference workspace: tile_pos | n_tiles | tile_base | partials (upper bound)
struct InferWS {
    uint16_t *tile_pos;
    int32_t *n_tiles, *tile_base;
    double *partial;
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
    x.tile_base = (int32_t *)take((size_t)(n + 1) * 4);
    x.partial = (double *)take((size_t)n * kMaxTiles * (is_default_bank(*c) ? 1 : 2) * c->n_steps * kNO * 8);
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
    return kMaxTiles * N * kTile * 2 + kMaxTiles * kTile * 2 + 4 + 4 + 4 + kNH * 2 + (kNH + 1) * 4 + cap * 2 +
           (N + 1) * 4 + cap * 2 + N * 8 + kMaxTiles * N * 8;
}

int64_t train_chunk(const snn_consts_t *c, int64_t n) {
    const size_t budget = (size_t)768 << 20;
    int64_t ch = (int64_t)(budget / train_ws_per_image(c));
    ch = std::max<int64_t>(1, std::min<int64_t>(ch, 1024));
    return std::min<int64_t>(ch, std::max<int64_t>(n, 1));
}

size_t train_ws(const snn_consts_t *c, int64_t chunk, TrainWS *out, char *base) {
    const size_t N = c->n_steps, cap = train_evcap(c), n = chunk;
    size_t off = 0;
    auto take = [&](size_t bytes) {
        char *p = base ? base + off : nullptr;
        off += al(bytes);
        return p;
    };
    TrainWS w;
    w.raster = (uint8_t *)take(n * kMaxTiles * N * kTile * 2);
    w.tile_pos = (uint16_t *)take(n * kMaxTiles * kTile * 2);
    w.n_tiles = (int32_t *)take(n * 4);
    w.tile_base = (int32_t *)take((n + 1) * 4);
    w.n_act = (int32_t *)take(n * 4);
    w.act_k = (uint16_t *)take(n * kNH * 2);
    w.act_off = (int32_t *)take(n * (kNH + 1) * 4);
    w.nsp = (uint16_t *)take(n * cap * 2);
    w.step_off = (int32_t *)take(n * (N + 1) * 4);
    w.step_k = (uint16_t *)take(n * cap * 2);
    w.norm = (double *)take(n * N * 8);
    w.wp = (double *)take(n * kMaxTiles * N * 8);
    w.evcap = (int64_t)cap;
    if (out) *out = w;
    return off;
}

cudaEvent_t g_ev_before = nullptr, g_ev_after = nullptr;  // snn_profile_events

int sm_count() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    return sms;
}

// prep -> tile scan -> hidden (persistent) [-> output]; raster etc. in A
template <bool TRACE, bool DEF, bool RASTER, bool GSUM, bool SGN>
int launch_batch(const BatchArgs &A, bool with_output, cudaStream_t st) {
    static int hid_blocks = 0;
    if (!hid_blocks) {
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&hid_blocks, k_hidden<TRACE, DEF, RASTER, GSUM, SGN>,
                                                          kThreads, 0) != cudaSuccess ||
            hid_blocks <= 0)
            hid_blocks = 4;
    }
    int rc;
    const unsigned n = (unsigned)A.n_images;
    k_prep<<<n, kThreads, 0, st>>>(A);
    if ((rc = cuda_check("k_prep"))) return rc;
    k_tile_scan<<<1, 1024, 0, st>>>(A);
    if ((rc = cuda_check("k_tile_scan"))) return rc;
    const int64_t max_groups = (2 * A.n_images * kMaxTiles + kWPC - 1) / kWPC;
    const unsigned grid = (unsigned)std::min<int64_t>((int64_t)hid_blocks * sm_count(), max_groups);
    if (g_ev_before) cudaEventRecord(g_ev_before, st);
    k_hidden<TRACE, DEF, RASTER, GSUM, SGN><<<grid, kThreads, 0, st>>>(A);
    if ((rc = cuda_check("k_hidden"))) return rc;
    if (g_ev_after) cudaEventRecord(g_ev_after, st);
    if (with_output) {
        k_output<<<(n + kOutWarps - 1) / kOutWarps, kOutWarps * 32, kOutSmemBytes, st>>>(A);
        if ((rc = cuda_check("k_output"))) return rc;
    }
    return SNN_OK;
}

// Picks the k_hidden instantiation: TRACE variants always use FP64 compares.
template <bool DEF, bool RASTER, bool GSUM>
int launch_fast(const BatchArgs &A, bool with_output, cudaStream_t st) {
    return signed_lif(A.c) ? launch_batch<false, DEF, RASTER, GSUM, true>(A, with_output, st)
                           : launch_batch<false, DEF, RASTER, GSUM, false>(A, with_output, st);
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
extern "C" const char *snn_last_error(void) { return g_err; }

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
    A.raster = out->raster;
    A.partial = w.partial;
    A.out = *out;
    const bool def = is_default_bank(*c);
    A.items_per_tile = def ? 1 : 2;
    const bool raster = out->raster != nullptr;
    if (out->v_hid) {
        if (raster) return def ? launch_batch<true, true, true, true, false>(A, true, s)
                               : launch_batch<true, false, true, true, false>(A, true, s);
        return def ? launch_batch<true, true, false, true, false>(A, true, s)
                   : launch_batch<true, false, false, true, false>(A, true, s);
    }
    if (raster) return def ? launch_fast<true, true, true>(A, true, s) : launch_fast<false, true, true>(A, true, s);
    return def ? launch_fast<true, false, true>(A, true, s) : launch_fast<false, false, true>(A, true, s);
}

extern "C" size_t snn_train_workspace(const snn_consts_t *c, int64_t n) {
    if (!c || n < 0 || c->n_steps <= 0) return 0;
    return train_ws(c, train_chunk(c, n), nullptr, nullptr);
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
    const NormadCaps caps = normad_caps(c);
    const size_t smem = normad_smem_bytes(c->n_steps, caps);
    if (smem > 220 * 1024) return set_error(SNN_EINVAL, "n_steps too large for the sequential NormAD CTA");
    const int64_t chunk = train_chunk(c, n);
    TrainArgs T;
    memset(&T, 0, sizeof(T));
    const size_t need = train_ws(c, chunk, &T.ws, (char *)d_ws);
    if (!d_ws || ws_bytes < need) return set_error(SNN_ENOMEM, "workspace too small");
    if (cudaFuncSetAttribute(k_normad, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return cuda_check("cudaFuncSetAttribute(k_normad)");
    T.c = *c;
    T.w = d_w;
    T.status = d_status;
    for (int64_t i0 = 0; i0 < n; i0 += chunk) {
        const int64_t cn = std::min(chunk, n - i0);
        BatchArgs A;
        memset(&A, 0, sizeof(A));
        A.c = *c;
        A.images = d_images + i0 * SNN_N_PIXELS;
        A.n_images = cn;
        A.w = d_w;
        A.ctab = d_ctab;
        A.raster = T.ws.raster;
        A.tile_pos = T.ws.tile_pos;
        A.n_tiles = T.ws.n_tiles;
        A.tile_base = T.ws.tile_base;
        A.items_per_tile = is_default_bank(*c) ? 1 : 2;
        if ((rc = is_default_bank(*c) ? launch_fast<true, true, false>(A, false, s)
                                      : launch_fast<false, true, false>(A, false, s)))
            return rc;
        T.n = cn;
        T.first = i0;
        T.labels = d_labels + i0;
        T.counts = d_counts + i0 * kNO;
        k_compact<<<(unsigned)cn, kCThreads, 0, s>>>(T);
        if ((rc = cuda_check("k_compact"))) return rc;
        k_normad<<<1, kTThreads, smem, s>>>(T, caps);
        if ((rc = cuda_check("k_normad"))) return rc;
    }
    return SNN_OK;
}
