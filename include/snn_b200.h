/*
 * snn_b200.h -- C ABI of the B200-native spiking-digit hot path.
 *
 * Drop-in boundary for the reference package `spikedigits`
 * (/root/reference/pkg/src/spikedigits).  The reference has no FFI: its hot
 * path sits behind Python functions, and each entry point below is what the
 * Python API mirror (paper_1711_03637_b200/) binds through ctypes to replace
 * one of them (see INTEGRATION.md for the bindings):
 *
 *   snn_input_table  <- network._input_tables           (network.py:224-245)
 *   snn_infer        <- network.run_presentation         (network.py:267-326)
 *                       network.forward_pass             (network.py:329-346)
 *                       evaluate.batch_counts            (evaluate.py:27-40)
 *   snn_train        <- normad.train_presentation        (normad.py:141-162)
 *                       normad.train_epoch               (normad.py:179-207)
 *
 * Conventions: all array pointers are DEVICE pointers owned by the caller;
 * `stream` is a cudaStream_t (NULL = legacy default stream).  Calls are
 * asynchronous on `stream` except where noted.  Arithmetic is IEEE float64
 * in the reference's SI units and operation order.  No torch types cross
 * this boundary.
 */
#ifndef SNN_B200_H
#define SNN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SNN_ABI_VERSION 2

#define SNN_IMAGE_SIDE 28
#define SNN_N_PIXELS 784
#define SNN_N_FILTERS 12
#define SNN_N_POSITIONS 676 /* 26 x 26 valid windows */
#define SNN_N_HIDDEN 8112   /* (row*26+col)*12 + filter, network.py:158 */
#define SNN_N_OUTPUTS 10
#define SNN_TILE 32          /* window positions per warp tile */
#define SNN_MAX_TILES 22     /* ceil(676 / 32) */
#define SNN_RASTER_CHUNK 8   /* steps per raster chunk (512 bytes per tile) */

/* status codes (int return values and d_status[0]) */
#define SNN_OK 0
#define SNN_ENOMEM 12
#define SNN_EINVAL 22
#define SNN_ENONFINITE 1001 /* weight update produced non-finite values (normad.py:122-124) */
#define SNN_ECUDA 1002

/* One LIF population, derived on the host exactly as neurons.lif_step does
 * (neurons.py:109-118): beta = dt*(2 - g*dt/C)/(2*C), refr = t_ref/dt. */
typedef struct snn_lif {
    double g;    /* leak conductance, S */
    double el;   /* rest / reset potential, V */
    double vt;   /* threshold, V */
    double beta; /* RK2 collapsed step factor */
    double refr; /* refractory / dt (float64, compared as step > last + refr) */
} snn_lif_t;

/* Everything the hot path reads from NetworkConfig / FilterBank / LearnConfig.
 * Decay factors are host libm exp() values (neurons.py:148-150, normad.py:82). */
typedef struct snn_consts {
    int32_t n_steps;        /* round(T/dt), network.py:148-150 */
    int32_t desired_period; /* steps between target spikes; 0 = no target (network.py:171-193) */
    double dt;
    double i0, ip;          /* pixel encoding i = i0 + k*ip (network.py:72-77) */
    snn_lif_t lif_in, lif_hid, lif_out;
    double decay_slow;      /* exp(-dt/5 ms)  */
    double decay_fast;      /* exp(-dt/1.25 ms) */
    double decay_learn;     /* exp(-dt/1 ms), normad.py:82 */
    double dhat_scale;      /* dt / C_out, normad.py:83 */
    double inhibition;      /* NetworkConfig.inhibition_weight (A per unit trace) */
    double learning_rate;   /* LearnConfig.learning_rate */
    double norm_eps;        /* LearnConfig.norm_epsilon */
    double taps[12][9];     /* FilterBank.weighted[f].ravel() (filters.py:57-60) */
} snn_consts_t;

/* Optional outputs of snn_infer; every pointer may be NULL except counts.
 * The hidden spike raster is compact and chunked by 8 steps: with
 * C = ceil(N / 8), image i owns the block that starts at byte
 * tile_base[i] * C * 512, laid out [chunk][tile][half][lane][8 steps]; the
 * byte for step chunk*8 + j is the 6-bit spike mask of features
 * half*6 .. half*6+5 of the lane's window (tile_pos); steps >= N read 0.
 * A raster buffer must hold n * 22 * C * 512 bytes (the upper bound). */
typedef struct snn_infer_out {
    int32_t *counts;     /* [n][10] output spike counts */
    uint8_t *raster;     /* compact hidden raster (see above) */
    uint16_t *tile_pos;  /* [n][22][32] window position of each lane (0xFFFF = none) */
    int32_t *n_tiles;    /* [n] tiles (32 active windows each) per image */
    int32_t *tile_base;  /* [n+1] exclusive prefix sum of n_tiles */
    uint16_t *out_raster;/* [n][N] 10-bit output spike masks */
    double *ff;          /* [n][N][10] feed-forward current c_hidden @ W */
    double *v_out;       /* [n][N][10] output membrane after each step */
    double *v_hid;       /* [n][N][8112] hidden membrane after each step (only
                            neurons of active windows are written) */
    int32_t *near_ties;  /* [n] output-layer steps whose threshold decision could
                            differ from the reference's: the output neuron is live
                            and |v - V_T| is within a rigorous bound of the
                            difference between the reference's c_hidden @ W
                            (dgemv, network.py:311) and this library's
                            event-driven sum, propagated through the LIF update
                            (DESIGN.md section 6.1).  0 on an image means its
                            output spikes are provably the reference's. */
    int32_t *hidden_redo;/* [1] windows the guard-band hidden kernel re-simulated
                            in float64; written by the last
                            hidden-layer launch of the call */
} snn_infer_out_t;

int snn_abi_version(void);
const char *snn_last_error(void);

/* Input-layer response table for the 256 pixel levels (replaces the
 * lru-cached network._input_tables).  d_ctab: [N][256] float64 kernel traces;
 * d_spk: [N][256] uint8 spike flags (may be NULL). */
int snn_input_table(const snn_consts_t *c, double *d_ctab, uint8_t *d_spk, void *stream);

/* Bytes of device workspace snn_infer needs for n images. */
size_t snn_infer_workspace(const snn_consts_t *c, int64_t n_images);

/* Batched inference: n independent presentations (uint8 [n][784] images,
 * float64 [8112][10] row-major weights, table from snn_input_table). */
int snn_infer(const snn_consts_t *c, const uint8_t *d_images, int64_t n_images,
              const double *d_weights, const double *d_ctab, const snn_infer_out_t *out,
              void *d_workspace, size_t workspace_bytes, void *stream);

/* Profiling hook: when set, every following snn_infer / snn_train call records
 * `before` (a cudaEvent_t) on its stream just before the fused hidden-layer
 * kernel (k_hidden) and `after` just after it, so a caller can time that
 * kernel alone with cudaEventElapsedTime.  Pass NULLs to disable. */
void snn_profile_events(void *before, void *after);

/* Profiling hook: with n_events >= 6 cudaEvent_t handles, every following
 * un-pipelined inference launch sequence records events[0] before k_prep,
 * [1] after k_prep, [2] after k_tile_scan, [3] after the hidden-layer kernel,
 * [4] after k_gsum and [5] after k_output on its stream, and [6] (optional)
 * between the guard-band hidden kernel and its float64 redo, so the caller can
 * time each kernel of a live call.  NULL / 0 disables. */
void snn_profile_stage_events(void *const *events, int n_events);

/* The tuning and profiling knobs below (snn_set_*, snn_normad_*) apply to the
 * calling thread's CURRENT CUDA device (cudaSetDevice): one process can drive
 * several GPUs with independent settings.  Function attributes and occupancy
 * are likewise cached per device. */

/* Tuning of snn_infer: calls with more than images_per_subbatch images (and
 * no caller-visible raster) are pipelined in sub-batches -- the hidden layer
 * of one sub-batch overlaps the contraction and output layer of the previous
 * one on an internal stream; 0 disables.  hidden_ctas_per_sm caps the
 * persistent k_hidden grid (0 = occupancy limit).  Defaults: 0, 0 (measured:
 * no gain on one B200 -- the persistent k_hidden leaves no room to overlap). */
void snn_set_pipeline(int64_t images_per_subbatch, int hidden_ctas_per_sm);

/* Hidden-layer kernel selection (all give the same raster bits).  Default
 * (enable = 1): with the default bank, a refractory span of 3 steps at every
 * step (t_ref/dt = 3) and N <= 200, the guard-band kernel -- float32 packed
 * pairs with a per-window float64 error bound, windows near a threshold
 * decision re-simulated in float64; otherwise the float64
 * kernel that keeps the whole input table in shared memory (one CTA of 20
 * warps per SM) when N <= 108, else the one that streams the table through a
 * ring.  The guard band is used for batches of >= 256 images (below that
 * the float64 kernel is faster); enable = 5 uses it at any batch size.
 * enable = 3: the float64 table-resident kernel (frozen spike masks)
 * instead of the guard-band kernel; enable = 2: float64 with per-neuron
 * refractory horizons; enable = 0: the float64 ring kernel. */
void snn_set_hidden_resident(int enable);

/* snn_train runs its sequential NormAD chain on a cluster of 8 CTAs that
 * keeps W in distributed shared memory.  enable = 4 (default): the kernel
 * whose output scan of image i+1 runs speculatively during image i's update
 * and is proven or redone (normad_spec.cuh; d_status[3] counts the redone
 * scans), when its shared memory fits, else as 1; 1 or 3: the cluster kernel
 * with the G partials pushed to the leader when its shared memory fits, else
 * pulled (2 forces pulling), else one CTA (0 forces it).  All give the same
 * weights (1-4 bit for bit). */
void snn_set_normad_cluster(int enable);

/* The output layer of batches of >= 256 images uses the lane-distributed
 * step (k_output_dist: each lane owns one inhibition trace; fewer FP64
 * instructions, the kernel is FP64-throughput bound there); enable = 0 forces
 * the replicated-trace step everywhere (same bits). */
void snn_set_output_dist(int enable);

/* Profiling hook: when d_clk (device, int64 [64][16]) is set, the cluster
 * NormAD kernel records clock64() at its phase boundaries for the first 64
 * images of each snn_train call (NULL disables).  Effective only in the
 * profiling build (-DSNN_NORMAD_PROFILE, build.py --profile); a no-op in the
 * product library. */
void snn_normad_phase_clocks(long long *d_clk);

/* Profiling only -- results are WRONG while set: the cluster NormAD kernel
 * skips phases (bit 0 output scan, 1 R adjoint, 2 dW, 3 G partials, 4 G
 * gather) so their cost can be measured by difference.  0 = off (default).
 * Effective only in the profiling build, like snn_normad_phase_clocks. */
void snn_normad_skip(int mask);

/* Images per NormAD launch chunk of an n-image snn_train call; 0 for
 * invalid arguments.  Each chunk runs 6 kernels (prep, tile scan, hidden,
 * compact, shard, NormAD).  When n exceeds one chunk, the first chunk is
 * min(chunk, 64) images and the preparation of chunk k+1 runs on an
 * auxiliary stream during chunk k's NormAD kernel (two workspace buffer
 * sets, see snn_train_workspace). */
int64_t snn_train_chunk(const snn_consts_t *c, int64_t n_images);

/* Bytes of device workspace snn_train needs for n images. */
size_t snn_train_workspace(const snn_consts_t *c, int64_t n_images);

/* Sequential online NormAD over n images in the given order, updating
 * d_weights in place (float64 [8112][10]).  d_counts: [n][10] pre-update
 * output counts.  d_status (int32[4], device): [0] status code, [1] index of
 * the failing image, [2] images completed, [3] output scans the speculative
 * kernel had to redo on the exact sums (telemetry).
 * On SNN_ENONFINITE the weights hold
 * the state before the failing image (the reference raises and discards it). */
int snn_train(const snn_consts_t *c, const uint8_t *d_images, const uint8_t *d_labels,
              int64_t n_images, double *d_weights, const double *d_ctab, int32_t *d_counts,
              int32_t *d_status, void *d_workspace, size_t workspace_bytes, void *stream);

/* Canvas preprocessing (replaces preprocess.preprocess_pipeline,
 * /root/reference/pkg/src/spikedigits/preprocess.py:110-115): n grayscale
 * canvases of any shape up to 1024 x 1024, row-major uint8, back to back in
 * d_pixels (canvas i starts at d_offsets[i], shape d_shapes[2i] x
 * d_shapes[2i+1], ink threshold d_thresholds[i] in 0..255) -> d_out
 * [n][28][28] uint8, bit-identical to the reference (binarize, crop to ink,
 * Pillow BILINEAR resize of the longer side to 20, centre of mass, 3x3
 * Gaussian blur).  blur3x3 (host, 9 doubles) is the reference's normalised
 * kernel.  d_status[i]: 0 ok, 1 blank drawing (BlankDrawingError), 2 shape
 * outside 1..1024.  One CTA per canvas. */
int snn_preprocess(const uint8_t *d_pixels, const int64_t *d_offsets, const int32_t *d_shapes,
                   const int32_t *d_thresholds, int64_t n, const double *blur3x3, uint8_t *d_out,
                   int32_t *d_status, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* SNN_B200_H */
