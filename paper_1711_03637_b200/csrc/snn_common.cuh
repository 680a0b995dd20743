// Shared device helpers for the spiking-digit kernels (sm_100a).
//
// All membrane / trace arithmetic uses explicit round-to-nearest intrinsics
// (__dadd_rn, __dmul_rn, ...), which nvcc never contracts into FMA, so every
// elementwise update is the exact float64 operation sequence numpy performs
// in the reference.  The only FMA is the 3x3 stencil, where OpenBLAS's dgemm
// (np.tensordot, network.py:220) is itself a k-ordered FMA chain.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "snn_b200.h"

namespace snn {

constexpr int kSide = SNN_IMAGE_SIDE;
constexpr int kFmap = 26;
constexpr int kNF = SNN_N_FILTERS;
constexpr int kNPos = SNN_N_POSITIONS;
constexpr int kNH = SNN_N_HIDDEN;
constexpr int kNO = SNN_N_OUTPUTS;
constexpr int kTile = SNN_TILE;
constexpr int kMaxTiles = SNN_MAX_TILES;
constexpr unsigned kFull = 0xffffffffu;

// LIF candidate potential, neurons.py:118-121:
//   v_new = max(v + beta*(I - g*(v - E_L)), E_L)   (five rounded ops, then clamp)
__device__ __forceinline__ double lif_candidate(double v, double drive, const snn_lif_t &p) {
    double t = __dsub_rn(v, p.el);
    t = __dmul_rn(p.g, t);
    t = __dsub_rn(drive, t);
    t = __dmul_rn(p.beta, t);
    double vn = __dadd_rn(v, t);
    return vn < p.el ? p.el : vn;  // np.maximum for finite operands
}

// First step at which a neuron that spiked at `step` is live again:
// live <=> step' > step + t_ref/dt in float64 (neurons.py:113)
//      <=> step' >= floor(step + refr) + 1.
__device__ __forceinline__ int next_live_step(int step, double refr) {
    return (int)floor(__dadd_rn((double)step, refr)) + 1;
}

// numpy's pairwise add-reduce for exactly 10 float64 values (c_out.sum()).
__device__ __forceinline__ double pairwise10(const double *x) {
    double r = __dadd_rn(__dadd_rn(__dadd_rn(x[0], x[1]), __dadd_rn(x[2], x[3])),
                         __dadd_rn(__dadd_rn(x[4], x[5]), __dadd_rn(x[6], x[7])));
    r = __dadd_rn(r, x[8]);
    return __dadd_rn(r, x[9]);
}

__device__ __forceinline__ double ldcg(const double *p) { return __ldcg(p); }

}  // namespace snn
