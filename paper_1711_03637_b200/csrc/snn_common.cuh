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

// ---------------------------------------------------------------------------
// Blackwell async-copy helpers: 1-D TMA bulk copy global -> shared completing
// on an mbarrier (SASS: UBLKCP / SYNCS.*).
namespace snn {

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// dst/src 16-byte aligned, bytes a multiple of 16
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// 16-byte cp.async (LDGSTS) global -> shared, L2 only
__device__ __forceinline__ void cp_async16(void *dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }

__device__ __forceinline__ void cp_async_wait_group1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}

__device__ __forceinline__ int warp_excl_scan_int(int x, int *total) {
    const int lane = threadIdx.x & 31;
    int inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(kFull, inc, o);
        if (lane >= o) inc += y;
    }
    *total = __shfl_sync(kFull, inc, 31);
    return inc - x;
}

}  // namespace snn
