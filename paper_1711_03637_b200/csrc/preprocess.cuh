// Canvas preprocessing on the GPU (SURVEY 8(f) "GPU preprocess"): a
// user-drawn grayscale canvas -> the 28x28 image the network takes, exactly
// as the reference's preprocess_pipeline
// (/root/reference/pkg/src/spikedigits/preprocess.py:110-115):
//   binarize (:31-35)  ->  crop to the ink's bounding box (:38-45)  ->  ink
//   255/0  ->  resize, longer side 20 (:48-63; Pillow BILINEAR on 8-bit
//   data: separable fixed-point passes, 22 fractional bits, restated from
//   libImaging/Resample.c)  ->  place by centre of mass in 28x28 (:66-90)  ->
//   normalised 3x3 Gaussian blur, rint, clip (:93-107).
// One CTA per canvas; canvases of any size up to 1024 x 1024.  Integer and
// fixed-point steps are exact; the centroid and the blur use the reference's
// float64 operation order, so outputs are bit-identical (oracle/
// preprocess_oracle.py, tests/golden/canvases.npz).
#pragma once

#include "snn_common.cuh"

namespace snn {

constexpr int kPThreads = 256;
constexpr int kPMaxSide = 1024;
constexpr int kPContent = 20;
constexpr int kPPrec = 22;  // Pillow's PRECISION_BITS for 8-bit data
constexpr int kPMaxTaps = 2 * kPMaxSide + 3 * kPContent + 64;  // sum over outputs of 2*ceil(support)+1

struct PreArgs {
    const uint8_t *pixels;    // all canvases, row-major, back to back
    const int64_t *offsets;   // [n] start of each canvas in pixels
    const int32_t *shapes;    // [n][2] (height, width)
    const int32_t *thresholds;  // [n]
    int64_t n;
    double blur[9];           // preprocess.py:93-96, computed on the host with numpy
    uint8_t *out;             // [n][28][28]
    int32_t *status;          // [n] 0 ok, 1 blank drawing, 2 bad shape
};

struct PreSmem {
    int box[4];                         // r0, r1, c0, c1 (half-open)
    int nb[2];                          // new_h, new_w
    int bounds[2][kPContent][2];        // per pass and output index: xmin, xmax
    int koff[2][kPContent + 1];         // start of each output index's taps in kk
    int kk[2][kPMaxTaps];               // fixed-point taps
    uint8_t tmp[kPMaxSide * kPContent]; // after the horizontal pass: [rows][new_w]
    uint8_t img[kPContent * kPContent]; // resized: [new_h][new_w]
    uint8_t placed[28 * 28];
    long long mass[3];                  // total, sum rowsum*r, sum colsum*c
};

// Resample.c precompute_coeffs + normalize_coeffs_8bpc (bilinear filter) for
// output index xx of an in -> out pass; written into S by one thread.
__device__ void pre_coeffs(int in, int out, int xx, int *bounds, int *kk) {
    const double scale = (double)in / (double)out;
    const double filterscale = scale > 1.0 ? scale : 1.0;
    const double support = filterscale, ss = 1.0 / filterscale;
    const double center = ((double)xx + 0.5) * scale;
    int xmin = (int)(center - support + 0.5);
    if (xmin < 0) xmin = 0;
    int xmax = (int)(center + support + 0.5);
    if (xmax > in) xmax = in;
    xmax -= xmin;
    double ww = 0.0;
    for (int x = 0; x < xmax; ++x) {
        double t = ((double)(x + xmin) - center + 0.5) * ss;
        if (t < 0.0) t = -t;
        ww += t < 1.0 ? 1.0 - t : 0.0;
    }
    for (int x = 0; x < xmax; ++x) {
        double t = ((double)(x + xmin) - center + 0.5) * ss;
        if (t < 0.0) t = -t;
        double w = t < 1.0 ? 1.0 - t : 0.0;
        if (ww != 0.0) w /= ww;
        kk[x] = w < 0 ? (int)(-0.5 + w * (double)(1 << kPPrec)) : (int)(0.5 + w * (double)(1 << kPPrec));
    }
    bounds[0] = xmin;
    bounds[1] = xmax;
}

__device__ __forceinline__ uint8_t clip8(int acc) {
    const int v = acc >> kPPrec;
    return (uint8_t)(v < 0 ? 0 : v > 255 ? 255 : v);
}

__global__ void __launch_bounds__(kPThreads) k_preprocess(const PreArgs P) {
    __shared__ PreSmem S;
    const int tid = threadIdx.x;
    const int64_t i = blockIdx.x;
    const int H = P.shapes[2 * i], Wd = P.shapes[2 * i + 1];
    uint8_t *out = P.out + i * 784;
    if (H < 1 || Wd < 1 || H > kPMaxSide || Wd > kPMaxSide) {
        for (int t = tid; t < 784; t += kPThreads) out[t] = 0;
        if (tid == 0) P.status[i] = 2;
        return;
    }
    const uint8_t *cv = P.pixels + P.offsets[i];
    const int thr = P.thresholds[i];
    if (tid == 0) {
        S.box[0] = H;
        S.box[1] = -1;
        S.box[2] = Wd;
        S.box[3] = -1;
    }
    __syncthreads();
    // ---- bounding box of the ink (pixels >= threshold)
    {
        int r0 = H, r1 = -1, c0 = Wd, c1 = -1;
        for (int p = tid; p < H * Wd; p += kPThreads)
            if (cv[p] >= thr) {
                const int r = p / Wd, c = p - r * Wd;
                r0 = min(r0, r);
                r1 = max(r1, r);
                c0 = min(c0, c);
                c1 = max(c1, c);
            }
        if (r1 >= 0) {
            atomicMin(&S.box[0], r0);
            atomicMax(&S.box[1], r1);
            atomicMin(&S.box[2], c0);
            atomicMax(&S.box[3], c1);
        }
    }
    __syncthreads();
    if (S.box[1] < 0) {  // BlankDrawingError
        for (int t = tid; t < 784; t += kPThreads) out[t] = 0;
        if (tid == 0) P.status[i] = 1;
        return;
    }
    const int r0 = S.box[0], c0 = S.box[2];
    const int ch = S.box[1] + 1 - r0, cw = S.box[3] + 1 - c0;
    // preprocess.py:56-61: the longer side -> 20, the other rounded, >= 1
    int nh, nw;
    if (ch >= cw) {
        nh = kPContent;
        nw = max(1, (int)floor((double)(cw * kPContent) / (double)ch + 0.5));
    } else {
        nw = kPContent;
        nh = max(1, (int)floor((double)(ch * kPContent) / (double)cw + 0.5));
    }
    const bool hpass = nw != cw, vpass = nh != ch;
    // ---- taps: one thread per output index of each pass
    if (tid == 0) {  // tap offsets (each output index spans at most 2*support+1 inputs)
        int o = 0;
        for (int xx = 0; xx <= nw; ++xx) {
            S.koff[0][xx] = o;
            if (xx < nw) o += (int)ceil((double)cw / nw > 1.0 ? (double)cw / nw : 1.0) * 2 + 1;
        }
        o = 0;
        for (int yy = 0; yy <= nh; ++yy) {
            S.koff[1][yy] = o;
            if (yy < nh) o += (int)ceil((double)ch / nh > 1.0 ? (double)ch / nh : 1.0) * 2 + 1;
        }
    }
    __syncthreads();
    if (hpass && tid < nw) pre_coeffs(cw, nw, tid, S.bounds[0][tid], S.kk[0] + S.koff[0][tid]);
    if (vpass && tid >= 32 && tid - 32 < nh) pre_coeffs(ch, nh, tid - 32, S.bounds[1][tid - 32], S.kk[1] + S.koff[1][tid - 32]);
    __syncthreads();
    // ---- horizontal pass on the ink (255 where >= threshold) -> tmp[ch][nw]
    for (int t = tid; t < ch * nw; t += kPThreads) {
        const int r = t / nw, xx = t - r * nw;
        const uint8_t *row = cv + (size_t)(r0 + r) * Wd + c0;
        if (hpass) {
            const int xmin = S.bounds[0][xx][0], xmax = S.bounds[0][xx][1];
            const int *k = S.kk[0] + S.koff[0][xx];
            int acc = 1 << (kPPrec - 1);
            for (int x = 0; x < xmax; ++x) acc += (row[xmin + x] >= thr ? 255 : 0) * k[x];
            S.tmp[t] = clip8(acc);
        } else {
            S.tmp[t] = row[xx] >= thr ? 255 : 0;
        }
    }
    __syncthreads();
    // ---- vertical pass -> img[nh][nw]
    for (int t = tid; t < nh * nw; t += kPThreads) {
        const int yy = t / nw, xx = t - yy * nw;
        if (vpass) {
            const int ymin = S.bounds[1][yy][0], ymax = S.bounds[1][yy][1];
            const int *k = S.kk[1] + S.koff[1][yy];
            int acc = 1 << (kPPrec - 1);
            for (int y = 0; y < ymax; ++y) acc += (int)S.tmp[(ymin + y) * nw + xx] * k[y];
            S.img[t] = clip8(acc);
        } else {
            S.img[t] = S.tmp[t];
        }
    }
    for (int t = tid; t < 784; t += kPThreads) S.placed[t] = 0;
    if (tid < 3) S.mass[tid] = 0;
    __syncthreads();
    // ---- centre of mass (exact integer sums, as numpy's float64 sums of integers)
    {
        long long tot = 0, rs = 0, cs = 0;
        for (int t = tid; t < nh * nw; t += kPThreads) {
            const int yy = t / nw, xx = t - yy * nw;
            const long long v = S.img[t];
            tot += v;
            rs += v * yy;
            cs += v * xx;
        }
        atomicAdd((unsigned long long *)&S.mass[0], (unsigned long long)tot);
        atomicAdd((unsigned long long *)&S.mass[1], (unsigned long long)rs);
        atomicAdd((unsigned long long *)&S.mass[2], (unsigned long long)cs);
    }
    __syncthreads();
    if (S.mass[0] == 0) {  // preprocess.py:78-79
        for (int t = tid; t < 784; t += kPThreads) out[t] = 0;
        if (tid == 0) P.status[i] = 1;
        return;
    }
    const double total = (double)S.mass[0];
    const double rbar = (double)S.mass[1] / total, cbar = (double)S.mass[2] / total;
    const double center = 13.5;
    const int dr = min(max((int)floor(center - rbar + 0.5), 0), 28 - nh);
    const int dc = min(max((int)floor(center - cbar + 0.5), 0), 28 - nw);
    for (int t = tid; t < nh * nw; t += kPThreads) {
        const int yy = t / nw, xx = t - yy * nw;
        S.placed[(dr + yy) * 28 + dc + xx] = S.img[t];
    }
    __syncthreads();
    // ---- blur (preprocess.py:99-107): out += k[a][b] * padded[..], a-major
    for (int t = tid; t < 784; t += kPThreads) {
        const int r = t / 28, c = t - r * 28;
        double acc = 0.0;
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int b = 0; b < 3; ++b) {
                const int rr = r + a - 1, cc = c + b - 1;
                const double x = (rr >= 0 && rr < 28 && cc >= 0 && cc < 28) ? (double)S.placed[rr * 28 + cc] : 0.0;
                acc = __dadd_rn(acc, __dmul_rn(P.blur[a * 3 + b], x));
            }
        const double v = rint(acc);
        out[t] = (uint8_t)(v < 0.0 ? 0.0 : v > 255.0 ? 255.0 : v);
    }
    if (tid == 0) P.status[i] = 0;
}

}  // namespace snn
