// metrics.cuh — evaluation metrics of the completed tensor:
//   RSE = ‖T − X‖/‖T‖, RMSE over the missing entries Ω^c (T = |Ω^c|), PSNR per band of the
//   last mode (peak 1, averaged over bands), SSIM per band for 3rd-order tensors (11×11
//   Gaussian window σ = 1.5, K1 = 0.01, K2 = 0.03, L = 1, valid windows; images smaller than
//   11 use one uniform full-image window), averaged over windows and bands.
// Deterministic: every sum is per CTA in fixed order, then combined in index order.
#pragma once

#include <math_constants.h>

#include "common.cuh"

namespace ifctn {

constexpr int kMetThreads = 256;

// grid = (chunks, bands): CTA (c, β) sums the fibres [β·fpb + c·chunk, …) of band β (band =
// last mode, so a band is a contiguous fibre range).  part[(β·chunks + c)·5 + ·] =
// [Σ d², Σ t², Σ_{Ω^c} d², |Ω^c|, Σ_band d²] with d = t − x.
template <typename T>
__global__ void __launch_bounds__(kMetThreads) metric_sums(const T* truth, const T* X, const uint32_t* bits,
                                                           int64_t I1, int64_t I1p, int64_t fpb, int64_t chunk,
                                                           double* part) {
    __shared__ double red[5][kMetThreads];
    const int64_t band = blockIdx.y, c = blockIdx.x;
    const int64_t f0 = band * fpb + c * chunk, f1 = min(band * fpb + fpb, f0 + chunk);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
    for (int64_t f = f0 + warp; f < f1; f += nw) {
        for (int64_t i1 = lane; i1 < I1; i1 += 32) {
            const double t = (double)truth[f * I1 + i1];
            const double d = t - (double)X[f * I1p + i1];
            const int64_t e = f * I1p + i1;
            const bool obs = (bits[e >> 5] >> (e & 31)) & 1u;
            s0 = fma(d, d, s0);
            s1 = fma(t, t, s1);
            if (!obs) {
                s2 = fma(d, d, s2);
                s3 += 1.0;
            }
        }
    }
    red[0][threadIdx.x] = s0;
    red[1][threadIdx.x] = s1;
    red[2][threadIdx.x] = s2;
    red[3][threadIdx.x] = s3;
    __syncthreads();
    for (int st = blockDim.x >> 1; st > 0; st >>= 1) {
        if ((int)threadIdx.x < st)
            for (int q = 0; q < 4; ++q) red[q][threadIdx.x] += red[q][threadIdx.x + st];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        double* o = part + (band * gridDim.x + c) * 5;
        o[0] = red[0][0];
        o[1] = red[1][0];
        o[2] = red[2][0];
        o[3] = red[3][0];
        o[4] = red[0][0];  // this band's Σ d² share
    }
}

// SSIM of one 16×16 tile of valid windows of band β (3rd-order tensors; image = modes 1, 2,
// both ≥ 11).  part[β·ntiles + tile] = Σ SSIM over the tile's windows.
constexpr int kSsimTile = 16, kSsimWin = 11;

__device__ __forceinline__ double ssim_value(double mt, double mx, double tt, double xx, double tx) {
    const double C1 = 0.01 * 0.01, C2 = 0.03 * 0.03;
    const double vt = tt - mt * mt, vx = xx - mx * mx, cov = tx - mt * mx;
    return ((2 * mt * mx + C1) * (2 * cov + C2)) / ((mt * mt + mx * mx + C1) * (vt + vx + C2));
}

template <typename T>
__global__ void __launch_bounds__(kSsimTile * kSsimTile) ssim_tiles(const T* truth, const T* X, int64_t I1,
                                                                     int64_t I1p, int64_t I2, int tiles_x,
                                                                     double* part) {
    constexpr int P = kSsimTile + kSsimWin - 1;
    __shared__ double pt[P][P], px[P][P];
    __shared__ double w1[kSsimWin];
    __shared__ double red[kSsimTile * kSsimTile];
    const int64_t band = blockIdx.y;
    const int tile = blockIdx.x;
    const int ty = tile / tiles_x, tx = tile % tiles_x;
    const int64_t o1 = (int64_t)tx * kSsimTile, o2 = (int64_t)ty * kSsimTile;  // first window origin
    const int tid = threadIdx.x;
    if (tid < kSsimWin) {  // normalised 1-D Gaussian, σ = 1.5 (the 2-D window is its outer product)
        double sum = 0.0;
        for (int k = 0; k < kSsimWin; ++k) sum += exp(-(double)((k - 5) * (k - 5)) / (2.0 * 1.5 * 1.5));
        w1[tid] = exp(-(double)((tid - 5) * (tid - 5)) / (2.0 * 1.5 * 1.5)) / sum;
    }
    // patch rows = mode-2 index i2, columns = mode-1 index i1
    for (int e = tid; e < P * P; e += blockDim.x) {
        const int r = e / P, q = e % P;
        const int64_t i1 = o1 + q, i2 = o2 + r;
        double tv = 0.0, xv = 0.0;
        if (i1 < I1 && i2 < I2) {
            tv = (double)truth[(band * I2 + i2) * I1 + i1];
            xv = (double)X[(band * I2 + i2) * I1p + i1];
        }
        pt[r][q] = tv;
        px[r][q] = xv;
    }
    __syncthreads();
    const int wy = tid / kSsimTile, wx = tid % kSsimTile;
    double v = 0.0;
    if (o1 + wx <= I1 - kSsimWin && o2 + wy <= I2 - kSsimWin) {
        double mt = 0, mx = 0, tt = 0, xx = 0, tx2 = 0;
        for (int r = 0; r < kSsimWin; ++r)
            for (int q = 0; q < kSsimWin; ++q) {
                const double w = w1[r] * w1[q];
                const double a = pt[wy + r][wx + q], b = px[wy + r][wx + q];
                mt = fma(w, a, mt);
                mx = fma(w, b, mx);
                tt = fma(w, a * a, tt);
                xx = fma(w, b * b, xx);
                tx2 = fma(w, a * b, tx2);
            }
        v = ssim_value(mt, mx, tt, xx, tx2);
    }
    red[tid] = v;
    __syncthreads();
    for (int st = blockDim.x >> 1; st > 0; st >>= 1) {
        if (tid < st) red[tid] += red[tid + st];
        __syncthreads();
    }
    if (tid == 0) part[band * gridDim.x + tile] = red[0];
}

// Images smaller than the window (a spatial size < 11): one uniform window over the whole
// band image.  part[β] = SSIM of band β.
template <typename T>
__global__ void __launch_bounds__(256) ssim_whole(const T* truth, const T* X, int64_t I1, int64_t I1p,
                                                  int64_t I2, double* part) {
    __shared__ double red[5][256];
    const int64_t band = blockIdx.x;
    double m[5] = {0, 0, 0, 0, 0};
    for (int64_t e = threadIdx.x; e < I1 * I2; e += blockDim.x) {
        const int64_t i2 = e / I1, i1 = e - i2 * I1;
        const double a = (double)truth[(band * I2 + i2) * I1 + i1];
        const double b = (double)X[(band * I2 + i2) * I1p + i1];
        m[0] += a;
        m[1] += b;
        m[2] += a * a;
        m[3] += b * b;
        m[4] += a * b;
    }
    for (int q = 0; q < 5; ++q) red[q][threadIdx.x] = m[q];
    __syncthreads();
    for (int st = blockDim.x >> 1; st > 0; st >>= 1) {
        if ((int)threadIdx.x < st)
            for (int q = 0; q < 5; ++q) red[q][threadIdx.x] += red[q][threadIdx.x + st];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const double n = (double)(I1 * I2);
        part[band] = ssim_value(red[0][0] / n, red[1][0] / n, red[2][0] / n, red[3][0] / n, red[4][0] / n);
    }
}

// Fixed-order combination of the partials of this rank into red[4 + 2·IN] (global band
// indices; bands of other ranks stay 0 so that the all-reduce sums them):
//   red[0..3] = [Σ d², Σ t², Σ_{Ω^c} d², |Ω^c|], red[4 + β] = Σ_band d², red[4 + IN + β] = Σ SSIM.
static __global__ void metric_reduce(const double* part, int64_t chunks, int64_t bl, int64_t boff, int64_t IN,
                              const double* spart, int64_t ntiles, double* red) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    for (int64_t q = 0; q < 4 + 2 * IN; ++q) red[q] = 0.0;
    for (int64_t b = 0; b < bl; ++b) {
        double bs = 0;
        for (int64_t c = 0; c < chunks; ++c) {
            const double* o = part + (b * chunks + c) * 5;
            for (int q = 0; q < 4; ++q) red[q] += o[q];
            bs += o[4];
        }
        red[4 + boff + b] = bs;
        if (spart) {
            double ss = 0;
            for (int64_t t = 0; t < ntiles; ++t) ss += spart[b * ntiles + t];
            red[4 + IN + boff + b] = ss;
        }
    }
}

// fin = [RSE, RMSE on Ω^c (NaN if Ω^c is empty), band-mean PSNR (+inf if a band is exact),
//        mean SSIM (NaN when not computed), Σ t², |Ω^c|]
static __global__ void metric_finish(const double* red, int64_t IN, double band_n, double nwin_total, double* fin) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const double d2 = red[0], t2 = red[1], m2 = red[2], mc = red[3];
    fin[0] = sqrt(d2) / sqrt(t2);
    fin[1] = mc > 0.0 ? sqrt(m2 / mc) : CUDART_NAN;
    double ps = 0.0;
    bool exact = false;
    for (int64_t b = 0; b < IN; ++b) {
        const double mse = red[4 + b] / band_n;
        if (mse > 0.0) ps += 10.0 * log10(1.0 / mse);
        else exact = true;
    }
    fin[2] = exact ? CUDART_INF : ps / (double)IN;
    double ss = 0.0;
    for (int64_t b = 0; b < IN; ++b) ss += red[4 + IN + b];
    fin[3] = nwin_total > 0.0 ? ss / nwin_total : CUDART_NAN;
    fin[4] = t2;
    fin[5] = mc;
}

}  // namespace ifctn
