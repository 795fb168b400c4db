// l2pass.cuh — step a2 for L2-resident tensors (C1–C4: X ≤ 48 MB stays in the 126 MB L2
// between passes): β(a,j) = Σ M·X, ω(a,j) = Σ M² of block (k,i) (Prop. 1 + Eq. 8, P:L224-243,
// P:L301-314; same arithmetic as fiber_walk.cuh) computed per KEPT VALUE v instead of per
// fibre range, so every CTA owns whole outputs: no partial-slot array, no second-stage reduce
// kernel (the HBM-streaming walk of fiber_walk.cuh cuts X into one contiguous range per warp,
// which for these sizes is ~1 stage per warp and leaves one partial per (warp, v) to reduce).
//
// A CTA (8 warps) handles `vpc` kept values with `wpv` warps each (vpc·wpv = 8); the warps of
// one v split its fibres r (the reduced outer indices, odometer order); Z CTAs per v split
// them further when there are too few v to fill the GPU — their partials (fp64) are summed
// in z order by the last CTA of v to arrive (deterministic).  Per fibre, with the outer
// indices i_q held by lane q (shuffled):
//     M(i_0) = s · Π_{q ∈ vec} H_{0,q}(i_0, i_q),  s = Π_{outer pairs {p,q} ≠ {k,i}} H_{p,q}(i_p, i_q)
// (vec = the outer modes other than the kept lane-pair partner; H_{0,q} columns are contiguous
// and zero on the pad rows, so pads weigh 0).  Loads are 16-B vectors straight from L2/L1.
//   KEPT1 (pair {0,m}): v = i_m, per-lane fp32 accumulators over the warp's fibres, fp64
//                        across warps and CTAs; outputs β(:, v) (I_1 values).
//   RED1  ({k,i} outer): v = (i_k, i_i), per-fibre fp32 lane partials summed in fp64.
#pragma once

#include "common.cuh"

namespace ifctn {

template <typename T>
struct L2Params {
    const T* X;
    const T* H;
    double* beta;
    double* omega;
    int I1, I1p, N;
    int64_t Ii, Ik;
    int kept1, kIsMode0;   // KEPT1: k == 0 (j = i_0, a = v) else (a = i_0, j = v)
    int m;                 // KEPT1: the kept outer mode; RED1: -1
    int k, i;              // RED1: v = i_k + I_k·i_i
    int64_t NV, FR, FRz;   // kept values, fibres per v, fibres per (v, z)
    int vpc, wpv, Z;
    int64_t fstride[MAXN];
    int nr;                // reduced outer modes (odometer, first fastest)
    int rmode[MAXN];
    int64_t rdim[MAXN];
    int nvec;              // vector factors H_{0,q}(:, i_q)
    int64_t vec_off[MAXN];
    int vec_mode[MAXN];
    int npair;             // scalar factors H_{p,q}(i_p, i_q), 1 ≤ p < q
    int64_t pair_off[MAXP], pair_ld[MAXP];
    int pair_p[MAXP], pair_q[MAXP];
    double* scr;           // Z > 1: NV·Z·(KEPT1 ? I1p : 1)·2 partials
    unsigned* cnt;         // Z > 1: NV arrival counters, zero between launches
};

constexpr int kL2Threads = 256;

// NCH: 16-byte chunks per lane (I1p ≤ 32·NCH·16/sizeof(T))
template <typename T, bool KEPT, int NCH>
__global__ void __launch_bounds__(kL2Threads) l2_contract(const __grid_constant__ L2Params<T> P) {
    constexpr int VE = 16 / (int)sizeof(T);  // elements per 16-byte chunk
    constexpr int NE = NCH * VE;             // elements per lane
    extern __shared__ __align__(16) double l2sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int vloc = warp / P.wpv, wv = warp % P.wpv;
    const int64_t v = (int64_t)blockIdx.x * P.vpc + vloc;
    const int z = blockIdx.y;
    const int I1p = P.I1p;
    bool ev[NCH];
#pragma unroll
    for (int c = 0; c < NCH; ++c) ev[c] = (c * 32 + lane) * VE < I1p;

    T sb[NE], sw[NE];  // KEPT1: per-element accumulators
#pragma unroll
    for (int e = 0; e < NE; ++e) sb[e] = sw[e] = T(0);
    double tb = 0.0, tw = 0.0;  // RED1
    // kept indices of v (lane q holds i_q)
    int kidx = 0;
    if (v < P.NV) {
        if (KEPT) {
            if (lane == P.m) kidx = (int)v;
        } else {
            if (lane == P.k) kidx = (int)(v % P.Ik);
            if (lane == P.i) kidx = (int)(v / P.Ik);
        }
    }
    const int64_t r0 = (int64_t)z * P.FRz, r1 = min(P.FR, r0 + P.FRz);
    for (int64_t r = r0 + wv; v < P.NV && r < r1; r += P.wpv) {
        // outer indices of fibre (v, r): lane q holds i_q
        int midx = kidx;
        {
            int rr = (int)r;
#pragma unroll
            for (int j = 0; j < MAXN; ++j)
                if (j < P.nr) {
                    const int rd = (int)P.rdim[j];
                    const int d = rr % rd;
                    rr /= rd;
                    if (lane == P.rmode[j]) midx = d;
                }
        }
        auto idx = [&](int q) { return __shfl_sync(0xffffffffu, midx, q); };
        int64_t f = 0;
        for (int q = 1; q < P.N; ++q) f += (int64_t)idx(q) * P.fstride[q];
        T sv[MAXP];  // all scalar loads in flight before the product
#pragma unroll
        for (int t = 0; t < MAXP; ++t)
            sv[t] = t < P.npair ? P.H[P.pair_off[t] + (int64_t)idx(P.pair_q[t]) * P.pair_ld[t] + idx(P.pair_p[t])] : T(1);
        T s = T(1);
#pragma unroll
        for (int t = 0; t < MAXP; ++t) s *= sv[t];
        const T* xf = P.X + f * I1p;
        const T* hc[MAXN];
#pragma unroll
        for (int t = 0; t < MAXN; ++t) hc[t] = P.H;
#pragma unroll
        for (int t = 0; t < MAXN; ++t)
            if (t < P.nvec) hc[t] = P.H + P.vec_off[t] + (int64_t)idx(P.vec_mode[t]) * I1p;
        T pb = T(0), pw = T(0);
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
            if (!ev[c]) continue;
            const int e0 = (c * 32 + lane) * VE;
            const float4 xq = *reinterpret_cast<const float4*>(xf + e0);
            const T* x = reinterpret_cast<const T*>(&xq);
            T w[VE];
#pragma unroll
            for (int u = 0; u < VE; ++u) w[u] = s;
#pragma unroll
            for (int t = 0; t < MAXN; ++t) {
                if (t < P.nvec) {
                    const float4 hq = *reinterpret_cast<const float4*>(hc[t] + e0);
                    const T* h = reinterpret_cast<const T*>(&hq);
#pragma unroll
                    for (int u = 0; u < VE; ++u) w[u] *= h[u];
                }
            }
#pragma unroll
            for (int u = 0; u < VE; ++u) {
                if (KEPT) {
                    sb[c * VE + u] = fma(w[u], x[u], sb[c * VE + u]);
                    sw[c * VE + u] = fma(w[u], w[u], sw[c * VE + u]);
                } else {
                    pb = fma(w[u], x[u], pb);
                    pw = fma(w[u], w[u], pw);
                }
            }
        }
        if (!KEPT) {
            tb += (double)pb;
            tw += (double)pw;
        }
    }
    // ---- combine the wpv warps of each v (fixed order), then the Z CTAs of v ------------
    __shared__ unsigned last;
    if constexpr (KEPT) {
        // l2sm: [8 warps][2][I1p] doubles
        double* mine = l2sm + (size_t)warp * 2 * I1p;
#pragma unroll
        for (int c = 0; c < NCH; ++c)
#pragma unroll
            for (int u = 0; u < VE; ++u) {
                const int e = (c * 32 + lane) * VE + u;
                if (e < I1p) {
                    mine[e] = (double)sb[c * VE + u];
                    mine[I1p + e] = (double)sw[c * VE + u];
                }
            }
        __syncthreads();
        // thread t: element e of v-local slot vl
        const int per = I1p;
        for (int q = threadIdx.x; q < P.vpc * per; q += blockDim.x) {
            const int vl = q / per, e = q - vl * per;
            const int64_t vv = (int64_t)blockIdx.x * P.vpc + vl;
            if (vv >= P.NV) continue;
            double b = 0.0, w = 0.0;
            for (int u = 0; u < P.wpv; ++u) {
                const double* src = l2sm + (size_t)(vl * P.wpv + u) * 2 * I1p;
                b += src[e];
                w += src[I1p + e];
            }
            if (P.Z == 1) {
                if (e < P.I1) {
                    const int64_t o = P.kIsMode0 ? ((int64_t)e * P.Ii + vv) : (vv * P.Ii + e);
                    P.beta[o] = b;
                    P.omega[o] = w;
                }
            } else {
                double* dst = P.scr + ((vv * P.Z + z) * I1p + e) * 2;
                dst[0] = b;
                dst[1] = w;
            }
        }
    } else {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            tb += __shfl_xor_sync(0xffffffffu, tb, o);
            tw += __shfl_xor_sync(0xffffffffu, tw, o);
        }
        if (lane == 0) {
            l2sm[2 * warp] = tb;
            l2sm[2 * warp + 1] = tw;
        }
        __syncthreads();
        if ((int)threadIdx.x < P.vpc) {
            const int vl = threadIdx.x;
            const int64_t vv = (int64_t)blockIdx.x * P.vpc + vl;
            if (vv < P.NV) {
                double b = 0.0, w = 0.0;
                for (int u = 0; u < P.wpv; ++u) {
                    b += l2sm[2 * (vl * P.wpv + u)];
                    w += l2sm[2 * (vl * P.wpv + u) + 1];
                }
                if (P.Z == 1) {
                    const int64_t o = (vv % P.Ik) * P.Ii + vv / P.Ik;  // j = i_k, a = i_i
                    P.beta[o] = b;
                    P.omega[o] = w;
                } else {
                    P.scr[(vv * P.Z + z) * 2] = b;
                    P.scr[(vv * P.Z + z) * 2 + 1] = w;
                }
            }
        }
    }
    if (P.Z == 1) return;
    // Z > 1 (one v per CTA): the last CTA of v to arrive sums the Z partials in z order
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = (atomicAdd(P.cnt + v, 1u) == (unsigned)(P.Z - 1)) ? 1u : 0u;
    __syncthreads();
    if (!last || v >= P.NV) return;
    __threadfence();
    const int per = KEPT ? I1p : 1;
    for (int e = threadIdx.x; e < per; e += blockDim.x) {
        double b = 0.0, w = 0.0;
        for (int zz = 0; zz < P.Z; ++zz) {
            const double* src = P.scr + ((v * P.Z + zz) * per + e) * 2;
            b += __ldcg(src);
            w += __ldcg(src + 1);
        }
        if (KEPT) {
            if (e < P.I1) {
                const int64_t o = P.kIsMode0 ? ((int64_t)e * P.Ii + v) : (v * P.Ii + e);
                P.beta[o] = b;
                P.omega[o] = w;
            }
        } else {
            const int64_t o = (v % P.Ik) * P.Ii + v / P.Ik;
            P.beta[o] = b;
            P.omega[o] = w;
        }
    }
    if (threadIdx.x == 0) P.cnt[v] = 0u;
}

}  // namespace ifctn
