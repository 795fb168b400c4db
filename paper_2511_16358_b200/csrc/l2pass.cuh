// l2pass.cuh — step a2 for L2-resident tensors (C1–C4: X ≤ 48 MB stays in the 126 MB L2
// between passes): β(a,j) = Σ M·X, ω(a,j) = Σ M² of block (k,i) (Prop. 1 + Eq. 8, P:L224-243,
// P:L301-314; same arithmetic as fiber_walk.cuh) computed per KEPT VALUE v instead of per
// fibre range, so every CTA owns whole outputs: no partial-slot array, no second-stage reduce
// kernel (the HBM-streaming walk of fiber_walk.cuh cuts X into one contiguous range per warp,
// which for these sizes is ~1 stage per warp and leaves one partial per (warp, v) to reduce).
//
// These passes are bound by L2 latency, not bandwidth (8–35 MB per pass), so both kernels are
// built around memory-level parallelism: a thread decodes U fibres, issues all their X loads
// (16-B vectors, L1-bypassing) and weight-factor loads before the first use, and the work
// split (host: Solver::make_l2) keeps every thread at one or two such rounds with all CTAs
// resident at once.
//
//   l2_kept (pair {0,m}, v = i_m): outputs β(:, v) — I_1 values per v.  A warp is CG chunk
//     lanes × 32/CG fibre lanes: lane (cl, fl) owns the 16-byte chunk cg·CG + cl of mode 1 and
//     walks the fibres r of v with a mixed-radix odometer (no divisions in the loop); per-lane
//     fp32 accumulators, then fp64 across fibre lanes (xor butterfly), warps and — when the
//     fibres of v are split over Z CTAs — the Z partials in z order by the last CTA to arrive
//     (deterministic).  Work item = (v, chunk group): blocks with few kept values (C3's 3-long
//     mode, C4's 4-long mode) still fill the GPU without deep partial sums.
//   l2_red ({k,i} outer, v = (i_k, i_i)): one scalar pair per v.  A warp takes whole fibres
//     (lane = chunk), U fibres in flight; the outer indices live one per lane (lane q holds
//     i_q) and the scalar factors are loaded one per lane and multiplied by a butterfly.
//
// With the outer indices i_q of a fibre,
//     M(i_0) = s · Π_{q ∈ vec} H_{0,q}(i_0, i_q),  s = Π_{outer pairs {p,q} ≠ {k,i}} H_{p,q}(i_p, i_q)
// (vec = the outer modes other than the kept lane-pair partner; H_{0,q} columns are contiguous
// and zero on the pad rows, so pads weigh 0).
#pragma once

#include "common.cuh"

namespace ifctn {

constexpr int MAXRD = MAXN - 2;                  // reduced outer modes of a KEPT block
constexpr int MAXJJ = MAXRD * (MAXRD - 1) / 2;   // pairs of them

template <typename T>
struct L2Params {
    const T* X;
    const T* H;
    double* beta;
    double* omega;
    int I1, I1p, N;
    int64_t Ii, Ik;
    int kept1, kIsMode0;   // KEPT: k == 0 (j = i_0, a = v) else (a = i_0, j = v)
    int m;                 // KEPT: the kept outer mode; RED: -1
    int k, i;              // RED: v = i_k + I_k·i_i
    int64_t NV, FR, FRz;   // kept values, fibres per v, fibres per (v, z)
    int Z;                 // CTAs per v-group along the fibres (grid.y)
    int64_t fstride[MAXN];
    int nr;                // reduced outer modes (odometer, first fastest)
    int rmode[MAXN];
    int rdim[MAXN];
    int rdiv[MAXN];        // Π of the faster reduced dims
    // ---- l2_red: warps per v, v per CTA; vector factors H_{0,q}(:, i_q), scalar factors
    int vpc, wpv;
    int nvec;
    int vec_off[MAXN];
    int npair;             // scalar factors H_{p,q}(i_p, i_q), 1 ≤ p < q
    int pair_off[MAXP], pair_ld[MAXP];
    int pair_p[MAXP], pair_q[MAXP];
    // ---- l2_kept: chunk groups, items (v, cg) per CTA, warps per item
    int CG, NCG, ipc, wpi;
    int64_t kf_stride;     // fibre-index stride of the kept mode m
    int rfs[MAXRD];        // fibre-index stride of reduced mode j
    int rv_off[MAXRD];     // H_{0,rmode[j]}: column i at rv_off + i·I1p
    int ks_off[MAXRD], ks_mv[MAXRD], ks_mj[MAXRD];  // H_{m,rmode[j]}(v, i_j) = H[off + v·mv + i_j·mj]
    int jj_off[MAXJJ], jj_ma[MAXJJ], jj_mb[MAXJJ];  // H_{rmode[j],rmode[j']} = H[off + i_j·ma + i_j'·mb]
    double* scr;           // Z > 1: grid.x·Z·(values per CTA)·2 partials
    unsigned* cnt;         // Z > 1: grid.x arrival counters, zero between launches
};

constexpr int kL2Threads = 256;
constexpr int kL2U = 4;  // fibres in flight per thread (kept) / per warp (red)

// Σ_z scr[z·stride] for z < Z in z order, the loads of 8 partials in flight at a time
__device__ __forceinline__ double l2_zsum(const double* p, int Z, int64_t stride) {
    double s = 0.0;
    for (int z0 = 0; z0 < Z; z0 += 8) {
        double v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = z0 + q < Z ? __ldcg(p + (int64_t)(z0 + q) * stride) : 0.0;
#pragma unroll
        for (int q = 0; q < 8; ++q)
            if (z0 + q < Z) s += v[q];
    }
    return s;
}

// ---- KEPT: pair {0, m}; NR = N − 2 reduced outer modes ----------------------------------------
template <typename T, int NR>
__global__ void __launch_bounds__(kL2Threads) l2_kept(const __grid_constant__ L2Params<T> P) {
    constexpr int VE = 16 / (int)sizeof(T);
    constexpr int U = kL2U;
    using V = typename VecT<T>::V;
    __shared__ double sm[8 * 2 * 32 * VE];  // [warp][β|ω][chunk lane · VE]
    __shared__ unsigned last;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int CG = P.CG, FL = 32 / CG, CGE = CG * VE;
    const int cl = lane & (CG - 1), fl = lane / CG;
    const int il = warp / P.wpi, wi = warp - il * P.wpi;
    const int64_t nitems = P.NV * P.NCG;
    const int64_t item = (int64_t)blockIdx.x * P.ipc + il;
    const bool item_ok = item < nitems;
    const int64_t v = item_ok ? item / P.NCG : 0;
    const int cg = item_ok ? (int)(item - v * P.NCG) : 0;
    const int z = blockIdx.y;
    const int I1p = P.I1p;
    const int e0 = (cg * CG + cl) * VE;
    const bool act = item_ok && e0 < I1p;
    const int slots = P.wpi * FL;  // fibres of the item per step
    const int r0 = (int)(z * P.FRz), r1 = (int)min(P.FR, (int64_t)r0 + P.FRz);
    int r = r0 + wi * FL + fl;

    // odometer digits of r and of the step (mixed radix rdim[0..NR))
    int dg[NR > 0 ? NR : 1], ds[NR > 0 ? NR : 1], dm[NR > 0 ? NR : 1];
    {
        int rr = min(r, (int)P.FR - 1), ss = slots;
#pragma unroll
        for (int j = 0; j < NR; ++j) {
            dm[j] = P.rdim[j];
            dg[j] = rr % dm[j];
            rr /= dm[j];
            ds[j] = ss % dm[j];
            ss /= dm[j];
        }
    }
    const T* __restrict__ Hb = P.H;
    const T* xb = P.X + (v * P.kf_stride) * I1p + e0;
    int ksb[NR > 0 ? NR : 1];
#pragma unroll
    for (int j = 0; j < NR; ++j) ksb[j] = P.ks_off[j] + (int)v * P.ks_mv[j];

    T sb[VE], sw[VE];
#pragma unroll
    for (int e = 0; e < VE; ++e) sb[e] = sw[e] = T(0);

    while (act && r < r1) {
        V xq[U];
        T s[U];
        int ho[U][NR > 0 ? NR : 1];
        bool val[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            val[u] = r + u * slots < r1;
            int f = 0;
            T sc = T(1);
            if (val[u]) {
#pragma unroll
                for (int j = 0; j < NR; ++j) {
                    f += dg[j] * P.rfs[j];
                    ho[u][j] = P.rv_off[j] + dg[j] * I1p + e0;
                    sc *= Hb[ksb[j] + dg[j] * P.ks_mj[j]];
                }
                int t = 0;
#pragma unroll
                for (int j = 0; j < NR; ++j)
#pragma unroll
                    for (int j2 = j + 1; j2 < NR; ++j2, ++t) sc *= Hb[P.jj_off[t] + dg[j] * P.jj_ma[t] + dg[j2] * P.jj_mb[t]];
                xq[u] = ld_stream(reinterpret_cast<const V*>(xb + (int64_t)f * I1p));
            } else {
                xq[u] = zero_v<T>();
#pragma unroll
                for (int j = 0; j < NR; ++j) ho[u][j] = 0;
            }
            s[u] = sc;
            // advance the odometer by one step (digits stay < dm: one conditional subtract)
            int carry = 0;
#pragma unroll
            for (int j = 0; j < NR; ++j) {
                int d = dg[j] + ds[j] + carry;
                carry = (j + 1 < NR && d >= dm[j]) ? 1 : 0;
                dg[j] = d - (carry ? dm[j] : 0);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (!val[u]) continue;
            T x[VE], w[VE];
            VecT<T>::get(xq[u], x);
#pragma unroll
            for (int e = 0; e < VE; ++e) w[e] = s[u];
#pragma unroll
            for (int j = 0; j < NR; ++j) {
                const V hq = *reinterpret_cast<const V*>(Hb + ho[u][j]);
                T h[VE];
                VecT<T>::get(hq, h);
#pragma unroll
                for (int e = 0; e < VE; ++e) w[e] *= h[e];
            }
#pragma unroll
            for (int e = 0; e < VE; ++e) {
                sb[e] = fma(w[e], x[e], sb[e]);
                sw[e] = fma(w[e], w[e], sw[e]);
            }
        }
        r += U * slots;
    }
    // ---- fibre lanes (xor butterfly, fp64), then the item's warps, then the Z CTAs -----------
    double db[VE], dw[VE];
#pragma unroll
    for (int e = 0; e < VE; ++e) {
        db[e] = (double)sb[e];
        dw[e] = (double)sw[e];
    }
    for (int o = CG; o < 32; o <<= 1) {
#pragma unroll
        for (int e = 0; e < VE; ++e) {
            db[e] += __shfl_xor_sync(0xffffffffu, db[e], o);
            dw[e] += __shfl_xor_sync(0xffffffffu, dw[e], o);
        }
    }
    if (fl == 0) {
#pragma unroll
        for (int e = 0; e < VE; ++e) {
            sm[(warp * 2 + 0) * CGE + cl * VE + e] = db[e];
            sm[(warp * 2 + 1) * CGE + cl * VE + e] = dw[e];
        }
    }
    __syncthreads();
    // thread q: item-local il2, β|ω, element el of the chunk group
    const int nout = P.ipc * 2 * CGE;
    auto emit = [&](int q, double val) {
        const int il2 = q / (2 * CGE), rem = q - il2 * 2 * CGE;
        const int bw = rem / CGE, el = rem - bw * CGE;
        const int64_t it2 = (int64_t)blockIdx.x * P.ipc + il2;
        if (it2 >= nitems) return;
        const int64_t v2 = it2 / P.NCG;
        const int e = (int)(it2 - v2 * P.NCG) * CGE + el;
        if (e >= P.I1) return;
        const int64_t o = P.kIsMode0 ? ((int64_t)e * P.Ii + v2) : (v2 * P.Ii + e);
        (bw ? P.omega : P.beta)[o] = val;
    };
    for (int q = threadIdx.x; q < nout; q += kL2Threads) {
        const int il2 = q / (2 * CGE), rem = q - il2 * 2 * CGE;
        double a = 0.0;
        for (int u = 0; u < P.wpi; ++u) a += sm[(il2 * P.wpi + u) * 2 * CGE + rem];
        if (P.Z == 1) emit(q, a);
        else P.scr[((int64_t)blockIdx.x * P.Z + z) * nout + q] = a;
    }
    if (P.Z == 1) return;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = (atomicAdd(P.cnt + blockIdx.x, 1u) == (unsigned)(P.Z - 1)) ? 1u : 0u;
    __syncthreads();
    if (!last) return;
    __threadfence();
    for (int q = threadIdx.x; q < nout; q += kL2Threads)
        emit(q, l2_zsum(P.scr + (int64_t)blockIdx.x * P.Z * nout + q, P.Z, nout));
    if (threadIdx.x == 0) P.cnt[blockIdx.x] = 0u;
}

// ---- RED: kept pair {k,i} both outer; NCH 16-byte chunks per lane ----------------------------
template <typename T, int NCH>
__global__ void __launch_bounds__(kL2Threads) l2_red(const __grid_constant__ L2Params<T> P) {
    constexpr int VE = 16 / (int)sizeof(T);
    constexpr int U = kL2U;
    using V = typename VecT<T>::V;
    __shared__ double sm[16];
    __shared__ unsigned last;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int vloc = warp / P.wpv, wv = warp - vloc * P.wpv;
    const int64_t v = (int64_t)blockIdx.x * P.vpc + vloc;
    const bool v_ok = v < P.NV;
    const int z = blockIdx.y;
    const int I1p = P.I1p;
    bool ev[NCH];
#pragma unroll
    for (int c = 0; c < NCH; ++c) ev[c] = (c * 32 + lane) * VE < I1p;
    // lane q holds outer index i_q: kept (fixed by v) or reduced (decoded from r)
    int kidx = 0, my_div = 1, my_dim = 1;
    bool my_red = false;
    if (v_ok) {
        if (lane == P.k) kidx = (int)(v % P.Ik);
        if (lane == P.i) kidx = (int)(v / P.Ik);
    }
#pragma unroll
    for (int j = 0; j < MAXN; ++j)
        if (j < P.nr && lane == P.rmode[j]) {
            my_div = P.rdiv[j];
            my_dim = P.rdim[j];
            my_red = true;
        }
    // lane t < npair loads scalar factor t
    const bool my_pair = lane < P.npair;
    const int pl = my_pair ? lane : 0;
    const int my_pp = P.pair_p[pl], my_pq = P.pair_q[pl], my_poff = P.pair_off[pl], my_pld = P.pair_ld[pl];
    const T* __restrict__ Hb = P.H;
    double tb = 0.0, tw = 0.0;
    const int r0 = (int)(z * P.FRz), r1 = (int)min(P.FR, (int64_t)r0 + P.FRz);
    for (int rb = r0 + wv; v_ok && rb < r1; rb += U * P.wpv) {
        V xq[U][NCH];
        T s[U];
        int ho[U][MAXN - 1];
        bool val[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int r = rb + u * P.wpv;
            val[u] = r < r1;
            const int rr = val[u] ? r : rb;
            const int midx = my_red ? (int)(((unsigned)rr / (unsigned)my_div) % (unsigned)my_dim) : kidx;
            int f = 0;
#pragma unroll
            for (int q = 1; q < MAXN; ++q) {
                ho[u][q - 1] = 0;
                if (q < P.N) {
                    const int iq = __shfl_sync(0xffffffffu, midx, q);
                    f += iq * (int)P.fstride[q];
                    ho[u][q - 1] = P.vec_off[q - 1] + iq * I1p;
                }
            }
            const int ip = __shfl_sync(0xffffffffu, midx, my_pp);
            const int iq2 = __shfl_sync(0xffffffffu, midx, my_pq);
            s[u] = my_pair ? Hb[my_poff + iq2 * my_pld + ip] : T(1);
            const T* xf = P.X + (int64_t)f * I1p;
#pragma unroll
            for (int c = 0; c < NCH; ++c)
                xq[u][c] = (ev[c] && val[u]) ? ld_stream(reinterpret_cast<const V*>(xf + (c * 32 + lane) * VE)) : zero_v<T>();
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) s[u] *= __shfl_xor_sync(0xffffffffu, s[u], o);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (!val[u]) continue;
            T pb = T(0), pw = T(0);
#pragma unroll
            for (int c = 0; c < NCH; ++c) {
                if (!ev[c]) continue;
                const int e0 = (c * 32 + lane) * VE;
                T x[VE], w[VE];
                VecT<T>::get(xq[u][c], x);
#pragma unroll
                for (int e = 0; e < VE; ++e) w[e] = s[u];
#pragma unroll
                for (int t = 0; t < MAXN - 1; ++t) {
                    if (t < P.nvec) {
                        const V hq = *reinterpret_cast<const V*>(Hb + ho[u][t] + e0);
                        T h[VE];
                        VecT<T>::get(hq, h);
#pragma unroll
                        for (int e = 0; e < VE; ++e) w[e] *= h[e];
                    }
                }
#pragma unroll
                for (int e = 0; e < VE; ++e) {
                    pb = fma(w[e], x[e], pb);
                    pw = fma(w[e], w[e], pw);
                }
            }
            tb += (double)pb;
            tw += (double)pw;
        }
    }
    // ---- lanes, then the wpv warps of each v (fixed order), then the Z CTAs -------------------
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        tb += __shfl_xor_sync(0xffffffffu, tb, o);
        tw += __shfl_xor_sync(0xffffffffu, tw, o);
    }
    if (lane == 0) {
        sm[2 * warp] = tb;
        sm[2 * warp + 1] = tw;
    }
    __syncthreads();
    auto emit = [&](int64_t vv, double b, double w) {
        const int64_t o = (vv % P.Ik) * P.Ii + vv / P.Ik;  // j = i_k, a = i_i
        P.beta[o] = b;
        P.omega[o] = w;
    };
    if ((int)threadIdx.x < P.vpc) {
        const int vl = threadIdx.x;
        const int64_t vv = (int64_t)blockIdx.x * P.vpc + vl;
        if (vv < P.NV) {
            double b = 0.0, w = 0.0;
            for (int u = 0; u < P.wpv; ++u) {
                b += sm[2 * (vl * P.wpv + u)];
                w += sm[2 * (vl * P.wpv + u) + 1];
            }
            if (P.Z == 1) {
                emit(vv, b, w);
            } else {
                double* dst = P.scr + (((int64_t)blockIdx.x * P.Z + z) * P.vpc + vl) * 2;
                dst[0] = b;
                dst[1] = w;
            }
        }
    }
    if (P.Z == 1) return;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = (atomicAdd(P.cnt + blockIdx.x, 1u) == (unsigned)(P.Z - 1)) ? 1u : 0u;
    __syncthreads();
    if (!last) return;
    __threadfence();
    if ((int)threadIdx.x < P.vpc) {
        const int vl = threadIdx.x;
        const int64_t vv = (int64_t)blockIdx.x * P.vpc + vl;
        if (vv < P.NV) {
            const double* src = P.scr + ((int64_t)blockIdx.x * P.Z * P.vpc + vl) * 2;
            emit(vv, l2_zsum(src, P.Z, (int64_t)P.vpc * 2), l2_zsum(src + 1, P.Z, (int64_t)P.vpc * 2));
        }
    }
    if (threadIdx.x == 0) P.cnt[blockIdx.x] = 0u;
}

}  // namespace ifctn
