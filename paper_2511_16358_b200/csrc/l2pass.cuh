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
#include "fiber_walk.cuh"

#include <type_traits>

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
    int rfs[MAXRD];        // fibre-index stride of reduced mode j
    int rfsI[MAXRD];       // the same in elements (· I1p)
    int nb0;               // l2_kept: runs along reduced mode r_0, ⌈rdim[0] / kL2RunU⌉
    int dsr[MAXRD];        // l2_kept: digits of the per-step run stride (radix nb0, rdim[1], …)
    int rv_off[MAXRD];     // H_{0,r_j}: column d at rv_off + d·I1p
    int jj_off[MAXJJ], jj_ma[MAXJJ], jj_mb[MAXJJ];  // H_{r_j,r_j'}(d_j, d_j') = H[off + d_j·ma + d_j'·mb]
    // scalar factors against the kept outer modes: KEPT: H_{m,r_j}(v, d) = H[ks_off + v·ks_mv + d·ks_mj];
    // RED: ks_* for mode k (index j = i_k), is_* for mode i (index a = i_i)
    int ks_off[MAXRD], ks_mv[MAXRD], ks_mj[MAXRD];
    int is_off[MAXRD], is_mv[MAXRD], is_mj[MAXRD];
    // ---- l2_kept: chunk groups, items (v, cg) per CTA, warps per item, table elements per item
    int CG, NCG, ipc, wpi;
    int lcg, lwpi;         // log2 of CG, wpi
    int tab_item;          // shared-memory elements per item: tables V_j, then the scalars A_j
    int asc_item;          // … of which scalars (Σ rdim, rounded up to a 16-byte multiple)
    int64_t kf_stride;     // fibre-index stride of the kept mode m
    // ---- l2_red: team size, H_{0,k} / H_{0,i} offsets
    int TL;
    int pk_off, pi_off;
    double* scr;           // Z > 1: grid.x·Z·(values per CTA)·2 partials
    unsigned* cnt;         // Z > 1: grid.x arrival counters, zero between launches
    // launch-time: bit 0 — the predecessor in the stream is a solve of the same sweep (it waits
    // for ITS predecessor before it lets this grid start, and writes no X), so nothing still
    // running can write X: the first rounds' X loads are issued before pdl_wait().  That solve
    // rewrites one pair matrix H_{k',i'} only; tables built from other pairs are staged before
    // the wait too: l2_kept bit 1+j — V_j (pair {0,r_j}), bit 4+j — A_j (pair {m,r_j});
    // l2_red bit 1 — P_v (pairs {0,k}, {0,i}).
    int x_early;
};

constexpr int kL2Threads = 256;
constexpr int kL2U = 4;  // cells in flight per thread (l2_red; l2_kept: l2_kept_u)
#ifndef IFCTN_L2_RUN_U
#define IFCTN_L2_RUN_U 8
#endif
constexpr int kL2RunU = IFCTN_L2_RUN_U;
#ifndef IFCTN_L2_MINB
#define IFCTN_L2_MINB 2
#endif
// rounds of X loads issued before griddepcontrol.wait (x_early): 2 for third-order tensors, 1 for
// fourth-order ones (A/B: the second round's 32 registers cost C4 188 -> 192 µs per sweep, and
// gain C2 58 -> 56, C2r 133 -> 130)
#ifndef IFCTN_L2_PRE3
#define IFCTN_L2_PRE3 2
#endif
#ifndef IFCTN_L2_PRE4
#define IFCTN_L2_PRE4 1
#endif

// per-thread asynchronous global → shared copies (LDGSTS)
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
template <typename T>
__device__ __forceinline__ void cp_async_scalar(uint32_t dst, const T* src) {
    if constexpr (sizeof(T) == 4) asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
    else asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}

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
// Dynamic shared memory: per item (v, cg) the weight tables of its chunk group,
//   V_j[d][e] = H_{0,r_j}(cg·CGE + e, d) · H_{m,r_j}(v, d),  d < rdim[j], e < CGE,
// so a cell (chunk, fibre) costs one 16-byte X load, NR 16-byte shared-memory reads and the
// NR(NR−1)/2 scalars H_{r_j,r_j'}(d_j, d_j').
template <typename T, int NR>
__global__ void __launch_bounds__(kL2Threads, IFCTN_L2_MINB) l2_kept(const __grid_constant__ L2Params<T> P) {
    constexpr int VE = 16 / (int)sizeof(T);
    constexpr int U = kL2RunU;
    constexpr int NRa = NR > 0 ? NR : 1;
    static_assert(NR >= 1 && NR <= 2, "l2_kept serves orders 3 and 4");
    constexpr int kL2Pre = NR == 1 ? IFCTN_L2_PRE3 : IFCTN_L2_PRE4;
    using V = typename VecT<T>::V;
    extern __shared__ __align__(16) unsigned char l2sm_raw[];
    __shared__ double sm[8 * 2 * 32 * VE];  // [warp][β|ω][chunk lane · VE]
    __shared__ unsigned last;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int CG = P.CG, lcg = P.lcg, FL = 32 >> lcg, CGE = CG * VE;
    const int cl = lane & (CG - 1), fl = lane >> lcg;
    const int il = warp >> P.lwpi, wi = warp - (il << P.lwpi);
    const int nitems = (int)P.NV * P.NCG;  // < 2^31 (host check)
    const int item = (int)blockIdx.x * P.ipc + il;
    const bool item_ok = item < nitems;
    const int v = item_ok ? item / P.NCG : 0;
    const int cg = item_ok ? item - v * P.NCG : 0;
    const int z = blockIdx.y;
    const int I1p = P.I1p;
    const int e0 = (cg * CG + cl) * VE;
    const bool act = item_ok && e0 < I1p;
    const int slots = P.wpi * FL;  // fibres of the item per step
    const int r0 = (int)(z * P.FRz), r1 = (int)min(P.FR, (int64_t)r0 + P.FRz);
    int r = r0 + wi * FL + fl;
    const T* __restrict__ Hb = P.H;

    // A thread's unit of work is a RUN: U consecutive values d0 = b·U + u of reduced mode r_0 (the
    // longest one, host order) at fixed higher digits — everything but the X cell, the V_0 row
    // and the scalars H_{r_0,r_j}(d0, d_j) is per run, and the cell addresses are base + u·stride.
    // Runs are numbered in mixed radix (nb0 = ⌈rdim[0]/U⌉, rdim[1], …) and walked by odometer.
    int dg[NRa], ds[NRa], dm[NRa], tb0[NRa], ab0[NRa];
    {
        int rr = min(r, (int)P.FR - 1), toff = cl * VE, aoff = P.tab_item - P.asc_item;
#pragma unroll
        for (int j = 0; j < NR; ++j) {
            dm[j] = j == 0 ? P.nb0 : P.rdim[j];
            dg[j] = j + 1 < NR ? rr % dm[j] : rr;
            rr /= dm[j];
            ds[j] = P.dsr[j];
            tb0[j] = toff;
            toff += P.rdim[j] * CGE;
            ab0[j] = aoff;
            aoff += P.rdim[j];
        }
    }
    const T* xb = P.X + ((int64_t)v * P.kf_stride) * I1p + e0;
    T* tab = reinterpret_cast<T*>(l2sm_raw) + (size_t)il * P.tab_item;
    const int rdim0 = NR > 0 ? P.rdim[0] : 1;
    const unsigned xst = NR > 0 ? (unsigned)P.rfsI[0] : 0u;  // X elements between cells of a run
    // X cells of the run the odometer stands on
    auto load_run = [&](V (&dst)[U]) {
        const int d0s = dg[0] * U;
        const int nv = min(U, rdim0 - d0s);
        unsigned xo = (unsigned)d0s * xst;
#pragma unroll
        for (int j = 1; j < NR; ++j) xo += (unsigned)(dg[j] * P.rfsI[j]);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            dst[u] = zero_v<T>();
            if (u < nv) dst[u] = ld_stream(reinterpret_cast<const V*>(xb + xo + (unsigned)u * xst));
        }
    };
    // next run of this thread
    auto next_run = [&]() {
        int carry = 0;
#pragma unroll
        for (int j = 0; j < NR; ++j) {
            int d = dg[j] + ds[j] + carry;
            carry = (j + 1 < NR && d >= dm[j]) ? 1 : 0;
            dg[j] = d - (carry ? dm[j] : 0);
        }
    };
    V xpre[kL2Pre][U];
    int npre = 0;
#ifndef IFCTN_EXP_NO_XEARLY
    if (P.x_early && act) {  // X is not written by anything still running (L2Params::x_early)
        int sv[NRa];
#pragma unroll
        for (int j = 0; j < NR; ++j) sv[j] = dg[j];
#pragma unroll
        for (int t = 0; t < kL2Pre; ++t)
            if (r + t * slots < r1) {
                load_run(xpre[t]);
                next_run();
                npre = t + 1;
            }
#pragma unroll
        for (int j = 0; j < NR; ++j) dg[j] = sv[j];
    }
#endif
    // ---- stage the item's tables (its wpi warps): asynchronous global → shared copies (LDGSTS,
    // all in flight at once), V_j[d][·] = H_{0,r_j}(chunk group, d) and A_j[d] = H_{m,r_j}(v, d);
    // phase 1 = the tables the running predecessor does not write (x_early), before the wait
    auto stage_tables = [&](int phase) {
        if (!item_ok) return;
        const int tid = wi * 32 + lane, nt = P.wpi * 32;
        int toff = 0, aoff = P.tab_item - P.asc_item;
#pragma unroll
        for (int j = 0; j < NR; ++j) {
            const int n = P.rdim[j] << lcg;
            if (((P.x_early >> (1 + j)) & 1) == phase)
                for (int q = tid; q < n; q += nt) {
                    const int d = q >> lcg, c2 = q - (d << lcg);
                    const int ee = (cg * CG + c2) * VE;
                    if (ee < I1p) cp_async16(smem_u32(tab + toff + q * VE), Hb + P.rv_off[j] + d * I1p + ee);
                    else *reinterpret_cast<V*>(tab + toff + q * VE) = zero_v<T>();
                }
            if (((P.x_early >> (4 + j)) & 1) == phase) {
                const int ksb = P.ks_off[j] + v * P.ks_mv[j];
                for (int d = tid; d < P.rdim[j]; d += nt) cp_async_scalar<T>(smem_u32(tab + aoff + d), Hb + ksb + d * P.ks_mj[j]);
            }
            toff += n * VE;
            aoff += P.rdim[j];
        }
    };
#ifdef IFCTN_EXP_L2_SKIP_STAGE
    if (P.I1 < 0)
#endif
    if (P.x_early >> 1) stage_tables(1);
    pdl_wait();
    pdl_launch();
#ifdef IFCTN_EXP_L2_SKIP_STAGE
    if (P.I1 < 0)
#endif
    stage_tables(0);
    cp_async_wait_all();
    __syncthreads();

    T sb[VE], sw[VE];
#pragma unroll
    for (int e = 0; e < VE; ++e) sb[e] = sw[e] = T(0);
    // one run; first > 0: its X cells were loaded before the wait (xpre[first − 1])
    auto do_run = [&](auto first) {
        const int d0s = dg[0] * U;
        const int nv = min(U, rdim0 - d0s);
        // loads of the run: X cells and the scalars H_{r_0,r_1}(d0, d_1)
        V xq[U];
        T p[U];
        if constexpr (decltype(first)::value > 0) {
#pragma unroll
            for (int u = 0; u < U; ++u) xq[u] = xpre[decltype(first)::value - 1][u];
        } else {
            load_run(xq);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            p[u] = T(1);
            if constexpr (NR == 2)
                if (u < nv) p[u] = Hb[P.jj_off[0] + (d0s + u) * P.jj_ma[0] + dg[1] * P.jj_mb[0]];
        }
        // run-constant part of the weight: V_1[d_1] · A_1[d_1]
        T bv[VE];
#pragma unroll
        for (int e = 0; e < VE; ++e) bv[e] = T(1);
        if constexpr (NR == 2) {
            T h1[VE];
            VecT<T>::get(*reinterpret_cast<const V*>(tab + tb0[1] + dg[1] * CGE), h1);
            scale<T, VE>(h1, tab[ab0[1] + dg[1]], bv);
        }
        const T* t0 = tab + tb0[0] + d0s * CGE;
        const T* a0 = tab + ab0[0] + d0s;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (u < nv) {
                T x[VE], h[VE], w[VE];
                VecT<T>::get(xq[u], x);
                VecT<T>::get(*reinterpret_cast<const V*>(t0 + u * CGE), h);
                if constexpr (NR == 2) {
                    T bp[VE];
                    scale<T, VE>(bv, p[u] * a0[u], bp);
                    mul<T, VE>(h, bp, w);
                } else {
                    scale<T, VE>(h, a0[u], w);
                }
                accumulate<T, VE>(w, x, sb, sw);
            }
        }
        next_run();
        r += slots;
    };
#ifdef IFCTN_EXP_L2_SKIP_MAIN  // timing experiments only (wrong results): fixed cost of the kernel
    if (P.I1 < 0)
#endif
    {
        if (npre > 0) do_run(std::integral_constant<int, 1>{});
        if constexpr (kL2Pre > 1)
            if (npre > 1) do_run(std::integral_constant<int, 2>{});
        while (act && r < r1) do_run(std::integral_constant<int, 0>{});
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
    const int lce = lcg + (VE == 4 ? 2 : 1);  // log2 CGE
    auto emit = [&](int q, double val) {
        const int il2 = q >> (lce + 1), rem = q - (il2 << (lce + 1));
        const int bw = rem >> lce, el = rem - (bw << lce);
        const int it2 = (int)blockIdx.x * P.ipc + il2;
        if (it2 >= nitems) return;
        const int v2 = it2 / P.NCG;
        const int e = (it2 - v2 * P.NCG) * CGE + el;
        if (e >= P.I1) return;
        const int64_t o = P.kIsMode0 ? ((int64_t)e * P.Ii + v2) : ((int64_t)v2 * P.Ii + e);
        (bw ? P.omega : P.beta)[o] = val;
    };
    for (int q = threadIdx.x; q < nout; q += kL2Threads) {
        const int il2 = q >> (lce + 1), rem = q - (il2 << (lce + 1));
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

// ---- RED: kept pair {k,i} both outer; NRR = N − 3 reduced outer modes -------------------------
// A team of TL threads (8 … 256) owns one v = (i_k, i_i) (one z-share of its fibres): the cells
// (fibre r, 16-byte chunk c) of v are dealt to the team's threads in flat order q = r·NC + c
// (coalesced: consecutive lanes read consecutive chunks), stepped without divisions.  The
// v-constant part of the weight, P_v(i_0) = H_{0,k}(i_0, j)·H_{0,i}(i_0, a), is staged once in
// shared memory per team; per cell: one X load, one shared-memory read, NRR vector loads
// H_{0,r}(c, d) and the scalars of the fibre.  Everything sums into one (β, ω) pair per v:
// per-cell fp32, then fp64 over the thread's cells, the team (xor butterfly, warps in order),
// and the Z CTAs in z order (last CTA to arrive).
template <typename T, int NRR>
__global__ void __launch_bounds__(kL2Threads, IFCTN_L2_MINB) l2_red(const __grid_constant__ L2Params<T> P) {
    constexpr int VE = 16 / (int)sizeof(T);
    constexpr int U = kL2U;
    constexpr int NRa = NRR > 0 ? NRR : 1;
    constexpr int NJJ = NRR * (NRR - 1) / 2;
    constexpr int kL2Pre = NRR == 0 ? IFCTN_L2_PRE3 : IFCTN_L2_PRE4;
    using V = typename VecT<T>::V;
    using A = std::conditional_t<(NRR >= 2), double, T>;  // orders ≥ 5: see l2_kept
    extern __shared__ __align__(16) unsigned char l2sm_raw[];
    __shared__ double sm[16];
    __shared__ unsigned last;
    const int TL = P.TL, tpc = kL2Threads / TL;
    const int team = threadIdx.x / TL, tl = threadIdx.x - team * TL;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t v = (int64_t)blockIdx.x * tpc + team;
    const bool v_ok = v < P.NV;
    const int z = blockIdx.y;
    const int I1p = P.I1p, NC = I1p / VE;
    const int jk = v_ok ? (int)(v % P.Ik) : 0, ai = v_ok ? (int)(v / P.Ik) : 0;
    const T* __restrict__ Hb = P.H;
    // ---- this thread's cells: q = tl + t·TL < ncell ---------------------------------------------
    const int r0 = (int)(z * P.FRz), r1 = (int)min(P.FR, (int64_t)r0 + P.FRz);
    const int ncell = v_ok ? (r1 - r0) * NC : 0;
    int q = tl;
    int c = tl % NC;
    const int dc = TL % NC;
    int dg[NRa], ds[NRa], dm[NRa], kb[NRa], ib[NRa];
    {
        int rr = min(r0 + tl / NC, (int)P.FR - 1), ss = TL / NC;
#pragma unroll
        for (int j = 0; j < NRR; ++j) {
            dm[j] = P.rdim[j];
            dg[j] = rr % dm[j];
            rr /= dm[j];
            ds[j] = ss % dm[j];
            ss /= dm[j];
            kb[j] = P.ks_off[j] + jk * P.ks_mv[j];
            ib[j] = P.is_off[j] + ai * P.is_mv[j];
        }
    }
    const T* xb = P.X + ((int64_t)jk * P.fstride[P.k] + (int64_t)ai * P.fstride[P.i]) * I1p;
    // next cell of this thread: chunk += dc (mod NC), fibre += ⌊TL/NC⌋ + wrap
    auto advance = [&](int& cc, int (&dd)[NRa]) {
        cc += dc;
        int carry = cc >= NC ? 1 : 0;
        cc -= carry ? NC : 0;
#pragma unroll
        for (int j = 0; j < NRR; ++j) {
            int d = dd[j] + ds[j] + carry;
            carry = (j + 1 < NRR && d >= dm[j]) ? 1 : 0;
            dd[j] = d - (carry ? dm[j] : 0);
        }
    };
    auto x_of = [&](int cc, const int (&dd)[NRa]) {
        int f = 0;
#pragma unroll
        for (int j = 0; j < NRR; ++j) f += dd[j] * P.rfs[j];
        return ld_stream(reinterpret_cast<const V*>(xb + (int64_t)f * I1p + cc * VE));
    };
    V xpre[kL2Pre][U];
    int npre = 0;
#ifndef IFCTN_EXP_NO_XEARLY
    if (P.x_early) {  // the first rounds' X cells before the wait (L2Params::x_early)
        int c2 = c, d2[NRa];
#pragma unroll
        for (int j = 0; j < NRa; ++j) d2[j] = j < NRR ? dg[j] : 0;
#pragma unroll
        for (int t = 0; t < kL2Pre; ++t)
            if (q + t * U * TL < ncell) {
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    xpre[t][u] = zero_v<T>();
                    if (q + (t * U + u) * TL < ncell) xpre[t][u] = x_of(c2, d2);
                    advance(c2, d2);
                }
                npre = t + 1;
            }
    }
#endif
    // ---- P_v into shared memory (before the wait when the running solve writes neither pair) ----
    T* pv = reinterpret_cast<T*>(l2sm_raw) + (size_t)team * I1p;
    const bool pv_early = (P.x_early >> 1) & 1;
    if (!pv_early) {
        pdl_wait();
        pdl_launch();
    }
    if (v_ok) {
        const T* hk = Hb + P.pk_off + jk * I1p;
        const T* hi = Hb + P.pi_off + ai * I1p;
        for (int c = tl; c < NC; c += TL) {
            const V a = *reinterpret_cast<const V*>(hk + c * VE);
            const V b = *reinterpret_cast<const V*>(hi + c * VE);
            T x[VE], y[VE];
            VecT<T>::get(a, x);
            VecT<T>::get(b, y);
#pragma unroll
            for (int e = 0; e < VE; ++e) x[e] *= y[e];
            *reinterpret_cast<V*>(pv + c * VE) = VecT<T>::make(x);
        }
    }
    if (pv_early) {
        pdl_wait();
        pdl_launch();
    }
    __syncthreads();
    double tb = 0.0, tw = 0.0;
    auto do_round = [&](auto first) {
        V xq[U], hq[U][NRa];
        A s[U];
        int co[U];
        bool val[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            val[u] = q + u * TL < ncell;
            co[u] = c * VE;
            A sc = A(1);
            if (val[u]) {
                T pvv[2 * NRa + (NJJ > 0 ? NJJ : 1)];
                int t = 0;
#pragma unroll
                for (int j = 0; j < NRR; ++j) {
                    pvv[t++] = Hb[kb[j] + dg[j] * P.ks_mj[j]];
                    pvv[t++] = Hb[ib[j] + dg[j] * P.is_mj[j]];
                }
                int t3 = 0;
#pragma unroll
                for (int j = 0; j < NRR; ++j)
#pragma unroll
                    for (int j2 = j + 1; j2 < NRR; ++j2, ++t3)
                        pvv[t++] = Hb[P.jj_off[t3] + dg[j] * P.jj_ma[t3] + dg[j2] * P.jj_mb[t3]];
#pragma unroll
                for (int j = 0; j < NRR; ++j) hq[u][j] = *reinterpret_cast<const V*>(Hb + P.rv_off[j] + dg[j] * I1p + co[u]);
                if constexpr (decltype(first)::value > 0) xq[u] = xpre[decltype(first)::value - 1][u];
                else xq[u] = x_of(c, dg);
#pragma unroll
                for (int t2 = 0; t2 < 2 * NRR + NJJ; ++t2) sc *= (A)pvv[t2];
            } else {
                xq[u] = zero_v<T>();
#pragma unroll
                for (int j = 0; j < NRR; ++j) hq[u][j] = zero_v<T>();
            }
            s[u] = sc;
            advance(c, dg);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (!val[u]) continue;
            T x[VE], pe[VE];
            A w[VE];
            VecT<T>::get(xq[u], x);
            const V pq = *reinterpret_cast<const V*>(pv + co[u]);
            VecT<T>::get(pq, pe);
#pragma unroll
            for (int e = 0; e < VE; ++e) w[e] = (A)pe[e] * s[u];
#pragma unroll
            for (int j = 0; j < NRR; ++j) {
                T h[VE];
                VecT<T>::get(hq[u][j], h);
#pragma unroll
                for (int e = 0; e < VE; ++e) w[e] *= (A)h[e];
            }
            A pb = A(0), pw = A(0);
#pragma unroll
            for (int e = 0; e < VE; ++e) {
                pb = fma(w[e], (A)x[e], pb);
                pw = fma(w[e], w[e], pw);
            }
            tb += (double)pb;
            tw += (double)pw;
        }
        q += U * TL;
    };
    if (npre > 0) do_round(std::integral_constant<int, 1>{});
    if constexpr (kL2Pre > 1)
        if (npre > 1) do_round(std::integral_constant<int, 2>{});
    while (q < ncell) do_round(std::integral_constant<int, 0>{});
    // ---- the team: lanes (xor butterfly inside the team), its warps in order, then the Z CTAs --
    for (int o = 1; o < 32 && o < TL; o <<= 1) {
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
    // the first lane of every team finishes its v
    if (tl == 0 && v_ok) {
        double b, w;
        if (TL <= 32) {
            b = tb;
            w = tw;
        } else {
            b = w = 0.0;
            const int w0 = threadIdx.x >> 5;
            for (int u = 0; u < TL / 32; ++u) {
                b += sm[2 * (w0 + u)];
                w += sm[2 * (w0 + u) + 1];
            }
        }
        if (P.Z == 1) {
            emit(v, b, w);
        } else {
            double* dst = P.scr + (((int64_t)blockIdx.x * P.Z + z) * tpc + team) * 2;
            dst[0] = b;
            dst[1] = w;
        }
    }
    if (P.Z == 1) return;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = (atomicAdd(P.cnt + blockIdx.x, 1u) == (unsigned)(P.Z - 1)) ? 1u : 0u;
    __syncthreads();
    if (!last) return;
    __threadfence();
    if ((int)threadIdx.x < tpc) {
        const int64_t vv = (int64_t)blockIdx.x * tpc + threadIdx.x;
        if (vv < P.NV) {
            const double* src = P.scr + ((int64_t)blockIdx.x * P.Z * tpc + threadIdx.x) * 2;
            emit(vv, l2_zsum(src, P.Z, (int64_t)tpc * 2), l2_zsum(src + 1, P.Z, (int64_t)tpc * 2));
        }
    }
    if (threadIdx.x == 0) P.cnt[blockIdx.x] = 0u;
}

// ---- a5 for L2-resident tensors: X ← Ω ? X : (t + ρX)/(1+ρ), t = Π_{p<q} H_{p,q} (Eq. 9 in
// reading R1) and the three norms of the sweep row ---------------------------------
// Same cell mapping as l2_kept with every outer mode "reduced": a CTA owns one chunk group of
// mode 1 and a z-share of all fibres; its tables V_q[d][e] = H_{0,q}(cg·CGE + e, d) sit in shared
// memory; per cell one X load, the Ω word, NO table reads, the NO(NO−1)/2 scalars H_{q,q'}, one
// X store.  Norm partials: fp32 per thread (≤ a few rounds), fp64 across lanes and warps in
// fixed order, one row per CTA for finalize_norms.
template <typename T>
struct L2RefillParams {
    T* X;
    const T* H;
    const uint32_t* mask;
    double* norms;        // 3 per CTA (grid.x·z + x)
    T rho, inv1p;
    int I1p;
    int64_t nfib, FRz;
    int CG, lcg, NCG;
    int dim[MAXN - 1];    // outer mode dims, mode order (fibre index = mixed radix, mode 2 fastest)
    int ds[MAXN - 1];     // digits of the per-step fibre stride 8·32/CG
    int tv_off[MAXN - 1]; // H_{0,q}
    int pp_off[MAXP], pp_ld[MAXP];  // H_{q,q'}(i_q, i_q') = H[off + i_q'·ld + i_q], pairs in (q, q') order
    int x_early;          // launch-time, as L2Params::x_early: bit 0 — first rounds' X and Ω loads before
                          // pdl_wait(); bit 1 — the H_{0,q} tables too (the running solve's pair has no mode 0)
};

template <typename T, int NO>
__global__ void __launch_bounds__(kL2Threads, IFCTN_L2_MINB) l2_refill(const __grid_constant__ L2RefillParams<T> P) {
    constexpr int VE = 16 / (int)sizeof(T);
    constexpr int U = kL2U;
    constexpr int NPP = NO * (NO - 1) / 2;
    constexpr int kL2Pre = NO <= 2 ? IFCTN_L2_PRE3 : IFCTN_L2_PRE4;
    using V = typename VecT<T>::V;
    extern __shared__ __align__(16) unsigned char l2sm_raw[];
    __shared__ double sm[8 * 3];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int CG = P.CG, lcg = P.lcg, FL = 32 >> lcg, CGE = CG * VE;
    const int cl = lane & (CG - 1), fl = lane >> lcg;
    const int cg = blockIdx.x, z = blockIdx.y;
    const int I1p = P.I1p;
    const int e0 = (cg * CG + cl) * VE;
    const bool act = e0 < I1p;
    const int slots = 8 * FL;
    const int f0 = (int)(z * P.FRz), f1 = (int)min(P.nfib, (int64_t)f0 + P.FRz);
    int f = f0 + warp * FL + fl;
    const T* __restrict__ Hb = P.H;
    T* tab = reinterpret_cast<T*>(l2sm_raw);
    T* xb = P.X + e0;
    V xpre[kL2Pre][U];
    uint32_t mpre[kL2Pre][U];
    int npre = 0;
#ifndef IFCTN_EXP_NO_XEARLY
    if (P.x_early && act) {
#pragma unroll
        for (int t = 0; t < kL2Pre; ++t)
            if (f + t * U * slots < f1) {
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int fu = f + (t * U + u) * slots;
                    xpre[t][u] = zero_v<T>();
                    mpre[t][u] = ~0u;
                    if (fu < f1) {
                        const unsigned g = (unsigned)fu * (unsigned)I1p + (unsigned)e0;
                        mpre[t][u] = P.mask[g >> 5] >> (g & 31u);
                        xpre[t][u] = *reinterpret_cast<const V*>(xb + (size_t)fu * I1p);
                    }
                }
                npre = t + 1;
            }
    }
#endif
    const bool tab_early = (P.x_early >> 1) & 1;
    if (!tab_early) {
        pdl_wait();
        pdl_launch();
    }
    // tables
    {
        int toff = 0;
#pragma unroll
        for (int q = 0; q < NO; ++q) {
            const int n = P.dim[q] << lcg;
            for (int t = threadIdx.x; t < n; t += kL2Threads) {
                const int d = t >> lcg, c2 = t - (d << lcg);
                const int ee = (cg * CG + c2) * VE;
                if (ee < I1p) cp_async16(smem_u32(tab + toff + t * VE), Hb + P.tv_off[q] + d * I1p + ee);
                else *reinterpret_cast<V*>(tab + toff + t * VE) = zero_v<T>();
            }
            toff += n * VE;
        }
        if (tab_early) {
            pdl_wait();
            pdl_launch();
        }
        cp_async_wait_all();
    }
    int dg[NO], dm[NO], ds[NO], tb0[NO];
    {
        int rr = min(f, (int)P.nfib - 1), toff = cl * VE;
#pragma unroll
        for (int q = 0; q < NO; ++q) {
            dm[q] = P.dim[q];
            ds[q] = P.ds[q];
            dg[q] = q + 1 < NO ? rr % dm[q] : rr;
            rr /= dm[q];
            tb0[q] = toff;
            toff += dm[q] * CGE;
        }
    }
    __syncthreads();
    Norms3<T> qn;
    auto do_round = [&](auto first) {
        V xq[U];
        T s[U];
        uint32_t mw[U];
        int so[U][NO];
        unsigned val = 0;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int fu = f + u * slots;
            const bool ok = fu < f1;
            val |= ok ? (1u << u) : 0u;
            T sc = T(1);
#pragma unroll
            for (int q = 0; q < NO; ++q) so[u][q] = tb0[q] + dg[q] * CGE;
            if (ok) {
                if constexpr (NPP > 0) {
                    T pv[NPP];
                    int t = 0;
#pragma unroll
                    for (int q = 0; q < NO; ++q)
#pragma unroll
                        for (int q2 = q + 1; q2 < NO; ++q2, ++t) pv[t] = Hb[P.pp_off[t] + dg[q2] * P.pp_ld[t] + dg[q]];
#pragma unroll
                    for (int t2 = 0; t2 < NPP; ++t2) sc *= pv[t2];
                }
                if constexpr (decltype(first)::value > 0) {
                    mw[u] = mpre[decltype(first)::value - 1][u];
                    xq[u] = xpre[decltype(first)::value - 1][u];
                } else {
                    const unsigned g = (unsigned)fu * (unsigned)I1p + (unsigned)e0;
                    mw[u] = P.mask[g >> 5] >> (g & 31u);
                    xq[u] = *reinterpret_cast<const V*>(xb + (size_t)fu * I1p);
                }
            } else {
                xq[u] = zero_v<T>();
                mw[u] = ~0u;
            }
            s[u] = sc;
            int carry = 0;
#pragma unroll
            for (int q = 0; q < NO; ++q) {
                int d = dg[q] + ds[q] + carry;
                carry = (q + 1 < NO && d >= dm[q]) ? 1 : 0;
                dg[q] = d - (carry ? dm[q] : 0);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (!(val & (1u << u))) continue;
            T x[VE], t[VE], xn[VE];
            VecT<T>::get(xq[u], x);
#pragma unroll
            for (int e = 0; e < VE; ++e) t[e] = s[u];
#pragma unroll
            for (int q = 0; q < NO; ++q) {
                T h[VE];
                VecT<T>::get(*reinterpret_cast<const V*>(tab + so[u][q]), h);
#pragma unroll
                for (int e = 0; e < VE; ++e) t[e] *= h[e];
            }
            refill_chunk<T, VE>(x, t, mw[u], P.rho, P.inv1p, xn, qn);
            *reinterpret_cast<V*>(xb + (size_t)(f + u * slots) * I1p) = VecT<T>::make(xn);
        }
        f += U * slots;
    };
    if (npre > 0) do_round(std::integral_constant<int, 1>{});
    if constexpr (kL2Pre > 1)
        if (npre > 1) do_round(std::integral_constant<int, 2>{});
    while (act && f < f1) do_round(std::integral_constant<int, 0>{});
    double n0 = qn.s0(), n1 = qn.s1(), n2 = qn.s2();
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        n0 += __shfl_xor_sync(0xffffffffu, n0, o);
        n1 += __shfl_xor_sync(0xffffffffu, n1, o);
        n2 += __shfl_xor_sync(0xffffffffu, n2, o);
    }
    if (lane == 0) {
        sm[warp * 3 + 0] = n0;
        sm[warp * 3 + 1] = n1;
        sm[warp * 3 + 2] = n2;
    }
    __syncthreads();
    if (threadIdx.x < 3) {
        double a = 0.0;
        for (int w = 0; w < 8; ++w) a += sm[w * 3 + threadIdx.x];
        P.norms[((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * 3 + threadIdx.x] = a;
    }
}

}  // namespace ifctn
