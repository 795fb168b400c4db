// fiber_pass.cuh — K2 (coefficient contraction, step a2) and K4 (model rebuild + masked
// refill + norms, step a5) as one streaming kernel family over X in fibre order.
//
// Paper: Prop. 1 gives the mode-k coefficient matrix Z_k = diag(vec S_k)·⊗G;
// Eq. 8 solves column j of G_{k,i} from (y_j ⊗ G_{i,k}) D.  Written out per
// entry, the only data-sized work is
//     β(a,j) = Σ_{i: i_i=a, i_k=j} M(i) X(i),   ω(a,j) = Σ_{i: i_i=a, i_k=j} M(i)²,
//     M(i) = Π_{{p,q}≠{k,i}} H_{p,q}(i_p,i_q),   H_{p,q} = G_{p,q}ᵀ G_{q,p},
// and Eq. 9 needs t(i) = Π_{p<q} H_{p,q}(i_p,i_q) per entry.  Z_k is never
// materialised: the weight of an entry is rebuilt from the (small, cache-resident) H.
//
// B200 mapping: one pass streams X once with 16-B loads; a "group" of
// `lanes` threads owns whole mode-1 fibres, each lane fixed mode-1 positions (CPL chunks of
// VW elements).  Within a "run" only the fast reduced index i_{r0} changes, so
//     M(i_1, fibre) = ws(i_1) · H_{0,r0}(i_1, i_{r0}) · sf(i_{r0})
// with ws (every slower factor, per lane, registers), one 16-B H column chunk per fibre and
// sf = Π_m H_{r0,m}(i_{r0}, i_m) precomputed per run into a per-group shared-memory vector
// by the group's lanes.  Reductions are deterministic: lane-local accumulation, one partial
// slot per (group, v) pair, and a fixed-order fp64 second stage (reduce_partials).
#pragma once

#include "common.cuh"

namespace ifctn {

template <typename T, int MODE, int CPL, bool SMEM>
__global__ void __launch_bounds__(kPassThreads, (CPL == 1 ? kPassMinBlocks : (CPL == 2 ? 2 : 1))) fiber_pass(const __grid_constant__ PassParams<T> P) {
    using VTr = VecT<T>;
    using V = typename VTr::V;
    constexpr int VW = VTr::W;
    constexpr int U = (CPL >= 4) ? 1 : (kUnroll / CPL);
    constexpr bool kContract = (MODE == PASS_KEPT1 || MODE == PASS_RED1);

    extern __shared__ __align__(16) unsigned char smem_raw[];
    const T* __restrict__ Hb = P.H;
    size_t sm_off = 0;
    if constexpr (SMEM) {
        V* s = reinterpret_cast<V*>(smem_raw);
        const V* g = reinterpret_cast<const V*>(P.H);
        for (int64_t e = threadIdx.x; e < P.hsize / VW; e += blockDim.x) s[e] = g[e];
        __syncthreads();
        Hb = reinterpret_cast<const T*>(smem_raw);
        sm_off = (size_t)P.hsize * sizeof(T);
    }
    const int lanes = P.lanes;
    const int lane = threadIdx.x & (lanes - 1);
    const int gin = threadIdx.x >> P.lane_shift;  // group index inside the CTA
    T* sfv = reinterpret_cast<T*>(smem_raw + sm_off) + (size_t)gin * P.sf_cap;

    const int group = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> P.lane_shift);
    if (group >= P.ngroups) return;
    const unsigned gmask = (lanes == 32) ? 0xffffffffu
                                         : (((1u << lanes) - 1u) << ((threadIdx.x & 31) & ~(lanes - 1)));

    // lane → chunk offsets (clamped so every load is in bounds; invalid chunks weigh 0)
    int cofs[CPL];
    bool cval[CPL];
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
        const int ch = lane + c * lanes;
        cval[c] = ch < P.nchunk;
        cofs[c] = (cval[c] ? ch : P.nchunk - 1) * VW;
    }

    // All fibre/index arithmetic is 32-bit (nfib < 2^31 is checked on the host); only
    // element offsets into X are 64-bit.
    const int f0 = group * (int)P.L;
    const int f1 = min(f0 + (int)P.L, (int)P.nfib);
    const int FR = (int)P.FR;
    const bool has_fast = P.nred > 0;
    const int fstep = has_fast ? (int)P.fstride[P.rmode[0]] : 0;
    const int64_t xstep = (int64_t)fstep * P.I1p;      // elements between consecutive fibres
    const int hstep = has_fast ? P.I1p : 0;            // H_{0,r0} column step (0: ones column)
    const int rdim0 = has_fast ? (int)P.rdim[0] : 1;

    double n0 = 0.0, n1 = 0.0, n2 = 0.0;  // REFILL: ‖ΔX‖², ‖X‖², ‖X_new − t‖²; OBJ: n2

    int pos = f0;
    int v = pos / FR;
    int r = pos - v * FR;
    while (pos < f1) {
        const int seg_end = min(f1, (v + 1) * FR);
        int ridx[MAXN];
        {
            int rr = r;
#pragma unroll
            for (int j = 0; j < MAXN; ++j) {
                ridx[j] = 0;
                if (j < P.nred) {
                    ridx[j] = rr % (int)P.rdim[j];
                    rr /= (int)P.rdim[j];
                }
            }
        }
        T sb[CPL][VW], sw[CPL][VW];  // segment accumulators (one kept value v)
#pragma unroll
        for (int c = 0; c < CPL; ++c)
#pragma unroll
            for (int e = 0; e < VW; ++e) sb[c][e] = sw[c][e] = T(0);

        while (pos < seg_end) {
            const int run = has_fast ? min(seg_end - pos, rdim0 - ridx[0]) : 1;
            // ---- run setup (rare path): indices of every outer mode, slow factors --------
            int idx[MAXN];
#pragma unroll
            for (int m = 0; m < MAXN; ++m) idx[m] = 0;
            if (P.nkept >= 1) idx[P.kmode[0]] = v % (int)P.kdim[0];
            if (P.nkept >= 2) idx[P.kmode[1]] = v / (int)P.kdim[0];
#pragma unroll
            for (int j = 0; j < MAXN; ++j)
                if (j < P.nred) idx[P.rmode[j]] = ridx[j];
            int fib = 0;
#pragma unroll
            for (int m = 1; m < MAXN; ++m)
                if (m <= P.nouter) fib += idx[m] * (int)P.fstride[m];

            T ws[CPL][VW];
#pragma unroll
            for (int c = 0; c < CPL; ++c)
#pragma unroll
                for (int e = 0; e < VW; ++e) ws[c][e] = T(1);
            for (int t = 0; t < P.nvs; ++t) {
                const T* base = Hb + P.vs_off[t] + (int64_t)idx[P.vs_mode[t]] * P.I1p;
#pragma unroll
                for (int c = 0; c < CPL; ++c) {
                    T h[VW];
                    VTr::get(*reinterpret_cast<const V*>(base + cofs[c]), h);
#pragma unroll
                    for (int e = 0; e < VW; ++e) ws[c][e] *= h[e];
                }
            }
            T ss = T(1);
            for (int t = 0; t < P.nss; ++t)
                ss *= Hb[P.ss_off[t] + (int64_t)idx[P.ss_q[t]] * P.ss_ld[t] + idx[P.ss_p[t]]];
#pragma unroll
            for (int c = 0; c < CPL; ++c)
#pragma unroll
                for (int e = 0; e < VW; ++e) ws[c][e] = cval[c] ? ws[c][e] * ss : T(0);
            const int ri0 = ridx[0];
            const T* hcol0 = Hb + (has_fast ? P.vf_off + (int64_t)ri0 * P.I1p : P.ones_off);

            // ---- the run, in sub-runs of ≤ sf_cap fibres --------------------------------
            T q0 = T(0), q1 = T(0), q2 = T(0);
            for (int sub = 0; sub < run; sub += P.sf_cap) {
                const int len = min(run - sub, P.sf_cap);
                __syncwarp(gmask);
                for (int q = lane; q < len; q += lanes) {
                    T f = T(1);
                    for (int t = 0; t < P.nsf; ++t)
                        f *= Hb[P.sf_off[t] + (int64_t)idx[P.sf_fixmode[t]] * P.sf_fixmul[t] +
                                (int64_t)(ri0 + sub + q) * P.sf_inc[t]];
                    sfv[q] = f;
                }
                __syncwarp(gmask);
                const int64_t ebase = (int64_t)(fib + sub * fstep) * P.I1p;
                const T* xp = P.X + ebase;
                T* xw = P.Xw + ebase;
                const T* hp = hcol0 + sub * hstep;

                auto body = [&](auto uu, int q) {
                    constexpr int UU = decltype(uu)::value;
                    V xv[UU][CPL];
                    uint32_t mb[UU][CPL];
#pragma unroll
                    for (int u = 0; u < UU; ++u) {
#pragma unroll
                        for (int c = 0; c < CPL; ++c) {
                            const int64_t eo = (int64_t)(q + u) * xstep + cofs[c];
                            if constexpr (kContract) xv[u][c] = ld_stream(reinterpret_cast<const V*>(xp + eo));
                            else if constexpr (MODE != PASS_MODEL) xv[u][c] = *reinterpret_cast<const V*>(xp + eo);
                            if constexpr (MODE == PASS_REFILL) {
                                const int64_t ge = ebase + eo;
                                mb[u][c] = __ldg(P.mask + (ge >> 5)) >> (ge & 31);
                            }
                        }
                    }
#pragma unroll
                    for (int u = 0; u < UU; ++u) {
                        const T sf = sfv[q + u];
                        const T* hq = hp + (q + u) * hstep;
#pragma unroll
                        for (int c = 0; c < CPL; ++c) {
                            T hf[VW], w[VW];
                            VTr::get(*reinterpret_cast<const V*>(hq + cofs[c]), hf);
#pragma unroll
                            for (int e = 0; e < VW; ++e) w[e] = ws[c][e] * (hf[e] * sf);
                            if constexpr (kContract) {
                                T x[VW];
                                VTr::get(xv[u][c], x);
#pragma unroll
                                for (int e = 0; e < VW; ++e) {
                                    sb[c][e] = fma(w[e], x[e], sb[c][e]);
                                    sw[c][e] = fma(w[e], w[e], sw[c][e]);
                                }
                            } else if constexpr (MODE == PASS_REFILL) {
                                T x[VW], xn[VW];
                                VTr::get(xv[u][c], x);
#pragma unroll
                                for (int e = 0; e < VW; ++e) x[e] = cval[c] ? x[e] : T(0);  // clamped lane
#pragma unroll
                                for (int e = 0; e < VW; ++e) {
                                    const bool obs = (mb[u][c] >> e) & 1u;
                                    xn[e] = obs ? x[e] : (w[e] + P.rho * x[e]) * P.inv1p;
                                    const T d = xn[e] - x[e];
                                    const T g = xn[e] - w[e];
                                    q0 = fma(d, d, q0);
                                    q1 = fma(x[e], x[e], q1);
                                    q2 = fma(g, g, q2);
                                }
                                if (cval[c])
                                    *reinterpret_cast<V*>(xw + (int64_t)(q + u) * xstep + cofs[c]) = VTr::make(xn);
                            } else if constexpr (MODE == PASS_OBJ) {
                                T x[VW];
                                VTr::get(xv[u][c], x);
#pragma unroll
                                for (int e = 0; e < VW; ++e) {
                                    const T g = (cval[c] ? x[e] : T(0)) - w[e];
                                    q2 = fma(g, g, q2);
                                }
                            } else {  // PASS_MODEL: dense user layout, scalar stores
                                if (cval[c]) {
                                    const int64_t fb = (ebase + (int64_t)(q + u) * xstep) / P.I1p;
#pragma unroll
                                    for (int e = 0; e < VW; ++e) {
                                        const int i1 = cofs[c] + e;
                                        if (i1 < P.I1) P.out[fb * P.I1 + i1] = w[e];
                                    }
                                }
                            }
                        }
                    }
                };
                int q = 0;
                for (; q + U <= len; q += U) body(std::integral_constant<int, U>{}, q);
                for (; q < len; ++q) body(std::integral_constant<int, 1>{}, q);
            }
            if constexpr (MODE == PASS_REFILL || MODE == PASS_OBJ) {
                n0 += (double)q0;
                n1 += (double)q1;
                n2 += (double)q2;
            }
            pos += run;
            if (has_fast) {  // odometer advance by `run`
                ridx[0] += run;
#pragma unroll
                for (int j = 0; j < MAXN - 1; ++j) {
                    if (j + 1 < P.nred && ridx[j] >= (int)P.rdim[j]) {
                        ridx[j] = 0;
                        ridx[j + 1] += 1;
                    }
                }
            }
        }
        // ---- flush the segment's partials into slot group + v ---------------------------
        if constexpr (MODE == PASS_KEPT1) {
            const int64_t slot = (int64_t)group + v;
#pragma unroll
            for (int c = 0; c < CPL; ++c) {
                if (cval[c]) {
                    const int64_t o = slot * P.Lv + cofs[c];
                    *reinterpret_cast<V*>(P.part_b + o) = VTr::make(sb[c]);
                    *reinterpret_cast<V*>(P.part_w + o) = VTr::make(sw[c]);
                }
            }
        } else if constexpr (MODE == PASS_RED1) {
            T tb = T(0), tw = T(0);
#pragma unroll
            for (int c = 0; c < CPL; ++c)
#pragma unroll
                for (int e = 0; e < VW; ++e) {
                    tb += sb[c][e];
                    tw += sw[c][e];
                }
            for (int off = lanes >> 1; off > 0; off >>= 1) {
                tb += __shfl_xor_sync(gmask, tb, off);
                tw += __shfl_xor_sync(gmask, tw, off);
            }
            if (lane == 0) {
                const int64_t slot = (int64_t)group + v;
                P.part_b[slot] = tb;
                P.part_w[slot] = tw;
            }
        }
        v += 1;
        r = 0;
    }
    if constexpr (MODE == PASS_REFILL || MODE == PASS_OBJ) {
        for (int off = lanes >> 1; off > 0; off >>= 1) {
            n0 += __shfl_xor_sync(gmask, n0, off);
            n1 += __shfl_xor_sync(gmask, n1, off);
            n2 += __shfl_xor_sync(gmask, n2, off);
        }
        if (lane == 0) {
            P.norms[(int64_t)group * 3 + 0] = n0;
            P.norms[(int64_t)group * 3 + 1] = n1;
            P.norms[(int64_t)group * 3 + 2] = n2;
        }
    }
}

}  // namespace ifctn
