// fiber_pass.cuh — K2 (coefficient contraction, step a2) and K4 (model rebuild + masked
// refill + norms, step a5) as one streaming kernel family over X in fibre order.
//
// Paper: Prop. 1 gives the mode-k coefficient matrix Z_k = diag(vec S_k)·⊗G;
// Eq. 8 solves column j of G_{k,i} from (y_j ⊗ G_{i,k}) D.  Written out per
// entry, the only data-sized work is
//     β(a,j) = Σ_{i: i_i=a, i_k=j} M(i) X(i),   ω(a,j) = Σ_{i: i_i=a, i_k=j} M(i)²,
//     M(i) = Π_{{p,q}≠{k,i}} H_{p,q}(i_p,i_q),   H_{p,q} = G_{p,q}ᵀ G_{q,p},
// and Eq. 9 needs t(i) = Π_{p<q} H_{p,q}(i_p,i_q) per entry.  Z_k is never
// materialised: the weight of an entry is rebuilt from the (small, on-chip) H matrices.
//
// B200 mapping: one pass streams X once with 16-B loads; a "group" of
// `lanes` threads owns whole mode-1 fibres, each lane fixed mode-1 positions (CPL chunks of
// VW elements), so the mode-1 part of the weight is a per-lane vector that changes only with
// the fast reduced mode r0 (one 16-B LDS per fibre) and everything slower is cached in
// registers.  Reductions are deterministic: lane-local accumulation, one partial slot per
// (group, v) pair, and a fixed-order fp64 second stage (reduce_partials).
#pragma once

#include "common.cuh"

namespace ifctn {

template <typename T, int MODE, int CPL, bool SMEM>
__global__ void __launch_bounds__(kPassThreads) fiber_pass(const __grid_constant__ PassParams<T> P) {
    using VTr = VecT<T>;
    using V = typename VTr::V;
    constexpr int VW = VTr::W;
    constexpr int U = (CPL >= 4) ? 1 : (kUnroll / CPL);

    extern __shared__ __align__(16) unsigned char smem_raw[];
    const T* __restrict__ Hb = P.H;
    if constexpr (SMEM) {
        V* s = reinterpret_cast<V*>(smem_raw);
        const V* g = reinterpret_cast<const V*>(P.H);
        for (int64_t e = threadIdx.x; e < P.hsize / VW; e += blockDim.x) s[e] = g[e];
        __syncthreads();
        Hb = reinterpret_cast<const T*>(smem_raw);
    }

    const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t group = gt >> P.lane_shift;
    const int lane = threadIdx.x & (P.lanes - 1);
    if (group >= P.ngroups) return;
    const unsigned gmask = (P.lanes == 32) ? 0xffffffffu
                                           : (((1u << P.lanes) - 1u) << ((threadIdx.x & 31) & ~(P.lanes - 1)));

    int chunk[CPL];
    bool cval[CPL];
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
        chunk[c] = lane + c * P.lanes;
        cval[c] = chunk[c] < P.nchunk;
    }

    const int64_t f0 = group * P.L;
    const int64_t f1 = min(f0 + P.L, P.nfib);
    const bool has_fast = P.nred > 0;
    const int64_t fstep = has_fast ? P.fstride[P.rmode[0]] : 0;

    // pass-level accumulators
    double n0 = 0.0, n1 = 0.0, n2 = 0.0;  // REFILL: ‖ΔX‖², ‖X‖², ‖X_new − t‖²; OBJ: n2

    int64_t pos = f0;
    int64_t v = pos / P.FR;
    int64_t r = pos - v * P.FR;
    while (pos < f1) {
        const int64_t seg_end = min(f1, (v + 1) * P.FR);
        int64_t kidx0 = 0, kidx1 = 0;
        if (P.nkept >= 1) {
            kidx0 = v % P.kdim[0];
            kidx1 = v / P.kdim[0];
        }
        int64_t ridx[MAXN];
        {
            int64_t rr = r;
#pragma unroll
            for (int j = 0; j < MAXN; ++j) {
                ridx[j] = 0;
                if (j < P.nred) {
                    ridx[j] = rr % P.rdim[j];
                    rr /= P.rdim[j];
                }
            }
        }
        // segment accumulators (one kept value v)
        T sb[CPL][VW], sw[CPL][VW];
#pragma unroll
        for (int c = 0; c < CPL; ++c)
#pragma unroll
            for (int e = 0; e < VW; ++e) sb[c][e] = sw[c][e] = T(0);

        int64_t remaining = seg_end - pos;
        while (remaining > 0) {
            const int64_t run = has_fast ? min(remaining, P.rdim[0] - ridx[0]) : 1;
            // ---- run setup (rare path): indices of every outer mode, slow factors --------
            int64_t idx[MAXN];
#pragma unroll
            for (int m = 0; m < MAXN; ++m) idx[m] = 0;
            if (P.nkept >= 1) idx[P.kmode[0]] = kidx0;
            if (P.nkept >= 2) idx[P.kmode[1]] = kidx1;
#pragma unroll
            for (int j = 0; j < MAXN; ++j)
                if (j < P.nred) idx[P.rmode[j]] = ridx[j];
            int64_t fib = 0;
#pragma unroll
            for (int m = 1; m < MAXN; ++m)
                if (m <= P.nouter) fib += idx[m] * P.fstride[m];

            T ws[CPL][VW];
#pragma unroll
            for (int c = 0; c < CPL; ++c)
#pragma unroll
                for (int e = 0; e < VW; ++e) ws[c][e] = T(1);
            for (int t = 0; t < P.nvs; ++t) {
                const T* base = Hb + P.vs_off[t] + idx[P.vs_mode[t]] * P.I1p;
#pragma unroll
                for (int c = 0; c < CPL; ++c) {
                    if (cval[c]) {
                        T h[VW];
                        VTr::get(*reinterpret_cast<const V*>(base + chunk[c] * VW), h);
#pragma unroll
                        for (int e = 0; e < VW; ++e) ws[c][e] *= h[e];
                    }
                }
            }
            T ss = T(1);
            for (int t = 0; t < P.nss; ++t) ss *= Hb[P.ss_off[t] + idx[P.ss_q[t]] * P.ss_ld[t] + idx[P.ss_p[t]]];
#pragma unroll
            for (int c = 0; c < CPL; ++c)
#pragma unroll
                for (int e = 0; e < VW; ++e) ws[c][e] = cval[c] ? ws[c][e] * ss : T(0);
            int64_t sfo[MAXSF], sfi[MAXSF];
#pragma unroll
            for (int t = 0; t < MAXSF; ++t) {
                sfo[t] = 0;
                sfi[t] = 0;
                if (t < P.nsf) {
                    sfo[t] = P.sf_off[t] + idx[P.sf_fixmode[t]] * P.sf_fixmul[t];
                    sfi[t] = P.sf_inc[t];
                }
            }
            const T* vfb = Hb + (has_fast ? P.vf_off : 0);
            const int64_t ri0 = ridx[0];

            // ---- hot loop: `run` fibres with only the fast index i_{r0} changing ----------
            // Phase 1 issues U·CPL independent 16-B loads of X (and mask words); phase 2
            // rebuilds each entry's weight from cached slow factors × one fast H column.
            T q0 = T(0), q1 = T(0), q2 = T(0);
            for (int64_t t0 = 0; t0 < run; t0 += U) {
                V xv[U][CPL];
                uint32_t mb[U][CPL];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const bool uv = (t0 + u) < run;
                    const int64_t fb = fib + (t0 + u) * fstep;
#pragma unroll
                    for (int c = 0; c < CPL; ++c) {
                        const bool ok = uv && cval[c];
                        const int64_t xo = fb * P.I1p + chunk[c] * VW;
                        if constexpr (MODE == PASS_KEPT1 || MODE == PASS_RED1) {
                            xv[u][c] = ok ? ld_stream(reinterpret_cast<const V*>(P.X + xo)) : zero_v<T>();
                        } else if constexpr (MODE == PASS_REFILL || MODE == PASS_OBJ) {
                            xv[u][c] = ok ? *reinterpret_cast<const V*>(P.X + xo) : zero_v<T>();
                        }
                        if constexpr (MODE == PASS_REFILL) {
                            mb[u][c] = ok ? (__ldg(P.mask + (xo >> 5)) >> (xo & 31)) : 0xffffffffu;
                        }
                    }
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const bool uv = (t0 + u) < run;
                    const int64_t ri = ri0 + t0 + u;
                    const int64_t fb = fib + (t0 + u) * fstep;
                    T sf = T(1);
                    if (has_fast) {
#pragma unroll
                        for (int t = 0; t < MAXSF; ++t)
                            if (t < P.nsf) sf *= Hb[sfo[t] + ri * sfi[t]];
                    }
#pragma unroll
                    for (int c = 0; c < CPL; ++c) {
                        const bool ok = uv && cval[c];
                        T hf[VW];
                        if (has_fast) {
                            VTr::get(*reinterpret_cast<const V*>(vfb + ri * P.I1p + chunk[c] * VW), hf);
                        } else {
#pragma unroll
                            for (int e = 0; e < VW; ++e) hf[e] = T(1);
                        }
                        T w[VW], x[VW];
#pragma unroll
                        for (int e = 0; e < VW; ++e) w[e] = ok ? ws[c][e] * (hf[e] * sf) : T(0);
                        if constexpr (MODE != PASS_MODEL) VTr::get(xv[u][c], x);
                        if constexpr (MODE == PASS_KEPT1 || MODE == PASS_RED1) {
#pragma unroll
                            for (int e = 0; e < VW; ++e) {
                                sb[c][e] = fma(w[e], x[e], sb[c][e]);
                                sw[c][e] = fma(w[e], w[e], sw[c][e]);
                            }
                        } else if constexpr (MODE == PASS_REFILL) {
                            if (ok) {
                                T xn[VW];
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
                                *reinterpret_cast<V*>(P.Xw + fb * P.I1p + chunk[c] * VW) = VTr::make(xn);
                            }
                        } else if constexpr (MODE == PASS_OBJ) {
#pragma unroll
                            for (int e = 0; e < VW; ++e) {
                                const T g = x[e] - w[e];
                                q2 = fma(g, g, q2);
                            }
                        } else {  // PASS_MODEL
                            if (ok) {
#pragma unroll
                                for (int e = 0; e < VW; ++e) {
                                    const int i1 = chunk[c] * VW + e;
                                    if (i1 < P.I1) P.out[fb * P.I1 + i1] = w[e];
                                }
                            }
                        }
                    }
                }
            }
            if constexpr (MODE == PASS_REFILL || MODE == PASS_OBJ) {
                n0 += (double)q0;
                n1 += (double)q1;
                n2 += (double)q2;
            }
            remaining -= run;
            pos += run;
            if (has_fast) {  // odometer advance by `run`
                ridx[0] += run;
#pragma unroll
                for (int j = 0; j < MAXN - 1; ++j) {
                    if (j + 1 < P.nred && ridx[j] >= P.rdim[j]) {
                        ridx[j] = 0;
                        ridx[j + 1] += 1;
                    }
                }
            }
        }
        // ---- flush the segment's partials into slot group + v ---------------------------
        if constexpr (MODE == PASS_KEPT1) {
            const int64_t slot = group + v;
#pragma unroll
            for (int c = 0; c < CPL; ++c) {
                if (cval[c]) {
                    const int64_t o = slot * P.Lv + chunk[c] * VW;
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
            for (int off = P.lanes >> 1; off > 0; off >>= 1) {
                tb += __shfl_xor_sync(gmask, tb, off);
                tw += __shfl_xor_sync(gmask, tw, off);
            }
            if (lane == 0) {
                const int64_t slot = group + v;
                P.part_b[slot] = tb;
                P.part_w[slot] = tw;
            }
        }
        v += 1;
        r = 0;
    }
    if constexpr (MODE == PASS_REFILL || MODE == PASS_OBJ) {
        for (int off = P.lanes >> 1; off > 0; off >>= 1) {
            n0 += __shfl_xor_sync(gmask, n0, off);
            n1 += __shfl_xor_sync(gmask, n1, off);
            n2 += __shfl_xor_sync(gmask, n2, off);
        }
        if (lane == 0) {
            P.norms[group * 3 + 0] = n0;
            P.norms[group * 3 + 1] = n1;
            P.norms[group * 3 + 2] = n2;
        }
    }
}

}  // namespace ifctn
