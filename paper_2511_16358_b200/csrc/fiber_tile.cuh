// fiber_tile.cuh — v-blocked (tiled) contraction pass for the blocks that KEEP mode 2
// (code mode 1, fibre stride 1).
//
// Same arithmetic as fiber_walk.cuh (β/ω of Eq. 8 from the leave-one-pair-out weights of
// Prop. 1).  Only the fibre order differs: in the plain walk the kept
// index is fixed inside a segment, so consecutive fibres of a run are I_1 fibres apart (one
// 256-B piece per 16 KB for C5) and DRAM locality suffers.  Here a warp walks TILES of
// F consecutive kept values v = i_1 (one contiguous TMA copy per stage) × a run of the fast
// reduced index i_{r0}; every lane keeps F/FP accumulator sets, one per kept value, and
//     M = ws(i_0 | slow) · H_{0,1}(i_0, v) · H_{0,r0}(i_0, i_{r0}) · sf(v, i_{r0})
// with both H column blocks resident in shared memory, ws in registers and the scalar
// factors touching mode 1 or r0 tabulated per tile in shared memory (sfv[f][t]).
// Partial slot of (warp g, v) = (g + vb)·F + f (reduce_partials with VB = F).
#pragma once

#include "fiber_walk.cuh"

namespace ifctn {

template <typename T, int MODE, int EPL, int LPF, bool HRES>
__device__ __forceinline__ void fiber_pass_vb_body(const PassParams<T>& P, unsigned char* smem_raw, int ncta) {
    static_assert(MODE == PASS_KEPT1 || MODE == PASS_RED1 || MODE == PASS_FUSED, "contraction passes only");
    static_assert(HRES, "the tiled pass keeps its H blocks resident");
    // PASS_FUSED: a5 refill of sweep s fused with block (0,1)'s a2 of sweep s+1 (K = {0,1}):
    // t = M·H_{0,1}(i_0, v), X_new written back and used for β.
    constexpr bool kFused = (MODE == PASS_FUSED);
    // KEPT1/FUSED tiles keep modes {1, 2} (code 0, 1): H_{0,1} is the excluded pair; RED1
    // tiles apply their H_{0,1} column at the flush
    using Cfg = PassCfg<T, EPL, LPF, true, true, kFused>;
    constexpr int D = Cfg::D, F = Cfg::F, FP = Cfg::FP, SR = Cfg::SR;
    constexpr int STAGE = Cfg::STAGE;
    constexpr int MWF = Cfg::MWF;
    constexpr int NS = F / FP;  // accumulator sets per lane
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nwarps = blockDim.x >> 5;
    const int fsub = lane / LPF;
    const int eb = (lane % LPF) * EPL;
    const int I1p = P.I1p;
    const int RL = P.sf_cap / F;  // tile run capacity (stages per tile)

    uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw) + warp * D;
    T* sfv = reinterpret_cast<T*>(smem_raw + P.sfv_off) + (size_t)warp * P.sfv_stride;
    T* hres = reinterpret_cast<T*>(smem_raw + P.hres_off);  // [H_{0,1} | H_{0,r0}]
    T* stg = reinterpret_cast<T*>(smem_raw + P.stage_off) + (size_t)warp * Cfg::RING;
    // warp setup; the resident H blocks are loaded after the producer's first D stages are
    // issued (their copies' latency overlaps the load), see the barrier below
    for (int e = lane; e < Cfg::RING; e += 32) stg[e] = T(0);
    if (lane == 0)
        for (int s = 0; s < D; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
    fence_proxy_async_smem();
    __syncwarp();

    // Dynamic schedule: the stage range is cut into P.ngroups fixed chunks of L/F stages;
    // warps claim chunks from a global counter (P.sched[0]).  A chunk's partial slots and norm
    // slot are indexed by the chunk, not by the warp, so the result does not depend on which
    // warp ran it.  The last warp to retire resets the counters for the next launch.
    const int nchunks = (int)P.ngroups;
    const int LQ = (int)(P.L / F);            // stages per chunk
    const int QT = (int)(P.nfib / F);         // stages in total
    int c_first = 0;
    if (lane == 0) c_first = (int)atomicAdd(P.sched, 1u);
    c_first = __shfl_sync(0xffffffffu, c_first, 0);

    const uint32_t bar0 = smem_u32(bars);
    const uint32_t stg0 = smem_u32(stg);
    const T* __restrict__ Hb = P.H;
    bool ev[EPL];
#pragma unroll
    for (int e = 0; e < EPL; ++e) ev[e] = eb + e < I1p;
    const bool lane_full = eb + EPL <= I1p;
    const int ebc = eb < I1p ? eb : 0;
    const int FR = (int)P.FR;
    const int kdim0 = (int)P.kdim[0];
    const int nb0 = (int)P.nb0;
    const int rdim0 = (int)P.rdim[0];
    const int fstep0 = (int)P.fstride[P.rmode[0]];
    const int h1step = P.vf_off >= 0 ? I1p : 0;      // H_{0,1} is a factor (not the kept pair)
    const T* h1 = hres + ebc;                         // H_{0,1} block or the ones column
    const T* h2 = hres + P.hres_elems + ebc;          // H_{0,r0} block
    const T* h3 = hres + P.hres_elems + P.hres2_elems + ebc;  // fused: H_{0,1} block
    const uint32_t rowbytes = (uint32_t)(I1p * sizeof(T));
    double n0 = 0.0, n1 = 0.0, n2 = 0.0;  // fused: ‖ΔX‖², ‖X‖², ‖X_new − t‖²

    // stages = positions q = vb·FR + r (r in odometer order, r0 fastest)
    auto decode = [&](int q, int& vb, int& b0, int& nvalid, int (&ridx)[MAXN]) {
        vb = q / FR;
        int r = q - vb * FR;
        b0 = (vb % nb0) * F;
        nvalid = min(F, kdim0 - b0);
        int fib = b0;  // fstride[1] == 1
        if (P.nkept >= 2) fib += (vb / nb0) * (int)P.fstride[P.kmode[1]];
#pragma unroll
        for (int j = 0; j < MAXN; ++j) {
            ridx[j] = 0;
            if (j < P.nred) {
                ridx[j] = r % (int)P.rdim[j];
                r /= (int)P.rdim[j];
                fib += ridx[j] * (int)P.fstride[P.rmode[j]];
            }
        }
        return fib;
    };

    // ---- producer (lane 0): one stage (F contiguous fibres) per position, D ahead --------
    // incremental odometer over r (rmode[0] fastest); full decode only when vb changes.  At
    // the end of its chunk the producer claims the next one (at most one chunk ahead of the
    // consumers, who adopt it from lane 0 when they finish theirs).
    int p_chunk = c_first;
    bool p_ahead = false;
    int pq = c_first < nchunks ? c_first * LQ : 0;
    int pq1 = c_first < nchunks ? min(pq + LQ, QT) : 0;
    uint32_t p_n = 0;
    int p_vb, p_b0, p_nvalid, p_ridx[MAXN];
    int p_fib = decode(pq, p_vb, p_b0, p_nvalid, p_ridx);
    auto produce = [&]() {
        if (pq >= pq1) {
            if (p_ahead || p_chunk >= nchunks) return;
            p_chunk = (int)atomicAdd(P.sched, 1u);
            p_ahead = true;
            if (p_chunk >= nchunks) return;
            pq = p_chunk * LQ;
            pq1 = min(pq + LQ, QT);
            p_fib = decode(pq, p_vb, p_b0, p_nvalid, p_ridx);
        }
        const int fib = p_fib;
        const int nvalid = p_nvalid;
        const int s = (int)(p_n % (uint32_t)D);
        const uint32_t bar = bar0 + 8u * (uint32_t)s;
        const uint32_t sx = stg0 + (uint32_t)(s * STAGE * (int)sizeof(T));
        fence_stage_refill();
        const int64_t pg0 = (int64_t)fib * I1p;
        uint32_t mbytes = 0;
        int64_t ma0 = 0;
        if constexpr (kFused) {
            if (SR == I1p) {
                mbytes = mask_span(pg0, (int64_t)nvalid * I1p, ma0);
            } else {
                for (int f = 0; f < nvalid; ++f) mbytes += mask_span(pg0 + (int64_t)f * I1p, I1p, ma0);
            }
        }
        mbar_arrive_expect_tx_a(bar, (uint32_t)nvalid * rowbytes + mbytes);
        if constexpr (kFused) {
            const uint32_t sm = sx + (uint32_t)(Cfg::XH * (int)sizeof(T));
            if (SR == I1p) {
                tma_g2s_a(sm, P.mask + ma0, mbytes, bar);
            } else {
                for (int f = 0; f < nvalid; ++f) {
                    const uint32_t b = mask_span(pg0 + (int64_t)f * I1p, I1p, ma0);
                    IFCTN_CHECK(ma0 + (int64_t)(b / 4) <= P.mask_cap && b <= (uint32_t)(MWF * 4), "tiled fibre mask words");
                    tma_g2s_a(sm + (uint32_t)(f * MWF * 4), P.mask + ma0, b, bar);
                }
            }
        }
        IFCTN_CHECK(((int64_t)fib + nvalid) * I1p <= P.x_cap, "tiled X range");
        IFCTN_CHECK(!kFused || SR != I1p || ma0 + (int64_t)(mbytes / 4) <= P.mask_cap, "tiled mask words");
        const T* xs = P.X + (int64_t)fib * I1p;
        if (SR == I1p) {
            tma_g2s_a(sx, xs, (uint32_t)nvalid * rowbytes, bar);
        } else {
            for (int f = 0; f < nvalid; ++f)
                tma_g2s_a(sx + (uint32_t)(f * SR * (int)sizeof(T)), xs + (int64_t)f * I1p, rowbytes, bar);
        }
        ++pq;
        ++p_n;
        if (pq >= pq1) return;
        // advance the odometer (fast path: the fastest reduced index does not wrap)
        if (p_ridx[0] + 1 < rdim0) {
            p_ridx[0] += 1;
            p_fib += fstep0;
            return;
        }
        bool wrapped = true;
#pragma unroll
        for (int j = 0; j < MAXN; ++j) {
            if (wrapped && j < P.nred) {
                p_ridx[j] += 1;
                p_fib += (int)P.fstride[P.rmode[j]];
                if (p_ridx[j] < (int)P.rdim[j]) {
                    wrapped = false;
                } else {
                    p_fib -= p_ridx[j] * (int)P.fstride[P.rmode[j]];
                    p_ridx[j] = 0;
                }
            }
        }
        if (wrapped) p_fib = decode(pq, p_vb, p_b0, p_nvalid, p_ridx);  // next kept block
    };
    if (lane == 0)
        for (int d = 0; d < D; ++d) produce();
    {
        const float4* s1 = reinterpret_cast<const float4*>(P.H + P.hres_src);
        const float4* s2 = reinterpret_cast<const float4*>(P.H + P.vf2_off);
        const float4* s3 = reinterpret_cast<const float4*>(P.H + P.h01_off);
        float4* dst = reinterpret_cast<float4*>(hres);
        const int n1 = (int)(P.hres_elems * sizeof(T) / 16), n2 = (int)(P.hres2_elems * sizeof(T) / 16);
        const int n3 = (int)(P.hres3_elems * sizeof(T) / 16);
        for (int e = threadIdx.x; e < n1 + n2 + n3; e += blockDim.x)
            dst[e] = e < n1 ? s1[e] : (e < n1 + n2 ? s2[e - n1] : s3[e - n1 - n2]);
    }
    __syncthreads();
    TL_STAMP(1);

    T sb[NS][EPL], sw[NS][EPL];
#pragma unroll
    for (int t = 0; t < NS; ++t)
#pragma unroll
        for (int e = 0; e < EPL; ++e) sb[t][e] = sw[t][e] = T(0);
    uint32_t cn = 0;
    for (int chunk = c_first; chunk < nchunks;) {
        const int group = chunk;  // partial-slot / norm-slot index
        int q = chunk * LQ;
        const int q1 = min(q + LQ, QT);
        while (q < q1) {
            int vb, b0, nvalid, ridx[MAXN];
            decode(q, vb, b0, nvalid, ridx);
            const int seg_end = min(q1, (vb + 1) * FR);           // end of this kept block
            const int rl = min(min(seg_end - q, rdim0 - ridx[0]), RL);  // tile: r0 run
            // ---- tile setup: slow factors and the (v, i_{r0}) scalar table --------------------
            int midx = 0;  // index of outer mode m held by lane m (see fiber_walk.cuh)
            if (P.nkept >= 2 && lane == P.kmode[1]) midx = vb / nb0;
#pragma unroll
            for (int j = 0; j < MAXN; ++j)
                if (j < P.nred && lane == P.rmode[j]) midx = ridx[j];
            auto idx = [&](int m) { return __shfl_sync(0xffffffffu, midx, m); };
            T ws[EPL];
#pragma unroll
            for (int e = 0; e < EPL; ++e) ws[e] = ev[e] ? T(1) : T(0);
            for (int t = 0; t < P.nvs; ++t) {
                const T* base = Hb + P.vs_off[t] + (int64_t)idx(P.vs_mode[t]) * I1p + eb;
#pragma unroll
                for (int e = 0; e < EPL; ++e)
                    if (ev[e]) ws[e] *= base[e];
            }
            T ss = T(1);
            for (int t = 0; t < P.nss; ++t)
                ss *= Hb[P.ss_off[t] + (int64_t)idx(P.ss_q[t]) * P.ss_ld[t] + idx(P.ss_p[t])];
#pragma unroll
            for (int e = 0; e < EPL; ++e) ws[e] *= ss;
            // scalar factors touching mode 1 or r0, factorised: sf(f,t) = A(v_f)·B(i_{r0,t})·C(v_f, i_{r0,t})
            //   A = Π_q H_{1,q}(v, i_q), B = Π_q H_{r0,q}(i_{r0}, i_q) (q fixed in the tile),
            //   C = H_{1,r0}(v, i_{r0}) unless {1, r0} is the kept pair.
            T* At = sfv + P.sf_cap;
            T* Bt = At + F;
            // table bases (uniform: the index shuffles need the whole warp)
            const T* ab[MAXSF];
            const T* bb[MAXSF];
#pragma unroll
            for (int u = 0; u < MAXSF; ++u) {
                ab[u] = Hb;
                bb[u] = Hb;
                if (u < P.nta) ab[u] = Hb + P.ta_off[u] + (int64_t)idx(P.ta_fix[u]) * P.ta_mul[u];
                if (u < P.nsf) bb[u] = Hb + P.sf_off[u] + (int64_t)idx(P.sf_fixmode[u]) * P.sf_fixmul[u];
            }
            if (lane < F) {
                T a = T(1);
                const int v = b0 + min(lane, nvalid - 1);
#pragma unroll
                for (int u = 0; u < MAXSF; ++u)
                    if (u < P.nta) a *= ab[u][(int64_t)v * P.ta_inc[u]];
                At[lane] = a;
            }
            for (int t = lane; t < rl; t += 32) {
                T b = T(1);
#pragma unroll
                for (int u = 0; u < MAXSF; ++u)
                    if (u < P.nsf) b *= bb[u][(int64_t)(ridx[0] + t) * P.sf_inc[u]];
                Bt[t] = b;
            }
            __syncwarp();
            {
                const T* cb = P.tc_off >= 0 ? Hb + P.tc_off + (int64_t)ridx[0] * P.tc_ld + b0 : nullptr;
                for (int e = lane; e < F * rl; e += 32) {
                    const int f = e % F, t = e / F;  // F is a power of two: shifts
                    T val = At[f] * Bt[t];
                    if (cb) val *= cb[(int64_t)t * P.tc_ld + min(f, nvalid - 1)];
                    sfv[t * F + f] = val;
                }
            }
            __syncwarp();
            const T* h2run = h2 + (int64_t)ridx[0] * I1p;
            const int64_t fib0 = kFused ? decode(q, vb, b0, nvalid, ridx) : 0;  // fused: X address
            const int fstep = fstep0;
            Norms3<T> qn;
            T* xw = kFused ? P.Xw + fib0 * I1p : nullptr;  // fused: X_new of the stage's first fibre
            for (int t = 0; t < rl; ++t) {
                const int s = (int)(cn % (uint32_t)D);
                mbar_wait_a(bar0 + 8u * (uint32_t)s, (cn / (uint32_t)D) & 1u);
                const T* sx = stg + s * STAGE;
                const uint32_t* smw = reinterpret_cast<const uint32_t*>(sx + Cfg::XH);
                T hr[EPL];
                lds_vec<T, EPL>(h2run + t * I1p, hr);
                T wr[EPL];
#pragma unroll
                for (int e = 0; e < EPL; ++e) wr[e] = ws[e] * hr[e];
#pragma unroll
                for (int st = 0; st < NS; ++st) {
                    const int f = st * FP + fsub;
                    if (f < nvalid) {
                        T w[EPL], x[EPL];
                        // RED1: the column H_{0,1}(·, v_f) is constant over the kept block, so it
                        // is applied to the accumulators at the flush (Σ h·u·x = h·Σ u·x,
                        // Σ (h·u)² = h²·Σ u²); KEPT1/FUSED: H_{0,1} is the excluded pair
                        scale<T, EPL>(wr, sfv[t * F + f], w);
                        lds_vec<T, EPL>(sx + f * SR + eb, x);
                        if constexpr (kFused) {
                            T h01[EPL], tt[EPL], xn[EPL];
                            lds_vec<T, EPL>(h3 + (b0 + f) * I1p, h01);
                            mul<T, EPL>(w, h01, tt);
                            // Ω bits: the staged word range starts at the 128-bit boundary at or
                            // below the stage's (merged) or the fibre's first element
                            const int fo = f * I1p;
                            const int sl = (int)((uint32_t)(xw - P.Xw) & 127u);
                            const uint32_t bits = (SR == I1p) ? mask_bits_l(smw, sl + fo + eb)
                                                              : mask_bits_l(smw + f * MWF, ((sl + fo) & 127) + eb);
                            if (P.full_norms) refill_chunk<T, EPL>(x, tt, bits, P.rho, P.inv1p, xn, qn);
                            else refill_lite<T, EPL>(x, tt, bits, P.rho, P.inv1p, xn, qn);
                            store_chunk<T, EPL>(xw + fo + eb, xn, lane_full, ev);
                            accumulate<T, EPL>(w, xn, sb[st], sw[st]);
                        } else {
                            accumulate<T, EPL>(w, x, sb[st], sw[st]);
                        }
                    }
                }
                __syncwarp();
                ++cn;
                if constexpr (kFused) xw += (int64_t)fstep * I1p;
                if (lane == 0) produce();
            }
            __syncwarp();  // sfv is rewritten by the next tile
            if constexpr (kFused) {
                n0 += qn.s0();
                n1 += qn.s1();
                n2 += qn.s2();
            }
            q += rl;
            if (q >= seg_end) {  // kept block finished (or range end): flush its F values
#pragma unroll
                for (int st = 0; st < NS; ++st) {
                    const int f = st * FP + fsub;
                    const int64_t slot = ((int64_t)group + vb) * F + f;
                    IFCTN_CHECK(f >= nvalid || (slot + 1) * P.Lv <= P.part_cap, "tiled slot");
                    if constexpr (MODE == PASS_KEPT1 || kFused) {
                        if (f < nvalid) {
                            T* pbd = P.part_b + slot * P.Lv + eb;
                            T* pwd = P.part_w + slot * P.Lv + eb;
                            if (lane_full) {
                                stg_vec<T, EPL>(pbd, sb[st]);
                                stg_vec<T, EPL>(pwd, sw[st]);
                            } else {
#pragma unroll
                                for (int e = 0; e < EPL; ++e)
                                    if (ev[e]) {
                                        pbd[e] = sb[st][e];
                                        pwd[e] = sw[st][e];
                                    }
                            }
                        }
                    } else {
                        T hf[EPL];
                        lds_vec<T, EPL>(h1 + (b0 + min(f, nvalid - 1)) * h1step, hf);
                        T tb = T(0), tw = T(0);
#pragma unroll
                        for (int e = 0; e < EPL; ++e) {
                            tb = fma(hf[e], sb[st][e], tb);
                            tw = fma(hf[e] * hf[e], sw[st][e], tw);
                        }
#pragma unroll
                        for (int o = LPF / 2; o > 0; o >>= 1) {  // the fibre's LPF lanes
                            tb += __shfl_xor_sync(0xffffffffu, tb, o);
                            tw += __shfl_xor_sync(0xffffffffu, tw, o);
                        }
                        if ((lane % LPF) == 0 && f < nvalid) {
                            P.part_b[slot] = tb;
                            P.part_w[slot] = tw;
                        }
                    }
#pragma unroll
                    for (int e = 0; e < EPL; ++e) sb[st][e] = sw[st][e] = T(0);
                }
            }
        }
        if constexpr (kFused) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                n0 += __shfl_xor_sync(0xffffffffu, n0, o);
                n1 += __shfl_xor_sync(0xffffffffu, n1, o);
                n2 += __shfl_xor_sync(0xffffffffu, n2, o);
            }
            if (lane == 0) {
                P.norms[(int64_t)group * 3 + 0] = n0;
                P.norms[(int64_t)group * 3 + 1] = n1;
                P.norms[(int64_t)group * 3 + 2] = n2;
            }
            n0 = n1 = n2 = 0.0;
        }
        // next chunk: the one the producer claimed
        int nx = 0;
        if (lane == 0) {
            nx = p_chunk;
            p_ahead = false;
        }
        chunk = __shfl_sync(0xffffffffu, nx, 0);
    }
    if (lane == 0) {
        const unsigned total = (unsigned)ncta * (unsigned)nwarps;
        if (atomicAdd(P.sched + 1, 1u) == total - 1) {
            P.sched[0] = 0u;
            P.sched[1] = 0u;
        }
    }
}

template <typename T, int MODE, int EPL, int LPF, bool HRES>
__global__ void __launch_bounds__(kPassThreads, kPassMinBlocks)
    fiber_pass_vb(const __grid_constant__ PassParams<T> P) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    TL_STAMP(0);
    fiber_pass_vb_body<T, MODE, EPL, LPF, HRES>(P, smem_raw, gridDim.x);
#ifdef IFCTN_EXP_TIMELINE
    __syncthreads();
#endif
    TL_STAMP(2);
}

}  // namespace ifctn
