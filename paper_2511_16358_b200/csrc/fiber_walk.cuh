// fiber_walk.cuh — K2 (coefficient contraction, step a2) and K4 (model rebuild + masked
// refill + norms, step a5) as one streaming kernel family over X in fibre order (the plain
// walk; fiber_tile.cuh is the tiled walk for blocks keeping mode 2).
//
// Paper: Prop. 1 gives the mode-k coefficient matrix Z_k = diag(vec S_k)·⊗G;
// Eq. 8 solves column j of G_{k,i} from (y_j ⊗ G_{i,k}) D.  Written out per
// entry, the only data-sized work is
//     β(a,j) = Σ_{i: i_i=a, i_k=j} M(i) X(i),   ω(a,j) = Σ_{i: i_i=a, i_k=j} M(i)²,
//     M(i) = Π_{{p,q}≠{k,i}} H_{p,q}(i_p,i_q),   H_{p,q} = G_{p,q}ᵀ G_{q,p},
// and Eq. 9 needs t(i) = Π_{p<q} H_{p,q}(i_p,i_q) per entry.  Z_k is never
// materialised: the weight of an entry is rebuilt from the (small, cache-resident) H.
//
// B200 mapping.  One warp owns a contiguous range of mode-1 fibres
// (a fibre = the I1p-padded line X(:, i_2..i_N)), walked as "runs" in which only the fast
// reduced index i_{r0} changes, so
//     M(i_1, fibre) = ws(i_1) · H_{0,r0}(i_1, i_{r0}) · sf(i_{r0})
// with ws (all slower factors, registers), the H_{0,r0} column of the fibre (resident in
// shared memory for the whole pass when it fits: HRES) and sf = Π_m H_{r0,m}(i_{r0}, i_m),
// precomputed per run into a per-warp shared-memory vector.  The warp works on FP = 32/LPF
// fibres per step: lane l serves step fibre l/LPF at mode-1 positions [(l mod LPF)·EPL, +EPL)
// (16-B shared-memory vectors; fp32 math in packed FMUL2/FFMA2 pairs).
// Data movement is a TMA pipeline that runs ahead across run and segment boundaries: lane 0
// (the producer, with its own copy of the fibre walker) issues cp.async.bulk copies of F
// fibres of X (and their H columns when !HRES; the Ω words for refills) per stage into a
// D-stage shared-memory ring guarded by mbarriers (4 KB × 2 stages, PassCfg PLAIN); all 32
// lanes consume.  The run-constant slow factor ws is applied once per run.  Reductions are
// deterministic: lane-local accumulation, one partial slot per (warp, v) pair, and a
// fixed-order fp64 second stage (reduce_partials, or the solve itself: block_solve).
#pragma once

#include "common.cuh"
#include "solve.cuh"

namespace ifctn {

template <typename T, int N>
__device__ __forceinline__ void lds_vec(const T* p, T (&o)[N]) {
    static_assert(N * sizeof(T) % 16 == 0, "16-B vectors only");
#pragma unroll
    for (int v = 0; v < N * (int)sizeof(T) / 16; ++v) {
        const float4 q = reinterpret_cast<const float4*>(p)[v];
        const T* t = reinterpret_cast<const T*>(&q);
#pragma unroll
        for (int e = 0; e < 16 / (int)sizeof(T); ++e) o[v * (16 / sizeof(T)) + e] = t[e];
    }
}

template <typename T, int N>
__device__ __forceinline__ void stg_vec(T* p, const T (&o)[N]) {
    static_assert(N * sizeof(T) % 16 == 0, "16-B vectors only");
#pragma unroll
    for (int v = 0; v < N * (int)sizeof(T) / 16; ++v) {
        float4 q;
        T* t = reinterpret_cast<T*>(&q);
#pragma unroll
        for (int e = 0; e < 16 / (int)sizeof(T); ++e) t[e] = o[v * (16 / sizeof(T)) + e];
        reinterpret_cast<float4*>(p)[v] = q;
    }
}

// w = ws ⊙ h · sf   (fp32: packed FMUL2 pairs)
template <typename T, int N>
__device__ __forceinline__ void weight(const T (&ws)[N], const T (&h)[N], T sf, T (&w)[N]) {
    if constexpr (sizeof(T) == 4 && N % 2 == 0) {
        const float2 s2 = make_float2(sf, sf);
#pragma unroll
        for (int e = 0; e < N; e += 2) {
            const float2 hs = __fmul2_rn(make_float2(h[e], h[e + 1]), s2);
            const float2 r = __fmul2_rn(make_float2(ws[e], ws[e + 1]), hs);
            w[e] = r.x;
            w[e + 1] = r.y;
        }
    } else {
#pragma unroll
        for (int e = 0; e < N; ++e) w[e] = ws[e] * (h[e] * sf);
    }
}

// w = ws · sf
template <typename T, int N>
__device__ __forceinline__ void scale(const T (&ws)[N], T sf, T (&w)[N]) {
    if constexpr (sizeof(T) == 4 && N % 2 == 0) {
        const float2 s2 = make_float2(sf, sf);
#pragma unroll
        for (int e = 0; e < N; e += 2) {
            const float2 r = __fmul2_rn(make_float2(ws[e], ws[e + 1]), s2);
            w[e] = r.x;
            w[e + 1] = r.y;
        }
    } else {
#pragma unroll
        for (int e = 0; e < N; ++e) w[e] = ws[e] * sf;
    }
}

// o = a ⊙ b
template <typename T, int N>
__device__ __forceinline__ void mul(const T (&a)[N], const T (&b)[N], T (&o)[N]) {
    if constexpr (sizeof(T) == 4 && N % 2 == 0) {
#pragma unroll
        for (int e = 0; e < N; e += 2) {
            const float2 r = __fmul2_rn(make_float2(a[e], a[e + 1]), make_float2(b[e], b[e + 1]));
            o[e] = r.x;
            o[e + 1] = r.y;
        }
    } else {
#pragma unroll
        for (int e = 0; e < N; ++e) o[e] = a[e] * b[e];
    }
}

// sb += w ⊙ x, sw += w ⊙ w   (fp32: packed FFMA2 pairs)
template <typename T, int N>
__device__ __forceinline__ void accumulate(const T (&w)[N], const T (&x)[N], T (&sb)[N], T (&sw)[N]) {
    if constexpr (sizeof(T) == 4 && N % 2 == 0) {
#pragma unroll
        for (int e = 0; e < N; e += 2) {
            const float2 w2 = make_float2(w[e], w[e + 1]);
            const float2 b = __ffma2_rn(w2, make_float2(x[e], x[e + 1]), make_float2(sb[e], sb[e + 1]));
            const float2 q = __ffma2_rn(w2, w2, make_float2(sw[e], sw[e + 1]));
            sb[e] = b.x;
            sb[e + 1] = b.y;
            sw[e] = q.x;
            sw[e + 1] = q.y;
        }
    } else {
#pragma unroll
        for (int e = 0; e < N; ++e) {
            sb[e] = fma(w[e], x[e], sb[e]);
            sw[e] = fma(w[e], w[e], sw[e]);
        }
    }
}

// Norm accumulators of the refill / objective passes (per run, then fp64): q0 = ‖ΔX‖²,
// q1 = ‖X‖², q2 = ‖X_new − t‖².  fp32 keeps (even, odd) element pairs for packed FFMA2.
template <typename T>
struct Norms3 {
    T q0 = T(0), q1 = T(0), q2 = T(0);
    __device__ double s0() const { return (double)q0; }
    __device__ double s1() const { return (double)q1; }
    __device__ double s2() const { return (double)q2; }
};
template <>
struct Norms3<float> {
    float2 q0 = make_float2(0.f, 0.f), q1 = make_float2(0.f, 0.f), q2 = make_float2(0.f, 0.f);
    __device__ double s0() const { return (double)q0.x + (double)q0.y; }
    __device__ double s1() const { return (double)q1.x + (double)q1.y; }
    __device__ double s2() const { return (double)q2.x + (double)q2.y; }
};

// Eq. 9 on EPL entries (reading R1: per-entry prox minimiser) plus the norm accumulators of
// the stop test and the objective.
template <typename T, int N>
__device__ __forceinline__ void refill_chunk(const T (&x)[N], const T (&t)[N], uint32_t bits, T rho,
                                             T inv1p, T (&xn)[N], Norms3<T>& q) {
    if constexpr (sizeof(T) == 4 && N % 2 == 0) {
        const float2 r2 = make_float2(rho, rho), i2 = make_float2(inv1p, inv1p);
        const float2 m1 = make_float2(-1.f, -1.f);
#pragma unroll
        for (int e = 0; e < N; e += 2) {
            const float2 x2 = make_float2(x[e], x[e + 1]), t2 = make_float2(t[e], t[e + 1]);
            const float2 u = __fmul2_rn(__ffma2_rn(r2, x2, t2), i2);  // (t + ρx)/(1 + ρ)
            xn[e] = ((bits >> e) & 1u) ? x[e] : u.x;
            xn[e + 1] = ((bits >> (e + 1)) & 1u) ? x[e + 1] : u.y;
            const float2 n2 = make_float2(xn[e], xn[e + 1]);
            const float2 d = __ffma2_rn(x2, m1, n2);  // x_new − x
            const float2 g = __ffma2_rn(t2, m1, n2);  // x_new − t
            q.q0 = __ffma2_rn(d, d, q.q0);
            q.q1 = __ffma2_rn(x2, x2, q.q1);
            q.q2 = __ffma2_rn(g, g, q.q2);
        }
    } else {
#pragma unroll
        for (int e = 0; e < N; ++e) {
            const bool obs = (bits >> e) & 1u;
            xn[e] = obs ? x[e] : fma(rho, x[e], t[e]) * inv1p;
            const T d = xn[e] - x[e];
            const T g = xn[e] - t[e];
            q.q0 = fma(d, d, q.q0);
            q.q1 = fma(x[e], x[e], q.q1);
            q.q2 = fma(g, g, q.q2);
        }
    }
}

// Eq. 9 for the fused pass (a5 of sweep s inside a2(0,1) of sweep s+1; only used when the
// sweep loop needs no stop test or trace): X_new plus q1 = ‖X_new‖², kept for the
// non-finite check of the finaliser.
template <typename T, int N>
__device__ __forceinline__ void refill_lite(const T (&x)[N], const T (&t)[N], uint32_t bits, T rho,
                                            T inv1p, T (&xn)[N], Norms3<T>& q) {
    if constexpr (sizeof(T) == 4 && N % 2 == 0) {
        const float2 r2 = make_float2(rho, rho), i2 = make_float2(inv1p, inv1p);
#pragma unroll
        for (int e = 0; e < N; e += 2) {
            const float2 x2 = make_float2(x[e], x[e + 1]), t2 = make_float2(t[e], t[e + 1]);
            const float2 u = __fmul2_rn(__ffma2_rn(r2, x2, t2), i2);  // (t + ρx)/(1 + ρ)
            xn[e] = ((bits >> e) & 1u) ? x[e] : u.x;
            xn[e + 1] = ((bits >> (e + 1)) & 1u) ? x[e + 1] : u.y;
            const float2 n2 = make_float2(xn[e], xn[e + 1]);
            q.q1 = __ffma2_rn(n2, n2, q.q1);
        }
    } else {
#pragma unroll
        for (int e = 0; e < N; ++e) {
            xn[e] = ((bits >> e) & 1u) ? x[e] : fma(rho, x[e], t[e]) * inv1p;
            q.q1 = fma(xn[e], xn[e], q.q1);
        }
    }
}

// objective pass: q2 += (x − t)²
template <typename T, int N>
__device__ __forceinline__ void objective_chunk(const T (&x)[N], const T (&t)[N], Norms3<T>& q) {
    if constexpr (sizeof(T) == 4 && N % 2 == 0) {
        const float2 m1 = make_float2(-1.f, -1.f);
#pragma unroll
        for (int e = 0; e < N; e += 2) {
            const float2 g = __ffma2_rn(make_float2(t[e], t[e + 1]), m1, make_float2(x[e], x[e + 1]));
            q.q2 = __ffma2_rn(g, g, q.q2);
        }
    } else {
#pragma unroll
        for (int e = 0; e < N; ++e) {
            const T g = x[e] - t[e];
            q.q2 = fma(g, g, q.q2);
        }
    }
}

template <typename T, int N>
__device__ __forceinline__ void store_chunk(T* dst, const T (&v)[N], bool full, const bool (&ev)[N]) {
    if (full) {
        stg_vec<T, N>(dst, v);
    } else {
#pragma unroll
        for (int e = 0; e < N; ++e)
            if (ev[e]) dst[e] = v[e];
    }
}

// Ω bits staged in shared memory (PassCfg MASK): `mw` holds the 16-B-aligned word range that
// starts at word (g0 >> 5) & ~3 of the fibre (or stage) whose first element is g0.
__device__ __forceinline__ uint32_t mask_bits_s(const uint32_t* mw, int64_t g0, int64_t ge) {
    const int lb = (int)(ge - (((g0 >> 5) & ~(int64_t)3) << 5));
    return __funnelshift_r(mw[lb >> 5], mw[(lb >> 5) + 1], (uint32_t)(lb & 31));
}

// same with the bit offset lb relative to the staged range's first word
__device__ __forceinline__ uint32_t mask_bits_l(const uint32_t* mw, int lb) {
    return __funnelshift_r(mw[lb >> 5], mw[(lb >> 5) + 1], (uint32_t)(lb & 31));
}

// Producer side: bytes of the aligned word range covering elements [g0, g0 + n) plus the
// funnel word, and its first word.
__device__ __forceinline__ uint32_t mask_span(int64_t g0, int64_t n, int64_t& a0) {
    a0 = (g0 >> 5) & ~(int64_t)3;
    const int64_t a1 = ((((g0 + n - 1) >> 5) + 2) + 3) & ~(int64_t)3;
    return (uint32_t)((a1 - a0) * 4);
}

// Fibre walker: positions pos = v·FR + r of one warp's range, cut into runs (consecutive
// fibres differing only in i_{r0}, at most sf_cap long).  32-bit index arithmetic
// (nfib < 2^31 is checked on the host).
struct Walker {
    int pos, f1, v, seg_end;
    int ridx[MAXN];
    int run_len, fib, ri0;
    bool new_seg, seg_last;
};

template <typename T>
__device__ __forceinline__ void walker_init(Walker& w, const PassParams<T>& P, int f0, int f1) {
    const int FR = (int)P.FR;
    w.pos = f0;
    w.f1 = f1;
    w.v = f0 / FR;
    int rr = f0 - w.v * FR;
#pragma unroll
    for (int j = 0; j < MAXN; ++j) {
        w.ridx[j] = 0;
        if (j < P.nred) {
            w.ridx[j] = rr % (int)P.rdim[j];
            rr /= (int)P.rdim[j];
        }
    }
    w.seg_end = min(f1, (w.v + 1) * FR);
    w.run_len = 0;
    w.fib = 0;
    w.ri0 = 0;
    w.new_seg = true;
    w.seg_last = false;
}

// Move past the current run and describe the next one; false when the range is exhausted.
template <typename T>
__device__ __forceinline__ bool walker_next(Walker& w, const PassParams<T>& P) {
    const bool has_fast = P.nred > 0;
    if (w.run_len > 0) {
        w.pos += w.run_len;
        if (w.pos >= w.seg_end) {
            w.v += 1;
#pragma unroll
            for (int j = 0; j < MAXN; ++j) w.ridx[j] = 0;
            w.seg_end = min(w.f1, (w.v + 1) * (int)P.FR);
            w.new_seg = true;
        } else {
            w.new_seg = false;
            w.ridx[0] += w.run_len;
#pragma unroll
            for (int j = 0; j < MAXN - 1; ++j) {
                if (j + 1 < P.nred && w.ridx[j] >= (int)P.rdim[j]) {
                    w.ridx[j] = 0;
                    w.ridx[j + 1] += 1;
                }
            }
        }
    }
    if (w.pos >= w.f1) return false;
    w.run_len = has_fast ? min(min(w.seg_end - w.pos, (int)P.rdim[0] - w.ridx[0]), P.sf_cap) : 1;
    w.seg_last = w.pos + w.run_len >= w.seg_end;
    int fib = 0;
    if (P.nkept >= 1) fib += (w.v % (int)P.kdim[0]) * (int)P.fstride[P.kmode[0]];
    if (P.nkept >= 2) fib += (w.v / (int)P.kdim[0]) * (int)P.fstride[P.kmode[1]];
#pragma unroll
    for (int j = 0; j < MAXN; ++j)
        if (j < P.nred) fib += w.ridx[j] * (int)P.fstride[P.rmode[j]];
    w.fib = fib;
    w.ri0 = w.ridx[0];
    return true;
}

// The body of one pass for CTA `cta` (the __global__ wrapper below).
template <typename T, int MODE, int EPL, int LPF, bool HRES>
__device__ __forceinline__ void fiber_pass_body(const PassParams<T>& P, unsigned char* smem_raw, int cta) {
    // PASS_FUSED = the a5 refill of sweep s fused with the a2 contraction of block (0,1) of
    // sweep s+1 (same G): X is read once and written once for both.
    constexpr bool kFused = (MODE == PASS_FUSED);
    constexpr bool kContract = (MODE == PASS_KEPT1 || MODE == PASS_RED1 || kFused);
    constexpr bool kNorms = (MODE == PASS_REFILL || MODE == PASS_OBJ || kFused);
    constexpr bool kLoadX = (MODE != PASS_MODEL);
    constexpr bool kMask = (MODE == PASS_REFILL || kFused);
    using Cfg = PassCfg<T, EPL, LPF, HRES, kLoadX, kMask, true>;
    constexpr int D = Cfg::D, F = Cfg::F, FP = Cfg::FP, SR = Cfg::SR, NROW = Cfg::NROW;
    constexpr int STAGE = Cfg::STAGE;  // elements per ring stage (X, H rows, Ω words)
    constexpr int MWF = Cfg::MWF;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nwarps = blockDim.x >> 5;
    const int fsub = lane / LPF;                 // fibre of the step served by this lane
    const int eb = (lane % LPF) * EPL;           // first mode-1 position of this lane
    const int I1p = P.I1p;

    uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw) + warp * D;
    T* sfv = reinterpret_cast<T*>(smem_raw + P.sfv_off) + (size_t)warp * P.sfv_stride;
    T* hres = reinterpret_cast<T*>(smem_raw + P.hres_off);
    T* stg = reinterpret_cast<T*>(smem_raw + P.stage_off) + (size_t)warp * Cfg::RING;

    // Warp setup: zero the ring (row tails past I1p must read as 0) and init the stage
    // barriers; the producer then issues its first D stages BEFORE the CTA loads the resident
    // H_{0,r0} block (HRES), so the first copies' latency overlaps that load.
    for (int e = lane; e < Cfg::RING; e += 32) stg[e] = T(0);
    if (lane == 0)
        for (int s = 0; s < D; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
    fence_proxy_async_smem();
    __syncwarp();

    const int group = cta * nwarps + warp;
    const bool active = group < P.ngroups;

    const uint32_t bar0 = smem_u32(bars);
    const uint32_t stg0 = smem_u32(stg);
    const T* __restrict__ Hb = P.H;
    bool ev[EPL];
#pragma unroll
    for (int e = 0; e < EPL; ++e) ev[e] = eb + e < I1p;
    const bool lane_full = eb + EPL <= I1p;
    const int ebc = eb < I1p ? eb : 0;               // clamped (HRES reads stay in bounds)

    const int f0 = active ? group * (int)P.L : 0;
    const int f1 = active ? min(f0 + (int)P.L, (int)P.nfib) : 0;
    const bool has_fast = P.nred > 0;
    const int fstep = has_fast ? (int)P.fstride[P.rmode[0]] : 0;
    const int64_t xstep = (int64_t)fstep * I1p;      // elements between consecutive fibres
    const int hstep = has_fast ? I1p : 0;            // H_{0,r0} column step (0: ones column)
    const uint32_t rowbytes = (uint32_t)(I1p * sizeof(T));
    const bool xmerge = (SR == I1p) && (fstep == 1);  // F fibres = one contiguous copy
    const bool hmerge = (SR == I1p) && has_fast;

    // ---- producer (lane 0): its own walker, D stages ahead of the consumers --------------
    Walker Pw;
    walker_init(Pw, P, f0, f1);
    int p_left = 0;          // fibres of the producer's current run not yet issued
    uint32_t p_n = 0;        // next stage sequence number
    const T* p_x = P.X;      // next X fibre of the producer's run
    const T* p_h = Hb;       // next H column of the producer's run (!HRES)
    auto produce = [&]() {
        if (p_left == 0) {
            if (!walker_next(Pw, P)) return;
            p_left = Pw.run_len;
            p_x = P.X + (int64_t)Pw.fib * I1p;
            p_h = Hb + (has_fast ? P.vf_off + (int64_t)Pw.ri0 * I1p : P.ones_off);
        }
        const int nf = min(F, p_left);
        const int s = (int)(p_n % (uint32_t)D);
        const uint32_t bar = bar0 + 8u * (uint32_t)s;
        const uint32_t sx = stg0 + (uint32_t)(s * STAGE * (int)sizeof(T));
        fence_stage_refill();
        uint32_t mbytes = 0;
        int64_t ma0 = 0;
        const int64_t pg0 = p_x - P.X;  // first element of the stage's first fibre
        if constexpr (kMask) {
            if (xmerge) {
                mbytes = mask_span(pg0, (int64_t)nf * I1p, ma0);
            } else {
                for (int f = 0; f < nf; ++f) mbytes += mask_span(pg0 + (int64_t)f * xstep, I1p, ma0);
            }
        }
        mbar_arrive_expect_tx_a(bar, (uint32_t)nf * rowbytes * (uint32_t)NROW + mbytes);
        if constexpr (kMask) {
            const uint32_t sm = sx + (uint32_t)(Cfg::XH * (int)sizeof(T));
            if (xmerge) {
                tma_g2s_a(sm, P.mask + ma0, mbytes, bar);
            } else {
                for (int f = 0; f < nf; ++f) {
                    const uint32_t b = mask_span(pg0 + (int64_t)f * xstep, I1p, ma0);
                    IFCTN_CHECK(ma0 + (int64_t)(b / 4) <= P.mask_cap && b <= (uint32_t)(MWF * 4), "plain fibre mask words");
                    tma_g2s_a(sm + (uint32_t)(f * MWF * 4), P.mask + ma0, b, bar);
                }
            }
        }
        IFCTN_CHECK(!kLoadX || (p_x - P.X) + (int64_t)(nf - 1) * xstep + I1p <= P.x_cap, "plain X range");
        IFCTN_CHECK(!kMask || !xmerge || ma0 + (int64_t)(mbytes / 4) <= P.mask_cap, "plain mask words");
        if constexpr (kLoadX) {
            if (xmerge) {
                tma_g2s_a(sx, p_x, (uint32_t)nf * rowbytes, bar);
            } else {
                for (int f = 0; f < nf; ++f)
                    tma_g2s_a(sx + (uint32_t)(f * SR * (int)sizeof(T)), p_x + (int64_t)f * xstep, rowbytes, bar);
            }
            p_x += (int64_t)nf * xstep;
        }
        if constexpr (!HRES) {
            const uint32_t sh = sx + (uint32_t)((kLoadX ? F * SR : 0) * (int)sizeof(T));
            if (hmerge) {
                tma_g2s_a(sh, p_h, (uint32_t)nf * rowbytes, bar);
            } else {
                for (int f = 0; f < nf; ++f)
                    tma_g2s_a(sh + (uint32_t)(f * SR * (int)sizeof(T)), p_h + (int64_t)f * hstep, rowbytes, bar);
            }
            p_h += (int64_t)nf * hstep;
        }
        p_left -= nf;
        ++p_n;
    };
    if (active && lane == 0)
        for (int d = 0; d < D; ++d) produce();
    if constexpr (HRES) {
        const float4* src = reinterpret_cast<const float4*>(P.H + P.hres_src);
        float4* dst = reinterpret_cast<float4*>(hres);
        for (int e = threadIdx.x; e < (int)(P.hres_elems * sizeof(T) / 16); e += blockDim.x) dst[e] = src[e];
    }
    __syncthreads();
    TL_STAMP(1);
    // ---- consumers (all lanes) ---------------------------------------------------------
    double n0 = 0.0, n1 = 0.0, n2 = 0.0;  // REFILL: ‖ΔX‖², ‖X‖², ‖X_new − t‖²; OBJ: n2
    T sb[EPL], sw[EPL];                     // segment accumulators (one kept value v)
    uint32_t cn = 0;                        // next stage to consume
    if (!active) return;
    Walker C;
    walker_init(C, P, f0, f1);
    while (walker_next(C, P)) {
        if (C.new_seg) {
#pragma unroll
            for (int e = 0; e < EPL; ++e) sb[e] = sw[e] = T(0);
        }
        // run setup (rare path): indices of every outer mode, slow factors, sf vector
        // index of outer mode m held by lane m, read with a shuffle (a runtime-indexed local
        // array would live in local memory)
        int midx = 0;
        if (P.nkept >= 1 && lane == P.kmode[0]) midx = C.v % (int)P.kdim[0];
        if (P.nkept >= 2 && lane == P.kmode[1]) midx = C.v / (int)P.kdim[0];
#pragma unroll
        for (int j = 0; j < MAXN; ++j)
            if (j < P.nred && lane == P.rmode[j]) midx = C.ridx[j];
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
        const int len = C.run_len, ri0 = C.ri0;
        {
            // per-run bases of the fast scalar factors (registers), then 32-bit offsets
            const T* sfb[MAXSF];
            int sfi[MAXSF];
#pragma unroll
            for (int t = 0; t < MAXSF; ++t) {
                sfb[t] = Hb;
                sfi[t] = 0;
                if (t < P.nsf) {
                    sfb[t] = Hb + P.sf_off[t] + (int64_t)idx(P.sf_fixmode[t]) * P.sf_fixmul[t] +
                             (int64_t)ri0 * P.sf_inc[t];
                    sfi[t] = (int)P.sf_inc[t];
                }
            }
            for (int q = lane; q < len; q += 32) {
                T f = T(1);
#pragma unroll
                for (int t = 0; t < MAXSF; ++t)
                    if (t < P.nsf) f *= sfb[t][q * sfi[t]];
                sfv[q] = f;
            }
        }
        __syncwarp();
        const int64_t ebase = (int64_t)C.fib * I1p;
        const T* hrun = hres + (HRES && has_fast ? ri0 * I1p : 0) + ebc;
        T h01v[EPL];  // fused: the excluded pair's column H_{0,m}(·, i_m) completes t = M·H_{0,m}
        if constexpr (kFused) {
            const T* hb = Hb + P.h01_off + (int64_t)idx(P.h01_mode) * I1p + eb;
#pragma unroll
            for (int e = 0; e < EPL; ++e) h01v[e] = ev[e] ? hb[e] : T(0);
        }

        Norms3<T> qn;
        // contraction: the run-constant slow factor ws is applied once per run —
        // Σ (ws·u)·x = ws·Σ u·x and Σ (ws·u)² = ws²·Σ u², u = H_{0,r0}·sf per entry
        T rb[EPL], rw[EPL];
#pragma unroll
        for (int e = 0; e < EPL; ++e) rb[e] = rw[e] = T(0);
        for (int off = 0; off < len; off += F) {
            const int nf = min(F, len - off);
            const int s = (int)(cn % (uint32_t)D);
            mbar_wait_a(bar0 + 8u * (uint32_t)s, (cn / (uint32_t)D) & 1u);
            const T* sx = stg + s * STAGE;
            const T* sh = sx + (kLoadX ? F * SR : 0);
            const uint32_t* smw = reinterpret_cast<const uint32_t*>(sx + Cfg::XH);
            const int64_t sg0 = ebase + (int64_t)off * xstep;  // stage's first element
#pragma unroll
            for (int st = 0; st < F / FP; ++st) {
                const int f = st * FP + fsub;
                if (f < nf) {
                    const T sf = sfv[off + f];
                    T h[EPL], w[EPL];
                    if constexpr (HRES) lds_vec<T, EPL>(hrun + (off + f) * hstep, h);
                    else lds_vec<T, EPL>(sh + f * SR + eb, h);
                    if constexpr (MODE == PASS_KEPT1 || MODE == PASS_RED1) scale<T, EPL>(h, sf, w);
                    else weight<T, EPL>(ws, h, sf, w);
                    if constexpr (kFused) {
                        T x[EPL], t[EPL], xn[EPL];
                        lds_vec<T, EPL>(sx + f * SR + eb, x);
#pragma unroll
                        for (int e = 0; e < EPL; ++e) t[e] = w[e] * h01v[e];
                        const int64_t gf = sg0 + (int64_t)f * xstep, ge = gf + eb;
                        const uint32_t bits = xmerge ? mask_bits_s(smw, sg0, ge) : mask_bits_s(smw + f * MWF, gf, ge);
                        if (P.full_norms) refill_chunk<T, EPL>(x, t, bits, P.rho, P.inv1p, xn, qn);
                        else refill_lite<T, EPL>(x, t, bits, P.rho, P.inv1p, xn, qn);
                        store_chunk<T, EPL>(P.Xw + ge, xn, lane_full, ev);
                        accumulate<T, EPL>(w, xn, sb, sw);
                    } else if constexpr (kContract) {
                        T x[EPL];
                        lds_vec<T, EPL>(sx + f * SR + eb, x);
                        accumulate<T, EPL>(w, x, rb, rw);
                    } else if constexpr (MODE == PASS_REFILL) {
                        T x[EPL], xn[EPL];
                        lds_vec<T, EPL>(sx + f * SR + eb, x);
                        const int64_t gf = sg0 + (int64_t)f * xstep, ge = gf + eb;
                        const uint32_t bits = xmerge ? mask_bits_s(smw, sg0, ge) : mask_bits_s(smw + f * MWF, gf, ge);
                        refill_chunk<T, EPL>(x, w, bits, P.rho, P.inv1p, xn, qn);
                        store_chunk<T, EPL>(P.Xw + ge, xn, lane_full, ev);
                    } else if constexpr (MODE == PASS_OBJ) {
                        T x[EPL];
                        lds_vec<T, EPL>(sx + f * SR + eb, x);
                        objective_chunk<T, EPL>(x, w, qn);
                    } else {  // PASS_MODEL: dense user layout, scalar stores
                        const int64_t fb = C.fib + (int64_t)(off + f) * fstep;
#pragma unroll
                        for (int e = 0; e < EPL; ++e)
                            if (eb + e < P.I1) P.out[fb * P.I1 + eb + e] = w[e];
                    }
                }
            }
            __syncwarp();
            ++cn;
            if (lane == 0) produce();
        }
        if constexpr (MODE == PASS_KEPT1 || MODE == PASS_RED1) {
#pragma unroll
            for (int e = 0; e < EPL; ++e) {
                sb[e] = fma(ws[e], rb[e], sb[e]);
                sw[e] = fma(ws[e] * ws[e], rw[e], sw[e]);
            }
        }
        if constexpr (kNorms) {
            n0 += qn.s0();
            n1 += qn.s1();
            n2 += qn.s2();
        }
        __syncwarp();  // sfv is rewritten by the next run
        // ---- flush the segment's partials into slot group + v ---------------------------
        if (C.seg_last) {
            if constexpr (MODE == PASS_KEPT1 || kFused) {
                // lanes serving the same mode-1 positions in different step fibres: sum them
#pragma unroll
                for (int o = 16; o >= LPF; o >>= 1)
#pragma unroll
                    for (int e = 0; e < EPL; ++e) {
                        sb[e] += __shfl_xor_sync(0xffffffffu, sb[e], o);
                        sw[e] += __shfl_xor_sync(0xffffffffu, sw[e], o);
                    }
                if (fsub == 0) {
                    IFCTN_CHECK(((int64_t)group + C.v + 1) * P.Lv <= P.part_cap, "plain KEPT1 slot");
                    T* pbd = P.part_b + ((int64_t)group + C.v) * P.Lv + eb;
                    T* pwd = P.part_w + ((int64_t)group + C.v) * P.Lv + eb;
                    if (lane_full) {
                        stg_vec<T, EPL>(pbd, sb);
                        stg_vec<T, EPL>(pwd, sw);
                    } else {
#pragma unroll
                        for (int e = 0; e < EPL; ++e)
                            if (ev[e]) {
                                pbd[e] = sb[e];
                                pwd[e] = sw[e];
                            }
                    }
                }
            } else if constexpr (MODE == PASS_RED1) {
                T tb = T(0), tw = T(0);
#pragma unroll
                for (int e = 0; e < EPL; ++e) {
                    tb += sb[e];
                    tw += sw[e];
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    tb += __shfl_xor_sync(0xffffffffu, tb, o);
                    tw += __shfl_xor_sync(0xffffffffu, tw, o);
                }
                if (lane == 0) {
                    const int64_t slot = (int64_t)group + C.v;
                    IFCTN_CHECK(slot < P.part_cap, "plain RED1 slot");
                    P.part_b[slot] = tb;
                    P.part_w[slot] = tw;
                }
            }
        }
    }
    if constexpr (kNorms) {
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
    }
}

template <typename T, int MODE, int EPL, int LPF, bool HRES>
__global__ void __launch_bounds__(kPassThreads, kPassMinBlocks) fiber_pass(const __grid_constant__ PassParams<T> P) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    TL_STAMP(0);
    fiber_pass_body<T, MODE, EPL, LPF, HRES>(P, smem_raw, blockIdx.x);
#ifdef IFCTN_EXP_TIMELINE
    __syncthreads();
#endif
    TL_STAMP(2);
}

}  // namespace ifctn
