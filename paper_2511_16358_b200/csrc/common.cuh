// common.cuh — shared constants, vector helpers and parameter blocks of the sm_100a kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdio>

#include "peer.cuh"

#include <type_traits>

namespace ifctn {

#ifdef IFCTN_EXP_TIMELINE  // diagnosis builds only: per-CTA %globaltimer stamps of the passes
static __device__ unsigned long long g_tl[3 * 4096];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define TL_STAMP(q) \
    if (threadIdx.x == 0 && blockIdx.x < 4096) g_tl[3 * blockIdx.x + (q)] = gtimer();
#else
#define TL_STAMP(q)
#endif


constexpr int MAXN = 6;                        // IFCTN_MAX_ORDER
constexpr int MAXP = MAXN * (MAXN - 1) / 2;    // pairs p<q
constexpr int MAXSF = MAXN - 2;                // pairs involving the fast mode r0 (outer)
constexpr int MAXR = 64;                       // IFCTN_MAX_RANK
constexpr int MAXR_SMALL = 9;                   // block_solve (registers) up to here, then block_solve_big
constexpr int kPassThreads = 256;              // fiber-pass CTA size
constexpr int kPassMinBlocks = 2;              // ≤ 128 registers: ≥ 16 warps per SM
#ifndef IFCTN_RING_D
#define IFCTN_RING_D 3
#endif
constexpr int kRingStages = IFCTN_RING_D;      // TMA ring depth per warp (stages in flight)

// Compile-time shape of one fibre-pass instance (fiber_pass.cuh): EPL mode-1 positions per
// lane, LPF lanes per fibre (FP = 32/LPF fibres per warp step), ring rows per fibre (X and,
// without a resident H block, the H column), F fibres per TMA stage (≈ 2 KB), D stages.
// MASK (refill passes): each stage also carries the Ω bit words of its fibres, MWF 32-bit
// words per fibre slot (16-B aligned copies that cover the fibre's bits plus the funnel
// word), or the whole stage's bits in one copy when its fibres are contiguous.
#ifndef IFCTN_PLAIN_STAGE
#define IFCTN_PLAIN_STAGE 4096
#endif
#ifndef IFCTN_PLAIN_D
#define IFCTN_PLAIN_D 2
#endif
// PLAIN: the plain fibre walk (its accumulators do not grow with F, so its stage size and
// ring depth are set separately: IFCTN_PLAIN_STAGE bytes, IFCTN_PLAIN_D stages)
template <typename T, int EPL, int LPF, bool HRES, bool LOADX, bool MASK = false, bool PLAIN = false>
struct PassCfg {
    static constexpr int FP = 32 / LPF;
    static constexpr int SR = LPF * EPL;  // shared-memory row stride (elements)
    static constexpr int NROW = (LOADX ? 1 : 0) + (HRES ? 0 : 1);
    static constexpr int ROWB = SR * (int)sizeof(T);
    static constexpr int SB = PLAIN ? IFCTN_PLAIN_STAGE : 2048;
    static constexpr int FK = (SB / (NROW > 0 ? NROW : 1) / ROWB) / FP;
    static constexpr int F = FP * (FK > 1 ? FK : 1);
    static constexpr int D = PLAIN ? IFCTN_PLAIN_D : kRingStages;
    static constexpr int XH = NROW * F * SR;                       // X/H elements per stage
    static constexpr int MWF = MASK ? ((SR / 32 + 9 + 3) & ~3) : 0;  // mask words per fibre
    static constexpr int MW = F * MWF;                             // mask words per stage
    static constexpr int STAGE = XH + MW * 4 / (int)sizeof(T);     // elements per stage
    static constexpr int RING = D * STAGE;                         // ring elements per warp
};

enum PassMode : int {
    PASS_KEPT1 = 0,   // a2, mode 1 (code mode 0) is one of the kept modes {k,i}
    PASS_RED1 = 1,    // a2, mode 1 is reduced
    PASS_REFILL = 2,  // a5: X update + norms
    PASS_OBJ = 3,     // f = ½‖X − t‖² only
    PASS_MODEL = 4,   // write t = iFCTN(G) in the user layout
    PASS_FUSED = 5,   // a5 of sweep s fused with a2 of block (0,1) of sweep s+1 (KEPT1 layout)
};

template <typename T> struct VecT;
template <> struct VecT<float> {
    using V = float4;
    static constexpr int W = 4;
    __device__ static inline void get(const V& v, float* o) { o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w; }
    __device__ static inline V make(const float* o) { return make_float4(o[0], o[1], o[2], o[3]); }
};
template <> struct VecT<double> {
    using V = double2;
    static constexpr int W = 2;
    __device__ static inline void get(const V& v, double* o) { o[0] = v.x; o[1] = v.y; }
    __device__ static inline V make(const double* o) { return make_double2(o[0], o[1]); }
};

template <typename T>
__device__ __forceinline__ typename VecT<T>::V zero_v() {
    T z[VecT<T>::W];
#pragma unroll
    for (int e = 0; e < VecT<T>::W; ++e) z[e] = T(0);
    return VecT<T>::make(z);
}

// Streaming 16-B load of X that must not displace the (small, reused) H/G working set in L1.
__device__ __forceinline__ float4 ld_stream(const float4* p) {
    float4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
    return r;
}
__device__ __forceinline__ double2 ld_stream(const double2* p) {
    double2 r;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];"
                 : "=d"(r.x), "=d"(r.y) : "l"(p));
    return r;
}

// ---- debug builds (IFCTN_DEBUG_CHECKS): device-side bounds checks on the computed indices
// of partial slots, TMA source ranges and mask words (compute-sanitizer is not available on
// the B200 pool); a failed check prints and traps the kernel.
#ifdef IFCTN_DEBUG_CHECKS
#define IFCTN_CHECK(cond, what)                                                              \
    do {                                                                                     \
        if (!(cond)) {                                                                       \
            printf("IFCTN_CHECK failed: %s (%s:%d) block %d thread %d\n", what, __FILE__,     \
                   __LINE__, (int)blockIdx.x, (int)threadIdx.x);                             \
            __trap();                                                                        \
        }                                                                                    \
    } while (0)
#else
#define IFCTN_CHECK(cond, what) \
    do {                        \
    } while (0)
#endif

// ---- TMA bulk copies + mbarriers (sm_90+ PTX; UBLKCP / SYNCS in sm_100a SASS) -------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_inval(uint64_t* bar) {
    asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// Before a TMA refills a ring slot the consumers only READ (their loads have retired: the
// values were used before the __syncwarp that precedes the refill), so no proxy fence is
// needed there; IFCTN_STAGE_FENCE restores it for experiments.
__device__ __forceinline__ void fence_stage_refill() {
#ifdef IFCTN_STAGE_FENCE
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
#endif
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
// global → shared bulk copy (TMA engine), completion counted on `bar` in bytes
__device__ __forceinline__ void tma_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// Blocking wait for phase `parity` of `bar`; the suspend-time hint lets the hardware park the
// warp until the phase completes instead of spinning on issue slots.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity), "r"(1000000u)
            : "memory");
    } while (!done);
}

// 32-bit shared-address variants (no generic→shared conversion in the hot loop)
__device__ __forceinline__ void mbar_arrive_expect_tx_a(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_g2s_a(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void mbar_wait_a(uint32_t bar, uint32_t parity) {
    uint32_t done;
    do {
#ifdef IFCTN_SPIN_WAIT
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(bar), "r"(parity)
            : "memory");
#else
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(bar), "r"(parity), "r"(1000000u)
            : "memory");
#endif
    } while (!done);
}

// ---- programmatic dependent launch (sm_90+): a kernel launched with the programmatic stream
// serialization attribute starts while its predecessor still runs; pdl_wait() blocks until the
// predecessor grid has completed and its memory is visible, pdl_launch() lets the successor's
// CTAs be scheduled.  Rule used here: wait FIRST, then launch — so everything older than the
// direct predecessor is complete when a kernel passes its wait, and only work that does not
// touch the predecessor's outputs (index arithmetic) sits before the wait.  Without the launch
// attribute both are no-ops.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// One fiber pass = one streaming sweep over the (local) X in fibre order.  A "fibre" is a
// mode-1 line X(:, i_2, …, i_N) stored contiguously with I1p ≥ I1 padded entries (pad = 0).
// Fibres are enumerated as pos = v·FR + r, v over the kept outer modes, r over the reduced
// outer modes in odometer order rmode[0] (fastest, "r0") … rmode[nred-1].
template <typename T>
struct PassParams {
    const T* H;          // all pairwise Grams H_{p,q} (p<q) in one buffer; H_{p,q}(a,b) at
    int64_t hsize;       //   off_{pq} + b·ld_p + a, ld_0 = I1p (pad rows zero), ld_p = I_p
    const T* X;          // internal padded X
    T* Xw;               // PASS_REFILL: X, updated in place
    const uint32_t* mask;// bit e of the padded layout = observed (pad bits = 1)
    T* part_b;           // PASS_KEPT1/RED1 partial slots, slot = group + v, Lv values each
    T* part_w;
    double* norms;       // PASS_REFILL/OBJ: 3 doubles per group
    T* out;              // PASS_MODEL: dense user layout
    T rho, inv1p;        // ρ and 1/(1+ρ)
    int I1, I1p;
    int64_t nfib, L, ngroups, NV, FR, Lv;
    int nkept;
    int kmode[2];
    int64_t kdim[2];
    int nred;
    int rmode[MAXN];
    int64_t rdim[MAXN];
    int64_t fstride[MAXN];   // fibre-index stride of each outer mode (index by mode)
    int nouter;              // N − 1
    // weight factors, classified on the host relative to r0
    int nvs;                 // slow vector factors H_{0,q}, q ≠ r0: column idx[q] of H_{0,q}
    int64_t vs_off[MAXN];
    int vs_mode[MAXN];
    int64_t vf_off;          // fast vector factor H_{0,r0} (valid iff nred > 0)
    int nss;                 // slow scalar factors H_{p,q}(i_p,i_q), p,q outer, ≠ r0
    int64_t ss_off[MAXP];
    int64_t ss_ld[MAXP];
    int ss_p[MAXP], ss_q[MAXP];
    int nsf;                 // fast scalar factors: pairs {r0, m}: H + off + idx[m]·mul + i_r0·inc
    int64_t sf_off[MAXSF];
    int sf_fixmode[MAXSF];
    int64_t sf_fixmul[MAXSF];
    int64_t sf_inc[MAXSF];
    int64_t ones_off;        // a column of I1p ones in H (the "fast factor" when nred == 0)
    int sf_cap;              // per-warp shared-memory slots for the fast scalar factors
    int64_t sfv_off, hres_off, stage_off;  // byte offsets in dynamic shared memory
    int64_t hres_src, hres_elems;          // resident H block (HRES): offset in H, elements
    // v-blocking (fiber_pass_vb only): mode 1 (code mode 1, fibre stride 1) is kept; runs are
    // F consecutive fibres i_1 ∈ [b·F, b·F+F) at one reduced position r; positions are
    // ((vb·FR + r)·F + f), vb = b + nb0·kidx1.
    int64_t nb0;
    int64_t vf2_off, hres2_elems;  // tiled pass: resident H_{0,r0} block after H_{0,1}
    int64_t h01_off, hres3_elems;  // fused pass: H_{0,m} of the first block's pair {0,m}
    int h01_mode;                  // (global offset; resident when tiled, m = 1), and m
    // tiled pass: scalar factors touching mode 1 (A: H_{1,q}, q fixed in the tile), r0 (B: the
    // sf_* lists) or both (C: H_{1,r0}, -1 when {1,r0} is the kept pair); value of an entry is
    // H[off + idx[fix]·mul + x·inc] with x = v (A) or i_{r0} (B)
    int nta;
    int64_t ta_off[MAXSF], ta_mul[MAXSF], ta_inc[MAXSF];
    int ta_fix[MAXSF];
    int64_t tc_off, tc_ld;
    int64_t sfv_stride;            // per-warp elements of the sf scratch
    unsigned* sched;               // tiled pass: [next chunk, retired warps], zero between launches
    int full_norms;                // fused pass: all three norms (traced sweeps), else ‖X_new‖² only
    int64_t part_cap, x_cap, mask_cap;  // element / word capacities (IFCTN_DEBUG_CHECKS)
};

template <typename T>
struct ReduceParams {
    const T* part_b;
    const T* part_w;
    double* beta;        // I_i × I_k column-major (a fastest)
    double* omega;
    int64_t FR, L, NV, Lv;
    int kept1;           // 1: KEPT1 layout, 0: RED1
    int I1;              // real mode-1 size (KEPT1)
    int64_t Ii;          // output leading dimension
    int kIsMode0;        // KEPT1: k == 0 (j = i_1, a = v) else (a = i_1, j = v)
    int kmode0IsK;       // RED1: kmode[0] == k
    int64_t kdim0;
    int64_t VB, nb0;     // v-blocking: block width (1 = off), blocks along kmode[0]
    // grid = (NV, ntile, Z): CTA (v, tile, z) sums elements [tile·ET, tile·ET+ET) of v over
    // its z-th share of the slots; Z > 1 combines the Z partials in z order in the last CTA
    // to arrive (scr/cnt), so the sum order is fixed for a given Z.
    int ET, ntile, Z;
    int64_t part_cap;    // partial-slot capacity (IFCTN_DEBUG_CHECKS)
    double* scr;         // ≥ NV·ntile·Z·ET·2 doubles when Z > 1
    unsigned* cnt;       // ≥ NV·ntile counters, zero between launches
};

template <typename T>
struct SolveParams {
    const double* beta;
    const double* omega;
    T* Gki;              // R × I_k (local columns)
    const T* Gik;        // R × I_i
    T* H;                // Hall
    int64_t h_off, h_ld; // H_{min,max}
    int k_lt_i;          // k < i: H(j,a) at a·ld + j; else H(a,j) at j·ld + a
    int64_t Ik, Ii;
    double rho;
    double* delta;       // per column ‖c_new − c_old‖²
    int* flags;          // flags[0] |= 1 on a non-positive pivot
    double* proj;        // multi-GPU: per column [Gram upper triangle, rhs] partials
    int use_peer;        // multi-GPU over peer memory (peer.cuh): PROJECT writes the exchange
    PeerCtx peer;        //   slot, FROM_PROJ publishes, waits and sums the ranks' slots itself
    int R;               // R_{k,i} (block_solve_big; block_solve has it as a template argument)
    int fused_reduce;    // block_solve: sum β(a,j), ω(a,j) from the a2 partial slots itself
    ReduceParams<T> red; //   (the reduce_partials launch of the block is then skipped)
    int ta;              // block_solve_big: columns a of G_{i,k} staged at once (≥ I_i: all)
    int mma;             // block_solve_big on the fp64 tensor cores: bit 0 — Gram/RHS (big_gram_mma; 9 < R ≤ 39),
                         //   bit 1 — the H-row refresh (any R)
};

}  // namespace ifctn
