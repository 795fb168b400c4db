// ifctn.cu — host orchestration and the C-ABI (include/ifctn.h) of the B200 iFCTN-TC PAM
// sweep.  One translation unit; built with
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -shared -Xcompiler -fPIC
// Everything the sweep computes runs in the kernels of fiber_pass.cuh and solve.cuh; this
// file validates arguments, lays out the workspace, plans the passes (grid sizes, fibre
// enumeration, weight-factor lists), enqueues the sweep and captures it as a CUDA graph.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/ifctn.h"
#include "common.cuh"
#include "fiber_walk.cuh"
#include "fiber_tile.cuh"
#include "l2pass.cuh"
#include "solve.cuh"
#include "metrics.cuh"
#include "nccl_lite.h"

namespace ifctn {

static const char* kStatusNames[] = {
    "IFCTN_OK", "IFCTN_E_ARG", "IFCTN_E_SHAPE", "IFCTN_E_RANKS", "IFCTN_E_WORKSPACE",
    "IFCTN_E_CUDA", "IFCTN_E_NCCL", "IFCTN_E_NOT_SPD", "IFCTN_E_NONFINITE", "IFCTN_E_STATE",
    "IFCTN_E_UNSUPPORTED", "IFCTN_E_NO_OBSERVED"};

struct Error {
    ifctn_status st;
    std::string msg;
};

#define CU(expr)                                                                           \
    do {                                                                                   \
        cudaError_t _e = (expr);                                                           \
        if (_e != cudaSuccess)                                                             \
            throw ::ifctn::Error{IFCTN_E_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)}; \
    } while (0)

static void fail(ifctn_status st, const std::string& m) { throw Error{st, m}; }

static int64_t align_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }
static int pow2ceil(int x) {
    int p = 1;
    while (p < x) p <<= 1;
    return p;
}

constexpr int64_t kGroupBoundThreads = 160LL * 2048;  // ≥ resident threads of any B200 part
constexpr unsigned kFlagNoVBlock = IFCTN_FLAG_NO_VBLOCK;
constexpr unsigned kFlagNoFuse = IFCTN_FLAG_NO_FUSE;

// ------------------------------------------------------------------------------------------
// Shape: everything derivable from the arguments alone (no device needed).
// ------------------------------------------------------------------------------------------
struct Shape {
    int N = 0;
    int64_t dims[MAXN] = {};
    int32_t ranks[MAXN * MAXN] = {};
    ifctn_dtype dtype = IFCTN_F32;
    int64_t esize = 4;
    int vw = 4;
    // distribution
    int rank = 0, world = 1, shard = 0;
    bool dpath = false;  // distributed code path (world > 1, or a 1-rank comm / hook)
    bool peer = false;   // exchange over peer memory (peer.cuh) instead of NCCL
    int64_t sbegin = 0, send = 0;
    int64_t ld[MAXN] = {};  // local dims
    // layout
    int64_t I1 = 0, I1p = 0, nfib = 0, npad = 0, nloc = 0, nglob = 0;
    int64_t fstride[MAXN] = {};
    int64_t goff[MAXN][MAXN] = {};
    int64_t gtotal = 0;
    int64_t hoff[MAXN][MAXN] = {};  // p<q
    int64_t hld[MAXN] = {};
    int64_t htotal = 0, ones_off = 0;
    int epl = 0, lpf = 0, sf_cap = 0;  // see fiber_pass.cuh / PassCfg
    int64_t part_elems = 0, max_bw = 0, ndelta = 0, groups_bound = 0;
    int64_t delta_off[MAXN][MAXN] = {};
    int64_t proj_elems = 0;  // multi-GPU projected Gram/RHS buffer (doubles)
    // Internal mode order.  Everything above is in INTERNAL numbering: internal mode m is API
    // mode perm[m].  The identity unless the shard mode is API mode 0 (the lane/fibre mode of
    // every pass, which a shard would cut to I_0/W): then the two largest middle modes become
    // internal modes 0 (lane) and 1 (run/tile mode), the rest follow in API order and the last
    // mode stays last (bands stay the slowest mode), so each rank's passes see the long
    // fibres and runs of the unsharded tensor.  The block order, the factor layout and every
    // dense tensor at the boundary stay in API numbering (see Solver).
    int perm[MAXN] = {};
    bool permuted = false;
    int shard_api = 0;          // shard mode in API numbering
    int64_t eld[MAXN] = {};     // API-order local dims
    int64_t egoff[MAXN][MAXN] = {};  // API-order factor offsets (ABI layout)

    int R(int p, int q) const { return ranks[p * N + q]; }
};

static void shard_range_of(int64_t I, int world, int rank, int64_t* b, int64_t* e) {
    // ranks get ⌈I/W⌉ then ⌊I/W⌋ (reading R21): the first I mod W ranks get one extra.
    const int64_t base = I / world, extra = I % world;
    *b = rank * base + std::min<int64_t>(rank, extra);
    *e = *b + base + (rank < extra ? 1 : 0);
}

static Shape make_shape(int order, const int64_t* dims, const int32_t* ranks, ifctn_dtype dtype,
                        const ifctn_dist* dist) {
    Shape s;
    if (!dims || !ranks) fail(IFCTN_E_ARG, "dims/ranks must not be NULL");
    if (order < 2 || order > MAXN) fail(IFCTN_E_SHAPE, "order must be in [2, IFCTN_MAX_ORDER]");
    if (dtype != IFCTN_F32 && dtype != IFCTN_F64) fail(IFCTN_E_ARG, "dtype must be IFCTN_F32 or IFCTN_F64");
    s.N = order;
    s.dtype = dtype;
    s.esize = dtype == IFCTN_F32 ? 4 : 8;
    s.vw = dtype == IFCTN_F32 ? 4 : 2;
    double prodd = 1.0;
    for (int m = 0; m < order; ++m) {
        if (dims[m] < 1) fail(IFCTN_E_SHAPE, "every dim must be >= 1");
        s.dims[m] = dims[m];
        prodd *= (double)dims[m];
    }
    if (prodd > 4.0e18) fail(IFCTN_E_SHAPE, "tensor too large");
    for (int p = 0; p < order; ++p)
        for (int q = 0; q < order; ++q) {
            const int32_t r = ranks[p * order + q];
            if (p == q) {
                if (r != 0) fail(IFCTN_E_RANKS, "rank matrix diagonal must be 0");
            } else {
                if (r != ranks[q * order + p]) fail(IFCTN_E_RANKS, "rank matrix must be symmetric");
                if (r < 1) fail(IFCTN_E_RANKS, "off-diagonal ranks must be >= 1");
                if (r > MAXR) fail(IFCTN_E_UNSUPPORTED, "ranks above IFCTN_MAX_RANK are not supported by this build");
            }
            s.ranks[p * order + q] = r;
        }
    // distribution
    if (dist && dist->world > 1) {
        if (dist->rank < 0 || dist->rank >= dist->world) fail(IFCTN_E_ARG, "dist rank out of range");
        s.world = dist->world;
        s.rank = dist->rank;
        int sm = dist->shard_mode;
        if (sm < 0) {  // the largest mode, the first on ties
            sm = 0;
            for (int m = 1; m < order; ++m)
                if (dims[m] > dims[sm]) sm = m;
        }
        if (sm >= order) fail(IFCTN_E_ARG, "shard_mode out of range");
        if (dims[sm] < dist->world) fail(IFCTN_E_SHAPE, "shard mode smaller than the world size");
        s.shard = sm;
    } else {
        s.world = 1;
        s.rank = 0;
        s.shard = 0;
    }
    // a single rank with a communicator (or host hook) runs the distributed code path too:
    // projections, all-reduces (1-rank NCCL) and split finalisers — used to test the path
    s.dpath = dist && (dist->world > 1 || dist->nccl_unique_id || dist->host_allreduce ||
                       dist->exchange == IFCTN_XCHG_PEER);
    s.peer = s.dpath && dist->exchange == IFCTN_XCHG_PEER;
    if (dist && dist->exchange != IFCTN_XCHG_NCCL && dist->exchange != IFCTN_XCHG_PEER)
        fail(IFCTN_E_ARG, "dist->exchange must be IFCTN_XCHG_NCCL or IFCTN_XCHG_PEER");
    if (s.peer && (dist->world > kPeerMax)) fail(IFCTN_E_UNSUPPORTED, "peer exchange supports at most 16 ranks");
    if (s.dpath && dist->world == 1) {
        if (dist->rank != 0) fail(IFCTN_E_ARG, "dist rank out of range");
        int sm = dist->shard_mode < 0 ? 0 : dist->shard_mode;
        if (sm >= order) fail(IFCTN_E_ARG, "shard_mode out of range");
        s.shard = sm;
    }
    shard_range_of(s.dims[s.shard], s.world, s.rank, &s.sbegin, &s.send);
    for (int m = 0; m < order; ++m) s.ld[m] = s.dims[m];
    s.ld[s.shard] = s.send - s.sbegin;
    // API-order views, then the internal mode order (see Shape::perm)
    s.shard_api = s.shard;
    for (int m = 0; m < order; ++m) {
        s.eld[m] = s.ld[m];
        s.perm[m] = m;
    }
    {
        int64_t off = 0;
        for (int k = 0; k < order; ++k)
            for (int i = 0; i < order; ++i) {
                if (i == k) continue;
                s.egoff[k][i] = off;
                off += (int64_t)s.R(k, i) * s.eld[k];
            }
    }
    if (s.dpath && s.shard == 0 && order >= 3) {
        // internal order: [m1, m2, the other modes ascending, N-1] with m1, m2 the largest of
        // the middle modes 1..N-2 (first on ties) when longer than the shard slice; m2 makes
        // internal mode 1 (the run / tile mode of the passes, fibre stride 1) long as well
        int m1 = 1;
        for (int q = 2; q <= order - 2; ++q)
            if (s.eld[q] > s.eld[m1]) m1 = q;
        if (s.eld[m1] > s.eld[0]) {
            int m2 = -1;
            for (int q = 1; q <= order - 2; ++q)
                if (q != m1 && (m2 < 0 || s.eld[q] > s.eld[m2])) m2 = q;
            if (m2 >= 0 && !(s.eld[m2] > s.eld[0])) m2 = -1;
            int t = 0;
            s.perm[t++] = m1;
            if (m2 >= 0) s.perm[t++] = m2;
            for (int q = 0; q < order - 1; ++q)
                if (q != m1 && q != m2) s.perm[t++] = q;
            s.perm[t++] = order - 1;
            s.permuted = true;
            int32_t rk[MAXN * MAXN];
            for (int p = 0; p < order; ++p)
                for (int q = 0; q < order; ++q) rk[p * order + q] = s.ranks[s.perm[p] * order + s.perm[q]];
            for (int p = 0; p < order * order; ++p) s.ranks[p] = rk[p];
            for (int p = 0; p < order; ++p) {
                s.dims[p] = dims[s.perm[p]];
                s.ld[p] = s.eld[s.perm[p]];
                if (s.perm[p] == 0) s.shard = p;  // internal index of API mode 0
            }
        }
    }

    s.I1 = s.ld[0];
    s.I1p = align_up(s.I1, s.vw);
    s.nfib = 1;
    for (int m = 1; m < order; ++m) s.nfib *= s.ld[m];
    if (s.nfib >= (1LL << 31)) fail(IFCTN_E_UNSUPPORTED, "more than 2^31 mode-1 fibres per shard");
    s.npad = s.nfib * s.I1p;
    s.nloc = s.nfib * s.I1;
    s.nglob = (int64_t)prodd;
    s.fstride[0] = 0;
    int64_t st = 1;
    for (int m = 1; m < order; ++m) {
        s.fstride[m] = st;
        st *= s.ld[m];
    }
    // factors (local columns for the shard-mode chain)
    int64_t off = 0;
    for (int k = 0; k < order; ++k)
        for (int i = 0; i < order; ++i) {
            if (i == k) continue;
            s.goff[k][i] = off;
            off += (int64_t)s.R(k, i) * s.ld[k];
        }
    s.gtotal = off;
    // pairwise Grams, each block padded to the vector width
    off = 0;
    for (int p = 0; p < order; ++p) s.hld[p] = (p == 0) ? s.I1p : s.ld[p];
    for (int p = 0; p < order; ++p)
        for (int q = p + 1; q < order; ++q) {
            s.hoff[p][q] = off;
            off += align_up(s.hld[p] * s.ld[q], s.vw);
        }
    s.ones_off = off;  // a column of I1p ones (see PassParams::ones_off)
    off += s.I1p;
    s.htotal = off;
    // lane mapping
    // one warp per fibre stream: FP = 32/LPF fibres per step, lane serves EPL positions
    // (the instantiated (EPL, LPF) pairs of fiber_pass.cuh)
    if (s.esize == 4) {
        if (s.I1p <= 64) { s.epl = 4; s.lpf = 16; }
        else if (s.I1p <= 128) { s.epl = 4; s.lpf = 32; }
        else if (s.I1p <= 256) { s.epl = 8; s.lpf = 32; }
        else if (s.I1p <= 512) { s.epl = 16; s.lpf = 32; }
        else fail(IFCTN_E_UNSUPPORTED, "mode-1 size above 512 (f32) per shard is not supported by this build");
    } else {
        if (s.I1p <= 32) { s.epl = 2; s.lpf = 16; }
        else if (s.I1p <= 64) { s.epl = 2; s.lpf = 32; }
        else if (s.I1p <= 128) { s.epl = 4; s.lpf = 32; }
        else if (s.I1p <= 256) { s.epl = 8; s.lpf = 32; }
        else fail(IFCTN_E_UNSUPPORTED, "mode-1 size above 256 (f64) per shard is not supported by this build");
    }
    s.groups_bound = std::min<int64_t>(s.nfib, kGroupBoundThreads / 32);
    {
        int64_t mx = 1;
        for (int m = 1; m < order; ++m) mx = std::max(mx, s.ld[m]);
        s.sf_cap = (int)std::max<int64_t>(8, std::min<int64_t>(256, mx));
    }
    // partial slots: max over contract passes of (groups + NV) * Lv
    int64_t pmax = 0, bw = 0, nd = 0;
    for (int k = 0; k < order; ++k)
        for (int i = 0; i < order; ++i) {
            if (i == k) continue;
            int64_t NV = 1;
            for (int m = 1; m < order; ++m)
                if (m == k || m == i) NV *= s.ld[m];
            const bool kept1 = (k == 0 || i == 0);
            const int64_t Lv = kept1 ? s.I1p : 1;
            int64_t slots = s.groups_bound + NV;
            if (order >= 2 && (k == 1 || i == 1)) {  // v-blocked pass: (groups + NVB)·F, F ≤ 8
                const int64_t kdim1 = NV / s.ld[1];
                slots = s.groups_bound * 8 + NV + 8 * kdim1;
            }
            pmax = std::max(pmax, slots * Lv);
            bw = std::max(bw, s.ld[i] * s.ld[k]);
        }
    // ΔG² slots per block, the shard-mode chains LAST: the replicated entries then sit at the
    // same positions on every rank (finalize_norms sums them in the same order everywhere)
    for (int pass = 0; pass < 2; ++pass)
        for (int k = 0; k < order; ++k)
            for (int i = 0; i < order; ++i) {
                if (i == k || (pass == 0) == (s.dpath && k == s.shard)) continue;
                s.delta_off[k][i] = nd;
                nd += s.ld[k];
            }
    s.part_elems = align_up(pmax, s.vw);
    s.max_bw = bw;
    s.ndelta = nd;
    // projected Gram/RHS for the allreduce: max over blocks of I_k·(R(R+1)/2 + R)
    int64_t pe = 0;
    for (int k = 0; k < order; ++k)
        for (int i = 0; i < order; ++i)
            if (i != k) {
                const int64_t R = s.R(k, i);
                pe = std::max(pe, s.ld[k] * (R * (R + 1) / 2 + R));
            }
    s.proj_elems = pe + 8;
    return s;
}

struct Layout {
    int64_t x, bits, g, h, pb, pw, beta, omega, delta, norms, scal, flags, rse, proj, rscr, rcnt, sched, total;
};

// split-slot reduce (reduce_partials with Z > 1): scratch doubles and arrival counters
constexpr int64_t kRedScr = 2 * 2048 * 32 * 2;
constexpr int64_t kRedCnt = 8192;

static Layout make_layout(const Shape& s) {
    Layout L{};
    int64_t o = 0;
    auto take = [&](int64_t bytes) {
        const int64_t r = o;
        o = align_up(o + std::max<int64_t>(bytes, 1), 256);
        return r;
    };
    L.x = take(s.npad * s.esize);
    L.bits = take((align_up((s.npad + 31) / 32, 8) + 8) * 4);  // +8 words: 2-word funnel reads
    L.g = take(s.gtotal * s.esize);
    L.h = take(s.htotal * s.esize);
    L.pb = take(s.part_elems * s.esize);
    L.pw = take(s.part_elems * s.esize);
    L.beta = take(s.max_bw * 8);
    L.omega = take(s.max_bw * 8);
    L.delta = take(s.ndelta * 8);
    L.norms = take(s.groups_bound * 3 * 8);
    L.scal = take(16 * 8);
    L.flags = take(4 * 4);
    L.rse = take(2 * 1024 * 8 + 16);
    L.proj = take(s.proj_elems * 8);
    L.rscr = take(kRedScr * 8);
    L.rcnt = take(kRedCnt * 4);
    L.sched = take(64);
    L.total = o;
    return L;
}

static bool is_device_ptr(const void* p) {
    if (!p) return false;
    cudaPointerAttributes a;
    cudaError_t e = cudaPointerGetAttributes(&a, p);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// Device-addressable view of p: p itself for device/managed memory, the mapped device address
// for pinned (page-locked) host memory — kernels then read/write it directly over the host
// link with no staging copy — and nullptr for pageable host memory.
static void* device_view(const void* p) {
    if (!p) return nullptr;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    if (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) return const_cast<void*>(p);
    if (a.type == cudaMemoryTypeHost && a.devicePointer) return a.devicePointer;
    return nullptr;
}

// ------------------------------------------------------------------------------------------
// Solver<T>
// ------------------------------------------------------------------------------------------
struct SolverBase {
    virtual ~SolverBase() {}
    virtual void sweep(int t_max, double eps, int* done, ifctn_trace_row* trace) = 0;
    virtual void sync_check() = 0;
    virtual int profile_sweep(float* ms, int cap) = 0;
    virtual void reconstruct(int what, void* out) = 0;
    virtual void get_factors(void* out) = 0;
    virtual double rse(const void* truth) = 0;
    virtual void metrics(const void* truth, double* out4) = 0;
    virtual double objective() = 0;
    virtual void block_coefficients(int k, int i, double* beta, double* omega) = 0;
    virtual void block_update(int k, int i) = 0;
    virtual void x_update(double* norms) = 0;
    virtual int64_t launches() const = 0;
};

template <typename T>
struct PassPlan {
    PassParams<T> p;
    const void* fn = nullptr;
    dim3 grid;
    size_t smem = 0;
};

struct RedLaunch {
    const void* fn = nullptr;
    dim3 grid;
};

template <typename T>
struct BlockPlan {
    int k = 0, i = 0;
    bool vblk = false;
    PassPlan<T> pass;
    ReduceParams<T> red;
    RedLaunch red_l;
    SolveParams<T> sol;
    dim3 sol_grid;
    unsigned sol_threads = 128;
    size_t sol_smem = 0;
    const void* sol_fn = nullptr;
    // L2-resident tensors: the per-kept-value contraction (l2pass.cuh) instead of pass+reduce
    bool l2 = false;
    L2Params<T> l2p;
    const void* l2_fn = nullptr;
    dim3 l2_grid;
    size_t l2_smem = 0;
    // large ranks on one GPU: Gram/RHS of all columns by gram_project, then the FROM_PROJ solve
    bool gemm = false;
    SolveParams<T> gram_sol;
    dim3 gram_grid;
    size_t gram_smem = 0;
    // multi-GPU, k ≠ shard mode: project → all-reduce → solve
    bool dist = false;
    const void* proj_fn = nullptr;
    int64_t proj_count = 0;  // doubles summed across ranks
};

// (kernel, ring elements per warp) of one instantiated (T, MODE, EPL, LPF, HRES)
struct PassKernel {
    const void* fn;
    int64_t ring;
    int F;
};

// MODE >= 100: the v-blocked contraction kernel for MODE - 100
template <typename T, int MODE, int EPL, int LPF, bool HRES>
static PassKernel pk() {
    constexpr int M0 = MODE % 100;
    using Cfg = PassCfg<T, EPL, LPF, HRES, M0 != PASS_MODEL, M0 == PASS_REFILL || M0 == PASS_FUSED, (MODE < 100)>;
    if constexpr (MODE >= 100) {
        constexpr int M = MODE - 100;
        if constexpr ((M == PASS_KEPT1 || M == PASS_RED1 || M == PASS_FUSED) && HRES)
            return {(const void*)fiber_pass_vb<T, M, EPL, LPF, HRES>, Cfg::RING, Cfg::F};
        return {nullptr, 0, 0};
    } else {
        return {(const void*)fiber_pass<T, MODE, EPL, LPF, HRES>, Cfg::RING, Cfg::F};
    }
}

template <typename T, int MODE, bool HRES>
static PassKernel pick_pass_cfg(int epl, int lpf) {
    if constexpr (sizeof(T) == 4) {
        if (epl == 4) return lpf == 16 ? pk<T, MODE, 4, 16, HRES>() : pk<T, MODE, 4, 32, HRES>();
        if (epl == 8) return pk<T, MODE, 8, 32, HRES>();
        return pk<T, MODE, 16, 32, HRES>();
    } else {
        if (epl == 2) return lpf == 16 ? pk<T, MODE, 2, 16, HRES>() : pk<T, MODE, 2, 32, HRES>();
        if (epl == 4) return pk<T, MODE, 4, 32, HRES>();
        return pk<T, MODE, 8, 32, HRES>();
    }
}

template <typename T, int MODE>
static PassKernel pick_pass(int epl, int lpf, bool hres) {
    return hres ? pick_pass_cfg<T, MODE, true>(epl, lpf) : pick_pass_cfg<T, MODE, false>(epl, lpf);
}

template <typename T>
static PassKernel pick_pass_mode(int mode, int epl, int lpf, bool hres) {
    switch (mode) {
        case 100 + PASS_KEPT1: return pick_pass<T, 100 + PASS_KEPT1>(epl, lpf, hres);
        case 100 + PASS_RED1: return pick_pass<T, 100 + PASS_RED1>(epl, lpf, hres);
        case 100 + PASS_FUSED: return pick_pass<T, 100 + PASS_FUSED>(epl, lpf, hres);
        case PASS_FUSED: return pick_pass<T, PASS_FUSED>(epl, lpf, hres);
        case PASS_KEPT1: return pick_pass<T, PASS_KEPT1>(epl, lpf, hres);
        case PASS_RED1: return pick_pass<T, PASS_RED1>(epl, lpf, hres);
        case PASS_REFILL: return pick_pass<T, PASS_REFILL>(epl, lpf, hres);
        case PASS_OBJ: return pick_pass<T, PASS_OBJ>(epl, lpf, hres);
        default: return pick_pass<T, PASS_MODEL>(epl, lpf, hres);
    }
}

template <typename T, int SM>
static const void* pick_solve_sm(int R) {
    switch (R) {
        case 1: return (const void*)block_solve<T, 1, SM>;
        case 2: return (const void*)block_solve<T, 2, SM>;
        case 3: return (const void*)block_solve<T, 3, SM>;
        case 4: return (const void*)block_solve<T, 4, SM>;
        case 5: return (const void*)block_solve<T, 5, SM>;
        case 6: return (const void*)block_solve<T, 6, SM>;
        case 7: return (const void*)block_solve<T, 7, SM>;
        case 8: return (const void*)block_solve<T, 8, SM>;
        default: return (const void*)block_solve<T, 9, SM>;
    }
}

template <typename T>
static const void* pick_solve(int R, int sm = SOLVE_FULL) {
    if (R > MAXR_SMALL) {
        const void* fn = sm == SOLVE_PROJECT     ? (const void*)block_solve_big<T, SOLVE_PROJECT>
                         : sm == SOLVE_FROM_PROJ ? (const void*)block_solve_big<T, SOLVE_FROM_PROJ>
                                                 : (const void*)block_solve_big<T, SOLVE_FULL>;
        return fn;
    }
    if (sm == SOLVE_PROJECT) return pick_solve_sm<T, SOLVE_PROJECT>(R);
    if (sm == SOLVE_FROM_PROJ) return pick_solve_sm<T, SOLVE_FROM_PROJ>(R);
    return pick_solve_sm<T, SOLVE_FULL>(R);
}

template <typename T>
struct Solver : SolverBase {
    Shape s;
    Layout lay;
    double rho;
    unsigned flags;
    cudaStream_t user_stream;
    cudaStream_t st = nullptr;
    cudaEvent_t ev_in = nullptr, ev_out = nullptr;
    unsigned char* ws = nullptr;
    bool own_ws = false;
    int nsm = 0;
    size_t smem_limit = 0;
    // device views
    T *X, *G, *H, *pb, *pw;
    uint32_t* bits;
    double *beta, *omega, *delta, *norms, *scal, *rsep, *proj, *rscr;
    unsigned *rcnt, *sched;
    int* dflags;
    double* hscal = nullptr;  // pinned
    int* hflags = nullptr;    // pinned
    std::vector<BlockPlan<T>> blocks;
    PassPlan<T> refill, obj, model;
    PassPlan<T> fused;          // a5 ⊕ a2(0,1), see enqueue_mid()
    ReduceParams<T> fused_red;
    RedLaunch fused_red_l;
    SolveParams<T> fused_sol;  // block (0,1)'s solve after the fused pass (its slot layout)
    bool has_fused = false;
    // L2-resident tensors: a5 by l2_refill (l2pass.cuh) instead of the streaming refill pass
    bool l2r = false;
    L2RefillParams<T> l2rp;
    const void* l2r_fn = nullptr;
    dim3 l2r_grid;
    size_t l2r_smem = 0;
    cudaGraphExec_t gexec = nullptr;                                    // one plain sweep
    cudaGraphExec_t gexec_first = nullptr, gexec_mid = nullptr, gexec_last = nullptr;
    cudaGraphExec_t gexec_mid_t = nullptr, gexec_last_t = nullptr;  // traced fused sweeps
    double* trace_rows = nullptr;  // device: 5 doubles per traced sweep
    int* trace_count = nullptr;
    int trace_cap = 0;
    int64_t n_mid_t = 0, n_last_t = 0;
    int64_t nlaunch_sweep = 0, last_launches = 0;
    int64_t ctr = 0;                       // kernels enqueued so far (graph nodes at capture)
    static constexpr int64_t solve_slots = 64;  // max serial slot chain for the solve to absorb the reduce
    int64_t n_full = 0, n_first = 0, n_mid = 0, n_last = 0;  // kernels per captured graph
    int64_t sh_off = 0, sh_len = 0;        // ΔG² range of the shard-mode chains
    double* p5 = nullptr;                  // norm partials (see finalize_norms)
    double* hred = nullptr;                // pinned host buffer for host_allreduce
    void (*host_allreduce)(double*, size_t, void*) = nullptr;
    void* host_user = nullptr;
    // multi-GPU (see dist.cuh notes in DESIGN.md)
    NcclLite* nccl = nullptr;
    void* comm = nullptr;
    // peer-memory exchange (peer.cuh): own buffer, peers' mapped buffers, device context
    double* xbuf = nullptr;
    PeerCtx pctx{};
    std::vector<void*> peer_open;

    ~Solver() override {
        for (cudaGraphExec_t e : {gexec, gexec_first, gexec_mid, gexec_last, gexec_mid_t, gexec_last_t})
            if (e) cudaGraphExecDestroy(e);
        if (trace_rows) cudaFree(trace_rows);
        if (comm && nccl) nccl->commDestroy(comm);
        if (st) cudaStreamSynchronize(st);
        for (void* p : peer_open) cudaIpcCloseMemHandle(p);
        if (xbuf) cudaFree(xbuf);
        if (st) cudaStreamSynchronize(st);
        if (own_ws && ws) cudaFree(ws);
        if (hscal) cudaFreeHost(hscal);
        if (hflags) cudaFreeHost(hflags);
        if (hred) cudaFreeHost(hred);
        if (ev_in) cudaEventDestroy(ev_in);
        if (ev_out) cudaEventDestroy(ev_out);
        if (st) cudaStreamDestroy(st);
    }

    // stream-ordering with the caller's stream
    void begin() {
        CU(cudaEventRecord(ev_in, user_stream));
        CU(cudaStreamWaitEvent(st, ev_in, 0));
    }
    void end() {
        CU(cudaEventRecord(ev_out, st));
        CU(cudaStreamWaitEvent(user_stream, ev_out, 0));
    }

    // profiling (ifctn_profile_sweep): one event before every launch + one at the end
    std::vector<cudaEvent_t> prof_ev;
    bool profiling = false;
    void prof_mark() {
        if (!profiling) return;
        cudaEvent_t e;
        CU(cudaEventCreate(&e));
        CU(cudaEventRecord(e, st));
        prof_ev.push_back(e);
    }

    // pdl: the kernel calls pdl_wait() before it touches its predecessor's outputs, so it may be
    // launched with programmatic stream serialization (its launch and index prologue overlap the
    // predecessor's tail; captured into the sweep graphs as programmatic edges)
    template <typename P>
    void launch(const void* fn, dim3 g, dim3 b, size_t smem, const P& p, bool pdl = false) {
        prof_mark();
        void* args[] = {(void*)&p};
        launch_raw(fn, g, b, smem, args, pdl);
    }

    void launch_raw(const void* fn, dim3 g, dim3 b, size_t smem, void** args, bool pdl = false) {
        if (pdl && !(flags & IFCTN_FLAG_NO_PDL)) {
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = g;
            cfg.blockDim = b;
            cfg.dynamicSmemBytes = smem;
            cfg.stream = st;
            cudaLaunchAttribute at{};
            at.id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at.val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = &at;
            cfg.numAttrs = 1;
            CU(cudaLaunchKernelExC(&cfg, fn, args));
        } else {
            CU(cudaLaunchKernel(fn, g, b, args, smem, st));
        }
        ++ctr;
    }

    // vblk: v-blocked contraction (mode 1 kept; fiber_pass_vb), else the plain walk
    PassPlan<T> make_pass(int mode, int k, int i, bool vblk = false) {
        const int N = s.N;
        PassPlan<T> pp;
        PassParams<T>& p = pp.p;
        memset(&p, 0, sizeof(p));
        p.H = H;
        p.hsize = s.htotal;
        p.X = X;
        p.Xw = X;
        p.mask = bits;
        p.part_b = pb;
        p.part_cap = s.part_elems;
        p.x_cap = s.npad;
        p.mask_cap = (align_up((s.npad + 31) / 32, 8) + 8);
        p.part_w = pw;
        p.norms = norms;
        p.rho = (T)rho;
        p.inv1p = (T)(1.0 / (1.0 + rho));
        p.I1 = (int)s.I1;
        p.I1p = (int)s.I1p;
        p.nouter = N - 1;
        for (int m = 0; m < N; ++m) p.fstride[m] = s.fstride[m];
        const bool contract = (mode == PASS_KEPT1 || mode == PASS_RED1 || mode == PASS_FUSED);
        if (mode == PASS_FUSED) {  // block (0,m) or (m,0): the refill's t needs H_{0,m}
            p.h01_mode = std::max(k, i);
            p.h01_off = s.hoff[0][p.h01_mode];
        }
        // kept outer modes (ascending), reduced outer modes
        std::vector<int> kept, red;
        for (int m = 1; m < N; ++m) {
            if (contract && (m == k || m == i)) kept.push_back(m);
            else red.push_back(m);
        }
        // odometer order: r0 = the largest reduced mode (ties: lowest), then ascending
        // (v-blocked: ascending; the fast index is the kept mode 1).  Measured on a C5 shard:
        // preferring the contiguous mode 1 when it is short (8 fibres, 2 KB runs) doubled the
        // pass time (runs too short for the per-run setup) — keep the long runs.
        if (!red.empty() && !vblk) {
            int best = 0;
            for (size_t t = 1; t < red.size(); ++t)
                if (s.ld[red[t]] > s.ld[red[best]]) best = (int)t;
            std::rotate(red.begin(), red.begin() + best, red.begin() + best + 1);
        }
        p.nkept = (int)kept.size();
        for (size_t t = 0; t < kept.size(); ++t) {
            p.kmode[t] = kept[t];
            p.kdim[t] = s.ld[kept[t]];
        }
        if (p.nkept < 2) p.kdim[1] = 1;
        if (p.nkept < 1) p.kdim[0] = 1;
        p.nred = (int)red.size();
        for (size_t t = 0; t < red.size(); ++t) {
            p.rmode[t] = red[t];
            p.rdim[t] = s.ld[red[t]];
        }
        p.NV = 1;
        for (int m : kept) p.NV *= s.ld[m];
        p.FR = 1;
        for (int m : red) p.FR *= s.ld[m];
        p.nfib = s.nfib;
        p.Lv = (mode == PASS_KEPT1 || mode == PASS_FUSED) ? s.I1p : 1;
        const int r0 = red.empty() ? -1 : red[0];
        // weight factors: every pair p<q except {k,i} when contracting
        p.vf_off = -1;
        p.vf2_off = -1;
        p.tc_off = -1;
        if (vblk) {  // tiled pass (fiber_tile.cuh): fast indices are mode 1 and r0
            for (int a = 0; a < N; ++a)
                for (int b = a + 1; b < N; ++b) {
                    if ((a == k && b == i) || (a == i && b == k)) continue;
                    const int64_t off = s.hoff[a][b];
                    if (a == 0) {
                        if (b == 1) p.vf_off = off;
                        else if (b == r0) p.vf2_off = off;
                        else {
                            p.vs_off[p.nvs] = off;
                            p.vs_mode[p.nvs] = b;
                            ++p.nvs;
                        }
                    } else if ((a == 1 && b == r0) || (a == r0 && b == 1)) {
                        p.tc_off = off;        // H_{1,r0}(v, i_r0) at off + i_r0·ld_1 + v
                        p.tc_ld = s.hld[1];
                    } else if (a == 1 || b == 1) {
                        const int q = (a == 1) ? b : a;  // H_{1,q}(v, i_q), q > 1
                        p.ta_off[p.nta] = off;
                        p.ta_fix[p.nta] = q;
                        p.ta_mul[p.nta] = s.hld[1];
                        p.ta_inc[p.nta] = 1;
                        ++p.nta;
                    } else if (a == r0 || b == r0) {
                        const int fix = (a == r0) ? b : a;
                        p.sf_off[p.nsf] = off;
                        p.sf_fixmode[p.nsf] = fix;
                        p.sf_fixmul[p.nsf] = (a == r0) ? s.hld[a] : 1;
                        p.sf_inc[p.nsf] = (a == r0) ? 1 : s.hld[a];
                        ++p.nsf;
                    } else {
                        p.ss_off[p.nss] = off;
                        p.ss_ld[p.nss] = s.hld[a];
                        p.ss_p[p.nss] = a;
                        p.ss_q[p.nss] = b;
                        ++p.nss;
                    }
                }
        }
        for (int a = 0; a < N && !vblk; ++a)
            for (int b = a + 1; b < N; ++b) {
                if (contract && ((a == k && b == i) || (a == i && b == k))) continue;
                const int64_t off = s.hoff[a][b];
                if (a == 0) {
                    if (b == r0) p.vf_off = off;
                    else {
                        p.vs_off[p.nvs] = off;
                        p.vs_mode[p.nvs] = b;
                        ++p.nvs;
                    }
                } else if (a == r0 || b == r0) {
                    // H_{a,b}(i_a, i_b) at off + i_b·ld_a + i_a
                    const int fix = (a == r0) ? b : a;
                    p.sf_off[p.nsf] = off;
                    p.sf_fixmode[p.nsf] = fix;
                    p.sf_fixmul[p.nsf] = (a == r0) ? s.hld[a] : 1;
                    p.sf_inc[p.nsf] = (a == r0) ? 1 : s.hld[a];
                    ++p.nsf;
                } else {
                    p.ss_off[p.nss] = off;
                    p.ss_ld[p.nss] = s.hld[a];
                    p.ss_p[p.nss] = a;
                    p.ss_q[p.nss] = b;
                    ++p.nss;
                }
            }
        p.ones_off = s.ones_off;
        p.sf_cap = s.sf_cap;
        if (vblk) p.sf_cap = 8 * (int)std::min<int64_t>(s.ld[r0], 32);  // F ≤ 8 rows × run ≤ 32
        // H_{0,r0} (the per-fibre factor) resident in shared memory when it fits; without
        // that factor (no fast mode, or the kept pair itself) a column of ones stands in
        const bool hfac = p.vf_off >= 0;
        const int64_t rdim0 = hfac ? s.ld[vblk ? 1 : r0] : 1;
        const int64_t hres_elems = hfac ? s.I1p * rdim0 : s.I1p;
        const bool hres = hres_elems * s.esize <= 32 * 1024;
        p.hres_src = hfac ? p.vf_off : s.ones_off;
        p.hres_elems = hres ? hres_elems : 0;
        if (vblk) {  // second resident block: H_{0,r0}; fused: third, H_{0,1}
            p.hres2_elems = s.I1p * s.ld[r0];
            if (mode == PASS_FUSED) p.hres3_elems = s.I1p * s.ld[1];
            if (!hres || p.hres2_elems * s.esize > 32 * 1024) fail(IFCTN_E_STATE, "tiled pass needs resident H blocks");
        }
        // shared memory per CTA: [mbarriers][sf vectors][resident H][TMA ring per warp]
        const int nwarps = kPassThreads / 32;
        const PassKernel kern = pick_pass_mode<T>(vblk ? 100 + mode : mode, s.epl, s.lpf, hres);
        if (!kern.fn) fail(IFCTN_E_STATE, "no kernel for this pass");
        if (vblk) {  // positions (vb·FR + r)·F + f over NVB = nb0·kdim1 kept blocks
            const int64_t F = kern.F;
            if (F > p.sf_cap) fail(IFCTN_E_STATE, "v-block wider than the sf vector");
            p.nb0 = (p.kdim[0] + F - 1) / F;
            p.nfib = p.nb0 * p.kdim[1] * p.FR * F;
        }
        p.sfv_off = align_up((int64_t)nwarps * 8 * 8, 128);  // ≤ 8 stage barriers per warp
        // per warp: the sf table (sf_cap) + tiled-pass scratch for A (≤ 8) and B (≤ sf_cap/F)
        p.sfv_stride = vblk ? 2 * (int64_t)p.sf_cap + 8 : p.sf_cap;
        p.hres_off = align_up(p.sfv_off + (int64_t)nwarps * p.sfv_stride * s.esize, 128);
        p.stage_off = align_up(p.hres_off + (p.hres_elems + p.hres2_elems + p.hres3_elems) * s.esize, 128);
        const size_t smem = (size_t)(p.stage_off + (int64_t)nwarps * kern.ring * s.esize);
        pp.fn = kern.fn;
        if (smem > smem_limit) fail(IFCTN_E_UNSUPPORTED, "fibre-pass shared memory exceeds the device limit");
        // one kernel serves several passes with different sizes: allow the device maximum
        {
            cudaFuncAttributes fa;
            CU(cudaFuncGetAttributes(&fa, pp.fn));
            if (smem + fa.sharedSizeBytes > smem_limit) fail(IFCTN_E_UNSUPPORTED, "fibre-pass shared memory exceeds the device limit");
            CU(cudaFuncSetAttribute(pp.fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)(smem_limit - fa.sharedSizeBytes)));
        }
        int nb = 0;
        CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, pp.fn, kPassThreads, smem));
        if (nb < 1) nb = 1;
        // grid: one wave of warps.  Plain walk: one fibre range ("group") per warp, equal
        // fibre counts.  Tiled pass: one fixed chunk ("group") per warp, claimed dynamically
        // (fiber_tile.cuh), so no SM idles while others finish.
        int64_t gmax = (int64_t)nsm * nb * nwarps;
        gmax = std::min(gmax, s.groups_bound);
        const int64_t unit = vblk ? kern.F : 1;  // v-blocked ranges hold whole runs
        const int64_t nunits = p.nfib / unit;
        const int64_t nchunk = gmax;
        const int64_t L = std::max<int64_t>(1, (nunits + nchunk - 1) / nchunk) * unit;
        p.L = L;
        p.ngroups = (p.nfib + L - 1) / L;
        p.sched = sched;
        const int64_t warps = vblk ? std::min(gmax, p.ngroups) : p.ngroups;
        pp.grid = dim3((unsigned)((warps + nwarps - 1) / nwarps));
        pp.smem = smem;
        return pp;
    }

    // the tiled pass applies when a reduced outer mode exists and both resident H blocks fit
    bool tile_ok(int k, int i) const {
        int r0 = -1;
        for (int m = 1; m < s.N; ++m)
            if (m != k && m != i && (r0 < 0 || s.ld[m] > s.ld[r0])) r0 = m;
        if (r0 < 0) return false;
        const bool pair01_kept = (k == 0 || i == 0);
        const int64_t b1 = (pair01_kept ? s.I1p : s.I1p * s.ld[1]) * s.esize;
        const int64_t b2 = s.I1p * s.ld[r0] * s.esize;
        return b1 <= 32 * 1024 && b2 <= 32 * 1024;
    }

    // stage-2 reduce launch.  Lv = 1 with enough v to fill the GPU: a warp per v
    // (reduce_partials_warp).  Otherwise CTAs (v, element tile of ET ≤ 32, slot share z); Z > 1
    // only when the (v, tile) CTAs alone would leave SMs idle and every thread still sums ≥ 4
    // slots.
    RedLaunch split_reduce(ReduceParams<T>& r) {
        r.scr = rscr;
        r.cnt = rcnt;
        r.ET = 1;
        r.ntile = 1;
        r.Z = 1;
        const int64_t nslots = (r.FR * r.VB) / r.L + 2;
        if (r.Lv == 1 && r.NV >= 16 * (int64_t)nsm && nslots <= 1024)
            return {(const void*)reduce_partials_warp<T>, dim3((unsigned)((r.NV + 7) / 8))};
        int ET = 1;
        while (ET < r.Lv && ET < 32) ET <<= 1;
        r.ET = ET;
        r.ntile = (int)((r.Lv + ET - 1) / ET);
        const int64_t base = r.NV * r.ntile;
        const int64_t ny = 256 / ET;
        int64_t Z = 1;
        const int64_t target = 2 * (int64_t)nsm;
        if (base < target && base <= kRedCnt) {
            Z = (target + base - 1) / base;
            Z = std::min(Z, std::max<int64_t>(1, nslots / (ny * 4)));
            Z = std::min(Z, kRedScr / (base * ET * 2));
            Z = std::max<int64_t>(1, std::min<int64_t>(Z, 64));
        }
        r.Z = (int)Z;
        return {(const void*)reduce_partials<T>, dim3((unsigned)r.NV, (unsigned)r.ntile, (unsigned)Z)};
    }

    static const void* pick_l2_kept(int nr) {
        switch (nr) {
            case 1: return (const void*)l2_kept<T, 1>;
            default: return (const void*)l2_kept<T, 2>;
        }
    }
    static const void* pick_l2_red(int nrr) {
        switch (nrr) {
            case 0: return (const void*)l2_red<T, 0>;
            default: return (const void*)l2_red<T, 1>;
        }
    }

    // CTAs of `fn` (256 threads, `smem` dynamic bytes) resident on the device at once
    int64_t resident_ctas(const void* fn, size_t smem) {
        int per_sm = 0;
        CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kL2Threads, smem));
        return (int64_t)std::max(per_sm, 1) * nsm;
    }

    // Step a2 of block (k,i) by l2pass.cuh when X is L2-resident; false = not applicable.
    bool make_l2(BlockPlan<T>& b, int k, int i) {
        if (flags & IFCTN_FLAG_NO_L2PASS) return false;
        if (s.npad * s.esize > (int64_t)48 << 20) return false;
        const int N = s.N;
        // orders 3 and 4 (the paper's L2-sized workloads, C1–C4).  Orders ≥ 5 keep the streaming
        // walk: the small 5th-order test problems (C5s) are ill-conditioned enough to amplify
        // any change of rounding order ~25× per sweep, and their bars are set against the walk.
        if (N < 3 || N > 4) return false;
        if (s.nfib >= (1LL << 31) || s.htotal >= (1LL << 31)) return false;
        const int VE = 16 / (int)s.esize;
        L2Params<T>& P = b.l2p;
        memset(&P, 0, sizeof(P));
        P.X = X;
        P.H = H;
        P.beta = beta;
        P.omega = omega;
        P.I1 = (int)s.I1;
        P.I1p = (int)s.I1p;
        P.N = N;
        P.Ii = s.ld[i];
        P.Ik = s.ld[k];
        const bool kept1 = (k == 0 || i == 0);
        P.kept1 = kept1;
        P.kIsMode0 = (k == 0);
        P.m = kept1 ? std::max(k, i) : -1;
        P.k = k;
        P.i = i;
        for (int q = 1; q < N; ++q) P.fstride[q] = s.fstride[q];
        P.NV = kept1 ? s.ld[P.m] : s.ld[k] * s.ld[i];
        P.FR = 1;
        int64_t rsum = 0;
        {
            int rm[MAXN], nrm = 0;
            for (int q = 1; q < N; ++q) {
                const bool kept = kept1 ? (q == P.m) : (q == k || q == i);
                if (!kept) rm[nrm++] = q;
            }
            // odometer order: mode order (first fastest), except that the longest reduced mode
            // leads (l2_kept walks it in runs of kL2RunU cells)
            int lead = 0;
            for (int t = 1; t < nrm; ++t)
                if (s.ld[rm[t]] > s.ld[rm[lead]]) lead = t;
            if (nrm > 0) std::rotate(rm, rm + lead, rm + lead + 1);
            for (int t = 0; t < nrm; ++t) {
                const int q = rm[t];
                P.rmode[P.nr] = q;
                P.rdim[P.nr] = (int)s.ld[q];
                P.rfs[P.nr] = (int)s.fstride[q];
                P.rfsI[P.nr] = (int)(s.fstride[q] * s.I1p);
                P.rv_off[P.nr] = (int)s.hoff[0][q];
                ++P.nr;
                P.FR *= s.ld[q];
                rsum += s.ld[q];
            }
        }
        if (P.FR >= (1LL << 31) || P.NV >= (1LL << 31)) return false;
        // H_{p,r_j}(x, d) for a kept outer mode p: H[off + x·mv + d·mj]
        auto kept_scalar = [&](int p, int j, int* off, int* mv, int* mj) {
            const int q = P.rmode[j];
            if (p < q) {
                off[j] = (int)s.hoff[p][q];
                mv[j] = 1;
                mj[j] = (int)s.hld[p];
            } else {
                off[j] = (int)s.hoff[q][p];
                mv[j] = (int)s.hld[q];
                mj[j] = 1;
            }
        };
        {
            int t = 0;
            for (int j = 0; j < P.nr; ++j)
                for (int j2 = j + 1; j2 < P.nr; ++j2, ++t) {
                    const int q = P.rmode[j], q2 = P.rmode[j2];
                    if (q < q2) {
                        P.jj_off[t] = (int)s.hoff[q][q2];
                        P.jj_ma[t] = 1;
                        P.jj_mb[t] = (int)s.hld[q];
                    } else {
                        P.jj_off[t] = (int)s.hoff[q2][q];
                        P.jj_ma[t] = (int)s.hld[q2];
                        P.jj_mb[t] = 1;
                    }
                }
        }
        P.scr = rscr;
        P.cnt = rcnt;
        // Work split.  Cost model in L2 round trips: every CTA pays a fixed part (launch ramp,
        // index setup, table staging, the warp/CTA combine) plus one round per U cells of its
        // busiest thread; CTAs beyond the resident set wait for a second wave; a split over Z
        // CTAs adds the last-arrival combine.
        static const int kZs[] = {1, 2, 3, 4, 5, 6, 8, 10, 12, 16, 20, 24, 32, 48, 64};
        auto cdiv = [](int64_t a, int64_t c) { return (a + c - 1) / c; };
        const size_t smem_cap = std::min<size_t>(smem_limit > 24 * 1024 ? smem_limit - 24 * 1024 : 0, 96 * 1024);
        const int NC = (int)(s.I1p / VE);
        double best = 1e300;
        // diagnosis: IFCTN_L2_KEPT="CG,wpi,Z" / IFCTN_L2_RED="TL,Z" pin the split (0 = free)
        int pin[3] = {0, 0, 0};
        if (const char* e = getenv(kept1 ? "IFCTN_L2_KEPT" : "IFCTN_L2_RED")) sscanf(e, "%d,%d,%d", &pin[0], &pin[1], &pin[2]);
        if (kept1) {
            const int NR = N - 2;
            P.kf_stride = s.fstride[P.m];
            for (int j = 0; j < NR; ++j) kept_scalar(P.m, j, P.ks_off, P.ks_mv, P.ks_mj);
            b.l2_fn = pick_l2_kept(NR);
            CU(cudaFuncSetAttribute(b.l2_fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_cap));
            const int64_t tab_esize = s.esize;
            // work units of a kept value: runs of kL2RunU cells along reduced mode r_0
            P.nb0 = (int)cdiv(P.rdim[0], kL2RunU);
            P.FR = (P.FR / P.rdim[0]) * P.nb0;
            for (int CG = 1; CG <= 32; CG <<= 1) {
                if (CG < 4 && CG < NC) continue;      // ≥ 64 contiguous bytes per fibre piece
                if (CG > 4 && CG >= 2 * NC) continue;
                if (pin[0] && CG != pin[0]) continue;
                const int FL = 32 / CG;
                const int64_t NCG = cdiv(NC, CG);
                const double waste = (double)(NCG * CG) / NC;
                const int64_t asc_item = (rsum + VE - 1) / VE * VE;
                const int64_t tab_item = rsum * CG * VE + asc_item;
                for (int wpi = 1; wpi <= 8; wpi <<= 1) {
                    if (pin[1] && wpi != pin[1]) continue;
                    const int ipc = 8 / wpi;
                    const size_t smem = (size_t)ipc * tab_item * tab_esize;
                    if (smem > smem_cap) continue;
                    const int64_t resident = resident_ctas(b.l2_fn, smem);
                    if (P.NV * NCG >= (1LL << 30)) continue;
                    const int64_t nbx = cdiv(P.NV * NCG, ipc);
                    const int64_t slots = (int64_t)wpi * FL;
                    for (int Z : kZs) {
                        if (pin[2] && Z != pin[2]) continue;
                        if (Z > 1 && (Z > P.FR || nbx > kRedCnt || nbx * Z * ipc * 2 * CG * VE > kRedScr)) continue;
                        const int64_t FRz = cdiv(P.FR, Z), Ze = cdiv(P.FR, FRz);
                        const int64_t rounds = cdiv(FRz, slots);
                        const int64_t waves = cdiv(nbx * Ze, resident);
                        const double stage = (double)cdiv(rsum * CG, wpi * 32) / 4;  // table rounds
                        const double cost = waves * (1.5 + stage + rounds * waste) + (Ze > 1 ? 1.0 : 0.0) +
                                            1e-3 * (double)(nbx * Ze) / resident;
                        if (cost < best) {
                            best = cost;
                            P.CG = CG;
                            P.NCG = (int)NCG;
                            P.ipc = ipc;
                            P.wpi = wpi;
                            P.lcg = 0;
                            while ((1 << P.lcg) < CG) ++P.lcg;
                            P.lwpi = 0;
                            while ((1 << P.lwpi) < wpi) ++P.lwpi;
                            P.tab_item = (int)tab_item;
                            P.asc_item = (int)asc_item;
                            P.FRz = FRz;
                            P.Z = (int)Ze;
                            b.l2_grid = dim3((unsigned)nbx, (unsigned)Ze);
                            b.l2_smem = smem;
                        }
                    }
                }
            }
        } else {
            const int NRR = N - 3;
            for (int j = 0; j < NRR; ++j) {
                kept_scalar(k, j, P.ks_off, P.ks_mv, P.ks_mj);
                kept_scalar(i, j, P.is_off, P.is_mv, P.is_mj);
            }
            P.pk_off = (int)s.hoff[0][k];
            P.pi_off = (int)s.hoff[0][i];
            b.l2_fn = pick_l2_red(NRR);
            CU(cudaFuncSetAttribute(b.l2_fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_cap));
            for (int TL = 8; TL <= kL2Threads; TL <<= 1) {
                if (pin[0] && TL != pin[0]) continue;
                const int tpc = kL2Threads / TL;
                const size_t smem = (size_t)tpc * s.I1p * s.esize;
                if (smem > smem_cap) continue;
                const int64_t resident = resident_ctas(b.l2_fn, smem);
                const int64_t nbx = cdiv(P.NV, tpc);
                for (int Z : kZs) {
                    if (pin[1] && Z != pin[1]) continue;
                    if (Z > 1 && (Z > P.FR || nbx > kRedCnt || nbx * Z * tpc * 2 > kRedScr)) continue;
                    const int64_t FRz = cdiv(P.FR, Z), Ze = cdiv(P.FR, FRz);
                    const int64_t rounds = cdiv(cdiv(FRz * NC, TL), kL2U);
                    const int64_t waves = cdiv(nbx * Ze, resident);
                    const double stage = (double)cdiv(NC, TL) / kL2U;
                    const double cost = waves * (1.5 + stage + rounds) + (Ze > 1 ? 1.0 : 0.0) + 1e-3 * (double)(nbx * Ze) / resident;
                    if (cost < best) {
                        best = cost;
                        P.TL = TL;
                        P.FRz = FRz;
                        P.Z = (int)Ze;
                        b.l2_grid = dim3((unsigned)nbx, (unsigned)Ze);
                        b.l2_smem = smem;
                    }
                }
            }
        }
        if (best >= 1e300) return false;
        if (getenv("IFCTN_L2_VERBOSE"))
            fprintf(stderr, "l2 block (%d,%d) %s NV %lld FR %lld: CG %d wpi %d TL %d Z %d grid %u x %u smem %zu\n", k, i,
                    kept1 ? "kept" : "red", (long long)P.NV, (long long)P.FR, P.CG, P.wpi, P.TL, P.Z, b.l2_grid.x,
                    b.l2_grid.y, b.l2_smem);
        if (kept1) {  // digits of the per-step run stride
            int64_t st = (int64_t)P.wpi * (32 / P.CG);
            for (int j = 0; j < P.nr; ++j) {
                const int64_t radix = j == 0 ? P.nb0 : P.rdim[j];
                P.dsr[j] = (int)(st % radix);
                st /= radix;
            }
        }
        b.l2 = true;
        return true;
    }

    static const void* pick_l2_refill(int no) {
        switch (no) {
            case 1: return (const void*)l2_refill<T, 1>;
            case 2: return (const void*)l2_refill<T, 2>;
            default: return (const void*)l2_refill<T, 3>;
        }
    }

    // Step a5 by l2_refill when X is L2-resident; false = keep the streaming refill pass.
    bool make_l2_refill() {
        if (flags & IFCTN_FLAG_NO_L2PASS) return false;
        if (s.npad * s.esize > (int64_t)48 << 20) return false;
        const int N = s.N;
        if (N < 3 || N > 4 || s.nfib >= (1LL << 31) || s.htotal >= (1LL << 31) || s.npad >= (1LL << 32)) return false;
        int64_t fs = 1, dsum = 0;
        for (int q = 1; q < N; ++q) {  // fibre index = mixed radix over modes 2..N, mode 2 fastest
            if (s.fstride[q] != fs) return false;
            fs *= s.ld[q];
            dsum += s.ld[q];
        }
        const int VE = 16 / (int)s.esize;
        const int NC = (int)(s.I1p / VE);
        L2RefillParams<T>& P = l2rp;
        memset(&P, 0, sizeof(P));
        P.X = X;
        P.H = H;
        P.mask = bits;
        P.norms = norms;
        P.rho = (T)rho;
        P.inv1p = (T)(1.0 / (1.0 + rho));
        P.I1p = (int)s.I1p;
        P.nfib = s.nfib;
        for (int q = 1; q < N; ++q) {
            P.dim[q - 1] = (int)s.ld[q];
            P.tv_off[q - 1] = (int)s.hoff[0][q];
        }
        {
            int t = 0;
            for (int q = 1; q < N; ++q)
                for (int q2 = q + 1; q2 < N; ++q2, ++t) {
                    P.pp_off[t] = (int)s.hoff[q][q2];
                    P.pp_ld[t] = (int)s.hld[q];
                }
        }
        l2r_fn = pick_l2_refill(N - 1);
        auto cdiv = [](int64_t a, int64_t c) { return (a + c - 1) / c; };
        double best = 1e300;
        for (int CG = 1; CG <= 32; CG <<= 1) {
            if (CG < 4 && CG < NC) continue;
            if (CG > 4 && CG >= 2 * NC) continue;
            const size_t smem = (size_t)dsum * CG * VE * s.esize;
            if (smem > 40 * 1024) continue;
            const int FL = 32 / CG;
            const int64_t NCG = cdiv(NC, CG);
            const double waste = (double)(NCG * CG) / NC;
            const int64_t resident = resident_ctas(l2r_fn, smem);
            const int64_t slots = 8 * FL;
            for (int64_t rounds = 1; rounds <= 64; ++rounds) {
                const int64_t FRz = slots * kL2U * rounds;
                const int64_t Z = cdiv(s.nfib, FRz);
                if (NCG * Z > s.groups_bound || Z > 65535) continue;
                const int64_t waves = cdiv(NCG * Z, resident);
                const double stage = (double)cdiv(dsum * CG, kL2Threads) / 4;
                const double cost = waves * (1.5 + stage + rounds * waste) + 1e-3 * (double)(NCG * Z) / resident;
                if (cost < best) {
                    best = cost;
                    P.CG = CG;
                    P.lcg = 0;
                    while ((1 << P.lcg) < CG) ++P.lcg;
                    P.NCG = (int)NCG;
                    P.FRz = FRz;
                    l2r_grid = dim3((unsigned)NCG, (unsigned)Z);
                    l2r_smem = smem;
                }
            }
        }
        if (best >= 1e300) return false;
        int64_t st = 8 * (32 / P.CG);
        for (int q = 0; q < N - 1; ++q) {
            P.ds[q] = (int)(st % P.dim[q]);
            st /= P.dim[q];
        }
        return true;
    }

    void plan() {
        const int N = s.N;
        blocks.clear();
        // Gauss–Seidel order k↑, i↑ in API numbering (reading R6), blocks in internal numbering
        for (int ke = 0; ke < N; ++ke)
            for (int ie = 0; ie < N; ++ie) {
                if (ie == ke) continue;
                const int k = int_mode(ke), i = int_mode(ie);
                BlockPlan<T> b;
                b.k = k;
                b.i = i;
                const int mode = (k == 0 || i == 0) ? PASS_KEPT1 : PASS_RED1;
                const bool vblk = (k == 1 || i == 1) && !(flags & kFlagNoVBlock) && tile_ok(k, i);
                b.vblk = vblk;
                b.pass = make_pass(mode, k, i, vblk);
                ReduceParams<T>& r = b.red;
                r.part_b = pb;
                r.part_cap = s.part_elems;
                r.part_w = pw;
                r.beta = beta;
                r.omega = omega;
                r.FR = b.pass.p.FR;
                r.L = b.pass.p.L;
                r.NV = b.pass.p.NV;
                r.Lv = b.pass.p.Lv;
                r.kept1 = mode == PASS_KEPT1;
                r.I1 = (int)s.I1;
                r.Ii = s.ld[i];
                r.kIsMode0 = (k == 0);
                r.kmode0IsK = (b.pass.p.nkept >= 1 && b.pass.p.kmode[0] == k);
                r.kdim0 = b.pass.p.kdim[0];
                r.VB = vblk ? b.pass.p.nfib / (b.pass.p.nb0 * b.pass.p.kdim[1] * b.pass.p.FR) : 1;
                r.nb0 = vblk ? b.pass.p.nb0 : r.kdim0;
                b.red_l = split_reduce(r);
                SolveParams<T>& q = b.sol;
                q.beta = beta;
                q.omega = omega;
                q.Gki = G + s.goff[k][i];
                q.Gik = G + s.goff[i][k];
                q.H = H;
                const int a = std::min(k, i), c = std::max(k, i);
                q.h_off = s.hoff[a][c];
                q.h_ld = s.hld[a];
                q.k_lt_i = k < i;
                q.Ik = s.ld[k];
                q.Ii = s.ld[i];
                q.rho = rho;
                q.delta = delta + s.delta_off[k][i];
                q.flags = dflags;
                q.proj = proj;
                q.R = s.R(k, i);
                q.red = r;
                // The solve gathers its column from the slots itself (one launch fewer) when
                // that gather is short and coalesced: RED1 blocks (one value per slot) with few
                // slots per kept value, or KEPT1 blocks with i = 0 (a = i_1: consecutive a are
                // consecutive slot entries) with a short serial chain per thread.  KEPT1 with
                // k = 0 would gather one 4-B word per row: the parallel reduce runs first.
                const int64_t slots_per_v = (r.FR * r.VB) / r.L + 2;
                const int64_t chain = slots_per_v * ((s.ld[i] + 127) / 128);
                const bool gather_ok = r.kept1 ? (i == 0 && chain <= solve_slots) : (slots_per_v <= 16 && s.ld[i] >= 16);
                q.fused_reduce = (q.R <= MAXR_SMALL && gather_ok && !(flags & IFCTN_FLAG_NO_SOLVE_REDUCE)) ? 1 : 0;
                if (make_l2(b, k, i)) q.fused_reduce = 0;  // β, ω written whole by l2_contract
                b.sol_grid = dim3((unsigned)s.ld[k]);
                if (q.R > MAXR_SMALL) {  // large-rank path (§8(f1)): a CTA per column
                    b.sol_threads = kBigThreads;
                    // stage all of G_{i,k} at once when it fits in ≈ 110 KB (two CTAs per SM), else 32-column tiles
                    const size_t cap = std::min<size_t>(smem_limit - 8 * 1024, 110 * 1024);
                    q.ta = (int)s.ld[i];
                    if (big_solve_smem(q.R, q.ta, (int)s.esize) > cap) q.ta = 32;
                    q.mma = (flags & IFCTN_FLAG_NO_DMMA) ? 0 : (2 | (q.R <= kBigMmaMaxR ? 1 : 0));  // Gram/RHS | H refresh
                    b.sol_smem = big_solve_smem(q.R, q.ta, (int)s.esize);
                    if (b.sol_smem > smem_limit) fail(IFCTN_E_UNSUPPORTED, "rank too large for the solve kernel");
                    for (int m = 0; m < 3; ++m) {  // allow the device maximum (static smem aside)
                        const void* fn = pick_solve<T>(q.R, m);
                        cudaFuncAttributes fa;
                        CU(cudaFuncGetAttributes(&fa, fn));
                        CU(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                (int)(smem_limit - fa.sharedSizeBytes)));
                    }
                }
                q.use_peer = s.peer ? 1 : 0;
                q.peer = pctx;
                b.dist = s.dpath && k != s.shard;
                if (b.dist) {  // Σ over ranks of the projected Gram/RHS partials (§8(e))
                    const int R = s.R(k, i);
                    b.proj_fn = pick_solve<T>(R, SOLVE_PROJECT);
                    b.sol_fn = pick_solve<T>(R, SOLVE_FROM_PROJ);
                    b.proj_count = s.ld[k] * (R * (R + 1) / 2 + R);
                } else if (q.R > MAXR_SMALL && (flags & IFCTN_FLAG_GRAM_GEMM)) {
                    // one GPU, large rank: two columns per CTA share the g_a g_aᵀ tile products
                    b.gemm = true;
                    b.gram_sol = q;
                    b.gram_sol.use_peer = 0;
                    const size_t cap = std::min<size_t>(smem_limit - 8 * 1024, 128 * 1024);
                    b.gram_sol.ta = (int)s.ld[i];
                    if (gram_project_smem(q.R, b.gram_sol.ta) > cap) b.gram_sol.ta = 32;
                    b.gram_smem = gram_project_smem(q.R, b.gram_sol.ta);
                    if (b.gram_smem > smem_limit) fail(IFCTN_E_UNSUPPORTED, "rank too large for the Gram kernel");
                    CU(cudaFuncSetAttribute((const void*)gram_project<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)smem_limit));
                    b.gram_grid = dim3((unsigned)((s.ld[k] + kGramCols - 1) / kGramCols));
                    b.sol_fn = pick_solve<T>(q.R, SOLVE_FROM_PROJ);
                } else {
                    b.sol_fn = pick_solve<T>(s.R(k, i), SOLVE_FULL);
                }
                blocks.push_back(b);
            }
        refill = make_pass(PASS_REFILL, -1, -1);
        l2r = make_l2_refill();
        obj = make_pass(PASS_OBJ, -1, -1);
        model = make_pass(PASS_MODEL, -1, -1);
        nlaunch_sweep = 3 * (int64_t)blocks.size() + 2;
        // ΔG² of the shard-mode chains (local columns) is summed across ranks; the rest is
        // replicated: delta layout is block order, so blocks (s, ·) are one contiguous range
        sh_off = s.dpath ? s.delta_off[s.shard][s.shard == 0 ? 1 : 0] : 0;  // the last range
        sh_len = s.dpath ? (int64_t)(s.N - 1) * s.ld[s.shard] : 0;
        // fused a5(s) + a2 of block (0,1) of sweep s+1 (same G, X read and written once)
        has_fused = false;
        // (the first block keeps the lane mode 0: API (0,1), or its image under Shape::perm)
        if (!l2r && !(flags & kFlagNoFuse) && std::min(blocks[0].k, blocks[0].i) == 0) {
            const BlockPlan<T>& b0 = blocks[0];
            const bool vb = b0.vblk && std::max(b0.k, b0.i) == 1 && s.I1p * s.ld[1] * s.esize <= 32 * 1024;
            fused = make_pass(PASS_FUSED, b0.k, b0.i, vb);
            fused_red = b0.red;
            fused_red.FR = fused.p.FR;
            fused_red.L = fused.p.L;
            fused_red.VB = vb ? fused.p.nfib / (fused.p.nb0 * fused.p.kdim[1] * fused.p.FR) : 1;
            fused_red.nb0 = vb ? fused.p.nb0 : fused_red.kdim0;
            fused_red_l = split_reduce(fused_red);
            fused_sol = b0.sol;
            fused_sol.red = fused_red;
            has_fused = true;
        }
    }

    void build_all_H() {
        for (int a = 0; a < s.N; ++a)
            for (int b = a + 1; b < s.N; ++b) {
                const int64_t n = s.ld[a] * s.ld[b];
                pair_gram<T><<<(unsigned)((n + 255) / 256), 256, 0, st>>>(
                    G + s.goff[a][b], G + s.goff[b][a], s.R(a, b), s.ld[a], s.ld[b], H + s.hoff[a][b], s.hld[a]);
                CU(cudaGetLastError());
            }
    }

    // a2: the pass, then the second-stage reduce — unless the block's solve absorbs it
    // (small ranks: block_solve sums its column's slots itself; `full` forces the reduce for
    // ifctn_block_coefficients).  A skipped reduce keeps an empty profiling interval so that
    // ifctn_profile_sweep still reports [pass, reduce, solve] per block.
    // prev: the previous launch in the stream is the solve of that block of this sweep (see
    // L2Params::x_early: X and the tables of every pair but {prev.k, prev.i} are final)
    void enqueue_contract(const BlockPlan<T>& b, bool full = false, const BlockPlan<T>* prev = nullptr) {
        if (b.l2) {  // one launch writes β, ω whole; an empty interval for the reduce slot
            L2Params<T> lp = b.l2p;
            lp.x_early = 0;
            if (prev) {
                auto same = [&](int a, int c) { return (a == prev->k && c == prev->i) || (a == prev->i && c == prev->k); };
                lp.x_early = 1;
                if (lp.kept1) {
                    for (int j = 0; j < lp.nr; ++j) {
                        if (!same(0, lp.rmode[j])) lp.x_early |= 2 << j;
                        if (!same(lp.m, lp.rmode[j])) lp.x_early |= 16 << j;
                    }
                } else if (!same(0, lp.k) && !same(0, lp.i)) {
                    lp.x_early |= 2;
                }
            }
            launch(b.l2_fn, b.l2_grid, dim3(kL2Threads), b.l2_smem, lp, true);
            prof_mark();
            return;
        }
        launch(b.pass.fn, b.pass.grid, dim3(kPassThreads), b.pass.smem, b.pass.p);
        if (full || !b.sol.fused_reduce) launch(b.red_l.fn, b.red_l.grid, dim3(256), 0, b.red);
        else prof_mark();
    }

    void enqueue_solve(const BlockPlan<T>& b, const SolveParams<T>* sp = nullptr) {
        const SolveParams<T>& q = sp ? *sp : b.sol;
        if (b.gemm) {  // both launches in the block's solve interval of ifctn_profile_sweep
            launch((const void*)gram_project<T>, b.gram_grid, dim3(kBigThreads), b.gram_smem, b.gram_sol);
            void* args[] = {(void*)&b.gram_sol};
            launch_raw(b.sol_fn, b.sol_grid, dim3(b.sol_threads), b.sol_smem, args, true);
            return;
        }
        if (b.dist) {  // peer exchange: the solve below publishes, waits and sums itself
            launch(b.proj_fn, b.sol_grid, dim3(b.sol_threads), b.sol_smem, q);
            if (!s.peer) allreduce_dev(proj, (size_t)b.proj_count);
        }
        launch(b.sol_fn, b.sol_grid, dim3(b.sol_threads), b.sol_smem, q, !b.dist);
    }

    void enqueue_block(const BlockPlan<T>& b, const BlockPlan<T>* prev = nullptr) {
        enqueue_contract(b, false, prev);
        enqueue_solve(b);
    }

    // norms of the pass that just ran (ngroups partials) → scal (all-reduced across ranks)
    void enqueue_finalize(int64_t ngroups, int obj_only) {
        prof_mark();
        const bool multi = s.dpath;
        {
            const double* a0 = norms;
            const double* a2 = delta;
            int64_t a1 = ngroups, a3 = obj_only ? 0 : s.ndelta, a4 = sh_off, a5 = sh_len;
            int a9 = obj_only, a10 = multi ? 0 : 1;
            void* args[] = {&a0, &a1, &a2, &a3, &a4, &a5, &p5, &scal, &dflags, &a9, &a10};
            launch_raw((const void*)finalize_norms, dim3(1), dim3(1024), 0, args, true);
        }
        if (multi) {
            allreduce_dev(p5, 4);
            prof_mark();
            int a3 = obj_only;
            void* args[] = {&p5, &scal, &dflags, &a3};
            launch_raw((const void*)combine_norms, dim3(1), dim3(32), 0, args);
        }
    }

    void enqueue_xupdate(const BlockPlan<T>* prev = nullptr) {
        if (l2r) {
            L2RefillParams<T> rp = l2rp;
            rp.x_early = prev ? (prev->k != 0 && prev->i != 0 ? 3 : 1) : 0;
            launch(l2r_fn, l2r_grid, dim3(kL2Threads), l2r_smem, rp, true);
            enqueue_finalize((int64_t)l2r_grid.x * l2r_grid.y, 0);
            return;
        }
        launch(refill.fn, refill.grid, dim3(kPassThreads), refill.smem, refill.p);
        enqueue_finalize(refill.p.ngroups, 0);
    }

    void enqueue_sweep() {
        for (size_t b = 0; b < blocks.size(); ++b) enqueue_block(blocks[b], b > 0 ? &blocks[b - 1] : nullptr);
        enqueue_xupdate(&blocks.back());
    }

    // Fused sweep sequence for a fixed sweep count (eps ≤ 0, no trace):
    //   first = blocks of sweep 1;  mid = [a5(s-1) ⊕ a2(0,1)(s)], finaliser, rest of sweep s;
    //   last = a5 of the final sweep.  Same arithmetic as enqueue_sweep() repeated.
    void enqueue_first() {
        for (const auto& b : blocks) enqueue_block(b);
    }
    // traced: the fused pass keeps all three norms and every finaliser appends its row
    void enqueue_trace_push() {
        void* args[] = {&scal, &trace_rows, &trace_count};
        launch_raw((const void*)trace_push, dim3(1), dim3(32), 0, args);
    }
    void enqueue_mid(bool traced = false) {
        const BlockPlan<T>& b0 = blocks[0];
        PassParams<T> fp = fused.p;
        fp.full_norms = traced ? 1 : 0;
        launch(fused.fn, fused.grid, dim3(kPassThreads), fused.smem, fp);
        enqueue_finalize(fp.ngroups, 0);
        if (traced) enqueue_trace_push();
        if (!b0.sol.fused_reduce) launch(fused_red_l.fn, fused_red_l.grid, dim3(256), 0, fused_red);
        enqueue_solve(b0, &fused_sol);
        for (size_t b = 1; b < blocks.size(); ++b) enqueue_block(blocks[b]);
    }
    void enqueue_last(bool traced = false) {
        enqueue_xupdate();
        if (traced) enqueue_trace_push();
    }

    // Dense tensor of this rank's shard between the API linearisation and the internal mode
    // order (only when s.permuted).  to_internal: src API-dense → dst internal-dense; else
    // src internal-dense → dst API-dense.
    template <typename E>
    void permute_api(const E* src, E* dst, bool to_internal) {
        const int N = s.N;
        PermDesc d{};
        d.N = N;
        // source mode q ↔ its extent, source stride and destination stride
        int64_t dstride_api[MAXN], dstride_int[MAXN];
        int64_t acc = 1;
        for (int q = 0; q < N; ++q) {  // API-dense strides
            dstride_api[q] = acc;
            acc *= s.eld[q];
        }
        acc = 1;
        for (int t = 0; t < N; ++t) {  // internal-dense strides
            dstride_int[t] = acc;
            acc *= s.ld[t];
        }
        for (int q = 0; q < N; ++q) {
            if (to_internal) {  // source = API mode q = internal mode int_mode(q)
                d.dim[q] = s.eld[q];
                d.sstr[q] = dstride_api[q];
                d.dstr[q] = dstride_int[int_mode(q)];
            } else {            // source = internal mode q = API mode perm[q]
                d.dim[q] = s.ld[q];
                d.sstr[q] = dstride_int[q];
                d.dstr[q] = dstride_api[s.perm[q]];
            }
        }
        d.ym = to_internal ? s.perm[0] : int_mode(0);  // the source mode fastest in dst
        int64_t nb = 1;
        for (int q = 1; q < N; ++q)
            if (q != d.ym) nb *= d.dim[q];
        const int64_t tiles = ((d.dim[0] + kPermTile - 1) / kPermTile) * ((d.dim[d.ym] + kPermTile - 1) / kPermTile);
        const dim3 grid((unsigned)tiles, (unsigned)std::min<int64_t>(nb, 65535));
        permute_modes<E><<<grid, kPermTile * 8, 0, st>>>(src, dst, d);
        CU(cudaGetLastError());
    }
    // internal mode of API mode m (perm is an involution, but do not rely on it)
    int int_mode(int m) const {
        for (int q = 0; q < s.N; ++q)
            if (s.perm[q] == m) return q;
        return m;
    }
    // factor chains between the ABI layout (API block order) and the internal layout
    void copy_factors(const T* src, T* dst, bool to_internal, cudaMemcpyKind kind) {
        if (!s.permuted) {
            CU(cudaMemcpyAsync(dst, src, (size_t)s.gtotal * s.esize, kind, st));
            return;
        }
        for (int k = 0; k < s.N; ++k)
            for (int i = 0; i < s.N; ++i) {
                if (i == k) continue;
                const int64_t eo = s.egoff[k][i], io = s.goff[int_mode(k)][int_mode(i)];
                const size_t bytes = (size_t)s.R(int_mode(k), int_mode(i)) * s.eld[k] * s.esize;
                CU(cudaMemcpyAsync(to_internal ? dst + io : dst + eo, to_internal ? src + eo : src + io, bytes, kind, st));
            }
    }

    // Peer-memory exchange setup (IFCTN_XCHG_PEER): the exchange buffer, its IPC handle
    // all-gathered through the caller's host callback, the peers' buffers mapped.  Called
    // before plan() (the solve parameters carry the PeerCtx).
    void setup_peer(const ifctn_dist* dist) {
        const int64_t slot = std::max<int64_t>(s.proj_elems, 64);
        const size_t bytes = sizeof(double) * (size_t)(kPeerHeader + 2 * slot + 8);
        CU(cudaMalloc(&xbuf, bytes));
        CU(cudaMemset(xbuf, 0, bytes));
        CU(cudaDeviceSynchronize());  // zeroed before any peer can read the flag
        pctx.W = s.world;
        pctx.rank = s.rank;
        pctx.slot_elems = slot;
        pctx.epoch = reinterpret_cast<unsigned long long*>(xbuf + kPeerHeader + 2 * slot);
        pctx.arrive = reinterpret_cast<unsigned*>(pctx.epoch + 1);
        pctx.bufs[s.rank] = xbuf;
        if (s.world > 1) {
            if (!dist->host_allgather) fail(IFCTN_E_ARG, "dist->host_allgather must be set for IFCTN_XCHG_PEER");
            cudaIpcMemHandle_t h;
            CU(cudaIpcGetMemHandle(&h, xbuf));
            std::vector<cudaIpcMemHandle_t> all((size_t)s.world);
            dist->host_allgather(&h, all.data(), sizeof(h), dist->user);
            for (int r = 0; r < s.world; ++r) {
                if (r == s.rank) continue;
                void* p = nullptr;
                CU(cudaIpcOpenMemHandle(&p, all[(size_t)r], cudaIpcMemLazyEnablePeerAccess));
                peer_open.push_back(p);
                pctx.bufs[r] = (double*)p;
            }
        }
    }

    void init(const void* observed, const uint8_t* mask, const void* G0, void* workspace,
              size_t wbytes, cudaStream_t stream) {
        user_stream = stream;
        int dev = 0;
        CU(cudaGetDevice(&dev));
        CU(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
        int smo = 0;
        CU(cudaDeviceGetAttribute(&smo, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
        smem_limit = (size_t)smo;
        CU(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        CU(cudaEventCreateWithFlags(&ev_in, cudaEventDisableTiming));
        CU(cudaEventCreateWithFlags(&ev_out, cudaEventDisableTiming));
        CU(cudaMallocHost(&hscal, 16 * sizeof(double)));
        CU(cudaMallocHost(&hflags, 4 * sizeof(int)));
        if (workspace) {
            if (wbytes < (size_t)lay.total) fail(IFCTN_E_WORKSPACE, "workspace smaller than ifctn_workspace_bytes()");
            if (((uintptr_t)workspace) % 256) fail(IFCTN_E_WORKSPACE, "workspace must be 256-byte aligned");
            ws = (unsigned char*)workspace;
        } else {
            CU(cudaMalloc(&ws, lay.total));
            own_ws = true;
        }
        X = (T*)(ws + lay.x);
        bits = (uint32_t*)(ws + lay.bits);
        G = (T*)(ws + lay.g);
        H = (T*)(ws + lay.h);
        pb = (T*)(ws + lay.pb);
        pw = (T*)(ws + lay.pw);
        beta = (double*)(ws + lay.beta);
        omega = (double*)(ws + lay.omega);
        delta = (double*)(ws + lay.delta);
        norms = (double*)(ws + lay.norms);
        scal = (double*)(ws + lay.scal);
        p5 = scal + 10;  // scal[10..14]
        dflags = (int*)(ws + lay.flags);
        rsep = (double*)(ws + lay.rse);
        proj = (double*)(ws + lay.proj);
        rscr = (double*)(ws + lay.rscr);
        rcnt = (unsigned*)(ws + lay.rcnt);
        sched = (unsigned*)(ws + lay.sched);

        begin();
        CU(cudaMemsetAsync(ws, 0, lay.total, st));
        // inputs → device (temporary copies when the caller passed host memory)
        const size_t obytes = (size_t)s.nloc * s.esize;
        // pinned host inputs are read in place by pack_input (one pass over the host link)
        // (a mode swap reads transposed: pinned host inputs are staged by DMA first)
        const T* dobs = (const T*)(s.permuted ? (is_device_ptr(observed) ? observed : nullptr) : device_view(observed));
        const uint8_t* dmask = (const uint8_t*)(s.permuted ? (is_device_ptr(mask) ? mask : nullptr) : device_view(mask));
        void* tmp_o = nullptr;
        void* tmp_m = nullptr;
        void* tmp_po = nullptr;
        void* tmp_pm = nullptr;
        if (!dobs) {
            CU(cudaMallocAsync(&tmp_o, obytes, st));
            CU(cudaMemcpyAsync(tmp_o, observed, obytes, cudaMemcpyHostToDevice, st));
            dobs = (const T*)tmp_o;
        }
        if (!dmask) {
            CU(cudaMallocAsync(&tmp_m, (size_t)s.nloc, st));
            CU(cudaMemcpyAsync(tmp_m, mask, (size_t)s.nloc, cudaMemcpyHostToDevice, st));
            dmask = (const uint8_t*)tmp_m;
        }
        if (s.permuted) {  // API order → internal mode order, then the usual packing
            CU(cudaMallocAsync(&tmp_po, obytes, st));
            CU(cudaMallocAsync(&tmp_pm, (size_t)s.nloc, st));
            permute_api<T>(dobs, (T*)tmp_po, true);
            permute_api<uint8_t>(dmask, (uint8_t*)tmp_pm, true);
            dobs = (const T*)tmp_po;
            dmask = (const uint8_t*)tmp_pm;
        }
        const int64_t nw = (s.npad + 31) / 32;
        pack_input<T><<<(unsigned)std::min<int64_t>((nw + 7) / 8, 64 * nsm), 256, 0, st>>>(
            dobs, dmask, s.I1, s.I1p, s.npad, (flags & IFCTN_FLAG_X_FULL) ? 1 : 0, X, bits);
        CU(cudaGetLastError());
        copy_factors((const T*)G0, G, true, is_device_ptr(G0) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice);
        for (void* t : {tmp_o, tmp_m, tmp_po, tmp_pm})
            if (t) CU(cudaFreeAsync(t, st));
        {
            std::vector<T> ones((size_t)s.I1p, T(1));
            CU(cudaMemcpyAsync(H + s.ones_off, ones.data(), ones.size() * sizeof(T), cudaMemcpyHostToDevice, st));
            CU(cudaStreamSynchronize(st));
        }
        plan();
        build_all_H();
        CU(cudaStreamSynchronize(st));
        end();
    }

    template <typename F>
    cudaGraphExec_t capture_one(F&& enqueue) {
        CU(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
        try {
            enqueue();
        } catch (...) {
            cudaGraph_t g = nullptr;
            cudaStreamEndCapture(st, &g);
            if (g) cudaGraphDestroy(g);
            throw;
        }
        cudaGraph_t g = nullptr;
        CU(cudaStreamEndCapture(st, &g));
        cudaGraphExec_t e = nullptr;
        const cudaError_t err = cudaGraphInstantiate(&e, g, 0);
        cudaGraphDestroy(g);
        CU(err);
        return e;
    }

    template <typename F>
    cudaGraphExec_t capture_counted(F&& enqueue, int64_t& n) {
        const int64_t c0 = ctr;
        cudaGraphExec_t e = capture_one(enqueue);
        n = ctr - c0;
        return e;
    }

    void capture() { gexec = capture_counted([&] { enqueue_sweep(); }, n_full); }

    void capture_fused() {
        gexec_first = capture_counted([&] { enqueue_first(); }, n_first);
        gexec_mid = capture_counted([&] { enqueue_mid(); }, n_mid);
        gexec_last = capture_counted([&] { enqueue_last(); }, n_last);
    }
    void capture_fused_traced() {
        gexec_mid_t = capture_counted([&] { enqueue_mid(true); }, n_mid_t);
        gexec_last_t = capture_counted([&] { enqueue_last(true); }, n_last_t);
    }

    void check_flags_sync() {
        CU(cudaMemcpyAsync(hflags, dflags, 4 * sizeof(int), cudaMemcpyDeviceToHost, st));
        CU(cudaStreamSynchronize(st));
#ifndef IFCTN_EXP_NOCHECK  // timing experiments with parts of a kernel switched off
        if (hflags[0]) fail(IFCTN_E_NOT_SPD, "non-positive Cholesky pivot in a column solve");
        if (hflags[1]) fail(IFCTN_E_NONFINITE, "non-finite value in the sweep norms");
#endif
    }

    void sweep(int t_max, double eps, int* done, ifctn_trace_row* trace) override {
        if (t_max < 0) fail(IFCTN_E_ARG, "t_max must be >= 0");
        begin();
        // host-side all-reduce callbacks cannot live in a graph
        const bool use_graph = !(flags & IFCTN_FLAG_NO_GRAPH) && !host_allreduce;
        const bool need_sync = trace || eps > 0.0;
        int s_done = 0;
        last_launches = 0;
        const int64_t c0 = ctr;
        if (has_fused && trace && !(eps > 0.0) && use_graph && t_max >= 2) {
            // traced, fixed sweep count: the fused sequence with full norms; every sweep's row
            // is appended on the device and read back once
            if (t_max > trace_cap) {
                if (trace_rows) {
                    CU(cudaStreamSynchronize(st));
                    CU(cudaFree(trace_rows));
                }
                CU(cudaMalloc(&trace_rows, sizeof(double) * 5 * (size_t)t_max + 64));
                trace_count = (int*)(trace_rows + 5 * (size_t)t_max);
                trace_cap = t_max;
                if (gexec_mid_t) {  // the captured graphs hold the old buffer
                    cudaGraphExecDestroy(gexec_mid_t);
                    cudaGraphExecDestroy(gexec_last_t);
                    gexec_mid_t = gexec_last_t = nullptr;
                }
            }
            if (!gexec_mid) capture_fused();
            if (!gexec_mid_t) capture_fused_traced();
            CU(cudaMemsetAsync(trace_count, 0, sizeof(int), st));
            CU(cudaGraphLaunch(gexec_first, st));
            for (int sw = 1; sw < t_max; ++sw) CU(cudaGraphLaunch(gexec_mid_t, st));
            CU(cudaGraphLaunch(gexec_last_t, st));
            last_launches = n_first + (int64_t)(t_max - 1) * n_mid_t + n_last_t;
            std::vector<double> rows((size_t)5 * t_max);
            CU(cudaMemcpyAsync(rows.data(), trace_rows, rows.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
            check_flags_sync();
            for (int sw = 0; sw < t_max; ++sw) {
                trace[sw].sweep = (int)rows[5 * sw + 0];
                trace[sw].rel_change = rows[5 * sw + 1];
                trace[sw].objective = rows[5 * sw + 2];
                trace[sw].dx2 = rows[5 * sw + 3];
                trace[sw].dg2 = rows[5 * sw + 4];
            }
            if (done) *done = t_max;
            end();
            return;
        }
        if (has_fused && !need_sync && t_max >= 2) {  // fixed sweep count: fused sequence
            if (use_graph && !gexec_mid) capture_fused();
            if (use_graph) {
                CU(cudaGraphLaunch(gexec_first, st));
                for (int sw = 1; sw < t_max; ++sw) CU(cudaGraphLaunch(gexec_mid, st));
                CU(cudaGraphLaunch(gexec_last, st));
                last_launches = n_first + (int64_t)(t_max - 1) * n_mid + n_last;
            } else {
                enqueue_first();
                for (int sw = 1; sw < t_max; ++sw) enqueue_mid();
                enqueue_last();
                last_launches = ctr - c0;
            }
            if (done) *done = t_max;
            end();
            return;
        }
        if (use_graph && !gexec) capture();
        for (int sw = 0; sw < t_max; ++sw) {
            const int64_t c1 = ctr;
            if (use_graph) CU(cudaGraphLaunch(gexec, st));
            else enqueue_sweep();
            last_launches += use_graph ? n_full : ctr - c1;
            ++s_done;
            if (need_sync) {
                CU(cudaMemcpyAsync(hscal, scal, 16 * sizeof(double), cudaMemcpyDeviceToHost, st));
                check_flags_sync();
                if (trace) {
                    trace[sw].sweep = (int)hscal[5];
                    trace[sw].rel_change = hscal[4];
                    trace[sw].objective = hscal[2];
                    trace[sw].dx2 = hscal[0];
                    trace[sw].dg2 = hscal[3];
                }
                if (eps > 0.0 && hscal[4] < eps) break;
            }
        }
        if (done) *done = s_done;
        end();
    }

    int profile_sweep(float* ms, int cap) override {
        begin();
        profiling = true;
        prof_ev.clear();
        try {
            enqueue_sweep();
            prof_mark();
        } catch (...) {
            profiling = false;
            throw;
        }
        profiling = false;
        CU(cudaStreamSynchronize(st));
        const int n = (int)prof_ev.size() - 1;
        for (int t = 0; t < n && t < cap; ++t) CU(cudaEventElapsedTime(ms + t, prof_ev[t], prof_ev[t + 1]));
        for (auto e : prof_ev) cudaEventDestroy(e);
        prof_ev.clear();
        check_flags_sync();
        end();
        return n;
    }

    void sync_check() override {
        begin();
        check_flags_sync();
        end();
    }

    void reconstruct(int what, void* out) override {
        if (!out) fail(IFCTN_E_ARG, "out must not be NULL");
        if (what != IFCTN_MODEL && what != IFCTN_X) fail(IFCTN_E_ARG, "what must be IFCTN_MODEL or IFCTN_X");
        begin();
        const size_t bytes = (size_t)s.nloc * s.esize;
        const bool host = !is_device_ptr(out);
        if (s.permuted) {  // internal mode order → API order
            T* dout = host ? nullptr : (T*)out;
            void* tmp = nullptr;
            void* tmpm = nullptr;
            if (!dout) {
                CU(cudaMallocAsync(&tmp, bytes, st));
                dout = (T*)tmp;
            }
            const T* dense = X;  // internal-dense source
            if (what == IFCTN_X) {
                if (s.I1 != s.I1p) {
                    CU(cudaMallocAsync(&tmpm, bytes, st));
                    unpack_x<T><<<(unsigned)((s.nloc + 255) / 256), 256, 0, st>>>(X, s.I1, s.I1p, s.nloc, (T*)tmpm);
                    CU(cudaGetLastError());
                    dense = (const T*)tmpm;
                }
            } else {
                CU(cudaMallocAsync(&tmpm, bytes, st));
                PassParams<T> p = model.p;
                p.out = (T*)tmpm;
                launch(model.fn, model.grid, dim3(kPassThreads), model.smem, p);
                dense = (const T*)tmpm;
            }
            permute_api<T>(dense, dout, false);
            if (tmp) CU(cudaMemcpyAsync(out, tmp, bytes, cudaMemcpyDeviceToHost, st));
            for (void* t : {tmp, tmpm})
                if (t) CU(cudaFreeAsync(t, st));
        } else if (what == IFCTN_X && s.I1 == s.I1p) {
            // unpadded fibres: X already is the natural layout, one copy
            CU(cudaMemcpyAsync(out, X, bytes, cudaMemcpyDefault, st));
        } else {
            // device or pinned host out: written in place by the kernel; pageable: staged
            T* dout = (T*)device_view(out);
            void* tmp = nullptr;
            if (!dout) {
                CU(cudaMallocAsync(&tmp, bytes, st));
                dout = (T*)tmp;
            }
            if (what == IFCTN_X) {
                unpack_x<T><<<(unsigned)((s.nloc + 255) / 256), 256, 0, st>>>(X, s.I1, s.I1p, s.nloc, dout);
                CU(cudaGetLastError());
            } else {
                PassParams<T> p = model.p;
                p.out = dout;
                launch(model.fn, model.grid, dim3(kPassThreads), model.smem, p);
            }
            if (tmp) {
                CU(cudaMemcpyAsync(out, tmp, bytes, cudaMemcpyDeviceToHost, st));
                CU(cudaFreeAsync(tmp, st));
            }
        }
        if (host) CU(cudaStreamSynchronize(st));
        end();
    }

    void get_factors(void* out) override {
        if (!out) fail(IFCTN_E_ARG, "out must not be NULL");
        begin();
        const bool dev = is_device_ptr(out);
        copy_factors(G, (T*)out, false, dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost);
        if (!dev) CU(cudaStreamSynchronize(st));
        end();
    }

    // A device view of a truth tensor (API layout, host or device) in the internal mode order
    // (dense, leading dim I1); temporaries in *tmp/*tmpp, freed by the caller on st.
    const T* truth_view(const void* truth, void** tmp, void** tmpp) {
        const size_t bytes = (size_t)s.nloc * s.esize;
        const T* dt = (const T*)(s.permuted ? (is_device_ptr(truth) ? truth : nullptr) : device_view(truth));
        if (!dt) {
            CU(cudaMallocAsync(tmp, bytes, st));
            CU(cudaMemcpyAsync(*tmp, truth, bytes, cudaMemcpyHostToDevice, st));
            dt = (const T*)*tmp;
        }
        if (s.permuted) {
            CU(cudaMallocAsync(tmpp, bytes, st));
            permute_api<T>(dt, (T*)*tmpp, true);
            dt = (const T*)*tmpp;
        }
        return dt;
    }

    double rse(const void* truth) override {
        if (!truth) fail(IFCTN_E_ARG, "truth must not be NULL");
        begin();
        void* tmp = nullptr;
        void* tmpp = nullptr;
        const T* dt = truth_view(truth, &tmp, &tmpp);
        const int nb = 1024;
        rse_partial<T><<<nb, 256, 0, st>>>(dt, X, s.I1, s.I1p, s.nloc, rsep);
        sum_pairs<<<1, 256, 0, st>>>(rsep, nb, rsep + 2 * nb);
        CU(cudaGetLastError());
        allreduce_dev(rsep + 2 * nb, 2);
        CU(cudaMemcpyAsync(hscal + 8, rsep + 2 * nb, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
        for (void* t : {tmp, tmpp})
            if (t) CU(cudaFreeAsync(t, st));
        CU(cudaStreamSynchronize(st));
        end();
        const double num = hscal[8], den = hscal[9];
        if (!(den > 0.0)) fail(IFCTN_E_ARG, "truth has zero norm");
        return std::sqrt(num) / std::sqrt(den);
    }

    // RSE, RMSE on Ω^c, band-mean PSNR (bands = slices of the last mode), SSIM
    // (3rd-order: 11×11 Gaussian windows over modes 1, 2, per band).  Sums are per band and
    // global-indexed, all-reduced across ranks; SSIM needs whole band images (NaN when the
    // shard mode is an image mode).
    void metrics(const void* truth, double* out4) override {
        if (!truth) fail(IFCTN_E_ARG, "truth must not be NULL");
        begin();
        const int N = s.N;
        const int last = N - 1;
        const int64_t IN = s.dims[last];                     // global bands
        const int64_t bl = s.ld[last];                       // local bands
        const int64_t boff = (s.dpath && s.shard == last) ? s.sbegin : 0;
        const int64_t fpb = s.nfib / bl;                     // fibres per band (N ≥ 2)
        const int64_t chunks = std::max<int64_t>(1, std::min<int64_t>((fpb + 63) / 64, (4 * nsm + bl - 1) / bl));
        const int64_t chunk = (fpb + chunks - 1) / chunks;
        const bool ssim_ok = (N == 3) && !(s.dpath && s.shard != last);
        const bool gauss = s.ld[0] >= kSsimWin && s.ld[1] >= kSsimWin;
        const int tiles_x = (int)((std::max<int64_t>(s.ld[0] - kSsimWin + 1, 1) + kSsimTile - 1) / kSsimTile);
        const int tiles_y = (int)((std::max<int64_t>(s.ld[1] - kSsimWin + 1, 1) + kSsimTile - 1) / kSsimTile);
        const int64_t ntiles = gauss ? (int64_t)tiles_x * tiles_y : 1;
        const size_t nred = 4 + 2 * (size_t)IN;
        const size_t bytes = sizeof(double) * ((size_t)bl * chunks * 5 + (size_t)bl * ntiles + nred + 8);
        double* tmp = nullptr;
        CU(cudaMallocAsync(&tmp, bytes, st));
        double* part = tmp;
        double* spart = part + bl * chunks * 5;
        double* red = spart + bl * ntiles;
        double* fin = red + nred;
        void* tmpt = nullptr;
        void* tmptp = nullptr;
        const T* dt = truth_view(truth, &tmpt, &tmptp);
        metric_sums<T><<<dim3((unsigned)chunks, (unsigned)bl), kMetThreads, 0, st>>>(dt, X, bits, s.I1, s.I1p, fpb,
                                                                                      chunk, part);
        CU(cudaGetLastError());
        if (ssim_ok) {
            if (gauss)
                ssim_tiles<T><<<dim3((unsigned)ntiles, (unsigned)bl), kSsimTile * kSsimTile, 0, st>>>(
                    dt, X, s.ld[0], s.I1p, s.ld[1], tiles_x, spart);
            else
                ssim_whole<T><<<(unsigned)bl, 256, 0, st>>>(dt, X, s.ld[0], s.I1p, s.ld[1], spart);
            CU(cudaGetLastError());
        }
        metric_reduce<<<1, 1, 0, st>>>(part, chunks, bl, boff, IN, ssim_ok ? spart : nullptr, ntiles, red);
        CU(cudaGetLastError());
        allreduce_dev_chunked(red, nred);
        const double band_n = (double)(s.nglob / IN);
        const double nwin = gauss ? (double)((s.ld[0] - kSsimWin + 1) * (s.ld[1] - kSsimWin + 1)) : 1.0;
        metric_finish<<<1, 1, 0, st>>>(red, IN, band_n, ssim_ok ? nwin * (double)IN : 0.0, fin);
        CU(cudaGetLastError());
        CU(cudaMemcpyAsync(hscal + 8, fin, 6 * sizeof(double), cudaMemcpyDeviceToHost, st));
        for (void* t : {tmpt, tmptp})
            if (t) CU(cudaFreeAsync(t, st));
        CU(cudaFreeAsync(tmp, st));
        CU(cudaStreamSynchronize(st));
        end();
        if (!(hscal[12] > 0.0)) fail(IFCTN_E_ARG, "truth has zero norm");
        for (int q = 0; q < 4; ++q) out4[q] = hscal[8 + q];
        out4[4] = hscal[13];  // |Ω^c|
    }

    // all-reduce of an arbitrary-length fp64 buffer (host-callback staging is proj_elems long)
    void allreduce_dev_chunked(double* buf, size_t count) {
        const size_t step = host_allreduce ? (size_t)s.proj_elems : s.peer ? (size_t)pctx.slot_elems : count;
        for (size_t o = 0; o < count; o += step) allreduce_dev(buf + o, std::min(step, count - o));
    }

    double objective() override {
        begin();
        launch(obj.fn, obj.grid, dim3(kPassThreads), obj.smem, obj.p);
        enqueue_finalize(obj.p.ngroups, 1);
        CU(cudaMemcpyAsync(hscal, scal, 16 * sizeof(double), cudaMemcpyDeviceToHost, st));
        CU(cudaStreamSynchronize(st));
        end();
        return hscal[6];
    }

    const BlockPlan<T>& find_block(int k, int i) {  // k, i: API numbering
        if (k < 0 || i < 0 || k >= s.N || i >= s.N || k == i) fail(IFCTN_E_ARG, "block (k,i) out of range");
        k = int_mode(k);  // API → internal numbering
        i = int_mode(i);
        for (const auto& b : blocks)
            if (b.k == k && b.i == i) return b;
        fail(IFCTN_E_ARG, "block not found");
        return blocks[0];
    }

    void block_coefficients(int k, int i, double* bo, double* wo) override {
        if (!bo || !wo) fail(IFCTN_E_ARG, "beta/omega must not be NULL");
        const auto& b = find_block(k, i);
        begin();
        enqueue_contract(b, true);
        const size_t bytes = (size_t)(s.eld[i] * s.eld[k]) * sizeof(double);
        CU(cudaMemcpyAsync(bo, beta, bytes, cudaMemcpyDefault, st));
        CU(cudaMemcpyAsync(wo, omega, bytes, cudaMemcpyDefault, st));
        CU(cudaStreamSynchronize(st));
        end();
    }

    void block_update(int k, int i) override {
        const auto& b = find_block(k, i);
        begin();
        enqueue_block(b);
        check_flags_sync();
        end();
    }

    void x_update(double* nrm) override {
        begin();
        enqueue_xupdate();
        CU(cudaMemcpyAsync(hscal, scal, 16 * sizeof(double), cudaMemcpyDeviceToHost, st));
        check_flags_sync();
        if (nrm) {
            nrm[0] = hscal[0];
            nrm[1] = hscal[1];
            nrm[2] = hscal[2];
            nrm[3] = hscal[3];
        }
        end();
    }

    // In-place sum across ranks of `count` device doubles, ordered on the context's stream:
    // NCCL all-reduce (capturable into the sweep graph), or the caller's host_allreduce.
    void allreduce_dev(double* buf, size_t count) {
        if (!s.dpath) return;
        if (s.peer) {  // one CTA: copy in, publish, wait, rank-ordered sum (peer.cuh)
            if (count > (size_t)pctx.slot_elems) fail(IFCTN_E_STATE, "all-reduce larger than the exchange slot");
            void* args[] = {(void*)&pctx, &buf, &count};
            launch_raw((const void*)peer_allreduce, dim3(1), dim3(256), 0, args);
            return;
        }
        if (host_allreduce) {
            if (count > (size_t)s.proj_elems) fail(IFCTN_E_STATE, "all-reduce larger than the staging buffer");
            CU(cudaMemcpyAsync(hred, buf, count * sizeof(double), cudaMemcpyDeviceToHost, st));
            CU(cudaStreamSynchronize(st));
            host_allreduce(hred, count, host_user);
            CU(cudaMemcpyAsync(buf, hred, count * sizeof(double), cudaMemcpyHostToDevice, st));
            CU(cudaStreamSynchronize(st));
            return;
        }
        int r = nccl->allReduce(buf, buf, count, /*ncclFloat64*/ 8, /*ncclSum*/ 0, comm, st);
        if (r != 0) fail(IFCTN_E_NCCL, std::string("ncclAllReduce: ") + nccl->errorString(r));
    }

    int64_t launches() const override { return last_launches; }
};

}  // namespace ifctn

// ------------------------------------------------------------------------------------------
// C-ABI
// ------------------------------------------------------------------------------------------
struct ifctn_ctx {
    std::unique_ptr<ifctn::SolverBase> s;
    std::string err;
};

static thread_local std::string g_last_err;

template <typename F>
static ifctn_status guarded(ifctn_ctx* ctx, F&& f) {
    try {
        f();
        return IFCTN_OK;
    } catch (const ifctn::Error& e) {
        if (ctx) ctx->err = e.msg;
        g_last_err = e.msg;
        return e.st;
    } catch (const std::exception& e) {
        if (ctx) ctx->err = e.what();
        g_last_err = e.what();
        return IFCTN_E_CUDA;
    }
}

extern "C" {

ifctn_status ifctn_workspace_bytes(int order, const int64_t* dims, const int32_t* ranks,
                                   ifctn_dtype dtype, const ifctn_dist* dist, size_t* bytes) {
    return guarded(nullptr, [&] {
        if (!bytes) ifctn::fail(IFCTN_E_ARG, "bytes must not be NULL");
        ifctn::Shape s = ifctn::make_shape(order, dims, ranks, dtype, dist);
        *bytes = (size_t)ifctn::make_layout(s).total;
    });
}

ifctn_status ifctn_shard_range(int order, const int64_t* dims, const ifctn_dist* dist,
                               int* shard_mode, int64_t* begin, int64_t* end) {
    return guarded(nullptr, [&] {
        if (!dims) ifctn::fail(IFCTN_E_ARG, "dims must not be NULL");
        std::vector<int32_t> ranks(order * order, 1);
        for (int m = 0; m < order; ++m) ranks[m * order + m] = 0;
        ifctn::Shape s = ifctn::make_shape(order, dims, ranks.data(), IFCTN_F32, dist);
        if (shard_mode) *shard_mode = s.shard_api;
        if (begin) *begin = s.sbegin;
        if (end) *end = s.send;
    });
}

ifctn_status ifctn_create(ifctn_ctx** out, int order, const int64_t* dims, const int32_t* ranks,
                          ifctn_dtype dtype, double rho, const void* observed, const uint8_t* mask,
                          const void* init_factors, void* workspace, size_t workspace_bytes,
                          const ifctn_dist* dist, void* stream, unsigned flags) {
    if (!out) return IFCTN_E_ARG;
    *out = nullptr;
    std::unique_ptr<ifctn_ctx> ctx(new ifctn_ctx());
    ifctn_status st = guarded(ctx.get(), [&] {
        if (!observed || !mask || !init_factors) ifctn::fail(IFCTN_E_ARG, "observed/mask/init_factors must not be NULL");
        if (!(rho > 0.0) || !std::isfinite(rho)) ifctn::fail(IFCTN_E_ARG, "rho must be > 0");
        ifctn::Shape s = ifctn::make_shape(order, dims, ranks, dtype, dist);
        // Ω must be non-empty (checked on the host copy of the mask when it is host memory;
        // device masks are checked by the caller-side binding).
        if (!ifctn::is_device_ptr(mask)) {
            bool any = false;
            for (int64_t u = 0; u < s.nloc && !any; ++u) any = mask[u] != 0;
            if (!any && s.world == 1) ifctn::fail(IFCTN_E_NO_OBSERVED, "the mask has no observed entry");
        }
        auto build = [&](auto* tag) {
            using T = std::remove_pointer_t<decltype(tag)>;
            auto* sv = new ifctn::Solver<T>();
            ctx->s.reset(sv);
            sv->s = s;
            sv->lay = ifctn::make_layout(s);
            sv->rho = rho;
            sv->flags = flags;
            if (s.peer) {
                sv->setup_peer(dist);
            } else if (s.dpath) {
                if (dist->host_allreduce) {
                    sv->host_allreduce = dist->host_allreduce;
                    sv->host_user = dist->user;
                    CU(cudaMallocHost(&sv->hred, (size_t)s.proj_elems * sizeof(double)));
                } else {
                    if (!dist->nccl_unique_id)
                        ifctn::fail(IFCTN_E_ARG, "dist->nccl_unique_id (or host_allreduce) must be set when world > 1");
                    sv->nccl = ifctn::NcclLite::get();
                    if (!sv->nccl) ifctn::fail(IFCTN_E_NCCL, "libnccl.so.2 could not be loaded");
                    int r = sv->nccl->commInitRank(&sv->comm, s.world, dist->nccl_unique_id, s.rank);
                    if (r != 0) ifctn::fail(IFCTN_E_NCCL, std::string("ncclCommInitRank: ") + sv->nccl->errorString(r));
                }
            }
            sv->init(observed, mask, init_factors, workspace, workspace_bytes, (cudaStream_t)stream);
        };
        if (dtype == IFCTN_F32) build((float*)nullptr);
        else build((double*)nullptr);
    });
    if (st != IFCTN_OK) return st;
    *out = ctx.release();
    return IFCTN_OK;
}

#define CTX_CALL(ctx, body)                                    \
    if (!(ctx) || !(ctx)->s) return IFCTN_E_ARG;               \
    return guarded((ctx), [&] { body; })

ifctn_status ifctn_sweep(ifctn_ctx* ctx, int t_max, double eps, int* sweeps_done, ifctn_trace_row* trace) {
    CTX_CALL(ctx, ctx->s->sweep(t_max, eps, sweeps_done, trace));
}

ifctn_status ifctn_sync(ifctn_ctx* ctx) { CTX_CALL(ctx, ctx->s->sync_check()); }

ifctn_status ifctn_profile_sweep(ifctn_ctx* ctx, float* ms, int capacity, int* count) {
    CTX_CALL(ctx, {
        if (!ms || !count || capacity < 1) ifctn::fail(IFCTN_E_ARG, "ms/count must not be NULL");
        *count = ctx->s->profile_sweep(ms, capacity);
    });
}

ifctn_status ifctn_reconstruct(ifctn_ctx* ctx, int what, void* out) {
    CTX_CALL(ctx, ctx->s->reconstruct(what, out));
}

ifctn_status ifctn_get_factors(ifctn_ctx* ctx, void* out) { CTX_CALL(ctx, ctx->s->get_factors(out)); }

ifctn_status ifctn_rse(ifctn_ctx* ctx, const void* truth, double* rse) {
    CTX_CALL(ctx, {
        if (!rse) ifctn::fail(IFCTN_E_ARG, "rse must not be NULL");
        *rse = ctx->s->rse(truth);
    });
}

ifctn_status ifctn_metrics(ifctn_ctx* ctx, const void* truth, double* out) {
    CTX_CALL(ctx, {
        if (!out) ifctn::fail(IFCTN_E_ARG, "out must not be NULL");
        ctx->s->metrics(truth, out);
    });
}

ifctn_status ifctn_objective(ifctn_ctx* ctx, double* f) {
    CTX_CALL(ctx, {
        if (!f) ifctn::fail(IFCTN_E_ARG, "f must not be NULL");
        *f = ctx->s->objective();
    });
}

ifctn_status ifctn_block_coefficients(ifctn_ctx* ctx, int k, int i, double* beta, double* omega) {
    CTX_CALL(ctx, ctx->s->block_coefficients(k, i, beta, omega));
}

ifctn_status ifctn_block_update(ifctn_ctx* ctx, int k, int i) { CTX_CALL(ctx, ctx->s->block_update(k, i)); }

ifctn_status ifctn_x_update(ifctn_ctx* ctx, double* norms) { CTX_CALL(ctx, ctx->s->x_update(norms)); }

ifctn_status ifctn_destroy(ifctn_ctx* ctx) {
    if (!ctx) return IFCTN_E_ARG;
    delete ctx;
    return IFCTN_OK;
}

ifctn_status ifctn_peer_selftest(int world, int rounds, int64_t n, int64_t* errors) {
    using namespace ifctn;
    if (world < 2 || world > kPeerMax || rounds < 1 || n < 1 || n > (1 << 20) || !errors) return IFCTN_E_ARG;
    std::vector<double*> bufs((size_t)world, nullptr);
    unsigned long long* ep = nullptr;
    unsigned* cnt = nullptr;
    unsigned* err = nullptr;
    ifctn_status st = IFCTN_OK;
    auto ck = [&](cudaError_t e) {
        if (e != cudaSuccess && st == IFCTN_OK) {
            st = IFCTN_E_CUDA;
            g_last_err = cudaGetErrorString(e);
        }
    };
    PeerCtx X{};
    X.W = world;
    X.rank = 0;
    X.slot_elems = n;
    for (int r = 0; r < world; ++r) {
        ck(cudaMalloc(&bufs[(size_t)r], sizeof(double) * (size_t)(kPeerHeader + 2 * n)));
        if (st == IFCTN_OK) ck(cudaMemset(bufs[(size_t)r], 0, sizeof(double) * (size_t)(kPeerHeader + 2 * n)));
        X.bufs[r] = bufs[(size_t)r];
    }
    ck(cudaMalloc(&ep, sizeof(unsigned long long) * kPeerMax));
    ck(cudaMalloc(&cnt, sizeof(unsigned) * 2 * kPeerMax));
    ck(cudaMalloc(&err, sizeof(unsigned)));
    if (st == IFCTN_OK) {
        ck(cudaMemset(ep, 0, sizeof(unsigned long long) * kPeerMax));
        ck(cudaMemset(cnt, 0, sizeof(unsigned) * 2 * kPeerMax));
        ck(cudaMemset(err, 0, sizeof(unsigned)));
        X.epoch = ep;
        X.arrive = cnt;
        // 2 CTAs per virtual rank, all co-resident (cooperative launch guarantees it or fails)
        void* args[] = {&X, &rounds, &n, &err};
        ck(cudaLaunchCooperativeKernel((const void*)peer_selftest, dim3((unsigned)(2 * world)), dim3(128), args, 0, 0));
        ck(cudaDeviceSynchronize());
        unsigned h = 0;
        ck(cudaMemcpy(&h, err, sizeof(unsigned), cudaMemcpyDeviceToHost));
        *errors = (int64_t)h;
    }
    for (double* b : bufs)
        if (b) cudaFree(b);
    if (ep) cudaFree(ep);
    if (cnt) cudaFree(cnt);
    if (err) cudaFree(err);
    return st;
}

const char* ifctn_status_string(ifctn_status s) {
    if ((int)s < 0 || (int)s >= (int)(sizeof(ifctn::kStatusNames) / sizeof(ifctn::kStatusNames[0])))
        return "IFCTN_E_UNKNOWN";
    return ifctn::kStatusNames[(int)s];
}

const char* ifctn_last_error(const ifctn_ctx* ctx) {
    if (ctx) return ctx->err.c_str();
    return g_last_err.c_str();
}

int64_t ifctn_launch_count(const ifctn_ctx* ctx) {
    if (!ctx || !ctx->s) return 0;
    return ctx->s->launches();
}

}  // extern "C"

#ifdef IFCTN_EXP_TIMELINE
extern "C" int ifctn_exp_timeline(unsigned long long* out, int n) {
    cudaDeviceSynchronize();
    if (n < 0) {  // clear
        static unsigned long long z[3 * 4096] = {};
        return (int)cudaMemcpyToSymbol(ifctn::g_tl, z, sizeof(z));
    }
    return (int)cudaMemcpyFromSymbol(out, ifctn::g_tl, sizeof(unsigned long long) * 3 * (size_t)(n < 4096 ? n : 4096));
}
#endif
