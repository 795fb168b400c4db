// sweep.cuh — persistent whole-sweep kernel.
//
// Small tensors (C1–C4) are bound by the per-kernel fixed costs of a sweep's 3·N(N−1)+2
// launches, not by bytes.  `sweep_persistent` runs t_max complete sweeps in ONE cooperative
// launch: the same device bodies as the individual kernels (fiber_pass_body,
// fiber_pass_vb_body, reduce_partials(_warp)_body, block_solve(_big)_body,
// finalize_norms_body), one op after another, separated by grid-wide barriers
// (cooperative_groups grid.sync).  Every op keeps the work split of its standalone launch
// (one wave of pass CTAs, virtual blocks for reduces and solves, 128 solve threads, 1024
// virtual finaliser threads), so the result is bit-identical to the plain (unfused) launch
// sequence.  Single GPU only.
#pragma once

#include <cooperative_groups.h>

#include "fiber_tile.cuh"
#include "fiber_walk.cuh"
#include "solve.cuh"

namespace ifctn {

enum SweepOpKind : int { OP_PASS = 0, OP_REDUCE = 1, OP_SOLVE = 2, OP_SOLVE_BIG = 3, OP_FINALIZE = 4 };

struct SweepOp {
    int kind;
    int variant;   // pass: mode·4 + vblk·2 + hres; reduce: 0 warp, 1 CTA; solve: R
    int idx;       // index into the op kind's parameter array
    int pad;
    int64_t nvb;   // virtual blocks (reduce: x·y·z; solve: columns)
    int gy, gz;    // reduce grid y, z
};

template <typename T>
struct SweepProg {
    const SweepOp* ops;
    int nops;
    const PassParams<T>* pass;
    const ReduceParams<T>* red;
    const SolveParams<T>* sol;
    // finaliser
    const double* norms;
    int64_t ngroups;
    const double* delta;
    int64_t ndelta;
    double* p5;
    double* scal;
    int* flags;
};

template <typename T, int EPL, int LPF>
__device__ __forceinline__ void run_pass(int variant, const PassParams<T>& P, unsigned char* sm, int cta, int ncta) {
    switch (variant) {
        case PASS_KEPT1 * 4 + 0: fiber_pass_body<T, PASS_KEPT1, EPL, LPF, false>(P, sm, cta); break;
        case PASS_KEPT1 * 4 + 1: fiber_pass_body<T, PASS_KEPT1, EPL, LPF, true>(P, sm, cta); break;
        case PASS_KEPT1 * 4 + 3: fiber_pass_vb_body<T, PASS_KEPT1, EPL, LPF, true>(P, sm, ncta); break;
        case PASS_RED1 * 4 + 0: fiber_pass_body<T, PASS_RED1, EPL, LPF, false>(P, sm, cta); break;
        case PASS_RED1 * 4 + 1: fiber_pass_body<T, PASS_RED1, EPL, LPF, true>(P, sm, cta); break;
        case PASS_RED1 * 4 + 3: fiber_pass_vb_body<T, PASS_RED1, EPL, LPF, true>(P, sm, ncta); break;
        case PASS_REFILL * 4 + 0: fiber_pass_body<T, PASS_REFILL, EPL, LPF, false>(P, sm, cta); break;
        case PASS_REFILL * 4 + 1: fiber_pass_body<T, PASS_REFILL, EPL, LPF, true>(P, sm, cta); break;
        default: break;
    }
}

// variant ≥ 16: warp per column (block_solve_w): warps 0–3 take columns 4·vb + warp
template <typename T>
__device__ __forceinline__ void run_solve_w(int R, const SolveParams<T>& P, int64_t vb, double* red, double* cs) {
    const int w = threadIdx.x >> 5;
    const int64_t j = vb * 4 + w;
    if (w >= 4 || j >= P.Ik) return;
    double* rw = red + w * 64;
    double* cw = cs + w * 16;
    switch (R) {
        case 1: block_solve_body<T, 1, SOLVE_FULL, true>(P, j, 32, rw, cw); break;
        case 2: block_solve_body<T, 2, SOLVE_FULL, true>(P, j, 32, rw, cw); break;
        case 3: block_solve_body<T, 3, SOLVE_FULL, true>(P, j, 32, rw, cw); break;
        case 4: block_solve_body<T, 4, SOLVE_FULL, true>(P, j, 32, rw, cw); break;
        case 5: block_solve_body<T, 5, SOLVE_FULL, true>(P, j, 32, rw, cw); break;
        case 6: block_solve_body<T, 6, SOLVE_FULL, true>(P, j, 32, rw, cw); break;
        case 7: block_solve_body<T, 7, SOLVE_FULL, true>(P, j, 32, rw, cw); break;
        case 8: block_solve_body<T, 8, SOLVE_FULL, true>(P, j, 32, rw, cw); break;
        default: block_solve_body<T, 9, SOLVE_FULL, true>(P, j, 32, rw, cw); break;
    }
}

template <typename T>
__device__ __forceinline__ void run_solve(int R, const SolveParams<T>& P, int64_t j, double* red, double* cs) {
    switch (R) {
        case 1: block_solve_body<T, 1, SOLVE_FULL>(P, j, 128, red, cs); break;
        case 2: block_solve_body<T, 2, SOLVE_FULL>(P, j, 128, red, cs); break;
        case 3: block_solve_body<T, 3, SOLVE_FULL>(P, j, 128, red, cs); break;
        case 4: block_solve_body<T, 4, SOLVE_FULL>(P, j, 128, red, cs); break;
        case 5: block_solve_body<T, 5, SOLVE_FULL>(P, j, 128, red, cs); break;
        case 6: block_solve_body<T, 6, SOLVE_FULL>(P, j, 128, red, cs); break;
        case 7: block_solve_body<T, 7, SOLVE_FULL>(P, j, 128, red, cs); break;
        case 8: block_solve_body<T, 8, SOLVE_FULL>(P, j, 128, red, cs); break;
        default: block_solve_body<T, 9, SOLVE_FULL>(P, j, 128, red, cs); break;
    }
}

template <typename T, int EPL, int LPF>
__global__ void __launch_bounds__(kPassThreads, kPassMinBlocks)
    sweep_persistent(const __grid_constant__ SweepProg<T> G, int nsweeps) {
    namespace cg = cooperative_groups;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    cg::grid_group grid = cg::this_grid();
    const int cta = blockIdx.x, ncta = gridDim.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double* scratch = reinterpret_cast<double*>(smem_raw);
    for (int sweep = 0; sweep < nsweeps; ++sweep) {
        for (int o = 0; o < G.nops; ++o) {
            const SweepOp op = G.ops[o];
            if (op.kind == OP_PASS) {
                run_pass<T, EPL, LPF>(op.variant, G.pass[op.idx], smem_raw, cta, ncta);
                __syncthreads();
                // retire this pass's stage barriers before the shared memory is reused
                if (lane == 0) {
                    // (8 barrier slots per warp are reserved; invalidate the ones a pass uses)
                    constexpr int DB = IFCTN_PLAIN_D > kRingStages ? IFCTN_PLAIN_D : kRingStages;
                    const int d = (op.variant & 2) ? kRingStages : IFCTN_PLAIN_D;
                    uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw) + warp * d;
                    for (int s = 0; s < d && s < DB; ++s) mbar_inval(bars + s);
                }
            } else if (op.kind == OP_REDUCE) {
                const ReduceParams<T>& P = G.red[op.idx];
                unsigned* last = reinterpret_cast<unsigned*>(scratch + 512);
                for (int64_t v = cta; v < op.nvb; v += ncta) {
                    if (op.variant == 0) {
                        reduce_partials_warp_body(P, v);
                    } else {
                        const int64_t nx = op.nvb / ((int64_t)op.gy * op.gz);
                        const int64_t x = v % nx, yz = v / nx;
                        reduce_partials_body(P, x, (int)(yz % op.gy), (int)(yz / op.gy), scratch, scratch + 256, last);
                    }
                    __syncthreads();
                }
            } else if (op.kind == OP_SOLVE) {
                const SolveParams<T>& P = G.sol[op.idx];
                for (int64_t j = cta; j < op.nvb; j += ncta) {
                    if (op.variant >= 16) run_solve_w<T>(op.variant - 16, P, j, scratch, scratch + 4 * 64);
                    else run_solve<T>(op.variant, P, j, scratch, scratch + 4 * 64);
                    __syncthreads();
                }
            } else if (op.kind == OP_SOLVE_BIG) {
                const SolveParams<T>& P = G.sol[op.idx];
                int* okp = reinterpret_cast<int*>(scratch);
                double* colb = scratch + 2;
                double* dinv = scratch + 2 + 128;
                double* bsm = scratch + 256;
                for (int64_t j = cta; j < op.nvb; j += ncta) {
                    block_solve_big_body<T, SOLVE_FULL>(P, j, bsm, okp, colb, dinv);
                    __syncthreads();
                }
            } else if (op.kind == OP_FINALIZE) {
                if (cta == 0)
                    finalize_norms_body(G.norms, G.ngroups, G.delta, G.ndelta, 0, 0, G.p5, G.scal, G.flags, 0, 1,
                                        scratch);
            }
            grid.sync();
        }
    }
}

// shared scratch of the non-pass ops (doubles): reduce 512 + flag, solve 8·44 + 8,
// finaliser 5·1024, big solve 256 + its staging
__host__ inline size_t sweep_scratch_bytes(size_t big_solve_smem) {
    size_t b = sizeof(double) * 5 * 1024;
    b = b > sizeof(double) * (256 + 8) + big_solve_smem ? b : sizeof(double) * (256 + 8) + big_solve_smem;
    return b;
}

}  // namespace ifctn
