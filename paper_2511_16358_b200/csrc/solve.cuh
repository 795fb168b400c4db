// solve.cuh — second-stage reduction of the K2 partials, K3 (Gram/RHS + ρI + batched SPD
// solve + H refresh, steps a3/a4), the per-sweep finaliser, and layout/RSE kernels.
#pragma once

#include "common.cuh"

namespace ifctn {

// ---- stage 2 of a2: fixed-order fp64 sum of the partial slots of every kept value v ------
// Slots of v are g + v for g in [⌊vFR/L⌋, ⌊((v+1)FR−1)/L⌋] (each group covers L fibres).
// v-blocking (fiber_pass_vb): v = (kidx0, kidx1) lies in block vb at offset vv; the warps that
// covered block vb are g0..g1 and their slot of v is (g + vb)·VB + vv.  VB = 1 is the plain
// layout (vb = v).  Returns the element offset of (v, first slot, e = 0) and the slot count.
template <typename T>
__device__ __forceinline__ int64_t slot_base(const ReduceParams<T>& P, int64_t v, int64_t& nslots) {
    const int64_t kx0 = v % P.kdim0, kx1 = v / P.kdim0;
    const int64_t vb = kx0 / P.VB + P.nb0 * kx1, vv = kx0 % P.VB;
    const int64_t g0 = (vb * P.FR * P.VB) / P.L;
    const int64_t g1 = ((vb + 1) * P.FR * P.VB - 1) / P.L;
    nslots = g1 - g0 + 1;
    return ((g0 + vb) * P.VB + vv) * P.Lv;
}

// β/ω destination of (v, e); −1 for the padding rows of mode 1
template <typename T>
__device__ __forceinline__ int64_t out_index(const ReduceParams<T>& P, int64_t v, int64_t e) {
    if (P.kept1) {
        if (e >= P.I1) return -1;
        return P.kIsMode0 ? (e * P.Ii + v) : (v * P.Ii + e);
    }
    const int64_t x0 = v % P.kdim0, x1 = v / P.kdim0;  // kmode[0], kmode[1] indices
    const int64_t j = P.kmode0IsK ? x0 : x1;
    const int64_t a = P.kmode0IsK ? x1 : x0;
    return j * P.Ii + a;
}

// Lv = 1 (RED1 blocks, many v with few slots each): one warp per v, lanes stride the slots,
// butterfly sum (fixed order).
template <typename T>
__device__ __forceinline__ void reduce_partials_warp_body(const ReduceParams<T>& P, int64_t bx) {
    const int64_t v = bx * 8 + (threadIdx.x >> 5);
    if (v >= P.NV) return;
    const int lane = threadIdx.x & 31;
    int64_t nslots;
    const int64_t base = slot_base(P, v, nslots);
    const int64_t stride = P.VB;  // Lv = 1: consecutive slots are VB elements apart
    IFCTN_CHECK(nslots < 1 || base + (nslots - 1) * stride < P.part_cap, "reduce_warp slots");
    double b = 0.0, w = 0.0;
    for (int64_t s = lane; s < nslots; s += 32) {
        b += (double)P.part_b[base + s * stride];
        w += (double)P.part_w[base + s * stride];
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        b += __shfl_xor_sync(0xffffffffu, b, off);
        w += __shfl_xor_sync(0xffffffffu, w, off);
    }
    if (lane == 0) {
        const int64_t o = out_index(P, v, 0);
        if (o >= 0) {
            P.beta[o] = b;
            P.omega[o] = w;
        }
    }
}

template <typename T>
__global__ void __launch_bounds__(256) reduce_partials_warp(const ReduceParams<T> P) {
    reduce_partials_warp_body(P, blockIdx.x);
}

// CTA (v = bx, element tile = by, slot share z = bz); sb, sw: 256 doubles of shared scratch
template <typename T>
__device__ __forceinline__ void reduce_partials_body(const ReduceParams<T>& P, int64_t bx, int by, int bz,
                                                     double* sb, double* sw, unsigned* last_flag) {
    const int64_t v = bx;
    int64_t nslots;
    const int64_t base = slot_base(P, v, nslots);
    // this CTA: elements e = tile·ET + tx, slots [s0, s1) split over ny = 256/ET thread rows
    const int ET = P.ET, ny = 256 / ET;
    const int tx = threadIdx.x % ET, ty = threadIdx.x / ET;
    const int z = bz;
    const int64_t chunk = (nslots + P.Z - 1) / P.Z;
    const int64_t s0 = z * chunk, s1 = min(nslots, s0 + chunk);
    const int64_t e = (int64_t)by * ET + tx;
    double b = 0.0, w = 0.0;
    if (e < P.Lv) {
        const int64_t stride = (int64_t)ny * P.VB * P.Lv;
        int64_t o = base + (s0 + ty) * P.VB * P.Lv + e;
        int64_t s = s0 + ty;
        // 4 independent loads in flight per thread; the adds stay in slot order
        for (; s + 3 * ny < s1; s += 4 * ny, o += 4 * stride) {
            const T b0 = P.part_b[o], b1 = P.part_b[o + stride], b2 = P.part_b[o + 2 * stride],
                    b3 = P.part_b[o + 3 * stride];
            const T w0 = P.part_w[o], w1 = P.part_w[o + stride], w2 = P.part_w[o + 2 * stride],
                    w3 = P.part_w[o + 3 * stride];
            b += (double)b0; b += (double)b1; b += (double)b2; b += (double)b3;
            w += (double)w0; w += (double)w1; w += (double)w2; w += (double)w3;
        }
        for (; s < s1; s += ny, o += stride) {
            b += (double)P.part_b[o];
            w += (double)P.part_w[o];
        }
    }
    sb[threadIdx.x] = b;
    sw[threadIdx.x] = w;
    __syncthreads();
    for (int st = ny >> 1; st > 0; st >>= 1) {
        if (ty < st) {
            sb[threadIdx.x] += sb[threadIdx.x + st * ET];
            sw[threadIdx.x] += sw[threadIdx.x + st * ET];
        }
        __syncthreads();
    }
    if (P.Z > 1) {
        // publish this z-share, last CTA of (v, tile) to arrive sums the Z shares in z order
        const int64_t id = (int64_t)by * P.NV + v;
        double* my = P.scr + ((id * P.Z + z) * ET) * 2;
        if (ty == 0) {
            my[2 * tx] = sb[tx];
            my[2 * tx + 1] = sw[tx];
        }
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) *last_flag = (atomicAdd(P.cnt + id, 1u) == (unsigned)(P.Z - 1));
        __syncthreads();
        if (!*last_flag) return;
        __threadfence();
        if (ty == 0) {
            double bb = 0.0, ww = 0.0;
            const double* p = P.scr + id * P.Z * ET * 2 + 2 * tx;
            for (int zz = 0; zz < P.Z; ++zz) {
                bb += __ldcg(p + zz * ET * 2);
                ww += __ldcg(p + zz * ET * 2 + 1);
            }
            sb[tx] = bb;
            sw[tx] = ww;
        }
        if (threadIdx.x == 0) P.cnt[id] = 0u;
    }
    if (ty == 0 && e < P.Lv) {
        const int64_t o = out_index(P, v, e);
        if (o >= 0) {
            P.beta[o] = sb[tx];
            P.omega[o] = sw[tx];
        }
    }
}

template <typename T>
__global__ void __launch_bounds__(256) reduce_partials(const ReduceParams<T> P) {
    __shared__ double sb[256], sw[256];
    __shared__ unsigned last;
    reduce_partials_body(P, blockIdx.x, blockIdx.y, blockIdx.z, sb, sw, &last);
}

__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) x += __shfl_xor_sync(0xffffffffu, x, off);
    return x;
}

// ---- a3 + a4: per column j of G_{k,i} (Eq. 8) -------------------------------
//   Gram_j = Σ_a ω(a,j) g_a g_aᵀ + ρI,  rhs_j = Σ_a β(a,j) g_a + ρ c_old,  g_a = G_{i,k}(:,a)
//   c = Gram_j⁻¹ rhs_j by Cholesky (fp64);  then row j of H_{k,i} = cᵀ G_{i,k} (refresh).
// SM = SOLVE_FULL: all of it.  Multi-GPU (k ≠ shard mode): SOLVE_PROJECT writes
// this rank's projected partial (Gram upper triangle, rhs) = Σ_{a local} …, the partials are
// summed across ranks (NCCL all-reduce), then SOLVE_FROM_PROJ adds ρI, ρc_old and solves.
enum SolveMode : int { SOLVE_FULL = 0, SOLVE_PROJECT = 1, SOLVE_FROM_PROJ = 2 };

// β(a,j), ω(a,j) of block (k,i) straight from the a2 partial slots (fixed slot order), for a
// solve that absorbs the second-stage reduction: the inverse of out_index().
template <typename T>
__device__ __forceinline__ void column_coeffs(const ReduceParams<T>& Q, int64_t j, int64_t a, double& b,
                                              double& w) {
    int64_t v, e;
    if (Q.kept1) {
        if (Q.kIsMode0) {
            e = j;
            v = a;
        } else {
            e = a;
            v = j;
        }
    } else {
        e = 0;
        v = Q.kmode0IsK ? (j + Q.kdim0 * a) : (a + Q.kdim0 * j);
    }
    int64_t nslots;
    const int64_t base = slot_base(Q, v, nslots) + e;
    const int64_t stride = Q.VB * Q.Lv;
    IFCTN_CHECK(nslots < 1 || base + (nslots - 1) * stride < Q.part_cap, "solve gather slots");
    // all loads of a group of 8 slots in flight before the (in-order) sums: one L2 round
    // trip per 8 slots instead of one per slot (predicated tail); same summation order
    double sb = 0.0, sw = 0.0;
    for (int64_t s = 0; s < nslots; s += 8) {
        const int64_t rem = nslots - s;
        T vb[8], vw[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            vb[q] = q < rem ? Q.part_b[base + (s + q) * stride] : T(0);
            vw[q] = q < rem ? Q.part_w[base + (s + q) * stride] : T(0);
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            if (q < rem) {
                sb += (double)vb[q];
                sw += (double)vw[q];
            }
        }
    }
    b = sb;
    w = sw;
}

template <typename T, int R, int SM>
// nthr (a multiple of 32, ≤ blockDim.x) threads take part; the others only pass the barriers.
// red: (nthr/32)·NA + NA doubles of shared scratch, cs: R.
__device__ __forceinline__ void block_solve_body(const SolveParams<T>& P, int64_t j, int nthr,
                                                 double* red, double* cs, const T* cold_pre = nullptr) {
    constexpr int NG = R * (R + 1) / 2;
    constexpr int NA = NG + R;
    constexpr int KEEP = 2;  // columns a of G_{i,k} kept in registers for the H refresh
    const int nw = nthr >> 5;
    const int tid = (int)threadIdx.x;
    const int ntot = (int)blockDim.x;
    double* sum = red + nw * NA;
    auto sync = [&]() { __syncthreads(); };
    // peer exchange (peer.cuh): the FROM_PROJ solve is the collective's consumer
    unsigned long long pe = 0;
    if constexpr (SM == SOLVE_FROM_PROJ)
        if (P.use_peer) {
            pe = peer_next_epoch(P.peer);
            peer_publish_wait(P.peer, pe);
        }
    double acc[NA];
#pragma unroll
    for (int t = 0; t < NA; ++t) acc[t] = 0.0;
    T gk[KEEP][R];  // this thread's a = tid + q·nthr (q < KEEP) columns, reused by the H refresh
    const int64_t na = (SM == SOLVE_FROM_PROJ || tid >= nthr) ? 0 : P.Ii;
    int q = 0;
    for (int64_t a = tid; a < na; a += nthr, ++q) {
        double b, w;
        if (P.fused_reduce) {
            column_coeffs(P.red, j, a, b, w);
        } else {
            b = P.beta[j * P.Ii + a];
            w = P.omega[j * P.Ii + a];
        }
        T gt[R];
#pragma unroll
        for (int r = 0; r < R; ++r) gt[r] = P.Gik[a * R + r];
        double g[R];
#pragma unroll
        for (int r = 0; r < R; ++r) g[r] = (double)gt[r];
        if (q < KEEP) {
#pragma unroll
            for (int qq = 0; qq < KEEP; ++qq)
                if (qq == q)
#pragma unroll
                    for (int r = 0; r < R; ++r) gk[qq][r] = gt[r];
        }
        int t = 0;
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
            for (int s = r; s < R; ++s) acc[t++] += w * g[r] * g[s];
#pragma unroll
        for (int r = 0; r < R; ++r) acc[NG + r] += b * g[r];
    }
    const int wid = tid >> 5, ln = tid & 31;
    if constexpr (SM != SOLVE_FROM_PROJ) {
#pragma unroll
        for (int t = 0; t < NA; ++t) {
            const double s = warp_sum(acc[t]);
            if (ln == 0 && wid < nw) red[wid * NA + t] = s;
        }
        sync();
        // entry t = Σ_q red[q][t], q ascending (one thread per entry)
        double* pdst = nullptr;
        if constexpr (SM == SOLVE_PROJECT) pdst = P.use_peer ? peer_my_slot(P.peer) : P.proj;
        for (int t = tid; t < NA; t += ntot) {
            double v = 0.0;
            for (int qw = 0; qw < nw; ++qw) v += red[qw * NA + t];
            if constexpr (SM == SOLVE_PROJECT) pdst[j * NA + t] = v;
            else sum[t] = v;
        }
        if constexpr (SM == SOLVE_PROJECT) return;
    } else {
        for (int t = tid; t < NA; t += ntot) sum[t] = P.use_peer ? peer_sum(P.peer, pe, j * NA + t) : P.proj[j * NA + t];
    }
    sync();
    if (tid == 0) {
        // Cholesky with reciprocal pivots (1/√d by rsqrt; no divisions), substitutions by
        // multiplication with the stored reciprocals
        double A[R][R], L[R][R], inv[R], y[R], c[R], cold[R];
        int t = 0;
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
            for (int s = r; s < R; ++s) {
                const double v = sum[t];
                A[r][s] = v;
                A[s][r] = v;
                ++t;
            }
        double rhs[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            cold[r] = (double)(cold_pre ? cold_pre[r] : P.Gki[j * R + r]);
            A[r][r] += P.rho;
            rhs[r] = sum[NG + r] + P.rho * cold[r];
        }
        bool ok = true;
#pragma unroll
        for (int cc = 0; cc < R; ++cc) {
            double d = A[cc][cc];
#pragma unroll
            for (int s = 0; s < cc; ++s) d = fma(-L[cc][s], L[cc][s], d);
            if (!(d > 0.0)) ok = false;
            inv[cc] = rsqrt(d > 0.0 ? d : 1.0);
#pragma unroll
            for (int r = cc + 1; r < R; ++r) {
                double v = A[r][cc];
#pragma unroll
                for (int s = 0; s < cc; ++s) v = fma(-L[r][s], L[cc][s], v);
                L[r][cc] = v * inv[cc];
            }
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
            double v = rhs[r];
#pragma unroll
            for (int s = 0; s < r; ++s) v = fma(-L[r][s], y[s], v);
            y[r] = v * inv[r];
        }
#pragma unroll
        for (int r = R - 1; r >= 0; --r) {
            double v = y[r];
#pragma unroll
            for (int s = r + 1; s < R; ++s) v = fma(-L[s][r], c[s], v);
            c[r] = v * inv[r];
        }
        if (!ok) {
            atomicOr(P.flags, 1);
#pragma unroll
            for (int r = 0; r < R; ++r) c[r] = cold[r];
        }
        double d2 = 0.0;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const T cT = (T)c[r];
            P.Gki[j * R + r] = cT;
            cs[r] = (double)cT;
            const double dd = (double)cT - cold[r];
            d2 += dd * dd;
        }
        P.delta[j] = d2;
    }
    sync();
    // H refresh: H_{k,i}(j, a) = Σ_r c_r G_{i,k}(r, a) — from the registers where kept
    double cr[R];
#pragma unroll
    for (int r = 0; r < R; ++r) cr[r] = cs[r];
    q = 0;
    for (int64_t a = tid; a < P.Ii; a += ntot, ++q) {
        T gt[R];
        if (ntot == nthr && na > 0 && q < KEEP) {
#pragma unroll
            for (int qq = 0; qq < KEEP; ++qq)
                if (qq == q)
#pragma unroll
                    for (int r = 0; r < R; ++r) gt[r] = gk[qq][r];
        } else {
#pragma unroll
            for (int r = 0; r < R; ++r) gt[r] = P.Gik[a * R + r];
        }
        double h = 0.0;
#pragma unroll
        for (int r = 0; r < R; ++r) h += cr[r] * (double)gt[r];
        const int64_t o = P.k_lt_i ? (P.h_off + a * P.h_ld + j) : (P.h_off + j * P.h_ld + a);
        P.H[o] = (T)h;
    }
    if constexpr (SM == SOLVE_FROM_PROJ)
        if (P.use_peer) peer_retire(P.peer, pe);
}

template <typename T, int R, int SM>
__global__ void __launch_bounds__(128) block_solve(const SolveParams<T> P) {
    constexpr int NA = R * (R + 1) / 2 + R;
    __shared__ double red[5 * NA];
    __shared__ double cs[R];
    // the column's old coefficients were written by this block's solve of the previous sweep (or
    // at create): at least two kernels back, complete before this grid could start — loaded
    // ahead of the wait, off the critical path
    T cold_pre[R];
    if (threadIdx.x == 0) {
#pragma unroll
        for (int r = 0; r < R; ++r) cold_pre[r] = P.Gki[(int64_t)blockIdx.x * R + r];
    }
    pdl_wait();
    pdl_launch();
    block_solve_body<T, R, SM>(P, blockIdx.x, 128, red, cs, cold_pre);
}

// ---- a3 + a4 for large ranks (the paper's grids reach R_{1,2} = 36) --------
// Same mathematics as block_solve (Eq. 8) with the rank a runtime value ≤ 64.
// One CTA (256 threads) per column j:
//   * G_{i,k} is staged in shared memory as fp64 in tiles of `ta` columns a — normally all of
//     it at once; the loads of a batch are all in flight before the stores; reused by the H
//     refresh;
//   * Gram_j = G_{i,k} diag(ω(:,j)) G_{i,k}ᵀ and rhs_j = G_{i,k} β(:,j): for R ≤ 39 one fp64
//     tensor-core product (big_gram_mma below: DMMA m8n8k4, K split over the 8 warps, partial
//     tiles summed in warp order through a scratch); else (and under IFCTN_FLAG_NO_DMMA) SIMT
//     register tiles: task = (4×4 tile of the Gram upper triangle, or a 4-row tile of the rhs;
//     a-residue h mod KS), KS = the a-split that fills the CTA; the KS partial tiles are added
//     in h order (fixed order, deterministic);
//   * + ρI, ρ c_old, then a right-looking Cholesky in 4×4 blocks over the whole CTA (thread 0
//     factors the diagonal block in registers with rsqrt pivots, one thread per row solves the
//     panel, all threads apply the rank-4 trailing update); rhsᵀ rides as row Rp of the matrix,
//     so the same panel/trailing steps perform the forward substitution L y = rhs;
//   * warp 0: back substitution Lᵀ c = y (lane owns rows lane, lane + 32; the pivot value is
//     broadcast by shuffle); ‖Δc‖²;
//   * row j of H_{k,i}: on DMMA (rows a in tiles of 8, c in column 0 of B), or 8 threads per a.
constexpr int kBigThreads = 256;
#ifndef IFCTN_BIG_MINB  // CTAs per SM the register allocation allows
#define IFCTN_BIG_MINB 1
#endif

constexpr int kBigMmaMaxR = 39;  // big_gram_mma: ≤ 15 output tiles (30 accumulators) per warp
constexpr int kBigTPR = 4;       // big_gram_mma: tiles per round of its cross-warp sum (scratch: 8 warps × 4 × 64)
__host__ __device__ inline int big_solve_rp(int R) { return (R + 3) & ~3; }
__host__ __device__ inline int big_solve_lda(int R) { return big_solve_rp(R) + 1; }  // odd: rows hit different banks
// shared memory: G tile (ta·R + Rp doubles) + fp64 [A: Rp + 1 rows of lda (row Rp: rhsᵀ), ω, β (ta each),
// rhs, c, c_old (Rp each), the mma path's cross-warp scratch]
__host__ __device__ inline size_t big_solve_smem(int R, int ta, int /*esize*/) {
    const int Rp = big_solve_rp(R);
    return sizeof(double) * ((size_t)ta * R + Rp + (size_t)(Rp + 1) * big_solve_lda(R) + 2 * (size_t)ta + 3 * (size_t)Rp +
                             (R <= kBigMmaMaxR ? (kBigThreads / 32) * kBigTPR * 64 + 1 : 0));
}

// G_{i,k}(:, a0 …) (n = na·R elements of T) into shared memory as fp64, followed by `pad` zeros
// (the tiles over-read 4-wide): 16-byte loads when the source allows, every load of a thread
// in flight before its stores (one L2 round trip for the whole tile).
template <typename T>
__device__ __forceinline__ void stage_factor_fp64(const T* src, int n, int pad, double* gs, int tid, int nthr) {
    constexpr int VE = 16 / (int)sizeof(T);
    const bool vec = ((reinterpret_cast<uintptr_t>(src) & 15) == 0);
    const int nv = vec ? n / VE : 0;
    using V = typename VecT<T>::V;
    for (int base = 0; base < nv; base += 8 * nthr) {
        V v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int e = base + u * nthr + tid;
            v[u] = e < nv ? reinterpret_cast<const V*>(src)[e] : zero_v<T>();
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int e = base + u * nthr + tid;
            if (e < nv) {
                T t[VE];
                VecT<T>::get(v[u], t);
#pragma unroll
                for (int q = 0; q < VE; ++q) gs[e * VE + q] = (double)t[q];
            }
        }
    }
    for (int base = nv * VE; base < n; base += 8 * nthr) {
        T v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int e = base + u * nthr + tid;
            v[u] = e < n ? src[e] : T(0);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int e = base + u * nthr + tid;
            if (e < n) gs[e] = (double)v[u];
        }
    }
    for (int e = n + tid; e < n + pad; e += nthr) gs[e] = 0.0;
}

// ---- a3 for large ranks on one GPU: Gram/RHS of every column as a register-tiled fp64 product --
// proj[j] = [Σ_a ω(a,j) g_a g_aᵀ (upper triangle, row-major), Σ_a β(a,j) g_a]  (Eq. 8)
// for two columns j per CTA: the 4×4 tile products g_a[r]·g_a[s] are formed once per a and
// shared by both columns (the per-column kernel was bound by the shared-memory reads of g_a:
// 9 loads per 20 fp64 operations; here 5 per 48).  Same task split and fixed-order a-partials
// as block_solve_big; block_solve_big<SOLVE_FROM_PROJ> then adds ρI, factors and solves.
constexpr int kGramCols = 2;
__host__ __device__ inline size_t gram_project_smem(int R, int ta) {
    const int Rp = big_solve_rp(R);
    const size_t gsz = (size_t)ta * R + Rp, psz = (size_t)16 * kGramCols * kBigThreads;  // staged factor | partial tiles
    return sizeof(double) * ((gsz > psz ? gsz : psz) + kGramCols * 2 * (size_t)ta);
}

template <typename T>
__global__ void __launch_bounds__(kBigThreads) gram_project(const SolveParams<T> P) {
    extern __shared__ __align__(16) double bsm[];
    const int R = P.R, Rp = big_solve_rp(R), TA = P.ta;
    const int NG = R * (R + 1) / 2, NA = NG + R;
    double* gs = bsm;                          // G_{i,k}(:, a0 .. a0+ta) as fp64, row stride R
    const size_t gsz = (size_t)TA * R + Rp, psz = (size_t)16 * kGramCols * kBigThreads;
    double* om = gs + (gsz > psz ? gsz : psz); // [a][col] ω, then β
    double* be = om + kGramCols * (size_t)TA;
    const int tid = threadIdx.x, nthr = blockDim.x;
#ifdef IFCTN_EXP_PHASE_CLOCKS
    long long gclk[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#define GCLK(q) if (blockIdx.x == 0 && threadIdx.x == 0) gclk[q] = clock64();
#else
#define GCLK(q)
#endif
    GCLK(0);
    const int64_t j0 = (int64_t)blockIdx.x * kGramCols;
    const int ncol = (int)min((int64_t)kGramCols, P.Ik - j0);
    const int nt = Rp / 4;
    const int ntg = nt * (nt + 1) / 2;
    const int ntasks = ntg + nt;
    const int KS = max(1, min(8, nthr / ntasks));
    const int task_t = tid % ntasks, task_h = tid / ntasks;
    const bool has_task = task_h < KS;
    const bool is_rhs = task_t >= ntg;
    int tr = 0, ts = 0;
    if (has_task) {
        if (is_rhs) {
            tr = task_t - ntg;
        } else {
            int q = task_t;
            while (q >= nt - tr) {
                q -= nt - tr;
                ++tr;
            }
            ts = tr + q;
        }
    }
    double acc[kGramCols][4][4];
#pragma unroll
    for (int c = 0; c < kGramCols; ++c)
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v) acc[c][u][v] = 0.0;
    for (int64_t a0 = 0; a0 < P.Ii; a0 += TA) {
        const int na = (int)min((int64_t)TA, P.Ii - a0);
        __syncthreads();
        stage_factor_fp64<T>(P.Gik + a0 * R, na * R, Rp, gs, tid, nthr);
        GCLK(1);
        for (int q = tid; q < na * kGramCols; q += nthr) {
            const int c = q / na, a = q - c * na;
            const bool okc = c < ncol;
            om[a * kGramCols + c] = okc ? P.omega[(j0 + c) * P.Ii + a0 + a] : 0.0;
            be[a * kGramCols + c] = okc ? P.beta[(j0 + c) * P.Ii + a0 + a] : 0.0;
        }
        __syncthreads();
        GCLK(2);
        if (has_task) {
            if (is_rhs) {
                for (int a = task_h; a < na; a += KS) {
                    const double* gr = gs + a * R + 4 * tr;
#pragma unroll
                    for (int c = 0; c < kGramCols; ++c) {
                        const double b = be[a * kGramCols + c];
#pragma unroll
                        for (int u = 0; u < 4; ++u) acc[c][u][0] = fma(b, gr[u], acc[c][u][0]);
                    }
                }
            } else {
#pragma unroll 2
                for (int a = task_h; a < na; a += KS) {
                    const double* gr = gs + a * R + 4 * tr;
                    const double* gc = gs + a * R + 4 * ts;
                    double q[4][4];
#pragma unroll
                    for (int u = 0; u < 4; ++u)
#pragma unroll
                        for (int v = 0; v < 4; ++v) q[u][v] = gr[u] * gc[v];
#pragma unroll
                    for (int c = 0; c < kGramCols; ++c) {
                        const double w = om[a * kGramCols + c];
#pragma unroll
                        for (int u = 0; u < 4; ++u)
#pragma unroll
                            for (int v = 0; v < 4; ++v) acc[c][u][v] = fma(w, q[u][v], acc[c][u][v]);
                    }
                }
            }
        }
    }
    GCLK(3);
    // partial tiles into shared memory (over the staged factor, no longer needed): element e of
    // thread tid at part[e·nthr + tid] (conflict-free); then entry (c, r, s) = Σ_h in h order
    __syncthreads();
    double* part = gs;
    if (has_task) {
#pragma unroll
        for (int c = 0; c < kGramCols; ++c)
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int v = 0; v < 4; ++v) part[(c * 16 + u * 4 + v) * nthr + tid] = acc[c][u][v];
    }
    __syncthreads();
    GCLK(4);
    for (int q = tid; q < 16 * kGramCols * ntasks; q += nthr) {
        const int e = q / ntasks, t = q - e * ntasks;
        const int c = e >> 4, u = (e >> 2) & 3, v = e & 3;
        if (c >= ncol) continue;
        int idx;
        if (t < ntg) {
            int r4 = 0, qq = t;
            while (qq >= nt - r4) {
                qq -= nt - r4;
                ++r4;
            }
            const int r = 4 * r4 + u, sc = 4 * (r4 + qq) + v;
            if (r > sc || sc >= R) continue;
            idx = r * R - r * (r - 1) / 2 + (sc - r);
        } else {
            const int r = 4 * (t - ntg) + u;
            if (v != 0 || r >= R) continue;
            idx = NG + r;
        }
        double sum = 0.0;
        for (int h = 0; h < KS; ++h) sum += part[e * nthr + h * ntasks + t];
        P.proj[(j0 + c) * NA + idx] = sum;
    }
    GCLK(5);
#ifdef IFCTN_EXP_PHASE_CLOCKS
    if (blockIdx.x == 0 && threadIdx.x == 0)
        printf("gram_project R=%d phases (cycles): stage %lld  om/be %lld  gram %lld  reduce %lld  out %lld\n", R,
               gclk[1] - gclk[0], gclk[2] - gclk[1], gclk[3] - gclk[2], gclk[4] - gclk[3], gclk[5] - gclk[4]);
#endif
}

// ---- a3 for large ranks on the fp64 tensor cores ---------------------------
// D(8×8) += A(8×4, row-major) · B(4×8, column-major), all fp64 (SASS DMMA.8x8x4): lane l holds
// A[l/4][l%4], B[l%4][l/4] and D[l/4][2(l%4)], D[l/4][2(l%4)+1].
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// [Gram_j | rhs_j] = Σ_a g_a · [ω(a,j) g_aᵀ | β(a,j)] (Eq. 8) as one fp64 product with
// M = R rows r, N = R + 1 columns (s < R: the Gram, s = R: the rhs), K = I_i, on m8n8k4 tiles:
// NRT row tiles; the column tiles are the same NRT (the rhs column rides in the last one's
// padding) or, when R = 8·NRT (EXTRA), one more.  Only tiles on or above the diagonal are
// computed.  Warp w takes the k-steps (4 values of a) w, w + 8, … of a staged tile and holds
// every output tile: per k-step NRT fragment loads of g (conflict-free for R ≡ 4 mod 8), two
// scalar loads and NRT multiplies feed NRT(NRT+1)/2 (+NRT) DMMAs.  The 8 warps' partial tiles
// are added into A / rhs in warp order (fixed order, deterministic).  a ≥ na reads row na − 1
// with zero weights; rows/columns ≥ R of the tiles read finite padding and are not stored.
// the later staging tiles of big_gram_mma (long modes only): a call, so that its loads in flight
// do not add to the registers of the loop that holds every output tile
template <typename T>
__device__ __noinline__ void stage_factor_fp64_call(const T* src, int n, int pad, double* gs, int tid, int nthr) {
    stage_factor_fp64<T>(src, n, pad, gs, tid, nthr);
}

template <typename T, int NRT, bool EXTRA>
__device__ __forceinline__ void big_gram_mma(const SolveParams<T>& P, int64_t j, double* gs, double* A,
                                             double* om, double* be, double* rhs, double* scr) {
    constexpr int NCT = NRT + (EXTRA ? 1 : 0);
    constexpr int NTILE = NRT * (NRT + 1) / 2 + (EXTRA ? NRT : 0);
    const int R = P.R, LDA = big_solve_lda(R), TA = P.ta;
    const int tid = threadIdx.x, nthr = blockDim.x, lane = tid & 31, wi = tid >> 5, nw = kBigThreads / 32;
    const int lk = lane & 3, lq = lane >> 2;
    double acc[NTILE][2];
#pragma unroll
    for (int t = 0; t < NTILE; ++t) acc[t][0] = acc[t][1] = 0.0;
    for (int64_t a0 = 0; a0 < P.Ii; a0 += TA) {
        const int na = (int)min((int64_t)TA, P.Ii - a0);
        if (a0 > 0) {
            __syncthreads();
            stage_factor_fp64_call<T>(P.Gik + a0 * R, na * R, big_solve_rp(R), gs, tid, nthr);
        }
        for (int a = tid; a < na; a += nthr) {
            om[a] = P.omega[j * P.Ii + a0 + a];
            be[a] = P.beta[j * P.Ii + a0 + a];
        }
        __syncthreads();
        for (int ks = wi; 4 * ks < na; ks += nw) {
            const int a = 4 * ks + lk;
            const bool in = a < na;
            const double w = in ? om[a] : 0.0, b = in ? be[a] : 0.0;
            const double* gr = gs + min(a, na - 1) * R + lq;
            double fa[NRT], fb[NCT];
#pragma unroll
            for (int t = 0; t < NRT; ++t) fa[t] = gr[8 * t];
#pragma unroll
            for (int t = 0; t < NRT; ++t) {
                const int s = 8 * t + lq;
                fb[t] = (t + 1 < NRT || s < R) ? w * fa[t] : (s == R ? b : 0.0);
            }
            if constexpr (EXTRA) fb[NRT] = lq == 0 ? b : 0.0;
            int t = 0;
#pragma unroll
            for (int tr = 0; tr < NRT; ++tr)
#pragma unroll
                for (int tc = tr; tc < NCT; ++tc, ++t) dmma884(acc[t][0], acc[t][1], fa[tr], fb[tc]);
        }
    }
    // rounds of kBigTPR tiles: every warp writes its partial tiles (16 bytes per lane, contiguous),
    // then one thread per entry sums the 8 partials in warp order and stores the entry
    constexpr int NQ = (NTILE + kBigTPR - 1) / kBigTPR;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        __syncthreads();
#pragma unroll
        for (int tt = 0; tt < kBigTPR; ++tt)
            if (q * kBigTPR + tt < NTILE)
                *reinterpret_cast<double2*>(scr + (wi * kBigTPR + tt) * 64 + 2 * lane) =
                    make_double2(acc[q * kBigTPR + tt][0], acc[q * kBigTPR + tt][1]);
        __syncthreads();
        const int tt = tid >> 6, idx = tid & 63, t = q * kBigTPR + tt;
        if (t < NTILE) {
            double v[kBigThreads / 32];
#pragma unroll
            for (int w8 = 0; w8 < kBigThreads / 32; ++w8) v[w8] = scr[(w8 * kBigTPR + tt) * 64 + idx];
            double sum = v[0];
#pragma unroll
            for (int w8 = 1; w8 < kBigThreads / 32; ++w8) sum += v[w8];
            int tr = 0, rem = t;  // tile t = (tr, tr + rem) in the order the k-loop enumerates them
            while (rem >= NCT - tr) {
                rem -= NCT - tr;
                ++tr;
            }
            const int r = 8 * tr + (idx >> 3), sc = 8 * (tr + rem) + (idx & 7);
            if (r < R && sc <= R && r <= sc) *(sc < R ? A + r * LDA + sc : rhs + r) = sum;
        }
    }
    __syncthreads();
}

#ifdef IFCTN_EXP_PHASE_CLOCKS  // diagnosis builds only: per-phase clocks of CTA 0
#define PHASE_CLK(q) \
    if (j == 0 && threadIdx.x == 0) clk[q] = clock64();
#else
#define PHASE_CLK(q)
#endif
template <typename T, int SM>
__device__ __forceinline__ void block_solve_big_body(const SolveParams<T>& P, int64_t j, double* bsm, int* okp) {
#ifdef IFCTN_EXP_PHASE_CLOCKS
    long long clk[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#endif
    PHASE_CLK(0);
    const int R = P.R, Rp = big_solve_rp(R), LDA = big_solve_lda(R), TA = P.ta;
    const int NG = R * (R + 1) / 2, NA = NG + R;
    double* gs = bsm;                      // G_{i,k}(:, a0 .. a0+ta) as fp64, row stride R
    double* A = gs + (size_t)TA * R + Rp;  // Gram (row-major, lda)
    double* om = A + (size_t)(Rp + 1) * LDA;  // ω(a, j); row Rp of A carries rhsᵀ through the factorisation
    double* be = om + TA;                  // β(a, j)
    double* rhs = be + TA;
    double* cv = rhs + Rp;
    double* cold = cv + Rp;
    double* scr = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(cold + Rp) + 15) & ~uintptr_t(15));  // big_gram_mma
    const int tid = threadIdx.x, nthr = blockDim.x, lane = tid & 31;
    const int nt = Rp / 4;
    const int ntg = nt * (nt + 1) / 2;     // Gram tiles; then nt rhs tiles
    const int ntasks = ntg + nt;
    const int KS = max(1, min(8, nthr / ntasks));   // a-split per tile
    const int task_t = tid % ntasks, task_h = tid / ntasks;
    const bool has_task = task_h < KS;
    const bool is_rhs = task_t >= ntg;
    const bool one_tile = (int64_t)TA >= P.Ii;
    int tr = 0, ts = 0;
    if (has_task) {
        if (is_rhs) {
            tr = task_t - ntg;
        } else {
            int q = task_t;
            while (q >= nt - tr) {
                q -= nt - tr;
                ++tr;
            }
            ts = tr + q;
        }
    }
    auto stage = [&](int64_t a0, int na) { stage_factor_fp64<T>(P.Gik + a0 * R, na * R, Rp, gs, tid, nthr); };
    // G_{i,k} was written by the solve of block (i,k): at least two kernels back, complete
    // before this grid could start — its first tile is staged ahead of the wait, while the
    // predecessor (the a2 pass of this block) still runs
    if constexpr (SM != SOLVE_FROM_PROJ) stage(0, (int)min((int64_t)TA, P.Ii));
    const T cold_pre = tid < R ? P.Gki[j * R + tid] : T(0);  // this block's previous solve: same argument
    pdl_wait();
    pdl_launch();
    unsigned long long pe = 0;  // peer exchange (peer.cuh): FROM_PROJ is the consumer
    if constexpr (SM == SOLVE_FROM_PROJ)
        if (P.use_peer) {
            pe = peer_next_epoch(P.peer);
            peer_publish_wait(P.peer, pe);
        }
    if constexpr (SM != SOLVE_FROM_PROJ) {
      // ≤ 15 output tiles per warp: R ≤ 39 (P.mma, set at plan time); else the SIMT tiles below
      bool by_mma = (P.mma & 1) != 0;
      if (by_mma) {
        PHASE_CLK(6);
        PHASE_CLK(7);
        switch ((R + 7) >> 3) {
            case 2: if (R & 7) big_gram_mma<T, 2, false>(P, j, gs, A, om, be, rhs, scr); else big_gram_mma<T, 2, true>(P, j, gs, A, om, be, rhs, scr); break;
            case 3: if (R & 7) big_gram_mma<T, 3, false>(P, j, gs, A, om, be, rhs, scr); else big_gram_mma<T, 3, true>(P, j, gs, A, om, be, rhs, scr); break;
            case 4: if (R & 7) big_gram_mma<T, 4, false>(P, j, gs, A, om, be, rhs, scr); else big_gram_mma<T, 4, true>(P, j, gs, A, om, be, rhs, scr); break;
            case 5: if (R & 7) big_gram_mma<T, 5, false>(P, j, gs, A, om, be, rhs, scr); else by_mma = false; break;
            default: by_mma = false;
        }
        PHASE_CLK(1);
      }
      if (!by_mma) {
        double acc[4][4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v) acc[u][v] = 0.0;
        for (int64_t a0 = 0; a0 < P.Ii; a0 += TA) {
            const int na = (int)min((int64_t)TA, P.Ii - a0);
            if (a0 > 0) {
                __syncthreads();
                stage(a0, na);
            }
            PHASE_CLK(6);
            for (int a = tid; a < na; a += nthr) {
                om[a] = P.omega[j * P.Ii + a0 + a];
                be[a] = P.beta[j * P.Ii + a0 + a];
            }
            __syncthreads();
            PHASE_CLK(7);
            if (has_task) {
                if (is_rhs) {
                    for (int a = task_h; a < na; a += KS) {
                        const double b = be[a];
                        const double* gr = gs + a * R + 4 * tr;
#pragma unroll
                        for (int u = 0; u < 4; ++u) acc[u][0] = fma(b, gr[u], acc[u][0]);
                    }
                } else {
                    for (int a = task_h; a < na; a += KS) {
                        const double w = om[a];
                        const double* gr = gs + a * R + 4 * tr;
                        const double* gc = gs + a * R + 4 * ts;
                        const double r0 = w * gr[0], r1 = w * gr[1], r2 = w * gr[2], r3 = w * gr[3];
                        const double c0 = gc[0], c1 = gc[1], c2 = gc[2], c3 = gc[3];
                        acc[0][0] = fma(r0, c0, acc[0][0]); acc[0][1] = fma(r0, c1, acc[0][1]);
                        acc[0][2] = fma(r0, c2, acc[0][2]); acc[0][3] = fma(r0, c3, acc[0][3]);
                        acc[1][0] = fma(r1, c0, acc[1][0]); acc[1][1] = fma(r1, c1, acc[1][1]);
                        acc[1][2] = fma(r1, c2, acc[1][2]); acc[1][3] = fma(r1, c3, acc[1][3]);
                        acc[2][0] = fma(r2, c0, acc[2][0]); acc[2][1] = fma(r2, c1, acc[2][1]);
                        acc[2][2] = fma(r2, c2, acc[2][2]); acc[2][3] = fma(r2, c3, acc[2][3]);
                        acc[3][0] = fma(r3, c0, acc[3][0]); acc[3][1] = fma(r3, c1, acc[3][1]);
                        acc[3][2] = fma(r3, c2, acc[3][2]); acc[3][3] = fma(r3, c3, acc[3][3]);
                    }
                }
            }
        }
        PHASE_CLK(1);
        // Gram, rhs = Σ_h partial tiles, h ascending (h = 0 assigns: no zero fill)
        for (int h = 0; h < KS; ++h) {
            __syncthreads();
            if (has_task && task_h == h) {
                if (is_rhs) {
#pragma unroll
                    for (int u = 0; u < 4; ++u) rhs[4 * tr + u] = (h ? rhs[4 * tr + u] : 0.0) + acc[u][0];
                } else {
#pragma unroll
                    for (int u = 0; u < 4; ++u)
#pragma unroll
                        for (int v = 0; v < 4; ++v) {
                            double* e = A + (4 * tr + u) * LDA + 4 * ts + v;
                            *e = (h ? *e : 0.0) + acc[u][v];
                        }
                }
            }
        }
        __syncthreads();
      }
        if constexpr (SM == SOLVE_PROJECT) {
            // this rank's partial [upper triangle (r ≤ s, row-major), rhs] for the all-reduce
            double* pdst = P.use_peer ? peer_my_slot(P.peer) : P.proj;
            for (int t = tid; t < NA; t += nthr) {
                double v;
                if (t < NG) {
                    int r = 0, q = t;
                    while (q >= R - r) {
                        q -= R - r;
                        ++r;
                    }
                    v = A[r * LDA + r + q];
                } else {
                    v = rhs[t - NG];
                }
                pdst[j * NA + t] = v;
            }
            return;
        }
        // lower triangle from the upper one (the Cholesky reads rows): thread rows
        for (int r = tid >> 3; r < R; r += nthr >> 3)
            for (int c = tid & 7; c < r; c += 8) A[r * LDA + c] = A[c * LDA + r];
    } else {
        if (one_tile) stage(0, (int)P.Ii);  // for the H refresh
        for (int t = tid; t < NA; t += nthr) {
            const double v = P.use_peer ? peer_sum(P.peer, pe, j * NA + t) : P.proj[j * NA + t];
            if (t < NG) {
                int r = 0, q = t;
                while (q >= R - r) {
                    q -= R - r;
                    ++r;
                }
                A[(r + q) * LDA + r] = v;  // lower triangle
            } else {
                rhs[t - NG] = v;
            }
        }
    }
    __syncthreads();
    PHASE_CLK(2);
    // + ρI, + ρ c_old
    if (tid < R) {
        const double co = (double)cold_pre;
        cold[tid] = co;
        A[tid * LDA + tid] += P.rho;
        rhs[tid] += P.rho * co;
    }
    __syncthreads();
    // Cholesky, right-looking in 4×4 blocks over all threads (lower triangle, in place; the
    // diagonal keeps 1/L(c,c)).  Rows/columns R..Rp-1 are padded with the identity.  Per block
    // b: thread 0 factors the 4×4 diagonal block in registers; one thread per row solves the
    // panel below it; all threads apply the rank-4 trailing update — 3 barriers per block.
    for (int r = R + tid; r < Rp; r += nthr)
        for (int c = 0; c <= r; ++c) A[r * LDA + c] = (c == r) ? 1.0 : 0.0;
    if (tid == 0) *okp = 1;
    __syncthreads();
    // Row Rp of the factored matrix is rhsᵀ: its panel solves and trailing updates ARE the forward
    // substitution L y = rhs (y ends up in A[Rp][·]), so only Lᵀ c = y remains for the one warp.
    for (int c = tid; c < Rp; c += nthr) A[Rp * LDA + c] = c < R ? rhs[c] : 0.0;
    __syncthreads();
    for (int c0 = 0; c0 < Rp; c0 += 4) {
        if (tid == 0) {
            double L[4][4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int v = 0; v < 4; ++v) L[u][v] = v <= u ? A[(c0 + u) * LDA + c0 + v] : 0.0;
            bool ok = true;
#pragma unroll
            for (int cc = 0; cc < 4; ++cc) {
                double d = L[cc][cc];
#pragma unroll
                for (int k = 0; k < cc; ++k) d = fma(-L[cc][k], L[cc][k], d);
                ok = ok && d > 0.0;
                const double inv = rsqrt(d > 0.0 ? d : 1.0);
                L[cc][cc] = inv;
#pragma unroll
                for (int r = cc + 1; r < 4; ++r) {
                    double v = L[r][cc];
#pragma unroll
                    for (int k = 0; k < cc; ++k) v = fma(-L[r][k], L[cc][k], v);
                    L[r][cc] = v * inv;
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int v = 0; v <= u; ++v) A[(c0 + u) * LDA + c0 + v] = L[u][v];
            if (!ok) *okp = 0;
        }
        __syncthreads();
        const int m = Rp - c0 - 4 + 1;  // trailing rows, the rhs row included
        if (tid < m) {                  // panel row r: x = a · L11⁻ᵀ
            const int r = c0 + 4 + tid;
            double x[4];
#pragma unroll
            for (int cc = 0; cc < 4; ++cc) {
                double v = A[r * LDA + c0 + cc];
#pragma unroll
                for (int k = 0; k < cc; ++k) v = fma(-x[k], A[(c0 + cc) * LDA + c0 + k], v);
                x[cc] = v * A[(c0 + cc) * LDA + c0 + cc];
            }
#pragma unroll
            for (int cc = 0; cc < 4; ++cc) A[r * LDA + c0 + cc] = x[cc];
        }
        __syncthreads();
        // trailing lower triangle (r, c), c0+4 ≤ c ≤ r: thread rows, 8 lanes over c
        for (int rr = tid >> 3; rr < m; rr += nthr >> 3) {
            const int r = c0 + 4 + rr;
            const double l0 = A[r * LDA + c0], l1 = A[r * LDA + c0 + 1], l2 = A[r * LDA + c0 + 2],
                         l3 = A[r * LDA + c0 + 3];
            for (int c = c0 + 4 + (tid & 7); c <= min(r, Rp - 1); c += 8) {
                const double* lc = A + c * LDA + c0;
                double v = A[r * LDA + c];
                v = fma(-l0, lc[0], v);
                v = fma(-l1, lc[1], v);
                v = fma(-l2, lc[2], v);
                v = fma(-l3, lc[3], v);
                A[r * LDA + c] = v;
            }
        }
        __syncthreads();
    }
    if (tid < 32) {
        const bool ok = *okp != 0;
        PHASE_CLK(3);
        // Lᵀ c = y with y (row Rp of the factored matrix) in registers (lane owns rows lane,
        // lane + 32) and the pivot value broadcast by shuffle; the L entries are independent loads
        double x0 = lane < R ? A[Rp * LDA + lane] : 0.0, x1 = lane + 32 < R ? A[Rp * LDA + lane + 32] : 0.0;  // y
        for (int r = R - 1; r >= 0; --r) {
            const double lr0 = lane < r ? A[r * LDA + lane] : 0.0;
            const double lr1 = lane + 32 < r ? A[r * LDA + lane + 32] : 0.0;
            const double own = (r < 32 ? x0 : x1) * A[r * LDA + r];
            const double c = __shfl_sync(0xffffffffu, own, r & 31);
            if (lane == (r & 31)) {
                if (r < 32) x0 = c;
                else x1 = c;
            }
            x0 = fma(-lr0, c, x0);
            x1 = fma(-lr1, c, x1);
        }
        if (lane < R) cv[lane] = x0;
        if (lane + 32 < R) cv[lane + 32] = x1;
        __syncwarp();
        if (!ok) {
            if (lane == 0) atomicOr(P.flags, 1);
            for (int r = lane; r < R; r += 32) cv[r] = cold[r];
        }
        __syncwarp();
        double d2 = 0.0;
        for (int r = lane; r < R; r += 32) {
            const T cT = (T)cv[r];
            P.Gki[j * R + r] = cT;
            const double dd = (double)cT - cold[r];
            d2 += dd * dd;
            cv[r] = (double)cT;
        }
        d2 = warp_sum(d2);
        if (lane == 0) P.delta[j] = d2;
        PHASE_CLK(4);
    }
    // H refresh: H_{k,i}(j, a) = Σ_r c_r G_{i,k}(r, a), 8 threads per a
    const int row8 = tid >> 3, sub8 = tid & 7;
    for (int64_t a0 = 0; a0 < P.Ii; a0 += TA) {
        const int na = (int)min((int64_t)TA, P.Ii - a0);
        __syncthreads();
        if (!one_tile) {
            stage(a0, na);
            __syncthreads();
        }
        if (P.mma & 2) {
            // on the fp64 tensor cores: rows a in tiles of 8 (M), r in steps of 4 (K), c in column
            // 0 of B; a warp keeps 4 row tiles in flight; lanes with l%4 = 0 hold column 0 of D
            const int wi = tid >> 5, lk = lane & 3, lq = lane >> 2;
            for (int rt = wi; rt * 8 < na; rt += 4 * (kBigThreads / 32)) {
                double d0[4] = {0.0, 0.0, 0.0, 0.0}, d1[4] = {0.0, 0.0, 0.0, 0.0};
                for (int r0 = 0; r0 < R; r0 += 4) {
                    const double b = (lq == 0 && r0 + lk < R) ? cv[r0 + lk] : 0.0;
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int a = (rt + u * (kBigThreads / 32)) * 8 + lq;
                        // rows ≥ na / entries r ≥ R: in-bounds shared memory times b = 0, or unused rows
                        const double g = gs[min(a, na - 1) * R + r0 + lk];
                        dmma884(d0[u], d1[u], g, b);
                    }
                }
                if (lk == 0) {
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int a = (rt + u * (kBigThreads / 32)) * 8 + lq;
                        if (a < na) {
                            const int64_t ag = a0 + a;
                            const int64_t o = P.k_lt_i ? (P.h_off + ag * P.h_ld + j) : (P.h_off + j * P.h_ld + ag);
                            P.H[o] = (T)d0[u];
                        }
                    }
                }
            }
        } else
        for (int a = row8; a < na; a += nthr >> 3) {
            double h = 0.0;
            for (int r = sub8; r < R; r += 8) h = fma(cv[r], gs[a * R + r], h);
            h += __shfl_xor_sync(0xffffffffu, h, 1);
            h += __shfl_xor_sync(0xffffffffu, h, 2);
            h += __shfl_xor_sync(0xffffffffu, h, 4);
            if (sub8 == 0) {
                const int64_t ag = a0 + a;
                const int64_t o = P.k_lt_i ? (P.h_off + ag * P.h_ld + j) : (P.h_off + j * P.h_ld + ag);
                P.H[o] = (T)h;
            }
        }
    }
    PHASE_CLK(5);
    if constexpr (SM == SOLVE_FROM_PROJ)
        if (P.use_peer) peer_retire(P.peer, pe);
#ifdef IFCTN_EXP_PHASE_CLOCKS
    if (j == 0 && threadIdx.x == 0)
        printf("big solve R=%d phases (cycles): stage %lld  om/be+sync %lld  gram %lld  reduce+sym %lld  chol %lld  subst %lld  H %lld\n", P.R,
               clk[6] - clk[0], clk[7] - clk[6], clk[1] - clk[7], clk[2] - clk[1], clk[3] - clk[2], clk[4] - clk[3], clk[5] - clk[4]);
#endif
}

template <typename T, int SM>
__global__ void __launch_bounds__(kBigThreads, IFCTN_BIG_MINB) block_solve_big(const SolveParams<T> P) {
    extern __shared__ __align__(16) double bsm[];
    __shared__ int ok;
    block_solve_big_body<T, SM>(P, blockIdx.x, bsm, &ok);  // waits for its predecessor itself
}

// ---- a1: build H_{p,q} = G_{p,q}ᵀ G_{q,p} for one pair (K=R skinny product; FMA pipes) ---
template <typename T>
__global__ void pair_gram(const T* Gpq, const T* Gqp, int R, int64_t Ip, int64_t Iq, T* H,
                          int64_t ld) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= Ip * Iq) return;
    const int64_t a = e % Ip, b = e / Ip;
    double s = 0.0;
    for (int r = 0; r < R; ++r) s += (double)Gpq[a * R + r] * (double)Gqp[b * R + r];
    H[b * ld + a] = (T)s;
}

// ---- per-sweep finaliser: fixed-order fp64 sums of the refill norms and ΔG² -------------
// part5 = [‖ΔX‖², ‖X‖², ‖X_new − t‖², ΣΔG² of this rank's sharded columns, ΣΔG² of the
// replicated blocks].  Multi-GPU: the first four are summed across ranks before combining.
__device__ __forceinline__ void combine_into(const double* p5, double* scal, int* flags, int obj_only) {
    if (obj_only) {
        scal[6] = 0.5 * p5[2];
        if (!isfinite(scal[6])) atomicOr(flags + 1, 1);
        return;
    }
    const double dx2 = p5[0], x2 = p5[1], f = 0.5 * p5[2], dg2 = p5[3] + p5[4];
    const double xn = sqrt(x2);
    scal[0] = dx2;
    scal[1] = x2;
    scal[2] = f;
    scal[3] = dg2;
    scal[4] = sqrt(dx2) / (xn > 0.0 ? xn : 1.0);
    scal[5] += 1.0;
    if (!isfinite(dx2) || !isfinite(x2) || !isfinite(f) || !isfinite(dg2)) atomicOr(flags + 1, 1);
}

// One CTA of 1024 threads: strided per-thread sums, then a shuffle tree per warp and one over
// the 32 warp sums (fixed order: deterministic).  s: 5·32 doubles of shared scratch.
__device__ __forceinline__ void finalize_norms_body(const double* norms, int64_t ngroups, const double* delta,
                                                    int64_t ndelta, int64_t sh_off, int64_t sh_len, double* p5,
                                                    double* scal, int* flags, int obj_only, int combine,
                                                    double* s) {
    const int vt = threadIdx.x, nt = blockDim.x;
    double a[5] = {0, 0, 0, 0, 0};
    for (int64_t g = vt; g < ngroups; g += nt) {  // L2 loads: written by other CTAs just now
        a[0] += __ldcg(norms + 3 * g + 0);
        a[1] += __ldcg(norms + 3 * g + 1);
        a[2] += __ldcg(norms + 3 * g + 2);
    }
    if (!obj_only)
        for (int64_t d = vt; d < ndelta; d += nt) {
            if (d >= sh_off && d < sh_off + sh_len) a[3] += delta[d];
            else a[4] += delta[d];
        }
    const int w = vt >> 5, ln = vt & 31;
#pragma unroll
    for (int q = 0; q < 5; ++q) {
        const double v = warp_sum(a[q]);
        if (ln == 0) s[q * 32 + w] = v;
    }
    __syncthreads();
    if (w == 0) {
        const int nw = nt >> 5;
#pragma unroll
        for (int q = 0; q < 5; ++q) {
            const double v = warp_sum(ln < nw ? s[q * 32 + ln] : 0.0);
            if (ln == 0) p5[q] = v;
        }
        if (ln == 0 && combine) combine_into(p5, scal, flags, obj_only);
    }
}

static __global__ void __launch_bounds__(1024) finalize_norms(const double* norms, int64_t ngroups,
                                                       const double* delta, int64_t ndelta,
                                                       int64_t sh_off, int64_t sh_len, double* p5,
                                                       double* scal, int* flags, int obj_only,
                                                       int combine) {
    __shared__ double s[5 * 32];
    pdl_wait();
    pdl_launch();
    finalize_norms_body(norms, ngroups, delta, ndelta, sh_off, sh_len, p5, scal, flags, obj_only, combine, s);
}

// traced fused sweeps: append this sweep's row {sweep, rel_change, objective, dx2, dg2} of
// scal to the device trace (read back once after the last sweep)
static __global__ void trace_push(const double* scal, double* rows, int* count) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const int c = *count;
    double* r = rows + 5 * (int64_t)c;
    r[0] = scal[5];
    r[1] = scal[4];
    r[2] = scal[2];
    r[3] = scal[0];
    r[4] = scal[3];
    *count = c + 1;
}

static __global__ void combine_norms(const double* p5, double* scal, int* flags, int obj_only) {
    if (threadIdx.x == 0 && blockIdx.x == 0) combine_into(p5, scal, flags, obj_only);
}

// ---- layout kernels ------------------------------------------------------------------------
// X⁽⁰⁾ = P_Ω(O) (zeros on Ω^c; reading R7) packed into the padded fibre layout + mask bits.
template <typename T>
__global__ void pack_input(const T* obs, const uint8_t* mask, int64_t I1, int64_t I1p,
                           int64_t npad, int xfull, T* X, uint32_t* bits) {
    // one warp per 32-element mask word: lane t loads element 32w + t (coalesced, so pinned
    // host inputs stream well over the host link) and the ballot is the word
    const int lane = threadIdx.x & 31;
    const int64_t nw = (npad + 31) / 32;
    const int64_t wstride = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); w < nw; w += wstride) {
        const int64_t e = w * 32 + lane;
        T x = T(0);
        bool m = true;
        if (e < npad) {
            const int64_t f = e / I1p, i1 = e - f * I1p;
            if (i1 < I1) {
                const int64_t u = f * I1 + i1;
                m = mask[u] != 0;
                x = (m || xfull) ? obs[u] : T(0);
            }
            X[e] = x;
        }
        const uint32_t b = __ballot_sync(0xffffffffu, m);
        if (lane == 0) bits[w] = b;
    }
}

// Mode permutation between the API linearisation and the internal mode order (Shape::perm):
// a batched 32×32 shared-memory transpose of the source's fastest mode (x) and the source
// mode that is fastest in the destination (y); every other mode is a batch index (decoded per
// tile).  Dense tensors on both sides; src mode q has extent dim[q], stride sstr[q] in the
// source and dstr[q] in the destination.  Coalesced reads along x and writes along y.
constexpr int kPermTile = 32;
struct PermDesc {
    int N, ym;
    int64_t dim[MAXN], sstr[MAXN], dstr[MAXN];
};
template <typename E>
__global__ void __launch_bounds__(kPermTile * 8) permute_modes(const E* __restrict__ src, E* __restrict__ dst,
                                                               const PermDesc d) {
    __shared__ E tile[kPermTile][kPermTile + 1];
    const int64_t X = d.dim[0], Y = d.dim[d.ym];
    const int64_t tx_n = (X + kPermTile - 1) / kPermTile;
    const int64_t x0 = (int64_t)(blockIdx.x % tx_n) * kPermTile, y0 = (int64_t)(blockIdx.x / tx_n) * kPermTile;
    int64_t nb = 1;
    for (int q = 1; q < d.N; ++q)
        if (q != d.ym) nb *= d.dim[q];
    const int tx = threadIdx.x % kPermTile, ty = threadIdx.x / kPermTile;
    for (int64_t bt = blockIdx.y; bt < nb; bt += gridDim.y) {
        int64_t r = bt, so = 0, dof = 0;
        for (int q = 1; q < d.N; ++q) {
            if (q == d.ym) continue;
            const int64_t c = r % d.dim[q];
            r /= d.dim[q];
            so += c * d.sstr[q];
            dof += c * d.dstr[q];
        }
        __syncthreads();
        for (int y = ty; y < kPermTile; y += 8) {
            const int64_t xx = x0 + tx, yy = y0 + y;
            if (xx < X && yy < Y) tile[y][tx] = src[so + xx + yy * d.sstr[d.ym]];
        }
        __syncthreads();
        for (int y = ty; y < kPermTile; y += 8) {
            const int64_t yy = y0 + tx, xx = x0 + y;
            if (xx < X && yy < Y) dst[dof + yy + xx * d.dstr[0]] = tile[tx][y];
        }
    }
}

template <typename T>
__global__ void unpack_x(const T* X, int64_t I1, int64_t I1p, int64_t n, T* out) {
    const int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= n) return;
    const int64_t f = u / I1, i1 = u - f * I1;
    out[u] = X[f * I1p + i1];
}

// RSE partial sums: ‖T − X‖² and ‖T‖² per CTA (fp64), fixed order.
template <typename T>
__global__ void __launch_bounds__(256) rse_partial(const T* truth, const T* X, int64_t I1,
                                                   int64_t I1p, int64_t n, double* part) {
    __shared__ double s0[256], s1[256];
    double a = 0.0, b = 0.0;
    // warps stride over mode-1 fibres, lanes over i_1 (coalesced, no index division)
    const int64_t nfib = n / I1;
    const int lane = threadIdx.x & 31;
    const int64_t wstride = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t f = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); f < nfib; f += wstride) {
        const T* tf = truth + f * I1;
        const T* xf = X + f * I1p;
        for (int64_t i1 = lane; i1 < I1; i1 += 32) {
            const double t = (double)tf[i1];
            const double d = t - (double)xf[i1];
            a += d * d;
            b += t * t;
        }
    }
    s0[threadIdx.x] = a;
    s1[threadIdx.x] = b;
    __syncthreads();
    for (int st = 128; st > 0; st >>= 1) {
        if ((int)threadIdx.x < st) {
            s0[threadIdx.x] += s0[threadIdx.x + st];
            s1[threadIdx.x] += s1[threadIdx.x + st];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        part[2 * blockIdx.x] = s0[0];
        part[2 * blockIdx.x + 1] = s1[0];
    }
}

// out[0..1] = Σ_i part[2i], Σ_i part[2i+1] in a fixed tree (one CTA of 256 threads): a thread sums
// its run of consecutive pairs in order, lanes by xor butterfly, the 8 warp sums in warp order
static __global__ void __launch_bounds__(256) sum_pairs(const double* part, int n, double* out) {
    __shared__ double sm[8][2];
    const int tid = threadIdx.x, per = (n + 255) / 256;
    double v[2][8];
    double a = 0.0, b = 0.0;
    for (int i0 = tid * per; i0 < min(n, (tid + 1) * per); i0 += 8) {
        const int m = min(8, min(n, (tid + 1) * per) - i0);
#pragma unroll
        for (int u = 0; u < 8; ++u) {  // loads in flight together, added in order
            v[0][u] = u < m ? part[2 * (i0 + u)] : 0.0;
            v[1][u] = u < m ? part[2 * (i0 + u) + 1] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            a += v[0][u];
            b += v[1][u];
        }
    }
    a = warp_sum(a);
    b = warp_sum(b);
    if ((tid & 31) == 0) {
        sm[tid >> 5][0] = a;
        sm[tid >> 5][1] = b;
    }
    __syncthreads();
    if (tid == 0) {
        a = b = 0.0;
        for (int w = 0; w < 8; ++w) {
            a += sm[w][0];
            b += sm[w][1];
        }
        out[0] = a;
        out[1] = b;
    }
}

}  // namespace ifctn
