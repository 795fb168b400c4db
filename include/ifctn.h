/*
 * ifctn.h — C-ABI of the B200 (sm_100a) iFCTN tensor-completion PAM sweep.
 *
 * Paper: "iFCTN" (arxiv 2511.16358), /root/reference/PAPER.md ("P:Lx-y" = line range).
 * The library implements Algorithm 1: given the observed tensor O, the sample
 * set Ω, the iFCTN-rank matrix R, ρ, t_max and ε, it runs PAM sweeps, each of which
 *   (a2) contracts the other factors' KR chains into the unfolding-free coefficients of
 *        block (k,i) (Prop. 1; Eq. 8),
 *   (a3/a4) forms the Gram matrix + RHS of the proximal LS subproblem (+ρI) and solves the
 *        small SPD systems column by column (Eq. 8),
 *   (a5) rebuilds the low-rank model and refills Ω^c (Eq. 9, read as the exact
 *        per-entry prox minimiser (t + ρx)/(1+ρ); reading R1).
 *
 * Conventions
 *   - Modes are 0-based in this API (paper mode k = API k+1).
 *   - Dense tensors (observed O, mask, truth, outputs) are mode-1-fastest (column-major):
 *     linear index = i_0 + I_0*(i_1 + I_1*(i_2 + …)).  Under sharding (dist != NULL,
 *     world > 1) every tensor argument is this rank's shard: the contiguous slice of the
 *     shard mode given by ifctn_shard_range(), in the same linearisation.
 *   - Factors: the N(N-1) matrices G_{k,i} ∈ R^{R_{k,i} × I_k}, concatenated
 *     in order k ascending, i ascending (i≠k); each column-major (r fastest).  Under
 *     sharding the chains G_{s,·} of the shard mode s hold only the local columns.
 *   - Element type: ifctn_dtype for O, truth, factors and outputs; the mask is uint8
 *     (nonzero = observed); coefficient outputs (β, ω) are float64.
 *   - Memory: every data pointer may be HOST or DEVICE memory; the library inspects it with
 *     cudaPointerGetAttributes and copies as needed (pinned host memory gives async copies).
 *     The caller owns every buffer it passes; the library never frees caller memory.
 *   - Ordering: all device work is enqueued on the stream given to ifctn_create.
 *
 * Errors: every function returns an ifctn_status; nothing throws across the ABI.  Arguments
 * are validated before any device work.  ifctn_last_error(ctx) gives a message for the
 * most recent failure on that context (a static string for a NULL ctx).
 */
#ifndef IFCTN_H
#define IFCTN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ifctn_ctx ifctn_ctx;

typedef enum {
    IFCTN_OK = 0,
    IFCTN_E_ARG = 1,         /* NULL pointer, ρ ≤ 0, bad enum, bad block index            */
    IFCTN_E_SHAPE = 2,       /* order < 2 or > IFCTN_MAX_ORDER, a dim < 1, size overflow   */
    IFCTN_E_RANKS = 3,       /* R not symmetric, diagonal ≠ 0, off-diagonal < 1 or > max   */
    IFCTN_E_WORKSPACE = 4,   /* caller workspace too small or misaligned                  */
    IFCTN_E_CUDA = 5,        /* CUDA runtime error (message in ifctn_last_error)           */
    IFCTN_E_NCCL = 6,        /* NCCL error (multi-GPU)                                     */
    IFCTN_E_NOT_SPD = 7,     /* non-positive Cholesky pivot (impossible in exact arith.)   */
    IFCTN_E_NONFINITE = 8,   /* NaN/Inf met in the sweep norms                             */
    IFCTN_E_STATE = 9,       /* call not valid in the context's state                      */
    IFCTN_E_UNSUPPORTED = 10,/* valid input this build does not handle (see message)       */
    IFCTN_E_NO_OBSERVED = 11 /* Ω is empty (Algorithm 1 needs at least one observation)   */
} ifctn_status;

typedef enum { IFCTN_F32 = 0, IFCTN_F64 = 1 } ifctn_dtype;

#define IFCTN_MAX_ORDER 6
#define IFCTN_MAX_RANK 64

/* ifctn_create flags */
#define IFCTN_FLAG_NONE 0u
#define IFCTN_FLAG_NO_GRAPH 1u /* run sweeps as plain launches instead of a CUDA graph     */
#define IFCTN_FLAG_X_FULL 2u   /* `observed` is a full X (values off Ω kept), for resume  */
#define IFCTN_FLAG_NO_VBLOCK 8u /* diagnostic: plain fibre walk for every block (no v-blocking) */
#define IFCTN_FLAG_NO_SOLVE_REDUCE 64u /* diagnostic: separate a2 reduce kernel even when the
                                        * small-rank solve can absorb it                     */
#define IFCTN_FLAG_NO_L2PASS 128u /* diagnostic: the HBM-streaming fibre walk for step a2 even
                                     when X is L2-resident (default there: one CTA per kept
                                     value, no partial slots; csrc/l2pass.cuh)               */
#define IFCTN_FLAG_NO_FUSE 16u  /* diagnostic: never fuse a sweep's X update into the next
                                   sweep's first block (see ifctn_sweep)                      */
#define IFCTN_FLAG_NO_PDL 512u /* diagnostic: plain stream order for every launch (default: the
                                  L2-pass, solve and finaliser kernels are launched with
                                  programmatic stream serialization and wait for their
                                  predecessor themselves, griddepcontrol.wait)              */
#define IFCTN_FLAG_NO_DMMA 1024u /* diagnostic: large ranks (R > 9) build Gram_j and rhs_j (R <= 39)
                                    and refresh the H row with SIMT fp64 code (default: the fp64
                                    tensor cores, mma m8n8k4 = SASS DMMA; same fp64 accuracy,
                                    another summation order)                                */
#define IFCTN_FLAG_GRAM_GEMM 256u /* experiment: large ranks (R > 9) build Gram_j and rhs_j of
                                     two columns per CTA in a separate register-tiled kernel
                                     (gram_project), then the FROM_PROJ solve; measured slower
                                     than the per-column solve on one GPU (C2r: 46.6 vs 42.0 us
                                     per block), so off by default                          */

/* Multi-GPU description (one process per GPU).  NULL or world == 1: single GPU.
 * Sharding: X and Ω are split along the shard mode s; the factor chains
 * G_{s,·} hold this rank's columns; every other factor is replicated.  Per block (k,i) with
 * k ≠ s each rank projects its partial (β, ω) onto the Gram/RHS of Eq. 8 (I_k·(R(R+1)/2+R)
 * doubles) and the partials are summed across ranks; blocks with k = s need no exchange.  */
typedef struct {
    const void* nccl_unique_id; /* ncclUniqueId (128 bytes), identical on all ranks       */
    int rank;
    int world;
    int shard_mode;             /* 0-based; -1 = the largest mode, the first on ties
                                   (SURVEY §8(e)).  When the shard mode is mode 0 (the
                                   fibre/lane mode of the passes) and order ≥ 3, the library
                                   stores the shard internally with mode 0 swapped for the
                                   largest of modes 1..N-2, so fibres stay long; every
                                   argument keeps the layout documented here.              */
    /* Optional: sum across ranks on the host instead of NCCL (several ranks driven from host
     * threads on one device in tests, or a custom transport).  Called synchronously with a
     * host buffer of `count` doubles that must be replaced by the element-wise sum over all
     * ranks.  NULL = NCCL (nccl_unique_id required).  Disables CUDA-graph capture.          */
    void (*host_allreduce)(double* buf, size_t count, void* user);
    void* user;
    /* exchange = IFCTN_XCHG_PEER: no NCCL.  The per-block Gram/RHS partials (and the sweep
     * norms, RSE and metric sums) are exchanged over peer memory of one node (NVLink /
     * NVSwitch): every rank's library-owned exchange buffer is exported with a CUDA IPC
     * handle, and the solve kernel of each block publishes, waits for its peers and sums their
     * partials in rank order itself (device-side all-reduce fused with the solve; see
     * paper_2511_16358_b200/csrc/peer.cuh).  host_allgather (called once, inside
     * ifctn_create, with this rank's 64-byte handle) must fill `all` with the world handles in
     * rank order — a host all-gather (e.g. torch.distributed.all_gather_object).  May be NULL
     * when world == 1.  Ranks must be on distinct GPUs of one node with peer access.        */
    int exchange;
    void (*host_allgather)(const void* mine, void* all, size_t bytes, void* user);
} ifctn_dist;

#define IFCTN_XCHG_NCCL 0 /* NCCL all-reduce launched on the context's stream (default)      */
#define IFCTN_XCHG_PEER 1 /* device-side exchange over peer memory (one node)                */

/* One row of the per-sweep trace (Algorithm 1 stop test P:L341-344, Lemma 2). */
typedef struct {
    int sweep;          /* 1-based sweep index s+1                                         */
    double rel_change;  /* ‖X^{s+1} − X^{s}‖_F / ‖X^{s}‖_F  (denominator 1 if ‖X^{s}‖ = 0)  */
    double objective;   /* F(M^{s+1}) = ½‖X^{s+1} − iFCTN(G^{s+1})‖²_F                     */
    double dx2;         /* ‖X^{s+1} − X^{s}‖²_F                                            */
    double dg2;         /* Σ_{k,i} ‖G^{s+1}_{k,i} − G^{s}_{k,i}‖²_F                        */
} ifctn_trace_row;

/* Which tensor ifctn_reconstruct writes. */
#define IFCTN_MODEL 0 /* iFCTN(G) = Π_{p<q} (G_{p,q}ᵀG_{q,p})(i_p,i_q)  (Def. 4, Eq. 5)       */
#define IFCTN_X 1     /* the current iterate X                                               */

/* Bytes of device workspace ifctn_create needs (caller may pass NULL to let the library
 * allocate it).  Independent of the device; deterministic in its arguments.             */
ifctn_status ifctn_workspace_bytes(int order, const int64_t* dims, const int32_t* ranks,
                                   ifctn_dtype dtype, const ifctn_dist* dist, size_t* bytes);

/* This rank's slice [*begin, *end) of the shard mode (P:silent; reading R21:
 * ranks get ⌈I_s/W⌉ then ⌊I_s/W⌋ slices) and the shard mode itself.                    */
ifctn_status ifctn_shard_range(int order, const int64_t* dims, const ifctn_dist* dist,
                               int* shard_mode, int64_t* begin, int64_t* end);

/* Create a solver context: Algorithm 1 "Input" + "Initialization".
 *   dims[order]         global mode sizes I_0..I_{N-1}
 *   ranks[order*order]  iFCTN-rank matrix R, row-major, symmetric, zero diagonal,
 *                       1 ≤ R_{p,q} ≤ IFCTN_MAX_RANK (Def. 4)
 *   rho                 proximal weight ρ > 0
 *   observed            O (this rank's shard); values off Ω are ignored unless
 *                       IFCTN_FLAG_X_FULL; X⁽⁰⁾ = P_Ω(O) with zeros on Ω^c (reading R7)
 *   mask                Ω as uint8, same layout, nonzero = observed
 *   init_factors        G⁰ in the factor layout above
 *   workspace           device memory of ≥ ifctn_workspace_bytes(), 256-B aligned, owned by
 *                       the caller and kept alive until ifctn_destroy; NULL = library-owned
 *   stream              cudaStream_t (NULL = legacy default stream)
 * The inputs are copied; the caller may free them after this returns.                  */
ifctn_status ifctn_create(ifctn_ctx** out, int order, const int64_t* dims,
                          const int32_t* ranks, ifctn_dtype dtype, double rho,
                          const void* observed, const uint8_t* mask, const void* init_factors,
                          void* workspace, size_t workspace_bytes, const ifctn_dist* dist,
                          void* stream, unsigned flags);

/* Run up to t_max PAM sweeps (Algorithm 1 while-loop).  eps ≤ 0 runs exactly
 * t_max sweeps and, with trace == NULL, returns without synchronising (device errors are
 * then reported by ifctn_sync).  eps > 0 stops after the first sweep with rel_change < eps.
 * trace (host, t_max rows) is filled when non-NULL.  *sweeps_done (may be NULL).
 * With eps ≤ 0 and t_max ≥ 2 the X update of sweep s and the first block of sweep s+1
 * run as one pass over X (they use the same factors); results are the same sweeps up to
 * floating-point summation order.  With a trace on that path the rows are gathered on the
 * device and read back once, after the last sweep (a single synchronisation).          */
ifctn_status ifctn_sweep(ifctn_ctx* ctx, int t_max, double eps, int* sweeps_done,
                         ifctn_trace_row* trace);

/* Wait for the context's stream and report deferred device errors (E_NOT_SPD, E_NONFINITE). */
ifctn_status ifctn_sync(ifctn_ctx* ctx);

/* Write IFCTN_MODEL or IFCTN_X (this rank's shard, dense layout) to out.                */
ifctn_status ifctn_reconstruct(ifctn_ctx* ctx, int what, void* out);

/* Copy the current factors (layout of init_factors) to out.                              */
ifctn_status ifctn_get_factors(ifctn_ctx* ctx, void* out);

/* RSE = ‖T − X‖_F / ‖T‖_F over the global tensor (denominator reading R10).
 * truth: this rank's shard.                                                              */
ifctn_status ifctn_rse(ifctn_ctx* ctx, const void* truth, double* rse);

/* f(G, X) = ½‖X − iFCTN(G)‖²_F of the current state.                            */
ifctn_status ifctn_objective(ifctn_ctx* ctx, double* f);

/* ---- step-level entry points (the rows of a sweep; used by parity tests) ------------- */

/* Step a2 for block (k,i): β(a,j) = Σ_{i_i=a, i_k=j} M X, ω(a,j) = Σ M² with
 * M = Π_{{p,q}≠{k,i}} (G_{p,q}ᵀG_{q,p})(i_p,i_q) (Prop. 1 + Eq. 8's D, y_j),
 * from the current state, no state change.  beta/omega: float64 I_i × I_k column-major
 * (a = i_i fastest); under sharding the local partial sums.                              */
ifctn_status ifctn_block_coefficients(ifctn_ctx* ctx, int k, int i, double* beta,
                                      double* omega);

/* Steps a2-a4 for block (k,i): new G_{k,i} from the current state (Eq. 8), H refreshed.  */
ifctn_status ifctn_block_update(ifctn_ctx* ctx, int k, int i);

/* Step a5: X ← P_Ω(X) + P_Ω^c((iFCTN(G) + ρX)/(1+ρ)); norms (host, may be NULL) gets
 * {‖ΔX‖², ‖X_old‖², ½‖X_new − iFCTN(G)‖², Σ‖ΔG‖² since the last X update}.             */
ifctn_status ifctn_x_update(ifctn_ctx* ctx, double* norms);

ifctn_status ifctn_destroy(ifctn_ctx* ctx);

const char* ifctn_status_string(ifctn_status s);
const char* ifctn_last_error(const ifctn_ctx* ctx);

/* Self-test of the peer-exchange protocol on the CURRENT device (test support): `world`
 * (2..16) virtual ranks run `rounds` exchanges of `n` doubles in ONE cooperative launch (ranks
 * whose kernels wait on one another must not be separate launches on one GPU), with the same
 * publish / wait / rank-ordered sum / epoch code as the library's solve kernels.  *errors =
 * number of mismatching sums (0 expected).  E_ARG for bad sizes, E_CUDA on launch failure. */
ifctn_status ifctn_peer_selftest(int world, int rounds, int64_t n, int64_t* errors);

/* Run ONE sweep as plain launches with a CUDA event before every kernel, on the context's
 * stream, and return each launch's device time in ms, in launch order:
 *   for every block (k asc, i asc, i≠k): [a2 fibre pass, a2 partial reduce, a3/a4 solve],
 *   then [a5 refill pass, norm finaliser].
 * *count = 3·N(N−1) + 2 (entries beyond `capacity` are dropped).  Advances the state by
 * one sweep exactly like ifctn_sweep(ctx, 1, 0, …).                                    */
ifctn_status ifctn_profile_sweep(ifctn_ctx* ctx, float* ms, int capacity, int* count);

/* Kernel launches the last ifctn_sweep enqueued (graph nodes count as launches).         */
int64_t ifctn_launch_count(const ifctn_ctx* ctx);

/* ---- Evaluation metrics ------------------------------------------
 * The paper's evaluation quantities of the current X against a truth tensor T (this rank's
 * shard, host or device, same layout as `observed`), computed on the device in fp64 and
 * all-reduced across ranks:
 *   out[0] RSE  = ‖T − X‖_F / ‖T‖_F (reading R10)
 *   out[1] RMSE = sqrt(Σ_{Ω^c} (T − X)² / |Ω^c|) over the missing entries (NaN if Ω^c = ∅)
 *   out[2] PSNR = mean over the bands (slices of the last mode) of 10·log10(1/MSE_band),
 *                 peak 1 (data in [0,1]); +inf when a band is reproduced exactly
 *   out[3] SSIM (3rd-order tensors): per band the image over modes 1 and 2, single-scale SSIM
 *                 with an 11×11 Gaussian window (σ = 1.5), K1 = 0.01, K2 = 0.03, L = 1, over
 *                 the valid windows (one uniform whole-image window when a side is < 11),
 *                 averaged over windows and bands; NaN for other orders or when the shard
 *                 mode is an image mode
 *   out[4] |Ω^c| (global)
 * Errors: E_ARG for NULL pointers or ‖T‖ = 0.                                              */
ifctn_status ifctn_metrics(ifctn_ctx* ctx, const void* truth, double* out);

/* ---- Sampling-set generators on the device -------------
 * The paper's two missingness protocols, random missing (RM) and fibre missing (FM), as
 * exact-count draws without replacement (reading R12): the selected set is the k
 * indices u with the smallest keys key(u) = fmix64(seed + (u+1)·0x9E3779B97F4A7C15), i.e. the
 * u-th output of the splitmix64 generator started at state `seed` (fmix64: z ^= z>>30,
 * z *= 0xBF58476D1CE4E5B9, z ^= z>>27, z *= 0x94D049BB133111EB, z ^= z>>31; all mod 2^64).
 * The keys are distinct (a bijection of u), so the set is unique; the result is
 * deterministic and bit-identical on every GPU.  Found by an on-device 8-bit radix select
 * (no host synchronisation); all work is enqueued on `stream` (cudaStream_t, NULL = legacy
 * default).  A 2 KB scratch is taken with cudaMallocAsync on that stream and freed on it.
 *
 * ifctn_mask_uniform: mask[u] = 1 for the `observed` selected indices of u ∈ [0, n), else 0.
 *   mask    DEVICE, n bytes, caller-owned (written in full)
 * ifctn_mask_fibres: whole mode-`mode` fibres (0-based) missing.  Fibre index of entry
 *   u = i_0 + I_0(i_1 + …) is its linear index with mode `mode` removed (remaining modes
 *   ascending, lowest fastest); the `missing_fibres` selected fibres (keys over the fibre
 *   index space [0, n/I_mode)) are 0 along their whole length, every other entry is 1.
 *   mask    DEVICE, Π dims bytes, mode-1-fastest, caller-owned (written in full)
 * Errors: E_ARG for a NULL/host mask, negative counts or a count above the population;
 * E_SHAPE for a dim < 1; E_CUDA for a launch or allocation failure.                       */
ifctn_status ifctn_mask_uniform(uint8_t* mask, int64_t n, int64_t observed, uint64_t seed, void* stream);
ifctn_status ifctn_mask_fibres(uint8_t* mask, int order, const int64_t* dims, int mode,
                               int64_t missing_fibres, uint64_t seed, void* stream);

/* ---- Multi-instance driver: the paper's rank-grid protocol -------------
 * The paper reports its runtimes "including the time required to tune all parameters"
 * over rank grids such as R_{1,2} ∈ {3,6,9,15,30,36}, R_{1,3} = R_{2,3} ∈ {3,6,9}
 * (P:L485-486).  ifctn_grid_run solves `count` independent instances that share O, Ω (and
 * the truth for the RSE) and differ in ranks, ρ and G⁰, `concurrency` of them at a time on
 * one GPU, each in its own context on its own CUDA stream (small instances are launch- and
 * latency-bound, so concurrent streams fill the GPU).  Instances run in waves of
 * `concurrency`; every instance is bit-identical to a lone ifctn_create + ifctn_sweep(t_max,
 * eps = 0) run (same kernels, deterministic reductions).  Workspaces are allocated once per
 * slot (the largest instance's size) and reused.  Multi-GPU: give every process its own
 * slice of the instance list (no communication; bench/grid.py partitions and gathers).
 *   observed, mask, truth   as in ifctn_create / ifctn_rse (host or device); truth may be
 *                           NULL (results[].rse = NaN)
 *   instances[count]        ranks (order×order), ρ and G⁰ of each instance (caller-owned)
 *   t_max                   sweeps per instance (≥ 1); no stop test
 *   concurrency             instances resident at once (≥ 1)
 *   results[count]          per instance: final RSE, objective ½‖X − t‖², device seconds of
 *                           its sweeps, and its status (the call returns the first failure) */
typedef struct {
    const int32_t* ranks;
    double rho;
    const void* init_factors;
} ifctn_instance;

typedef struct {
    double rse;
    double objective;
    double seconds;
    int status;
} ifctn_instance_result;

ifctn_status ifctn_grid_run(int order, const int64_t* dims, ifctn_dtype dtype,
                            const void* observed, const uint8_t* mask, const void* truth,
                            const ifctn_instance* instances, int count, int t_max,
                            int concurrency, ifctn_instance_result* results);

#ifdef __cplusplus
}
#endif
#endif /* IFCTN_H */
