/*
 * ifctn_oracle.c — float64 CPU ORACLE for the iFCTN-TC PAM sweep.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load this library. The product path
 * (paper_2511_16358_b200/) never links, imports or executes anything here, and this
 * file shares no code, header, table or helper with the CUDA path.
 *
 * It is the plain, slow, obviously-correct statement of what the sweep computes,
 * written from the paper (arxiv 2511.16358, /root/reference/PAPER.md = "P:L…"):
 *
 *   - Def. 4 / Eq. 5: t(i_1..i_N) = Σ_r Π_{k} Π_{i≠k} G_{k,i}(r_{k,i}, i_k).
 *     Each rank index r_{p,q} occurs in exactly two factors (G_{p,q} and G_{q,p}), so the
 *     nested sum factorises into t(i) = Π_{p<q} H_{p,q}(i_p,i_q), H_{p,q} = G_{p,q}ᵀG_{q,p}.
 *     The factorised form is what the oracle evaluates; tests pin it to a literal Eq. 5
 *     nested sum (oracle/brute.py) on tiny inputs.
 *   - PAM scheme, Gauss–Seidel order k ascending, i ascending.
 *   - Eq. 8: column-wise closed form of the G_{k,i} subproblem, written as the
 *     normal equations (A_jᵀA_j + ρI) c = A_jᵀ x_j + ρ c_old with A_jᵀA_j = Σ_a ω(a,j) g_a g_aᵀ
 *     and A_jᵀx_j = Σ_a β(a,j) g_a (g_a = G_{i,k}(:,a)); tests pin this to a dense
 *     Prop. 1 Z_k construction (oracle/brute.py).
 *   - Eq. 9 read as the exact per-entry prox minimiser (t + ρx)/(1+ρ) on Ω^c
 *     (reading R1); X on Ω is left untouched (= O bit for bit).
 *   - Algorithm 1 and Lemma 2: sufficient decrease is asserted
 *     on every sweep.
 *
 * Conventions: modes are 0-based here (paper mode k = code k+1);
 * tensors are mode-1-fastest (column-major) and unpadded; G is the concatenation of the
 * N(N-1) matrices G_{k,i} (k ascending, i ascending, i≠k), each R_{k,i}×I_k column-major
 * (r fastest); H_{p,q} (p<q) is I_p×I_q column-major; β_{k,i}, ω_{k,i} are I_i×I_k
 * column-major (a = i_i fastest, j = i_k).
 *
 * Parallelism: optional OpenMP over contiguous chunks of the linear index with
 * thread-private accumulators merged in thread order (deterministic for a fixed thread
 * count); orc_set_threads(1) is the serial reference.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_MAXN 8

static int g_threads = 1;

void orc_set_threads(int t) { g_threads = t < 1 ? 1 : t; }
int orc_get_threads(void) { return g_threads; }

/* ---- shape helpers --------------------------------------------------------------- */

static int64_t prod_dims(int N, const int64_t* dims) {
    int64_t n = 1;
    for (int m = 0; m < N; ++m) n *= dims[m];
    return n;
}

/* Number of cherry-factor parameters: Σ_k Σ_{i≠k} R_{k,i} I_k  (Eq. 3). */
int64_t orc_num_params(int N, const int64_t* dims, const int32_t* ranks) {
    int64_t s = 0;
    for (int k = 0; k < N; ++k)
        for (int i = 0; i < N; ++i)
            if (i != k) s += (int64_t)ranks[k * N + i] * dims[k];
    return s;
}

/* Offset of G_{k,i} inside the concatenated factor array (k asc, i asc, i≠k). */
int64_t orc_factor_offset(int N, const int64_t* dims, const int32_t* ranks, int k, int i) {
    int64_t off = 0;
    for (int kk = 0; kk < N; ++kk)
        for (int ii = 0; ii < N; ++ii) {
            if (ii == kk) continue;
            if (kk == k && ii == i) return off;
            off += (int64_t)ranks[kk * N + ii] * dims[kk];
        }
    return -1;
}

/* Pair index of (p,q), p<q, in lexicographic order. */
static int pair_index(int N, int p, int q) {
    int idx = 0;
    for (int a = 0; a < N; ++a)
        for (int b = a + 1; b < N; ++b) {
            if (a == p && b == q) return idx;
            ++idx;
        }
    return -1;
}

/* ---- a1: pairwise Gram H_{p,q} = G_{p,q}ᵀ G_{q,p}  (Def. 4 / Eq. 5, P:L193-200;
 *          also the factors of S_k in Prop. 1) ------------------------------ */
void orc_pair_gram(int N, const int64_t* dims, const int32_t* ranks, const double* G,
                   int p, int q, double* H) {
    const int R = ranks[p * N + q];
    const double* Gpq = G + orc_factor_offset(N, dims, ranks, p, q); /* R × I_p */
    const double* Gqp = G + orc_factor_offset(N, dims, ranks, q, p); /* R × I_q */
    for (int64_t b = 0; b < dims[q]; ++b)
        for (int64_t a = 0; a < dims[p]; ++a) {
            double s = 0.0;
            for (int r = 0; r < R; ++r) s += Gpq[r + (int64_t)R * a] * Gqp[r + (int64_t)R * b];
            H[a + dims[p] * b] = s;
        }
}

/* All P = N(N-1)/2 pairwise Grams, each malloc'ed; Hs[pair_index(p,q)]. */
static double** all_grams(int N, const int64_t* dims, const int32_t* ranks, const double* G) {
    int P = N * (N - 1) / 2;
    double** Hs = (double**)calloc((size_t)P, sizeof(double*));
    for (int p = 0; p < N; ++p)
        for (int q = p + 1; q < N; ++q) {
            int id = pair_index(N, p, q);
            Hs[id] = (double*)malloc(sizeof(double) * (size_t)(dims[p] * dims[q]));
            orc_pair_gram(N, dims, ranks, G, p, q, Hs[id]);
        }
    return Hs;
}

static void free_grams(int N, double** Hs) {
    int P = N * (N - 1) / 2;
    for (int i = 0; i < P; ++i) free(Hs[i]);
    free(Hs);
}

static void decode(int64_t lin, int N, const int64_t* dims, int64_t* idx) {
    for (int m = 0; m < N; ++m) {
        idx[m] = lin % dims[m];
        lin /= dims[m];
    }
}

static void advance(int N, const int64_t* dims, int64_t* idx) {
    for (int m = 0; m < N; ++m) {
        if (++idx[m] < dims[m]) return;
        idx[m] = 0;
    }
}

/* Product of H_{p,q}(i_p,i_q) over all pairs p<q except the pair {skip_a, skip_b}
 * (pass skip_a = skip_b = -1 to keep every pair).  This is t(i) (Def. 4 closed form) or
 * the leave-one-pair-out weight M^{(k,i)}(i) of Eq. 8's D·(y_j ⊗ ·). */
static double pair_product(int N, const int64_t* dims, double* const* Hs, const int64_t* idx,
                           int skip_a, int skip_b) {
    double m = 1.0;
    int id = 0;
    for (int p = 0; p < N; ++p)
        for (int q = p + 1; q < N; ++q, ++id) {
            if ((p == skip_a && q == skip_b) || (p == skip_b && q == skip_a)) continue;
            m *= Hs[id][idx[p] + dims[p] * idx[q]];
        }
    return m;
}

static double load_x(const void* X, int x_is_f32, int64_t lin) {
    return x_is_f32 ? (double)((const float*)X)[lin] : ((const double*)X)[lin];
}

static int nthreads_for(int64_t n) {
    int t = g_threads;
    if (n < 4096) t = 1;
    return t;
}

/* ---- iFCTN model t = iFCTN(G)  (Def. 4, Eq. 5; closed form pinned by brute Eq. 5) ---- */
void orc_model(int N, const int64_t* dims, const int32_t* ranks, const double* G, double* t) {
    double** Hs = all_grams(N, dims, ranks, G);
    const int64_t n = prod_dims(N, dims);
    const int T = nthreads_for(n);
#pragma omp parallel num_threads(T)
    {
        int tid = 0, nt = 1;
#ifdef _OPENMP
        tid = omp_get_thread_num();
        nt = omp_get_num_threads();
#endif
        int64_t lo = n * tid / nt, hi = n * (tid + 1) / nt;
        int64_t idx[ORC_MAXN];
        decode(lo, N, dims, idx);
        for (int64_t lin = lo; lin < hi; ++lin) {
            t[lin] = pair_product(N, dims, Hs, idx, -1, -1);
            advance(N, dims, idx);
        }
    }
    free_grams(N, Hs);
}

/* Model entry at one multi-index (for sampled checks at full size). */
double orc_model_at(int N, const int64_t* dims, const int32_t* ranks, const double* G,
                    const int64_t* idx) {
    double m = 1.0;
    for (int p = 0; p < N; ++p)
        for (int q = p + 1; q < N; ++q) {
            const int R = ranks[p * N + q];
            const double* Gpq = G + orc_factor_offset(N, dims, ranks, p, q);
            const double* Gqp = G + orc_factor_offset(N, dims, ranks, q, p);
            double s = 0.0;
            for (int r = 0; r < R; ++r) s += Gpq[r + (int64_t)R * idx[p]] * Gqp[r + (int64_t)R * idx[q]];
            m *= s;
        }
    return m;
}

/* ---- a2: coefficient contraction of block (k,i)  (Prop. 1; Eq. 8)
 *   β(a,j) = Σ_{i: i_i=a, i_k=j} M^{(k,i)}(i) X(i),   ω(a,j) = Σ_{i: i_i=a, i_k=j} M^{(k,i)}(i)²
 * with M^{(k,i)} = Π_{{p,q}≠{k,i}} H_{p,q}(i_p,i_q). Outputs are I_i × I_k column-major.  */
void orc_block_contract(int N, const int64_t* dims, const int32_t* ranks, const double* G,
                        const void* X, int x_is_f32, int k, int i, double* beta, double* omega) {
    double** Hs = all_grams(N, dims, ranks, G);
    const int64_t n = prod_dims(N, dims);
    const int64_t nout = dims[i] * dims[k];
    const int T = nthreads_for(n);
    double* pb = (double*)calloc((size_t)(T * nout), sizeof(double));
    double* pw = (double*)calloc((size_t)(T * nout), sizeof(double));
#pragma omp parallel num_threads(T)
    {
        int tid = 0, nt = 1;
#ifdef _OPENMP
        tid = omp_get_thread_num();
        nt = omp_get_num_threads();
#endif
        double* b = pb + (int64_t)tid * nout;
        double* w = pw + (int64_t)tid * nout;
        int64_t lo = n * tid / nt, hi = n * (tid + 1) / nt;
        int64_t idx[ORC_MAXN];
        decode(lo, N, dims, idx);
        for (int64_t lin = lo; lin < hi; ++lin) {
            double m = pair_product(N, dims, Hs, idx, k, i);
            int64_t o = idx[i] + dims[i] * idx[k];
            b[o] += m * load_x(X, x_is_f32, lin);
            w[o] += m * m;
            advance(N, dims, idx);
        }
    }
    for (int64_t o = 0; o < nout; ++o) {
        double sb = 0.0, sw = 0.0;
        for (int t = 0; t < T; ++t) {
            sb += pb[(int64_t)t * nout + o];
            sw += pw[(int64_t)t * nout + o];
        }
        beta[o] = sb;
        omega[o] = sw;
    }
    free(pb);
    free(pw);
    free_grams(N, Hs);
}

/* Same contraction for one output (a,j) only: sums over the n/(I_i I_k) entries with
 * i_i = a, i_k = j. Used for sampled parity checks at full size. */
void orc_block_contract_at(int N, const int64_t* dims, const int32_t* ranks, const double* G,
                           const void* X, int x_is_f32, int k, int i, int64_t a, int64_t j,
                           double* beta, double* omega) {
    double** Hs = all_grams(N, dims, ranks, G);
    int64_t rdims[ORC_MAXN];
    int rmodes[ORC_MAXN], nr = 0;
    for (int m = 0; m < N; ++m)
        if (m != k && m != i) { rmodes[nr] = m; rdims[nr] = dims[m]; ++nr; }
    int64_t nred = prod_dims(nr, rdims);
    int64_t stride[ORC_MAXN];
    stride[0] = 1;
    for (int m = 1; m < N; ++m) stride[m] = stride[m - 1] * dims[m - 1];
    const int T = nthreads_for(nred);
    double* pb = (double*)calloc((size_t)T, sizeof(double));
    double* pw = (double*)calloc((size_t)T, sizeof(double));
#pragma omp parallel num_threads(T)
    {
        int tid = 0, nt = 1;
#ifdef _OPENMP
        tid = omp_get_thread_num();
        nt = omp_get_num_threads();
#endif
        int64_t lo = nred * tid / nt, hi = nred * (tid + 1) / nt;
        int64_t ridx[ORC_MAXN], idx[ORC_MAXN];
        decode(lo, nr, rdims, ridx);
        double sb = 0.0, sw = 0.0;
        for (int64_t r = lo; r < hi; ++r) {
            idx[k] = j;
            idx[i] = a;
            for (int t = 0; t < nr; ++t) idx[rmodes[t]] = ridx[t];
            int64_t lin = 0;
            for (int m = 0; m < N; ++m) lin += idx[m] * stride[m];
            double mm = pair_product(N, dims, Hs, idx, k, i);
            sb += mm * load_x(X, x_is_f32, lin);
            sw += mm * mm;
            advance(nr, rdims, ridx);
        }
        pb[tid] = sb;
        pw[tid] = sw;
    }
    double sb = 0.0, sw = 0.0;
    for (int t = 0; t < T; ++t) { sb += pb[t]; sw += pw[t]; }
    *beta = sb;
    *omega = sw;
    free(pb);
    free(pw);
    free_grams(N, Hs);
}

/* ---- a3/a4: Gram/RHS + ρI and the SPD solve for one column j of G_{k,i}
 *   (Eq. 8):  (Σ_a ω(a,j) g_a g_aᵀ + ρI) c = Σ_a β(a,j) g_a + ρ c_old,
 *   g_a = G_{i,k}(:,a) (R × I_i column-major).  Plain Cholesky LLᵀ, then two triangular
 *   solves.  Returns 0, or 7 if a pivot is not positive (impossible in exact arithmetic
 *   for ρ > 0).                                                                          */
int orc_column_solve(int R, int64_t I_i, const double* Gik, const double* beta_col,
                     const double* omega_col, const double* c_old, double rho, double* c_new) {
    double A[64 * 64], L[64 * 64], b[64], y[64];
    if (R > 64) return 1;
    for (int r = 0; r < R; ++r) {
        b[r] = rho * c_old[r];
        for (int s = 0; s < R; ++s) A[r + R * s] = (r == s) ? rho : 0.0;
    }
    for (int64_t a = 0; a < I_i; ++a) {
        const double* g = Gik + (int64_t)R * a;
        for (int r = 0; r < R; ++r) {
            b[r] += beta_col[a] * g[r];
            for (int s = 0; s < R; ++s) A[r + R * s] += omega_col[a] * g[r] * g[s];
        }
    }
    memset(L, 0, sizeof(L));
    for (int c = 0; c < R; ++c) {
        double d = A[c + R * c];
        for (int s = 0; s < c; ++s) d -= L[c + R * s] * L[c + R * s];
        if (!(d > 0.0)) return 7;
        L[c + R * c] = sqrt(d);
        for (int r = c + 1; r < R; ++r) {
            double v = A[r + R * c];
            for (int s = 0; s < c; ++s) v -= L[r + R * s] * L[c + R * s];
            L[r + R * c] = v / L[c + R * c];
        }
    }
    for (int r = 0; r < R; ++r) { /* L y = b */
        double v = b[r];
        for (int s = 0; s < r; ++s) v -= L[r + R * s] * y[s];
        y[r] = v / L[r + R * r];
    }
    for (int r = R - 1; r >= 0; --r) { /* Lᵀ c = y */
        double v = y[r];
        for (int s = r + 1; s < R; ++s) v -= L[s + R * r] * c_new[s];
        c_new[r] = v / L[r + R * r];
    }
    return 0;
}

/* One block update of G_{k,i} (PAM step; Eq. 8): contraction from the
 * current (most recent) factors, then every column solved from the same state (columns are
 * separable), then G_{k,i} overwritten. *dG2 += ‖G_new − G_old‖²_F.            */
int orc_block_update(int N, const int64_t* dims, const int32_t* ranks, double* G, const void* X,
                     int x_is_f32, int k, int i, double rho, double* dG2) {
    const int R = ranks[k * N + i];
    const int64_t Ii = dims[i], Ik = dims[k];
    double* beta = (double*)malloc(sizeof(double) * (size_t)(Ii * Ik));
    double* omega = (double*)malloc(sizeof(double) * (size_t)(Ii * Ik));
    orc_block_contract(N, dims, ranks, G, X, x_is_f32, k, i, beta, omega);
    double* Gki = G + orc_factor_offset(N, dims, ranks, k, i);
    const double* Gik = G + orc_factor_offset(N, dims, ranks, i, k);
    double* Gnew = (double*)malloc(sizeof(double) * (size_t)(R * Ik));
    int st = 0;
    for (int64_t j = 0; j < Ik && st == 0; ++j)
        st = orc_column_solve(R, Ii, Gik, beta + Ii * j, omega + Ii * j, Gki + (int64_t)R * j,
                              rho, Gnew + (int64_t)R * j);
    if (st == 0) {
        double d = 0.0;
        for (int64_t e = 0; e < (int64_t)R * Ik; ++e) {
            double diff = Gnew[e] - Gki[e];
            d += diff * diff;
            Gki[e] = Gnew[e];
        }
        if (dG2) *dG2 += d;
    }
    free(Gnew);
    free(beta);
    free(omega);
    return st;
}

/* ---- a5: X update (Eq. 9 read as the per-entry prox minimiser) plus norms.
 *   On Ω^c: X_new = (t + ρ X)/(1+ρ); on Ω: X untouched (X = O there, Alg. 1).
 *   out[0] = ‖X_new − X‖², out[1] = ‖X‖² (old X, the stop-test denominator P:L343),
 *   out[2] = f(G, X_new) = ½‖X_new − t‖².                                        */
void orc_refill(int N, const int64_t* dims, const int32_t* ranks, const double* G, double* X,
                const uint8_t* mask, double rho, double* out) {
    double** Hs = all_grams(N, dims, ranks, G);
    const int64_t n = prod_dims(N, dims);
    const int T = nthreads_for(n);
    double* part = (double*)calloc((size_t)(3 * T), sizeof(double));
#pragma omp parallel num_threads(T)
    {
        int tid = 0, nt = 1;
#ifdef _OPENMP
        tid = omp_get_thread_num();
        nt = omp_get_num_threads();
#endif
        int64_t lo = n * tid / nt, hi = n * (tid + 1) / nt;
        int64_t idx[ORC_MAXN];
        decode(lo, N, dims, idx);
        double dx2 = 0.0, x2 = 0.0, f2 = 0.0;
        for (int64_t lin = lo; lin < hi; ++lin) {
            double t = pair_product(N, dims, Hs, idx, -1, -1);
            double x = X[lin];
            double xn = mask[lin] ? x : (t + rho * x) / (1.0 + rho);
            dx2 += (xn - x) * (xn - x);
            x2 += x * x;
            f2 += (xn - t) * (xn - t);
            X[lin] = xn;
            advance(N, dims, idx);
        }
        part[3 * tid + 0] = dx2;
        part[3 * tid + 1] = x2;
        part[3 * tid + 2] = f2;
    }
    out[0] = out[1] = out[2] = 0.0;
    for (int t = 0; t < T; ++t) {
        out[0] += part[3 * t + 0];
        out[1] += part[3 * t + 1];
        out[2] += part[3 * t + 2];
    }
    out[2] *= 0.5;
    free(part);
    free_grams(N, Hs);
}

/* f(G, X) = ½‖X − iFCTN(G)‖²_F. */
double orc_objective(int N, const int64_t* dims, const int32_t* ranks, const double* G,
                     const double* X) {
    const int64_t n = prod_dims(N, dims);
    double* t = (double*)malloc(sizeof(double) * (size_t)n);
    orc_model(N, dims, ranks, G, t);
    double s = 0.0;
    for (int64_t e = 0; e < n; ++e) s += (X[e] - t[e]) * (X[e] - t[e]);
    free(t);
    return 0.5 * s;
}

/* X⁽⁰⁾ = P_Ω(O), zero on Ω^c (Alg. 1 initialisation P:L334; reading R7). */
void orc_init_x(int64_t n, const void* O, int o_is_f32, const uint8_t* mask, double* X) {
    for (int64_t e = 0; e < n; ++e) X[e] = mask[e] ? load_x(O, o_is_f32, e) : 0.0;
}

/* RSE = ‖X_true − X‖_F / ‖X_true‖_F (denominator reading R10). */
double orc_rse(int64_t n, const double* truth, const double* X) {
    double num = 0.0, den = 0.0;
    for (int64_t e = 0; e < n; ++e) {
        num += (truth[e] - X[e]) * (truth[e] - X[e]);
        den += truth[e] * truth[e];
    }
    return sqrt(num) / sqrt(den);
}

/* ---- one PAM sweep = Algorithm 1 lines 2-5 --------------------------------
 *   for k, for i≠k: block update (most recent values); then X update (Eq. 9);
 *   Lemma 2:  F_prev − F ≥ (ρ/2)(‖ΔX‖² + Σ‖ΔG‖²) − slack.
 *   *F_prev is updated to F on return.  row[0..3] = rel_change, F, ‖ΔX‖², Σ‖ΔG‖².
 *   Returns 0, 3 (Lemma 2 violated) or 7 (non-SPD).                                      */
int orc_sweep(int N, const int64_t* dims, const int32_t* ranks, double* G, double* X,
              const uint8_t* mask, double rho, double* F_prev, double* row, int check_lemma2) {
    double dG2 = 0.0;
    for (int k = 0; k < N; ++k)
        for (int i = 0; i < N; ++i) {
            if (i == k) continue;
            int st = orc_block_update(N, dims, ranks, G, X, 0, k, i, rho, &dG2);
            if (st) return st;
        }
    double out[3];
    orc_refill(N, dims, ranks, G, X, mask, rho, out);
    const double xnorm = sqrt(out[1]);
    const double rel = sqrt(out[0]) / (xnorm > 0.0 ? xnorm : 1.0); /* reading R9 */
    const double F = out[2];
    int status = 0;
    if (check_lemma2 && F_prev) {
        const int64_t n = prod_dims(N, dims);
        const double u = 1.1102230246251565e-16;
        double scale = fabs(*F_prev) > 1.0 ? fabs(*F_prev) : 1.0;
        double slack = 1e-12 * scale + 4.0 * (double)n * u * scale; /* reading R16 */
        if (*F_prev - F < 0.5 * rho * (out[0] + dG2) - slack) status = 3;
    }
    if (F_prev) *F_prev = F;
    if (row) {
        row[0] = rel;
        row[1] = F;
        row[2] = out[0];
        row[3] = dG2;
    }
    return status;
}

/* Full Algorithm 1 run: X⁽⁰⁾ = P_Ω(O); up to t_max sweeps; stop when rel < eps (eps ≤ 0
 * runs exactly t_max sweeps).  trace (optional) gets 4 doubles per sweep.  Returns the
 * number of sweeps done (≥0) or −status on an error.                                    */
int orc_solve(int N, const int64_t* dims, const int32_t* ranks, double* G, double* X,
              const uint8_t* mask, double rho, int t_max, double eps, double* trace,
              int check_lemma2) {
    double F = orc_objective(N, dims, ranks, G, X);
    for (int s = 0; s < t_max; ++s) {
        double row[4];
        int st = orc_sweep(N, dims, ranks, G, X, mask, rho, &F, row, check_lemma2);
        if (trace) memcpy(trace + 4 * s, row, sizeof(row));
        if (st) return -st;
        if (eps > 0.0 && row[0] < eps) return s + 1;
    }
    return t_max;
}
