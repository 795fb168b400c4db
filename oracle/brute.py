"""L0 "brute" oracle tier: literal, exponential-cost numpy statements of the paper's
definitions, for TINY inputs only (n·ΠR ≲ 1e6).

TEST INFRASTRUCTURE ONLY (see oracle/oracle.py). This file shares no code with the C oracle
(ifctn_oracle.c) nor with the CUDA path; it exists to pin the C oracle to the paper:

  * eq5_entry / eq5_tensor  — Def. 4, Eq. 5 nested sum over every rank index
  * khatri_rao             — P:L69, c_{(i-1)n+j,l} = a_{il} b_{jl}
  * unfold / fold          — mode-n unfolding X_(n), mode-1-fastest columns
  * cherry_tensor          — Def. 2, Eq. 2: (G_(k))ᵀ = M_N ⊙ … ⊙ M_{k+1} ⊙ M_{k-1} ⊙ … ⊙ M_1
  * build_S / build_Z      — Prop. 1, Eq. 6
  * dense_column_update    — Eq. 8 subproblem solved as a dense ridge LS on the
                             materialised coefficient matrix A_j = Z_k L_j
  * dense_sweep            — Algorithm 1 sweep built from dense_column_update
  * remark1_*              — Def. 3 / Remark 1 cherry product and its matricisation

Modes are 0-based in code (paper mode k = code k+1). Factor layout: list-of-dicts
``G[(k, i)]`` = R_{k,i} × I_k numpy array.
"""
from __future__ import annotations

import itertools

import numpy as np


# ---- basic multilinear algebra ---------------------------------------------------------

def khatri_rao(A, B):
    """A (m×r) ⊙ B (n×r) → (mn×r), row (i-1)n+j = a_i ∘ b_j."""
    m, r = A.shape
    n, r2 = B.shape
    assert r == r2
    C = np.zeros((m * n, r))
    for i in range(m):
        for j in range(n):
            C[i * n + j, :] = A[i, :] * B[j, :]
    return C


def khatri_rao_chain(mats):
    out = mats[0]
    for M in mats[1:]:
        out = khatri_rao(out, M)
    return out


def kron_chain(mats):
    out = mats[0]
    for M in mats[1:]:
        out = np.kron(out, M)
    return out


def unfold(X, n):
    """Mode-n unfolding X_(n) ∈ R^{I_n × Π_{m≠n} I_m}; remaining modes ascending with the
    lowest mode fastest (the convention under which Eq. 2/6/7 are consistent, reading R13)."""
    return np.reshape(np.moveaxis(X, n, 0), (X.shape[n], -1), order="F")


def fold(M, n, shape):
    rest = [shape[m] for m in range(len(shape)) if m != n]
    Y = np.reshape(M, [shape[n]] + rest, order="F")
    return np.moveaxis(Y, 0, n)


def vec(X):
    return np.reshape(X, -1, order="F")


# ---- Def. 4 / Eq. 5 --------------------------------------------------------------------

def pairs(N):
    return [(p, q) for p in range(N) for q in range(p + 1, N)]


def eq5_entry(G, dims, ranks, idx):
    """Eq. 5 literally: Σ over every r_{p,q} (p<q) of Π_k Π_{i≠k} G_{k,i}(r_{k,i}, i_k)."""
    N = len(dims)
    prs = pairs(N)
    total = 0.0
    for rs in itertools.product(*[range(int(ranks[p][q])) for (p, q) in prs]):
        r = {}
        for (p, q), v in zip(prs, rs):
            r[(p, q)] = v
            r[(q, p)] = v
        term = 1.0
        for k in range(N):
            for i in range(N):
                if i != k:
                    term *= G[(k, i)][r[(k, i)], idx[k]]
        total += term
    return total


def eq5_tensor(G, dims, ranks):
    X = np.zeros(dims)
    for idx in itertools.product(*[range(d) for d in dims]):
        X[idx] = eq5_entry(G, dims, ranks, idx)
    return X


# ---- Def. 2 / Eq. 2: cherry tensor -----------------------------------------------------

def cherry_tensor(k, mats, Ik):
    """mats: dict i -> M_i (R_i × I_k), i ≠ k (0..N-1). Returns the mode-k cherry tensor of
    size R_1 × … × I_k × … × R_N whose mode-k unfolding satisfies Eq. 2."""
    N = len(mats) + 1
    order_desc = [i for i in range(N - 1, -1, -1) if i != k]
    GkT = khatri_rao_chain([mats[i] for i in order_desc])  # (ΠR_i × I_k), P:L69 with r = I_k
    shape = [mats[i].shape[0] if i != k else Ik for i in range(N)]
    return fold(GkT.T, k, shape)


def cherry_tensor_elementwise(k, mats, Ik):
    """Rank-one slice statement: 𝒢(r_1..i_k..r_N) = Π_{i≠k} M_i(r_i, i_k)."""
    N = len(mats) + 1
    shape = [mats[i].shape[0] if i != k else Ik for i in range(N)]
    T = np.zeros(shape)
    for idx in itertools.product(*[range(s) for s in shape]):
        v = 1.0
        for i in range(N):
            if i != k:
                v *= mats[i][idx[i], idx[k]]
        T[idx] = v
    return T


# ---- Prop. 1 ---------------------------------------------------------------------------

def build_S(G, dims, k):
    """S_k = ∘_{i<j, i,j≠k} reshape(G_{i,j}ᵀ G_{j,i}) over the modes ≠ k."""
    N = len(dims)
    rest = [m for m in range(N) if m != k]
    S = np.ones([dims[m] for m in rest])
    for (p, q) in pairs(N):
        if k in (p, q):
            continue
        Hpq = G[(p, q)].T @ G[(q, p)]
        shape = [1] * len(rest)
        shape[rest.index(p)] = dims[p]
        shape[rest.index(q)] = dims[q]
        S = S * Hpq.reshape(shape)
    return S


def build_Z(G, dims, k):
    """Z_k = diag(vec(S_k)) · ⊗_{i∈{N..1}∖k} G_{i,k}ᵀ  (Eq. 6)."""
    N = len(dims)
    S = build_S(G, dims, k)
    K = kron_chain([G[(i, k)].T for i in range(N - 1, -1, -1) if i != k])
    return vec(S)[:, None] * K


def kr_chain_T(G, dims, k):
    """(𝒢_(k))ᵀ = G_{k,N} ⊙ … ⊙ G_{k,1} (skip k), as (ΠR × I_k) — Eq. 2 applied to 𝐆_k."""
    N = len(dims)
    return khatri_rao_chain([G[(k, m)] for m in range(N - 1, -1, -1) if m != k])


def L_map(G, dims, k, i, j):
    """Linear map c ↦ column j of the KR chain with G_{k,i}(:,j) replaced by c:
    (⊗_{m>i} g_m) ⊗ I_R ⊗ (⊗_{m<i} g_m), m ≠ k descending, g_m = G_{k,m}(:,j)."""
    N = len(dims)
    mats = []
    for m in range(N - 1, -1, -1):
        if m == k:
            continue
        if m == i:
            mats.append(np.eye(G[(k, i)].shape[0]))
        else:
            mats.append(G[(k, m)][:, j:j + 1])
    return kron_chain(mats)


def dense_column_update(G, dims, X, k, i, j, rho):
    """Eq. 8 subproblem for column j as a dense ridge least squares:
    min_c ½‖x_j − A_j c‖² + ρ/2‖c − c_old‖², A_j = Z_k L_j, x_j = column j of X_(k)ᵀ.
    Solved with numpy.linalg.lstsq on the stacked system [A_j; √ρ I] c ≈ [x_j; √ρ c_old]."""
    Z = build_Z(G, dims, k)
    A = Z @ L_map(G, dims, k, i, j)
    x = unfold(X, k).T[:, j]
    c_old = G[(k, i)][:, j]
    R = A.shape[1]
    As = np.vstack([A, np.sqrt(rho) * np.eye(R)])
    bs = np.concatenate([x, np.sqrt(rho) * c_old])
    c, *_ = np.linalg.lstsq(As, bs, rcond=None)
    return c, A, x


def dense_block_update(G, dims, X, k, i, rho):
    """All columns of G_{k,i} from the same state (columns separable)."""
    new = np.zeros_like(G[(k, i)])
    for j in range(dims[k]):
        new[:, j], _, _ = dense_column_update(G, dims, X, k, i, j, rho)
    return new


def dense_sweep(G, dims, X, mask, rho):
    """Algorithm 1 lines 2-5 with dense ridge solves and Eq. 9 as the prox minimiser."""
    N = len(dims)
    G = {key: v.copy() for key, v in G.items()}
    for k in range(N):
        for i in range(N):
            if i != k:
                G[(k, i)] = dense_block_update(G, dims, X, k, i, rho)
    ranks = [[0 if p == q else G[(p, q)].shape[0] for q in range(N)] for p in range(N)]
    t = eq5_tensor(G, dims, ranks)
    Xn = np.where(mask, X, (t + rho * X) / (1.0 + rho))
    return G, Xn


# ---- Def. 3 / Remark 1 -----------------------------------------------------------------

def remark1_elementwise(A1, A3, B1, B2):
    """Cherry product of a mode-2 cherry tensor 𝒜 (P×I×R; factors A_1 (P×I), A_3 (R×I)) and
    a mode-3 cherry tensor ℬ (Q×R×J; factors B_1 (Q×J), B_2 (R×J)), contracting the shared R:
    C(i,j,k,l) = Σ_r 𝒜(i,j,r) ℬ(k,r,l)  with the tensors materialised from their rank-one
    slices (Def. 2)."""
    I = A1.shape[1]
    J = B1.shape[1]
    Acal = cherry_tensor_elementwise(1, {0: A1, 2: A3}, I)   # P × I × R
    Bcal = cherry_tensor_elementwise(2, {0: B1, 1: B2}, J)   # Q × R × J
    return np.einsum("ijr,krl->ijkl", Acal, Bcal)


def remark1_matrix(A1, A3, B1, B2):
    """C = diag(vec(A_3ᵀB_2)) (B_1 ⊗ A_1)ᵀ, rows (j,l) j-fastest, cols (i,k) i-fastest."""
    return vec(A3.T @ B2)[:, None] * np.kron(B1, A1).T


# ---- helpers to move between the flat layout and dict-of-matrices ----------------------

def factors_from_flat(Gflat, dims, ranks):
    N = len(dims)
    G = {}
    off = 0
    for k in range(N):
        for i in range(N):
            if i == k:
                continue
            R = int(ranks[k][i])
            G[(k, i)] = np.asarray(Gflat[off:off + R * dims[k]], dtype=np.float64).reshape(dims[k], R).T.copy()
            off += R * dims[k]
    return G


def factors_to_flat(G, dims):
    N = len(dims)
    out = []
    for k in range(N):
        for i in range(N):
            if i != k:
                out.append(np.asarray(G[(k, i)]).T.reshape(-1))
    return np.concatenate(out)
