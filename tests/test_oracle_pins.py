"""Pins of the float64 oracle (oracle/) to things other than itself (-m "not gpu").

Each test pins one part of the oracle to a value the paper prints, a closed form, a
textbook special case, brute force on tiny inputs (oracle/brute.py, an independent literal
statement of Eq. 5 / Prop. 1 / Eq. 8), or an invariant the paper proves (Lemma 2).
"""
import json
import os

import numpy as np
import pytest

from oracle import brute
from oracle import oracle as O
from synth import make_config, make_problem

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


def rand_problem(dims, R, seed=0, scale=1.0):
    rng = np.random.default_rng(seed)
    N = len(dims)
    if np.isscalar(R):
        ranks = np.full((N, N), R, dtype=np.int32)
    else:
        ranks = np.asarray(R, dtype=np.int32)
    np.fill_diagonal(ranks, 0)
    sh = O.Shape(dims, ranks)
    G = rng.standard_normal(O.num_params(sh)) * scale
    X = rng.standard_normal(sh.n)
    return sh, ranks, G, X


def tensor_from_flat(x, dims):
    return np.reshape(x, dims, order="F")


# ---------------------------------------------------------------- model t = iFCTN(G) ---

@pytest.mark.parametrize("dims,R", [((3, 4, 2), [[0, 2, 3], [2, 0, 1], [3, 1, 0]]),
                                    ((2, 3, 2, 2), 2), ((2, 2, 2, 2, 2), [[0, 2, 1, 2, 1],
                                                                           [2, 0, 2, 1, 1],
                                                                           [1, 2, 0, 2, 2],
                                                                           [2, 1, 2, 0, 1],
                                                                           [1, 1, 2, 1, 0]])])
def test_model_matches_eq5_nested_sum(dims, R):
    """Closed form Π_{p<q} H_{p,q} == literal Eq. 5 nested sum."""
    sh, ranks, G, _ = rand_problem(dims, R, seed=1)
    t = O.model(sh, G)
    Gd = brute.factors_from_flat(G, dims, ranks)
    T = brute.eq5_tensor(Gd, dims, ranks)
    np.testing.assert_allclose(t, brute.vec(T), rtol=0, atol=1e-12 * max(1, np.abs(T).max()))


def test_model_all_ones_closed_form():
    """All-ones factors: every H entry equals R_{p,q}, so t ≡ Π_{p<q} R_{p,q}."""
    dims = (3, 5, 2, 4)
    R = [[0, 2, 3, 1], [2, 0, 2, 4], [3, 2, 0, 2], [1, 4, 2, 0]]
    sh = O.Shape(dims, R)
    t = O.model(sh, np.ones(O.num_params(sh)))
    assert np.all(t == 2 * 3 * 1 * 2 * 4 * 2)


def test_model_multilinear_and_model_at():
    """Scaling G_{1,2} by c scales t by c (multilinearity of Eq. 5); model_at == model."""
    sh, ranks, G, _ = rand_problem((4, 3, 5), 2, seed=2)
    t = O.model(sh, G)
    G2 = G.copy()
    off = O.factor_offset(sh, 0, 1)
    G2[off:off + 2 * 4] *= 3.0
    np.testing.assert_allclose(O.model(sh, G2), 3.0 * t, rtol=1e-14)
    idx = (3, 1, 4)
    assert abs(O.model_at(sh, G, idx) - t[3 + 4 * (1 + 3 * 4)]) <= 1e-14 * abs(t).max()


def test_model_mode_permutation_consistency():
    """Permuting modes (and relabelling factors/ranks) permutes the reconstruction."""
    dims = (3, 4, 2)
    sh, ranks, G, _ = rand_problem(dims, [[0, 2, 3], [2, 0, 1], [3, 1, 0]], seed=3)
    T = tensor_from_flat(O.model(sh, G), dims)
    perm = (2, 0, 1)
    Gd = brute.factors_from_flat(G, dims, ranks)
    dims_p = tuple(dims[m] for m in perm)
    ranks_p = ranks[np.ix_(perm, perm)]
    Gp = {(a, b): Gd[(perm[a], perm[b])] for a in range(3) for b in range(3) if a != b}
    shp = O.Shape(dims_p, ranks_p)
    Tp = tensor_from_flat(O.model(shp, brute.factors_to_flat(Gp, dims_p)), dims_p)
    np.testing.assert_allclose(Tp, np.transpose(T, perm), rtol=1e-13, atol=1e-13)


def test_kr_gram_identity():
    """(A⊙B)ᵀ(A⊙B) = AᵀA ∘ BᵀB (textbook; why the pairwise form exists)."""
    rng = np.random.default_rng(4)
    A, B = rng.standard_normal((5, 3)), rng.standard_normal((4, 3))
    C = brute.khatri_rao(A, B)
    np.testing.assert_allclose(C.T @ C, (A.T @ A) * (B.T @ B), rtol=1e-13)


# ------------------------------------------------------- cherry tensors, Prop. 1, Remark 1 -

def test_cherry_tensor_eq2_rank_one_slices():
    """Eq. 2 (KR chain + fold) == the rank-one-slice statement."""
    rng = np.random.default_rng(5)
    Ik = 3
    mats = {0: rng.standard_normal((2, Ik)), 2: rng.standard_normal((3, Ik)),
            3: rng.standard_normal((2, Ik))}
    a = brute.cherry_tensor(1, mats, Ik)
    b = brute.cherry_tensor_elementwise(1, mats, Ik)
    np.testing.assert_allclose(a, b, rtol=0, atol=1e-15)
    for m in range(Ik):  # every mode-k slice has rank one
        s = np.linalg.svd(b[:, m, :, :].reshape(2, -1), compute_uv=False)
        assert s[1] <= 1e-12 * s[0]


@pytest.mark.parametrize("dims,R", [((3, 4, 2), 2), ((2, 3, 2, 3), [[0, 2, 1, 2], [2, 0, 2, 1],
                                                                     [1, 2, 0, 2], [2, 1, 2, 0]])])
def test_prop1_unfolding_identity(dims, R):
    """(X_(k))ᵀ = Z_k (𝒢_(k))ᵀ for every k (Prop. 1 / Eq. 7), X from Eq. 5."""
    sh, ranks, G, _ = rand_problem(dims, R, seed=6)
    Gd = brute.factors_from_flat(G, dims, ranks)
    X = brute.eq5_tensor(Gd, dims, ranks)
    for k in range(len(dims)):
        lhs = brute.unfold(X, k).T
        rhs = brute.build_Z(Gd, dims, k) @ brute.kr_chain_T(Gd, dims, k)
        np.testing.assert_allclose(lhs, rhs, rtol=0, atol=1e-12 * np.abs(X).max())


def test_remark1_matricised_cherry_product():
    """Remark 1: C = diag(vec(A_3ᵀB_2))(B_1⊗A_1)ᵀ, entrywise."""
    rng = np.random.default_rng(7)
    P, I, R, Q, J = 2, 3, 2, 3, 2
    A1, A3 = rng.standard_normal((P, I)), rng.standard_normal((R, I))
    B1, B2 = rng.standard_normal((Q, J)), rng.standard_normal((R, J))
    C = brute.remark1_elementwise(A1, A3, B1, B2)           # (P, I, Q, J)
    M = brute.remark1_matrix(A1, A3, B1, B2)                # (IJ, PQ)
    for i in range(P):
        for j in range(I):
            for k in range(Q):
                for l in range(J):
                    assert abs(C[i, j, k, l] - M[j + I * l, i + P * k]) < 1e-13
                    assert abs(C[i, j, k, l] - A1[i, j] * B1[k, l] * (A3.T @ B2)[j, l]) < 1e-13


# ---------------------------------------------------- a2: coefficient contraction (β, ω) ---

CONTRACT_CASES = [((3, 4, 2), 2), ((2, 3, 2, 3), 2), ((2, 2, 3, 2, 2), [[0, 2, 1, 2, 1],
                                                                         [2, 0, 2, 1, 1],
                                                                         [1, 2, 0, 2, 2],
                                                                         [2, 1, 2, 0, 1],
                                                                         [1, 1, 2, 1, 0]])]


@pytest.mark.parametrize("dims,R", CONTRACT_CASES)
def test_block_contraction_vs_dense_Zk(dims, R):
    """A_jᵀA_j = G_{i,k} diag(ω(:,j)) G_{i,k}ᵀ and A_jᵀx_j = G_{i,k} β(:,j) with A_j = Z_k L_j
    materialised from Prop. 1 (dense, brute tier)."""
    sh, ranks, G, X = rand_problem(dims, R, seed=8)
    Gd = brute.factors_from_flat(G, dims, ranks)
    Xt = tensor_from_flat(X, dims)
    N = len(dims)
    for k in range(N):
        for i in range(N):
            if i == k:
                continue
            beta, omega = O.block_contract(sh, G, X, k, i)
            Gik = Gd[(i, k)]
            for j in range(dims[k]):
                _, A, x = brute.dense_column_update(Gd, dims, Xt, k, i, j, 0.1)
                np.testing.assert_allclose(A.T @ A, Gik @ np.diag(omega[:, j]) @ Gik.T,
                                           rtol=1e-11, atol=1e-11)
                np.testing.assert_allclose(A.T @ x, Gik @ beta[:, j], rtol=1e-11, atol=1e-11)


def test_block_contraction_N3_is_a_gemm():
    """Special case: N=3, block (1,2): ω = (H_23∘H_23)(H_13∘H_13)ᵀ (plain BLAS matmul),
    β(a,j) = Σ_m H_13(j,m) H_23(a,m) X(j,a,m) (einsum). H from numpy G ᵀG."""
    dims = (5, 6, 4)
    sh, ranks, G, X = rand_problem(dims, [[0, 2, 3], [2, 0, 2], [3, 2, 0]], seed=9)
    Gd = brute.factors_from_flat(G, dims, ranks)
    H13 = Gd[(0, 2)].T @ Gd[(2, 0)]
    H23 = Gd[(1, 2)].T @ Gd[(2, 1)]
    beta, omega = O.block_contract(sh, G, X, 0, 1)
    np.testing.assert_allclose(omega, (H23 * H23) @ (H13 * H13).T, rtol=1e-13)
    Xt = tensor_from_flat(X, dims)
    np.testing.assert_allclose(beta, np.einsum("jm,am,jam->aj", H13, H23, Xt), rtol=1e-12,
                               atol=1e-12)


def test_block_contraction_all_ones():
    """All-ones factors: ω ≡ (Π_{pairs≠{k,i}} R)² Π_{m≠k,i} I_m; β = M·(marginal sums of X)."""
    dims = (3, 4, 2, 5)
    R = [[0, 2, 3, 1], [2, 0, 2, 4], [3, 2, 0, 2], [1, 4, 2, 0]]
    sh = O.Shape(dims, R)
    rng = np.random.default_rng(10)
    X = rng.standard_normal(sh.n)
    G = np.ones(O.num_params(sh))
    Xt = tensor_from_flat(X, dims)
    k, i = 2, 0
    M = 2 * 1 * 2 * 4 * 2          # all pair ranks except R_{1,3} = 3
    beta, omega = O.block_contract(sh, G, X, k, i)
    assert np.all(omega == M * M * dims[1] * dims[3])
    marg = Xt.sum(axis=(1, 3))     # (I_1, I_3) indexed [a=i_1, j=i_3]
    np.testing.assert_allclose(beta, M * marg, rtol=1e-13)


def test_block_contract_at_matches_full():
    sh, ranks, G, X = rand_problem((4, 3, 5, 2), 2, seed=11)
    beta, omega = O.block_contract(sh, G, X.astype(np.float32), 3, 1)
    for (a, j) in [(0, 0), (2, 1), (1, 1)]:
        b, w = O.block_contract_at(sh, G, X.astype(np.float32), 3, 1, a, j)
        assert abs(b - beta[a, j]) < 1e-12 * max(1, abs(b))
        assert abs(w - omega[a, j]) < 1e-12 * max(1, abs(w))


# -------------------------------------------------------------- a3/a4: column solve ---

@pytest.mark.parametrize("dims,R", CONTRACT_CASES[:2])
def test_column_update_vs_dense_ridge_ls(dims, R):
    """Eq. 8 column (oracle normal equations + Cholesky) == dense ridge LS on A_j (lstsq)."""
    sh, ranks, G, X = rand_problem(dims, R, seed=12)
    Gd = brute.factors_from_flat(G, dims, ranks)
    Xt = tensor_from_flat(X, dims)
    for (k, i) in [(0, 1), (1, 0), (2, 1), (len(dims) - 1, 0)]:
        beta, omega = O.block_contract(sh, G, X, k, i)
        for j in range(dims[k]):
            st, c = O.column_solve(Gd[(i, k)], beta[:, j], omega[:, j], Gd[(k, i)][:, j], 0.1)
            assert st == 0
            c_ref, _, _ = brute.dense_column_update(Gd, dims, Xt, k, i, j, 0.1)
            np.testing.assert_allclose(c, c_ref, rtol=1e-8, atol=1e-8)


def test_column_update_large_rho_returns_c_old():
    """ρ → ∞: the prox term dominates and c → c_old (O(1/ρ))."""
    sh, ranks, G, X = rand_problem((3, 4, 2), 2, seed=13)
    Gd = brute.factors_from_flat(G, (3, 4, 2), ranks)
    beta, omega = O.block_contract(sh, G, X, 0, 2)
    g = Gd[(2, 0)]
    for j in range(3):
        c_old = Gd[(0, 2)][:, j]
        st, c = O.column_solve(g, beta[:, j], omega[:, j], c_old, 1e8)
        # c − c_old = (A+ρI)⁻¹(b − A c_old) ⇒ ‖c − c_old‖ ≤ ‖b − A c_old‖/ρ
        A = g @ np.diag(omega[:, j]) @ g.T
        bound = np.linalg.norm(g @ beta[:, j] - A @ c_old) / 1e8
        assert np.linalg.norm(c - c_old) <= bound * (1 + 1e-6) + 1e-15
        assert bound < 1e-4


def test_block_update_first_order_condition():
    """At the block minimiser: ∇_{G_{k,i}} f + ρ (G_new − G_old) = 0, by central
    finite differences of f computed with the brute Eq. 5 tensor."""
    dims = (3, 2, 3)
    sh, ranks, G, X = rand_problem(dims, 2, seed=14)
    rho = 0.3
    k, i = 1, 2
    Gold = G.copy()
    Gnew = G.copy()
    st, _ = O.block_update(sh, Gnew, X, k, i, rho)
    assert st == 0
    Xt = tensor_from_flat(X, dims)

    def f(Gflat):
        T = brute.eq5_tensor(brute.factors_from_flat(Gflat, dims, ranks), dims, ranks)
        return 0.5 * np.sum((Xt - T) ** 2)

    off = O.factor_offset(sh, k, i)
    h = 1e-6
    for e in range(off, off + 2 * dims[k]):
        gp, gm = Gnew.copy(), Gnew.copy()
        gp[e] += h
        gm[e] -= h
        grad = (f(gp) - f(gm)) / (2 * h)
        assert abs(grad + rho * (Gnew[e] - Gold[e])) < 1e-5 * max(1.0, abs(grad))


def test_block_update_matches_dense_block():
    dims = (3, 4, 2, 2)
    sh, ranks, G, X = rand_problem(dims, 2, seed=15)
    Gd = brute.factors_from_flat(G, dims, ranks)
    for (k, i) in [(0, 3), (2, 1)]:
        Gn = G.copy()
        O.block_update(sh, Gn, X, k, i, 0.1)
        ref = brute.dense_block_update(Gd, dims, tensor_from_flat(X, dims), k, i, 0.1)
        np.testing.assert_allclose(O.factor(sh, Gn, k, i), ref, rtol=1e-8, atol=1e-9)


# -------------------------------------------------------------------- a5: X update ---

def test_refill_scalar_minimiser_golden():
    """Eq. 9 as the prox minimiser: t=0.3, x=0.9, ρ=0.1 → 0.354545… (golden fixture)."""
    g = GOLDEN["x_update_scalar_example"]
    sh = O.Shape((1, 1), [[0, 1], [1, 0]])
    G = np.array([g["t"], 1.0])   # G_{1,2} = [t], G_{2,1} = [1] → t = 0.3
    X = np.array([g["x_old"]])
    dx2, x2, f = O.refill(sh, G, X, np.zeros(1, np.uint8), g["rho"])
    assert abs(X[0] - g["x_new"]) < 1e-15
    assert abs(x2 - 0.81) < 1e-15 and abs(dx2 - (g["x_new"] - 0.9) ** 2) < 1e-15
    assert abs(f - 0.5 * (g["x_new"] - 0.3) ** 2) < 1e-15


def test_refill_limits_and_feasibility():
    sh, ranks, G, X = rand_problem((4, 3, 5), 2, seed=16)
    t = O.model(sh, G)
    mask = (np.arange(sh.n) % 3 == 0).astype(np.uint8)
    X0 = X.copy()
    X1 = X.copy()
    O.refill(sh, G, X1, mask, 1e-300)          # ρ → 0: the model on Ω^c
    np.testing.assert_allclose(X1[mask == 0], t[mask == 0], rtol=1e-14)
    assert np.array_equal(X1[mask == 1].view(np.uint64), X0[mask == 1].view(np.uint64))
    X2 = t.copy()
    O.refill(sh, G, X2, mask, 0.1)             # t == X: fixed point
    np.testing.assert_allclose(X2, t, rtol=1e-15)


# ------------------------------------------------------------------ whole sweep ---

def test_sweep_matches_dense_sweep():
    """Oracle sweep (factorised Eq. 8) == Algorithm 1 built from dense Prop. 1 ridge solves."""
    dims = (3, 4, 3)
    sh, ranks, G, X = rand_problem(dims, 2, seed=17)
    mask = (np.random.default_rng(17).random(sh.n) < 0.5).astype(np.uint8)
    Gd = brute.factors_from_flat(G, dims, ranks)
    Gref, Xref = brute.dense_sweep(Gd, dims, tensor_from_flat(X, dims), mask.reshape(dims, order="F").astype(bool), 0.1)
    Gc, Xc = G.copy(), X.copy()
    F = O.objective(sh, Gc, Xc)
    st, F1, row = O.sweep(sh, Gc, Xc, mask, 0.1, F)
    assert st == 0
    np.testing.assert_allclose(Gc, brute.factors_to_flat(Gref, dims), rtol=1e-8, atol=1e-9)
    np.testing.assert_allclose(Xc, brute.vec(Xref), rtol=1e-8, atol=1e-9)


@pytest.mark.parametrize("name", ["C1", "C2s", "C3s", "C4s", "C5s"])
def test_lemma2_monotone_and_feasible(name):
    """Lemma 2 sufficient decrease every sweep (asserted inside orc_sweep), F monotone, and
    X[Ω] == O[Ω] bit for bit after every sweep."""
    p = make_config(name)
    sh = O.Shape(p.dims, p.ranks)
    G = p.G0.astype(np.float64)
    X = O.init_x(p.observed, p.mask)
    F = O.objective(sh, G, X)
    Fs = [F]
    obs = p.mask.astype(bool)
    for s in range(6):
        st, F, row = O.sweep(sh, G, X, p.mask, p.rho, F, True)
        assert st == 0, f"Lemma 2 violated at sweep {s}"
        Fs.append(F)
        assert np.array_equal(X[obs], p.observed[obs].astype(np.float64))
    assert all(Fs[s + 1] <= Fs[s] for s in range(len(Fs) - 1))


def test_stationary_at_exact_optimum():
    """Fully observed exact model initialised at the truth: one sweep changes nothing."""
    dims = (4, 5, 3)
    sh, ranks, G, _ = rand_problem(dims, 2, seed=18)
    X = O.model(sh, G)
    mask = np.ones(sh.n, np.uint8)
    G1, X1 = G.copy(), X.copy()
    st, F, row = O.sweep(sh, G1, X1, mask, 0.1, 0.0, False)
    assert np.abs(G1 - G).max() < 1e-10 and np.abs(X1 - X).max() < 1e-10


def test_order2_reduces_to_eckart_young():
    """N=2, full mask: PAM is proximal ALS for a rank-R matrix factorisation; its limit error
    is the Eckart–Young value √(Σ_{r>R} σ_r²) of the SVD (textbook)."""
    rng = np.random.default_rng(19)
    I1, I2, R = 12, 10, 2
    M = rng.standard_normal((I1, I2))
    sh = O.Shape((I1, I2), [[0, R], [R, 0]])
    G = rng.standard_normal(O.num_params(sh))
    X = M.reshape(-1, order="F").copy()
    r, trace = O.solve(sh, G, X, np.ones(I1 * I2, np.uint8), 1e-3, 3000, 0.0, True)
    assert r == 3000
    s = np.linalg.svd(M, compute_uv=False)
    ey = np.sqrt(np.sum(s[R:] ** 2))
    err = np.sqrt(2 * trace[-1, 1])
    assert abs(err - ey) < 1e-7 * ey


def test_serial_equals_threaded():
    p = make_config("C2s")
    sh = O.Shape(p.dims, p.ranks)
    out = []
    for t in (1, 4):
        O.set_threads(t)
        G = p.G0.astype(np.float64)
        X = O.init_x(p.observed, p.mask)
        F = O.objective(sh, G, X)
        for _ in range(2):
            st, F, _ = O.sweep(sh, G, X, p.mask, p.rho, F, True)
        out.append((G, X))
    O.set_threads(1)
    np.testing.assert_allclose(out[0][0], out[1][0], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(out[0][1], out[1][1], rtol=1e-12, atol=1e-12)


def test_exact_recovery_C1_recipe():
    """C1 recipe (20³, ranks 2, 30% observed, N(0,1) init) run long: the truth is recovered
    to rounding level (SURVEY §8(c) whole-sweep pin (v)). The problem is nonconvex: with
    this recipe seeds 1 and 4 of 0..4 reach exact recovery, the others stall at RSE ≈ 1
    (recorded in DESIGN.md); any dropped term or wrong index breaks exact recovery."""
    p = make_config("C1", seed=4)
    sh = O.Shape(p.dims, p.ranks)
    G = p.G0.astype(np.float64)
    X = O.init_x(p.observed, p.mask)
    r, trace = O.solve(sh, G, X, p.mask, p.rho, 300, 0.0, True)
    assert r == 300
    assert O.rse(p.truth, X) < 1e-10


# ------------------------------------------------- init and RSE (hand values) ---

def test_init_x_zeroes_unobserved_entries():
    """X⁽⁰⁾ = P_Ω(O) (Alg. 1 initialisation; reading R7): entries off Ω are 0 even
    when O carries (nonzero) values there; entries on Ω are O bit for bit (f64 and f32)."""
    O64 = np.array([1.5, -2.0, 3.25, 7.0, -0.125], dtype=np.float64)
    m = np.array([1, 0, 1, 0, 1], dtype=np.uint8)
    X = O.init_x(O64, m)
    assert X.tolist() == [1.5, 0.0, 3.25, 0.0, -0.125]
    O32 = np.array([0.1, 9.0, -0.3], dtype=np.float32)
    X = O.init_x(O32, np.array([0, 1, 1], np.uint8))
    assert X[0] == 0.0 and X[1] == 9.0 and X[2] == float(np.float32(-0.3))


def test_rse_denominator_is_the_truth_norm():
    """RSE = ‖T − X‖_F / ‖T‖_F (reading R10).  T = [3, 4], X = [3, 0]: ‖T − X‖ = 4,
    ‖T‖ = 5 → 0.8; the paper's printed ‖X‖ denominator would give 4/3 and a squared or
    unsquared-numerator slip 16/25 or 16/5 — all separated by this hand value."""
    T = np.array([3.0, 4.0])
    X = np.array([3.0, 0.0])
    assert O.rse(T, X) == 0.8
    # exact recovery and the all-zero estimate
    assert O.rse(T, T.copy()) == 0.0
    assert O.rse(T, np.zeros(2)) == 1.0


# ---------------------------------------------------------- paper-printed counts ---

def test_storage_counts_golden():
    """iFCTN 4344, FCTN 8688, Tucker 4856, TT 23319 on 256×256×31."""
    g = GOLDEN["storage_cost_256x256x31"]
    dims = g["dims"]
    sh = O.Shape(dims, np.full((3, 3), g["ifctn_ranks_all"]))
    assert O.num_params(sh) == g["ifctn_params"]
    assert make_config("C2").G0.size == g["ifctn_params"]
    r = g["fctn_ranks_all"]
    assert sum(d * r * r for d in dims) == g["fctn_params"]          # Σ_k I_k Π_{i≠k} R
    tr = g["tucker_ranks"]
    assert int(np.prod(tr)) + sum(d * t for d, t in zip(dims, tr)) == g["tucker_params"]
    tt = [1] + g["tt_ranks"] + [1]
    assert sum(tt[m] * dims[m] * tt[m + 1] for m in range(3)) == g["tt_params"]
