"""Pin the oracle restatement (oracle/gnp_oracle.c) before trusting it.

(1) bit-for-bit against the golden vectors the unmodified reference produced
    (tests/golden/make_golden.py), (2) the reference's own known-answer tests
    restated (tests/test_gnn.cpp, tests/test_krylov.cpp, tests/test_sparse_core.cpp),
(3) live against oracle/_ref where it is built.
"""
import math

import numpy as np
import pytest
from conftest import csr_of, f32, golden

from oracle import Csr


def csr_np(n, triplets):
    r, c, v = zip(*triplets) if triplets else ((), (), ())
    return np.array(r, np.int64), np.array(c, np.int64), np.array(v, np.float64), n


# ------------------------------------------------------------------ golden
def test_nonsym1138_gamma_hash(oc):
    g = golden("nonsym1138.npz")
    a = csr_of("a", g)
    assert a.n == 1138 and a.nnz == 7966
    assert oc.gershgorin_gamma(a) == float(g["gamma"])
    assert oc.csr_hash(a) == int(g["hash"])
    assert oc.csr_hash(oc.prescale(a, float(g["gamma"]))) == int(g["ahat_hash"])


def test_c1_matrix_params_apply_bitwise(oc):
    g = golden("c1.npz")
    a = oc.gen_convection_diffusion(64, 0.0)
    assert a.nnz == 20224
    assert oc.csr_hash(a) == int(g["hash"])
    assert oc.gershgorin_gamma(a) == float(g["gamma"]) == 8.0
    ah = oc.prescale(a, 8.0)
    assert oc.csr_hash(ah) == int(g["ahat_hash"])
    p = oc.init_params(16, 32, 8, 0)
    assert len(p) == 5265
    assert np.array_equal(p, g["params"])
    assert np.array_equal(oc.gaussian_vector(1, a.n), g["b"])
    out = oc.gnn_apply(ah.rounded_f32(), (16, 32, 8), f32(p), g["b"])
    assert np.array_equal(out, g["out"])


def test_c1_gmres_history_bitwise(oc):
    g = golden("c1.npz")
    ah = oc.prescale(oc.gen_convection_diffusion(64, 0.0), 8.0)
    s = oc.fgmres(ah, g["b"], maxiters=100, restart=10)
    gg = golden("c1_gmres.npz")
    assert s["status"] == str(gg["status"])
    assert np.array_equal(np.array([h[:2] for h in s["history"]]), gg["hist"])
    assert np.array_equal(s["x"], gg["x"])


def test_small_forward_backward_bitwise(oc):
    g = golden("small_fwd_bwd.npz")
    a = csr_of("a", g)
    out, grads = oc.gnn_forward_backward(a, (3, 4, 2), g["params"], g["b"], g["gout"])
    assert np.array_equal(out, g["out"])
    assert np.array_equal(grads, g["grads"])


def test_train_step_bitwise(oc):
    g = golden("train_step.npz")
    a = csr_of("a", g)
    x, b = oc.gaussian_batch(a, 3, 0, 4)
    assert np.array_equal(x, g["x"]) and np.array_equal(b, g["b"])
    loss, grads, out = oc.batch_loss_grads(a, (4, 8, 2), g["params"], x, b, 4, want_out=True)
    assert loss == float(g["loss"])
    assert np.array_equal(grads, g["grads"])
    assert np.array_equal(out, g["out"])
    z = np.zeros_like(grads)
    p, m1, m2, t = oc.adam_step((4, 8, 2), g["params"], grads, z, z, 0, 1e-3)
    assert t == 1
    assert np.array_equal(p, g["p_after"]) and np.array_equal(m1, g["m1"]) and np.array_equal(m2, g["m2"])


def test_trained_preconditioner_fgmres_history(oc):
    g = golden("trained_conv5.npz")
    a = oc.gen_convection_diffusion(5, 0.2)
    ah = oc.prescale(a, oc.gershgorin_gamma(a))
    b = oc.spmv(ah, np.ones(ah.n))
    s = oc.fgmres(ah, b, kind=1, dims=(4, 8, 2), params=g["params"], maxiters=50)
    assert s["status"] == str(g["status"]) == "converged"
    assert np.array_equal(np.array([h[:2] for h in s["history"]]), g["hist"])
    assert s["history"][-1][0] == 49  # converges at 49 in f64


# ------------------------------------------------------------------ reference KATs restated
def test_tiny_network_hand_computed(oc):
    # tests/test_gnn.cpp:135-162
    a = oc.csr_from_triplets(2, [0, 0, 1], [0, 1, 1], [0.5, 0.25, 0.5])
    p = np.array([0.3, 0.1, 1.2, 0.05, 0.7, 0.4, 0.9, 0.02, 1.1, 0.03])
    b = np.array([1.0, 2.0])
    tau = math.sqrt(5.0)
    s = math.sqrt(2.0) / tau
    relu = lambda x: max(x, 0.0)  # noqa: E731
    v = [s * 1.0, s * 2.0]
    x1 = [relu(vi * 0.3 + 0.1) * 1.2 + 0.05 for vi in v]
    ax = [0.5 * x1[0] + 0.25 * x1[1], 0.5 * x1[1]]
    conv = [relu(x1[i] * 0.7 + ax[i] * 0.4) for i in range(2)]
    want = [(relu(c * 0.9 + 0.02) * 1.1 + 0.03) * (tau / math.sqrt(2.0)) for c in conv]
    out = oc.gnn_apply(a, (1, 1, 1), p, b)
    for i in range(2):
        assert abs(out[i] - want[i]) <= 1e-14 * abs(want[i])


def test_zero_input_and_zero_head(oc):
    # tests/test_gnn.cpp:117-133
    eye = oc.csr_from_triplets(5, range(5), range(5), [1.0] * 5)
    p = oc.init_params(4, 4, 2, 1)
    assert np.all(oc.gnn_apply(eye, (4, 4, 2), p, np.zeros(5)) == 0.0)
    p2 = p.copy()
    p2[-5:] = 0.0  # dec2 (4) + dec2_bias
    b = oc.gaussian_vector(3, 5)
    assert np.all(oc.gnn_apply(eye, (4, 4, 2), p2, b) == 0.0)


def test_positive_homogeneity(oc):
    # tests/test_gnn.cpp:164-178
    a = oc.gen_convection_diffusion(4, 0.3)
    p = oc.init_params(4, 6, 3, 8)
    b = oc.gaussian_vector(9, a.n)
    base = oc.gnn_apply(a, (4, 6, 3), p, b)
    for alpha in (0.5, 10.0, 1e6):
        out = oc.gnn_apply(a, (4, 6, 3), p, alpha * b)
        assert np.all(np.abs(out - alpha * base) <= 1e-12 * alpha * (1 + np.abs(base)))


def test_backward_matches_finite_differences(oc):
    # tests/test_gnn.cpp:180-220 (kink-aware central differences)
    g = golden("small_fwd_bwd.npz")
    a = csr_of("a", g)
    a = Csr(a.n, a.row_ptr, a.col_idx, a.values)
    n = 40  # keep it small: leading 40x40 block of the fixture matrix
    rp = np.minimum(a.row_ptr[: n + 1], a.row_ptr[n])
    keep = [k for k in range(int(rp[-1])) if a.col_idx[k] < n]
    rows = np.repeat(np.arange(n), np.diff(a.row_ptr[: n + 1]))
    r = rows[keep] if len(keep) else []
    sm = oc.csr_from_triplets(n, r, a.col_idx[keep], a.values[keep])
    dims = (3, 4, 2)
    p = oc.init_params(*dims, 4)
    b = oc.gaussian_vector(12, n)
    gv = oc.gaussian_vector(13, n)
    out, grads = oc.gnn_forward_backward(sm, dims, p, b, gv)
    f0 = float(out @ gv)
    h = 1e-6
    checked = skipped = 0
    for k in range(len(p)):
        q = p.copy()
        q[k] += h
        fp = float(oc.gnn_apply(sm, dims, q, b) @ gv)
        q[k] -= 2 * h
        fm = float(oc.gnn_apply(sm, dims, q, b) @ gv)
        fwd, bwd = (fp - f0) / h, (f0 - fm) / h
        if abs(fwd - bwd) > 1e-3 * max(1.0, abs(fwd), abs(bwd)):
            skipped += 1
            continue
        fd = (fp - fm) / (2 * h)
        assert abs(fd - grads[k]) / max(1.0, abs(fd), abs(grads[k])) <= 1e-5
        checked += 1
    assert skipped <= 8 and checked >= len(p) - 8


def test_l1_loss_hand_examples(oc):
    # tests/test_gnn.cpp:242-284
    eye = oc.csr_from_triplets(2, [0, 1], [0, 1], [1.0, 1.0])
    loss, g = oc.l1_residual_loss(eye, np.array([1.0, 0.0]), np.zeros(2), 1)
    assert loss == 1.0 and g[0] == 1.0 and g[1] == 0.0
    out = np.array([3.0, 0.0, 0.0, -2.0])  # col-major 2x2
    loss, g = oc.l1_residual_loss(eye, out, np.zeros(4), 2)
    assert abs(loss - 2.5) <= 1e-15 and g[0] == 0.5 and g[3] == -0.5
    a = oc.csr_from_triplets(2, [0, 0, 1], [0, 1, 1], [2.0, -3.0, 4.0])
    loss, g = oc.l1_residual_loss(a, np.array([1.0, 0.0]), np.zeros(2), 1)
    assert loss == 2.0 and g[0] == 2.0 and g[1] == -3.0


def test_adam_closed_forms(oc):
    # tests/test_gnn.cpp:286-315
    p = oc.init_params(3, 4, 2, 21)
    z = np.zeros_like(p)
    q, m1, m2, t = p, z, z, 0
    for _ in range(3):
        q, m1, m2, t = oc.adam_step((3, 4, 2), q, z, m1, m2, t, 1e-3)
    assert np.array_equal(q, p) and t == 3
    gr = oc.gaussian_vector(22, len(p)) * 10.0
    q, *_ = oc.adam_step((3, 4, 2), p, gr, z, z, 0, 1e-3)
    want = p - 1e-3 * gr / (np.abs(gr) + 1e-8)
    assert np.all(np.abs(q - want) <= 1e-15 + 1e-12 * np.abs(want))


def test_lstsq_hand_values(oc):
    # tests/test_krylov.cpp:118-149
    y, tr, s = oc.hessenberg_lstsq(np.array([1.0, 0.0]), 1, 3.0)
    assert abs(y[0] - 3.0) < 1e-12 and abs(tr) < 1e-12 and not s
    y, tr, s = oc.hessenberg_lstsq(np.array([1.0, 1.0]), 1, 1.0)
    assert abs(y[0] - 0.5) < 1e-14 and abs(tr - 1 / math.sqrt(2)) < 1e-14


def test_fgmres_iteration_pins(oc):
    # tests/test_krylov.cpp:151-171, 198-219
    rng = np.random.default_rng(21)
    m = rng.uniform(-1, 1, (8, 8))
    np.fill_diagonal(m, 0)
    np.fill_diagonal(m, 2 * (np.abs(m).sum(1) + 0.5))
    r, c = np.nonzero(m)
    a = oc.csr_from_triplets(8, r, c, m[r, c])
    b = oc.gaussian_vector(21, 8)
    inv = np.linalg.inv(m)
    s = oc.fgmres(a, b, kind=2, params=inv.flatten(order="F"))
    assert s["status"] == "converged" and s["history"][-1][0] == 1
    d = oc.csr_from_triplets(2, [0, 1], [0, 1], [1.0, 2.0])
    s = oc.fgmres(d, np.ones(2))
    assert s["status"] == "converged" and s["history"][-1][0] == 2
    cd = oc.prescale(oc.gen_convection_diffusion(6, 0.4), 1.0)
    bb = oc.spmv(cd, np.ones(cd.n))
    plain = oc.fgmres(cd, bb)
    ident = oc.fgmres(cd, bb, kind=3)
    assert [h[1] for h in plain["history"]] == [h[1] for h in ident["history"]]


# ------------------------------------------------------------------ live vs reference
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_restatement_equals_reference_live(oc, ref, seed):
    a = ref.gen_random_nonsymmetric(150 + 37 * seed, 5, 1.4, 100 + seed)
    assert np.array_equal(oc.csr_from_triplets(a.n, *_triplets(a)).values, a.values)
    ah = ref.prescale(a, ref.gershgorin_gamma(a))
    assert oc.gershgorin_gamma(a) == ref.gershgorin_gamma(a)
    assert oc.csr_hash(ah) == ref.csr_hash(ah)
    t1, t2 = oc.transpose(ah), ref.transpose(ah)
    assert np.array_equal(t1.row_ptr, t2.row_ptr) and np.array_equal(t1.col_idx, t2.col_idx)
    dims = (5, 7, 3)
    p = ref.init_params(*dims, seed)
    assert np.array_equal(p, oc.init_params(*dims, seed))
    b = ref.gaussian_vector(seed + 10, a.n)
    assert np.array_equal(oc.gnn_apply(ah, dims, p, b), ref.gnn_apply(ah, dims, p, b))
    x, bb = ref.gaussian_batch(ah, seed, 1, 3)
    assert np.array_equal(oc.gaussian_batch(ah, seed, 1, 3)[1], bb)
    l1, g1 = oc.batch_loss_grads(ah, dims, p, x, bb, 3)
    l2, g2 = ref.batch_loss_grads(ah, dims, p, x, bb, 3)
    assert l1 == l2 and np.array_equal(g1, g2)
    s1 = oc.fgmres(ah, b, kind=1, dims=dims, params=p, maxiters=25, restart=7)
    s2 = ref.fgmres(ah, b, kind=1, dims=dims, params=p, maxiters=25, restart=7)
    assert s1["status"] == s2["status"]
    assert [h[:2] for h in s1["history"]] == [h[:2] for h in s2["history"]]


def _triplets(a):
    rows = np.repeat(np.arange(a.n), np.diff(a.row_ptr))
    perm = np.random.default_rng(0).permutation(a.nnz)  # shuffled input order
    return rows[perm], a.col_idx[perm], a.values[perm]


# ------------------------------------------------------------------ spectral sampler
# src/sampler.cpp:10-83, src/svd.cpp:10-80; known-answer tests restate
# tests/test_sampler.cpp:47-226.
def _csr_diag(vals):
    n = len(vals)
    return Csr(n, np.arange(n + 1, dtype=np.int64), np.arange(n, dtype=np.int64), np.array(vals, np.float64))


def _in_range(vk, k, x):
    n = x.size
    V = vk[: n * k].reshape(k, n).T
    r = x - V @ (V.T @ x)
    return np.linalg.norm(r) <= 1e-10 * np.linalg.norm(x)


def test_sampler_identity_breaks_down_at_step_one(oc):
    s = oc.spectral_sampler(_csr_diag([1.0] * 4), 3, 0)  # test_sampler.cpp:69-75
    assert s["k"] == 1 and s["m_eff"] == 1
    assert abs(s["s"][0] - 1.0) <= 1e-12


def test_jacobi_svd_eigen_oracle(oc):
    # test_sampler.cpp:47-67: (HᵀH - s²I) v = 0 for the right singular vectors
    a = _csr_diag([1.0, 2.0, 3.0])
    v, h, k, _ = oc.arnoldi_cycle(a, oc.gaussian_vector(9, 3), 3)
    H = h.reshape(3, 4).T  # (m+1) x m col-major
    u, s, zv = oc.jacobi_svd(H.T.ravel(), 4, 3)
    Z = zv.reshape(3, 3).T
    hth = H.T @ H
    for q in range(3):
        lam = s[q] ** 2
        assert np.max(np.abs(hth @ Z[:, q] - lam * Z[:, q])) <= 1e-10 * (1 + lam)
    assert list(s) == sorted(s, reverse=True)


def test_sampler_matches_reference_bitwise(oc, ref):
    a = ref.gen_random_nonsymmetric(50, 6, 1.3, 13)  # test_sampler.cpp:77-110
    s1, s2 = oc.spectral_sampler(a, 40, 21), ref.spectral_sampler(a, 40, 21)
    assert (s1["k"], s1["m_eff"]) == (s2["k"], s2["m_eff"]) == (40, s2["m_eff"])
    for key in ("v", "zsv", "s"):
        assert np.array_equal(s1[key], s2[key]), key
    V = s1["v"].reshape(40, 50).T
    assert np.max(np.abs(V.T @ V - np.eye(40))) <= 1e-10
    Z = s1["zsv"].reshape(40, 40).T
    assert np.max(np.abs(Z.T @ Z - np.eye(40))) <= 1e-10
    # the SVD of a random tall matrix, bitwise
    g = np.random.default_rng(3).standard_normal((9, 7))
    r1, r2 = oc.jacobi_svd(g.T.ravel(), 9, 7), ref.jacobi_svd(g.T.ravel(), 9, 7)
    assert all(np.array_equal(p, q) for p, q in zip(r1, r2))


@pytest.mark.parametrize("skip", [0, 2])
def test_assemble_batch_matches_reference(oc, ref, skip):
    a = ref.gen_random_nonsymmetric(20, 4, 1.5, 2)  # test_sampler.cpp:182-216
    s = oc.spectral_sampler(a, 8, 1)
    x1, b1 = oc.assemble_batch(a, s, 42, skip, 16, 8)
    x2, b2 = ref.assemble_batch(a, 8, 1, 42, skip, 16, 8)
    assert np.array_equal(x1, x2) and np.array_equal(b1, b2)
    for k in range(16):
        assert np.array_equal(b1[k * 20:(k + 1) * 20], oc.spmv(a, x1[k * 20:(k + 1) * 20]))
    assert all(_in_range(s["v"], s["k"], x1[k * 20:(k + 1) * 20]) for k in range(8))
    assert not _in_range(s["v"], s["k"], x1[15 * 20:16 * 20])
    with pytest.raises(Exception):
        oc.assemble_batch(a, s, 42, 0, 0, 0)
    with pytest.raises(Exception):
        oc.assemble_batch(a, s, 42, 0, 2, 3)
    # spectral_count = 0 is the Gaussian batch
    assert np.array_equal(oc.assemble_batch(a, s, 5, 1, 3, 0)[0], oc.gaussian_batch(a, 5, 1, 3)[0])


def test_spectral_golden(oc):
    g = golden("spectral.npz")
    a = oc.prescale(oc.gen_convection_diffusion(16, 0.5), float(g["gamma"]))
    s = oc.spectral_sampler(a, int(g["m"]), int(g["seed"]))
    assert (s["k"], s["m_eff"]) == (int(g["k"]), int(g["m_eff"]))
    assert np.array_equal(s["s"], g["s"])
    x, b = oc.assemble_batch(a, s, int(g["batch_seed"]), 1, int(g["batch"]), int(g["spectral"]))
    assert np.array_equal(x, g["x"]) and np.array_equal(b, g["b"])


# ------------------------------------------- full-size parity support (r02)
# Content hashes of the BASELINE config matrices at their full sizes (n, nnz,
# FNV-1a of the CSR as src/csr.cpp:152-173), shared by the oracle's
# restatement of the generators and the product's gnpc_csr_generate.
FULL_SIZE = [
    ("c2_convdiff3d", 64, 10.0, 0.0, 0, 262144, 1810432),
    ("c3_varcoeff2d", 512, 2.0, 0.0, 2, 262144, 1308672),
    ("c4_powerlaw", 1 << 20, 2.2, 0.0, 4, 1048576, 17069302),
    ("c5_aniso9pt", 2048, 1e-3, 30.0, 0, 4194304, 37724164),
]


@pytest.mark.parametrize("kind,size,p0,p1,seed", [
    ("c2_convdiff3d", 9, 10.0, 0.0, 0), ("c3_varcoeff2d", 33, 2.0, 0.0, 2),
    ("c4_powerlaw", 4000, 2.2, 0.0, 4), ("c5_aniso9pt", 37, 1e-3, 30.0, 0)])
def test_config_generators_bitwise_small(oc, capi, kind, size, p0, p1, seed):
    a = oc.gen_named(kind, size, p0, p1, seed)
    rp, ci, v = capi.Csr.generate(kind, size, p0, p1, seed).arrays()
    assert np.array_equal(a.row_ptr, rp) and np.array_equal(a.col_idx, ci)
    assert np.array_equal(a.values, v)


@pytest.mark.parametrize("kind,size,p0,p1,seed,n,nnz", FULL_SIZE)
def test_config_generators_full_size_hash(oc, capi, kind, size, p0, p1, seed, n, nnz):
    a = oc.gen_named(kind, size, p0, p1, seed)
    g = capi.Csr.generate(kind, size, p0, p1, seed)
    assert (a.n, a.nnz) == (n, nnz) == g.info()
    assert oc.csr_hash(a) == g.hash()
    assert oc.gershgorin_gamma(a) == g.gamma()


@pytest.mark.parametrize("dims", [(16, 32, 8), (32, 32, 8), (5, 7, 3)])
def test_streaming_apply_bitwise(oc, dims):
    a = oc.gen_named("c4_powerlaw", 3000, 2.2, 0.0, 4)
    ah = oc.prescale(a, oc.gershgorin_gamma(a)).rounded_f32()
    p = f32(oc.init_params(*dims, 1))
    b = oc.gaussian_vector(2, ah.n)
    want = oc.gnn_apply(ah, dims, p, b)
    for t in (1, 3, 8):
        assert np.array_equal(oc.gnn_apply_mt(ah, dims, p, b, threads=t), want)
    assert np.all(oc.gnn_apply_mt(ah, dims, p, np.zeros(ah.n), threads=4) == 0.0)


def test_streaming_apply_equals_reference_live(oc, ref):
    a = oc.gen_named("c5_aniso9pt", 40, 1e-3, 30.0)
    ah = oc.prescale(a, oc.gershgorin_gamma(a)).rounded_f32()
    p = f32(oc.init_params(32, 32, 8, 0))
    b = oc.gaussian_vector(3, ah.n)
    assert np.array_equal(oc.gnn_apply_mt(ah, (32, 32, 8), p, b, threads=5),
                          ref.gnn_apply(ah, (32, 32, 8), p, b))


def test_parallel_batch_grads_bitwise(oc, ref):
    a = oc.gen_named("c3_varcoeff2d", 20, 2.0, 0.0, 2)
    ah = oc.prescale(a, oc.gershgorin_gamma(a)).rounded_f32()
    dims, B = (32, 32, 3), 6
    p = f32(oc.init_params(*dims, 0))
    x, b = oc.gaussian_batch(ah, 3, 0, B)
    l0, g0, o0 = oc.batch_loss_grads(ah, dims, p, x, b, B, want_out=True)
    for t in (1, 4):
        l1, g1, o1 = oc.batch_loss_grads_mt(ah, dims, p, x, b, B, want_out=True, threads=t)
        assert l1 == l0 and np.array_equal(g1, g0) and np.array_equal(o1, o0)
    lr, gr = ref.batch_loss_grads(ah, dims, p, x, b, B)
    assert lr == l0 and np.array_equal(gr, g0)


def test_fgmres_threaded_and_callback_operators_bitwise(oc):
    a = oc.prescale(oc.gen_convection_diffusion(16, 0.3), 8.0)
    dims = (4, 8, 2)
    p = oc.init_params(*dims, 0)
    b = oc.gaussian_vector(1, a.n)
    r1 = oc.fgmres(a, b, kind=1, dims=dims, params=p, maxiters=30, restart=10)
    r2 = oc.fgmres(a, b, kind=lambda v: oc.gnn_apply(a, dims, p, v), maxiters=30, restart=10)
    oc.set_threads(4)
    try:
        r3 = oc.fgmres(a, b, kind=1, dims=dims, params=p, maxiters=30, restart=10)
    finally:
        oc.set_threads(1)
    for r in (r2, r3):
        assert r["status"] == r1["status"]
        assert [h[:2] for h in r["history"]] == [h[:2] for h in r1["history"]]
        assert np.array_equal(r["x"], r1["x"])
