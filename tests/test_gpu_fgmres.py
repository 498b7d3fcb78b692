"""GPU parity of the device-resident FGMRES (through the C ABI) against the
oracle: status, iteration counts (±1 with the fp32 GNP, exact without a
preconditioner), histories, and the reference's Krylov pins."""
import numpy as np
import pytest
from conftest import f32, golden, rel_l2

pytestmark = pytest.mark.gpu


def dev_csr(capi, a):
    return capi.Csr.from_arrays(a.n, a.row_ptr, a.col_idx, a.values)


def dense_dominant(n, seed):
    rng = np.random.default_rng(seed)
    m = rng.uniform(-1, 1, (n, n))
    np.fill_diagonal(m, 0)
    np.fill_diagonal(m, 2 * (np.abs(m).sum(1) + 0.5))
    return m


def csr_dense(oc, m):
    r, c = np.nonzero(m)
    return oc.csr_from_triplets(m.shape[0], r, c, m[r, c])


def test_c1_gmres_matches_golden(capi, oc, cuda):
    g = golden("c1.npz")
    gg = golden("c1_gmres.npz")
    ah = oc.prescale(oc.gen_convection_diffusion(64, 0.0), 8.0)
    s = capi.fgmres(dev_csr(capi, ah), g["b"], rtol=1e-8, maxiters=100, restart=10)
    assert s["status"] == str(gg["status"])
    h = np.array([e[:2] for e in s["history"]])
    assert h.shape == gg["hist"].shape
    assert np.array_equal(h[:, 0], gg["hist"][:, 0])
    assert np.allclose(h[:, 1], gg["hist"][:, 1], rtol=1e-6, atol=0)
    assert np.linalg.norm(s["x"] - gg["x"]) / np.linalg.norm(gg["x"]) < 1e-6


@pytest.mark.parametrize("n,restart", [(100, 10), (300, 7), (1000, 30)])
def test_gmres_random_vs_oracle(capi, oc, gnp, cuda, n, restart):
    from oracle import Csr

    g = gnp.gen_random_nonsymmetric(n, 6, 1.5, 42)
    a = Csr(g.n, np.array(g.row_ptr), np.array(g.col_idx), np.array(g.values))
    a32 = a.rounded_f32()
    b = oc.spmv(a32, np.ones(n))
    want = oc.fgmres(a32, b, rtol=1e-10, maxiters=200, restart=restart)
    got = capi.fgmres(dev_csr(capi, a32), b, rtol=1e-10, maxiters=200, restart=restart)
    assert got["status"] == want["status"] == "converged"
    assert got["history"][-1][0] == want["history"][-1][0]
    assert np.linalg.norm(got["x"] - np.ones(n)) / np.sqrt(n) < 1e-8


def test_exact_inverse_one_iteration(capi, oc, cuda):
    # tests/test_krylov.cpp:151-162 with a host FlexibleOperator
    m = f32(dense_dominant(8, 21))  # the device holds Â in fp32: make it exact
    a = csr_dense(oc, m)
    inv = np.linalg.inv(m)
    b = np.random.default_rng(1).standard_normal(8)
    s = capi.fgmres(dev_csr(capi, a), b, host_op=lambda v: inv @ v)
    assert s["status"] == "converged" and s["history"][-1][0] == 1
    assert s["history"][-1][1] <= 1e-10


def test_diag_converges_at_two(capi, oc, cuda):
    # tests/test_krylov.cpp:164-171
    d = oc.csr_from_triplets(2, [0, 1], [0, 1], [1.0, 2.0])
    s = capi.fgmres(dev_csr(capi, d), np.ones(2))
    assert s["status"] == "converged" and s["history"][-1][0] == 2


def test_identity_matrix_one_iteration(capi, oc, cuda):
    # tests/test_krylov.cpp:213-219
    eye = oc.csr_from_triplets(5, range(5), range(5), [1.0] * 5)
    s = capi.fgmres(dev_csr(capi, eye), np.arange(1.0, 6.0))
    assert s["status"] == "converged" and s["history"][-1][0] == 1


def test_gmres_equals_fgmres_identity(capi, oc, cuda):
    # tests/test_krylov.cpp:198-211
    a = oc.prescale(oc.gen_convection_diffusion(12, 0.4), 1.0)
    b = oc.spmv(a, np.ones(a.n))
    A = dev_csr(capi, a)
    plain = capi.fgmres(A, b, maxiters=60)
    flex = capi.fgmres(A, b, maxiters=60, host_op=lambda v: v)
    assert len(plain["history"]) == len(flex["history"])
    for p, f in zip(plain["history"], flex["history"]):
        assert abs(p[1] - f[1]) <= 1e-13 * max(1.0, p[1])


def test_linear_preconditioner_equals_gmres_on_am(capi, oc, cuda):
    # tests/test_krylov.cpp:248-271
    m = f32(dense_dominant(20, 31))
    a = csr_dense(oc, m)
    # power-of-two diagonal scaling keeps A·M exact in fp32 on the device
    dinv = 2.0 ** -np.round(np.log2(np.diag(m)))
    b = np.random.default_rng(2).standard_normal(20)
    flex = capi.fgmres(dev_csr(capi, a), b, maxiters=20, host_op=lambda v: dinv * v)
    am = m * dinv[None, :]
    plain = capi.fgmres(dev_csr(capi, csr_dense(oc, am)), b, maxiters=20)
    L = min(len(plain["history"]), len(flex["history"]))
    for i in range(L):
        assert abs(plain["history"][i][1] - flex["history"][i][1]) <= 1e-10 * max(1.0, plain["history"][i][1])


def test_tracked_residual_monotone_and_restart_true_residual(capi, oc, cuda):
    # tests/test_krylov.cpp:221-246
    a = oc.prescale(oc.gen_convection_diffusion(12, 0.5), 1.0)
    b = oc.spmv(a, np.ones(a.n))
    s = capi.fgmres(dev_csr(capi, a), b, maxiters=60, restart=10)
    prev = s["history"][0][1]
    for it, rel, _ in s["history"]:
        if it % 10 == 0 and it > 0:
            assert rel <= prev * (1 + 1e-10)
            prev = rel
    s = capi.fgmres(dev_csr(capi, a), b, maxiters=20, restart=20)
    h = [e[1] for e in s["history"]]
    assert all(h[i] <= h[i - 1] * (1 + 1e-12) for i in range(1, len(h)))


def test_timeout_and_errors(capi, oc, cuda):
    a = oc.prescale(oc.gen_convection_diffusion(20, 0.5), 1.0)
    b = oc.spmv(a, np.ones(a.n))
    s = capi.fgmres(dev_csr(capi, a), b, maxiters=1000000, timeout_secs=0.0)
    assert s["status"] == "timeout"
    with pytest.raises(capi.GnpcError) as e:
        capi.fgmres(dev_csr(capi, a), np.zeros(a.n))
    assert e.value.code == 1


def test_trained_gnp_converges_within_one_iteration(capi, oc, cuda):
    # tests/test_gnn.cpp:393-413 with the reference-trained params (golden)
    g = golden("trained_conv5.npz")
    a = oc.gen_convection_diffusion(5, 0.2)
    ah = oc.prescale(a, oc.gershgorin_gamma(a)).rounded_f32()
    b = oc.spmv(ah, np.ones(ah.n))
    A = dev_csr(capi, ah)
    m = capi.Model(A, (4, 8, 2), g["params"])
    # This case sits at the edge of convergence: the reference needs 49 (f64
    # inputs) / 50 (fp32-rounded inputs) iterations, and an fp32 emulation of M
    # in numpy needs 59 — a 1e-7 perturbation of M moves it by ~10 iterations.
    # So here the bar is convergence to the same tolerance; iteration parity is
    # pinned on the fast-converging case below (SURVEY §7 hard part 1).
    s = capi.fgmres(A, b, model=m, maxiters=80)
    assert s["status"] == "converged"
    assert s["history"][-1][1] <= 1e-8
    assert s["history"][-1][0] <= 80


def test_trained_gnp_iteration_parity(capi, oc, cuda):
    # reference-trained GNP (600 steps): 12 FGMRES iterations vs 32 for GMRES
    g = golden("trained_conv8.npz")
    a = oc.gen_convection_diffusion(8, 0.3)
    ah = oc.prescale(a, oc.gershgorin_gamma(a)).rounded_f32()
    b = oc.spmv(ah, np.ones(ah.n))
    A = dev_csr(capi, ah)
    m = capi.Model(A, (8, 16, 4), g["params"])
    s = capi.fgmres(A, b, model=m, maxiters=100, restart=20)
    assert s["status"] == str(g["status"]) == "converged"
    assert abs(s["history"][-1][0] - int(g["hist"][-1][0])) <= 1
    assert s["history"][-1][1] <= 1e-8
    assert np.max(np.abs(s["x"] - 1.0)) < 1e-6


def test_c1_seed0_gnp_fgmres_vs_oracle(capi, oc, cuda):
    g = golden("c1.npz")
    ah = oc.prescale(oc.gen_convection_diffusion(64, 0.0), 8.0)
    A = dev_csr(capi, ah)
    m = capi.Model(A, (16, 32, 8), g["params"])
    s = capi.fgmres(A, g["b"], model=m, rtol=1e-8, maxiters=100, restart=10)
    want = oc.fgmres(ah, g["b"], kind=1, dims=(16, 32, 8), params=f32(g["params"]),
                     rtol=1e-8, maxiters=100, restart=10)
    assert s["status"] == want["status"] == "maxiters"
    assert s["history"][-1][0] == want["history"][-1][0] == 100
    assert abs(s["history"][-1][1] - want["history"][-1][1]) <= 0.05 * want["history"][-1][1]


def test_python_solve_drop_in(gnp, cuda):
    # tests/python/test_smoke.py:41-49 / 52-65 through the module
    a = gnp.prescale(gnp.gen_convection_diffusion(8, 0.3), gnp.gershgorin_gamma(gnp.gen_convection_diffusion(8, 0.3)))
    b = gnp.spmv(a, [1.0] * a.n)
    for precond in ("none", "jacobi"):
        out = gnp.solve(a, b, precond=precond, maxiters=200)
        assert out["status"] == "converged"
        assert out["history"][-1][1] <= 1e-8
        assert max(abs(v - 1.0) for v in out["x"]) < 1e-6


def test_fused_apply_after_mid_cycle_stop(capi, oc, cuda):
    # d = 16 applies run as one persistent launch with grid barriers; a device
    # solve that stops mid-cycle skips the rest of the cycle's applies, which
    # must keep the barrier counter consistent for later applies
    g = golden("c1.npz")
    ah = oc.prescale(oc.gen_convection_diffusion(64, 0.0), 8.0)
    A = dev_csr(capi, ah)
    m = capi.Model(A, (16, 32, 8), g["params"])
    r5 = capi.fgmres(A, g["b"], model=m, rtol=1e-30, maxiters=5, restart=10)["history"][-1][1]
    for _ in range(2):
        s = capi.fgmres(A, g["b"], model=m, rtol=r5 * 1.0001, maxiters=100, restart=10)
        assert s["status"] == "converged" and s["history"][-1][0] <= 5
    y = m.apply(g["b"])
    assert rel_l2(y, g["out"]) < 1e-5


@pytest.mark.parametrize("n_grid", [64, 23])
def test_onchip_mgs_variant_matches(capi, oc, gnp, cuda, n_grid):
    # k_krylov_ortho_onchip (w in registers + shared memory; taken for n too
    # long for the register variant, e.g. C5) forced at C2 size and at an
    # odd size in a subprocess, against the default variant and the oracle
    import json
    import os
    import subprocess
    import sys

    code = r"""
import json, sys, numpy as np
sys.path.insert(0, "."); sys.path.insert(0, "oracle")
from paper_2406_00809_b200 import capi
import oracle
oc = oracle.restatement()
a0 = oc.gen_named("c2_convdiff3d", %d, 10.0)
a = oc.prescale(a0, oc.gershgorin_gamma(a0)).rounded_f32()
b = oc.spmv(a, oc.gaussian_vector(1, a.n))
A = capi.Csr.from_arrays(a.n, a.row_ptr, a.col_idx, a.values)
s = capi.fgmres(A, b, rtol=1e-8, maxiters=120, restart=30)
m = capi.Model(A, (16, 32, 8), oc.init_params(16, 32, 8, 0).astype(np.float32).astype(np.float64))
g = capi.fgmres(A, b, model=m, rtol=1e-8, maxiters=40, restart=30)
print(json.dumps({"h": [e[1] for e in s["history"]], "st": s["status"], "hg": [e[1] for e in g["history"]],
                  "re": s["reorth_steps"]}))
""" % n_grid
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for force in ("0", "1"):
        env = dict(os.environ, GNPC_FORCE_ONCHIP_MGS=force)
        r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True,
                           timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(json.loads(r.stdout.strip().splitlines()[-1]))
    d, o = outs
    assert d["st"] == o["st"] and len(d["h"]) == len(o["h"]) and len(d["hg"]) == len(o["hg"])
    for x, y in zip(d["h"], o["h"]):  # GMRES: only the MGS reduction order differs
        assert abs(x - y) <= 1e-9 * max(abs(y), 1e-300) + 1e-15
    for x, y in zip(d["hg"], o["hg"]):  # fp32 GNP: rounding flips inside M can follow
        assert abs(x - y) <= 1e-4 * abs(y)
    # and the oracle's GMRES on the same system
    a0 = oc.gen_named("c2_convdiff3d", n_grid, 10.0)
    a = oc.prescale(a0, oc.gershgorin_gamma(a0)).rounded_f32()
    b = oc.spmv(a, oc.gaussian_vector(1, a.n))
    want = oc.fgmres(a, b, rtol=1e-8, maxiters=120, restart=30)
    assert want["status"] == o["st"] and len(want["history"]) == len(o["h"])
    assert abs(want["history"][-1][1] - o["h"][-1]) <= 1e-6 * want["history"][-1][1]


def test_fgmres_on_length_sorted_ragged_matrix(capi, oc, gnp, cuda):
    # power-law rows (the C4 generator at 2^12): the apply inside FGMRES runs
    # on length-sorted nodes (gather b / scatter M(b)), the SpMV and the MGS
    # on the natural order; against the oracle's f64 FGMRES on the same
    # fp32-rounded inputs, and against the natural-order apply bit for bit
    import os

    from oracle import Csr

    a0 = gnp.generate("c4_powerlaw", 1 << 12, 2.2, 0.0, 4)
    a = Csr(a0.n, np.array(a0.row_ptr), np.array(a0.col_idx), np.array(a0.values))
    ah = oc.prescale(a, oc.gershgorin_gamma(a)).rounded_f32()
    dims = (16, 32, 8)
    p = f32(oc.init_params(*dims, 0))
    b = oc.spmv(ah, oc.gaussian_vector(2, ah.n))
    res = []
    for nosort in (False, True):
        if nosort:
            os.environ["GNPC_NO_ROWSORT"] = "1"
        try:
            A = dev_csr(capi, ah)
            m = capi.Model(A, dims, p)
            s = capi.fgmres(A, b, model=m, rtol=1e-6, maxiters=40, restart=20)
            assert bool(A.layout_flags() & 32) == (not nosort)
            res.append(s)
        finally:
            os.environ.pop("GNPC_NO_ROWSORT", None)
    want = oc.fgmres(ah, b, kind=1, dims=dims, params=p, rtol=1e-6, maxiters=40, restart=20)
    s = res[0]
    assert s["status"] == want["status"]
    assert abs(s["history"][-1][0] - want["history"][-1][0]) <= 1
    hw = np.array([h[1] for h in want["history"]])
    hs = np.array([h[1] for h in s["history"]])
    k = min(len(hw), len(hs))
    assert np.max(np.abs(hs[:k] - hw[:k]) / hw[:k]) <= 5e-2
    # same bits as the natural order: the permuted apply changes no sum
    assert np.array_equal(res[0]["x"], res[1]["x"])
    assert [h[1] for h in res[0]["history"]] == [h[1] for h in res[1]["history"]]
