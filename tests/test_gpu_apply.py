"""GPU parity of the GNP apply M(b) (sm_100a kernels, through the C ABI)
against the oracle.  Tolerance (north_star): fp32 arithmetic with fp32
accumulation must land within 1e-4 relative error of the f64 reference on the
same fp32-rounded inputs; expected level ~1e-6."""
import math

import numpy as np
import pytest
from conftest import csr_of, f32, golden, max_rel, rel_l2

from oracle import Csr

pytestmark = pytest.mark.gpu
TOL = 1e-4


def dev_csr(capi, a: Csr):
    return capi.Csr.from_arrays(a.n, a.row_ptr, a.col_idx, a.values)


def check(y, want, tol=TOL):
    assert rel_l2(y, want) <= tol, rel_l2(y, want)
    assert max_rel(y, want) <= tol, max_rel(y, want)


def test_c1_apply_matches_golden(capi, oc, cuda):
    g = golden("c1.npz")
    ah = oc.prescale(oc.gen_convection_diffusion(64, 0.0), 8.0)
    m = capi.Model(dev_csr(capi, ah), (16, 32, 8), g["params"])
    y = m.apply(g["b"])
    check(y, g["out"])
    assert rel_l2(y, g["out"]) < 1e-5  # expected ~1e-6


def test_nonsym1138_apply(capi, oc, cuda):
    g = golden("nonsym1138.npz")
    a = csr_of("a", g)
    ah = oc.prescale(a, float(g["gamma"]))
    ga = golden("nonsym1138_apply.npz")
    m = capi.Model(dev_csr(capi, ah), (16, 32, 8), ga["params32"])
    check(m.apply(ga["b"]), ga["out"])


def test_odd_dims_apply(capi, cuda):
    g = golden("small_fwd_bwd.npz")
    a = csr_of("a", g)
    m = capi.Model(dev_csr(capi, a), (3, 4, 2), g["params"])
    check(m.apply(g["b"]), g["out"])


def test_tiny_hand_computed(capi, oc, cuda):
    # tests/test_gnn.cpp:135-162 in fp32
    a = oc.csr_from_triplets(2, [0, 0, 1], [0, 1, 1], [0.5, 0.25, 0.5])
    p = np.array([0.3, 0.1, 1.2, 0.05, 0.7, 0.4, 0.9, 0.02, 1.1, 0.03])
    y = capi.Model(dev_csr(capi, a), (1, 1, 1), p).apply(np.array([1.0, 2.0]))
    want = oc.gnn_apply(a, (1, 1, 1), p, np.array([1.0, 2.0]))
    assert np.all(np.abs(y - want) <= 1e-6 * np.abs(want))


def test_zero_input_and_zero_head(capi, oc, cuda):
    a = oc.prescale(oc.gen_convection_diffusion(16, 0.3), 8.6)
    p = oc.init_params(4, 4, 2, 1)
    m = capi.Model(dev_csr(capi, a), (4, 4, 2), p)
    assert np.all(m.apply(np.zeros(a.n)) == 0.0)
    p2 = p.copy()
    p2[-5:] = 0.0
    m2 = capi.Model(dev_csr(capi, a), (4, 4, 2), p2)
    assert np.all(m2.apply(oc.gaussian_vector(3, a.n)) == 0.0)


def test_positive_homogeneity(capi, oc, cuda):
    a = oc.prescale(oc.gen_convection_diffusion(32, 0.3), 8.6)
    p = oc.init_params(16, 32, 8, 8)
    m = capi.Model(dev_csr(capi, a), (16, 32, 8), p)
    b = oc.gaussian_vector(9, a.n)
    base = m.apply(b)
    for alpha in (0.5, 10.0, 1e6):
        # τ is formed in f64, so only the fp32 rounding of v = (√n/τ) b moves
        assert rel_l2(m.apply(alpha * b), alpha * base) <= 1e-6


@pytest.mark.parametrize("d,h,L", [(16, 32, 8), (32, 32, 8), (8, 16, 3), (5, 7, 2), (64, 32, 2)])
def test_widths_vs_oracle(capi, oc, gnp, cuda, d, h, L):
    a0 = gnp.generate("c3_varcoeff2d", 48, 2.0, 0.0, 2)
    a = Csr(a0.n, np.array(a0.row_ptr), np.array(a0.col_idx), np.array(a0.values))
    ah = oc.prescale(a, oc.gershgorin_gamma(a)).rounded_f32()
    p = f32(oc.init_params(d, h, L, 3))
    b = oc.gaussian_vector(4, a.n)
    want = oc.gnn_apply(ah, (d, h, L), p, b)
    check(capi.Model(dev_csr(capi, ah), (d, h, L), p).apply(b), want)


def test_powerlaw_long_rows_vs_oracle(capi, oc, gnp, cuda):
    a0 = gnp.generate("c4_powerlaw", 1 << 15, 2.2, 0.0, 4)
    a = Csr(a0.n, np.array(a0.row_ptr), np.array(a0.col_idx), np.array(a0.values))
    assert np.diff(a.row_ptr).max() > 512  # exercises the long-row path
    ah = oc.prescale(a, oc.gershgorin_gamma(a)).rounded_f32()
    p = f32(oc.init_params(16, 32, 8, 0))
    b = oc.gaussian_vector(4, a.n)
    want = oc.gnn_apply(ah, (16, 32, 8), p, b)
    check(capi.Model(dev_csr(capi, ah), (16, 32, 8), p).apply(b), want)


def test_c2_full_size_vs_oracle(capi, oc, gnp, cuda):
    # BASELINE config 2 at its full size (oracle: a few seconds)
    a0 = gnp.generate("c2_convdiff3d", 64, 10.0)
    a = Csr(a0.n, np.array(a0.row_ptr), np.array(a0.col_idx), np.array(a0.values))
    assert a.n == 262144 and a.nnz == 1810432
    ah = oc.prescale(a, oc.gershgorin_gamma(a)).rounded_f32()
    p = f32(oc.init_params(16, 32, 8, 0))
    b = oc.gaussian_vector(1, a.n)
    want = oc.gnn_apply(ah, (16, 32, 8), p, b)
    check(capi.Model(dev_csr(capi, ah), (16, 32, 8), p).apply(b), want)


def test_c5_full_size_properties(capi, gnp, cuda):
    # config 5 (n = 4.19M, d = 32) is too large for the f64 oracle in seconds:
    # size-independent properties instead — determinism, homogeneity, zero map.
    a = capi.Csr.generate("c5_aniso9pt", 2048, 1e-3, 30.0)
    ah = a.prescale(a.gamma())
    n, nnz = ah.info()
    assert n == 4194304 and nnz == 37724164
    m = capi.Model(ah, (32, 32, 8), capi.init_params(32, 32, 8, 0))
    b = np.random.default_rng(3).standard_normal(n)
    y1 = m.apply(b)
    y2 = m.apply(b)
    assert np.array_equal(y1, y2)
    assert np.all(np.isfinite(y1)) and np.linalg.norm(y1) > 0
    assert rel_l2(m.apply(4.0 * b), 4.0 * y1) <= 1e-6
    assert np.all(m.apply(np.zeros(n)) == 0.0)


def test_c5_reduced_grid_vs_oracle(capi, oc, gnp, cuda):
    a0 = gnp.generate("c5_aniso9pt", 256, 1e-3, 30.0)
    a = Csr(a0.n, np.array(a0.row_ptr), np.array(a0.col_idx), np.array(a0.values))
    ah = oc.prescale(a, oc.gershgorin_gamma(a)).rounded_f32()
    p = f32(oc.init_params(32, 32, 8, 0))
    b = oc.gaussian_vector(3, a.n)
    check(capi.Model(dev_csr(capi, ah), (32, 32, 8), p).apply(b), oc.gnn_apply(ah, (32, 32, 8), p, b))


def test_device_f32_entry_matches_host_entry(capi, oc, cuda):
    import torch

    g = golden("c1.npz")
    ah = oc.prescale(oc.gen_convection_diffusion(64, 0.0), 8.0)
    m = capi.Model(dev_csr(capi, ah), (16, 32, 8), g["params"])
    bt = torch.tensor(g["b"], dtype=torch.float32, device="cuda")
    out = torch.empty_like(bt)
    m.apply_device_f32(bt.data_ptr(), out.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    check(out.double().cpu().numpy(), g["out"])


def test_python_module_drop_in(gnp, oc, cuda):
    g = golden("c1.npz")
    a = gnp.prescale(gnp.gen_convection_diffusion(64, 0.0), 8.0)
    p = gnp.params_from_flat(g["params"].tolist(), 16, 32, 8)
    y = np.array(gnp.gnn_apply(a, p, g["b"].tolist()))
    check(y, g["out"])
    assert math.isfinite(float(np.sum(y)))
