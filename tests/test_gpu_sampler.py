"""GPU parity of the spectral sampler (src/sampler.cpp:10-83): the Arnoldi
cycle runs on the device (fp32 Â values, fp64 basis, device MGS reduction
order), the SVD and sampling on the host.  Against the oracle on the same
fp32-rounded matrix the basis agrees to reduction-order level (1e-10 here);
batches drawn from the product's own factors are bit-identical to the
oracle's sampling of those factors."""
import numpy as np
import pytest
from conftest import golden, rel_l2

pytestmark = pytest.mark.gpu


def dev_csr(capi, a):
    return capi.Csr.from_arrays(a.n, a.row_ptr, a.col_idx, a.values)


@pytest.mark.parametrize("grid,m,seed", [(16, 20, 7), (24, 40, 1)])
def test_device_sampler_matches_oracle(capi, oc, cuda, grid, m, seed):
    a = oc.prescale(oc.gen_convection_diffusion(grid, 0.5), 8.0).rounded_f32()
    s = capi.Sampler(dev_csr(capi, a), m, seed)
    want = oc.spectral_sampler(a, m, seed)
    assert (s.k, s.m_eff) == (want["k"], want["m_eff"])
    v, z, sv = s.factors()
    assert np.max(np.abs(sv - want["s"]) / want["s"][0]) <= 1e-10
    # basis columns: orthonormal, and equal to the oracle's to rounding
    V = v.reshape(s.k, a.n).T
    assert np.max(np.abs(V.T @ V - np.eye(s.k))) <= 1e-10
    assert rel_l2(v, want["v"]) <= 1e-9
    # batches from these factors: bitwise the oracle's sampling of them
    fac = {"v": v, "zsv": z, "s": sv, "k": s.k, "m_eff": s.m_eff}
    x1, b1 = capi.assemble_batch(s.csr, s, 9, 1, 8, 4)
    x2, b2 = oc.assemble_batch(a, fac, 9, 1, 8, 4)
    assert np.array_equal(x1, x2) and np.array_equal(b1, b2)


def test_device_sampler_golden(capi, oc, cuda):
    g = golden("spectral.npz")  # the reference, unrounded f64 matrix
    a = oc.prescale(oc.gen_convection_diffusion(16, 0.5), float(g["gamma"]))
    A = dev_csr(capi, a)
    s = capi.Sampler(A, int(g["m"]), int(g["seed"]))
    assert (s.k, s.m_eff) == (int(g["k"]), int(g["m_eff"]))
    _, _, sv = s.factors()
    assert np.max(np.abs(sv - g["s"]) / g["s"][0]) <= 1e-6  # fp32 Â vs f64
    x, b = capi.assemble_batch(A, s, int(g["batch_seed"]), 1, int(g["batch"]), int(g["spectral"]))
    assert rel_l2(x, g["x"]) <= 1e-5 and rel_l2(b, g["b"]) <= 1e-5
    spec = int(g["spectral"]) * a.n  # Gaussian columns: the same Rng stream, bitwise
    assert np.array_equal(x[spec:], g["x"][spec:]) and np.array_equal(b[spec:], g["b"][spec:])


def test_sampler_identity_breakdown(capi, cuda):
    n = 4
    A = capi.Csr.from_arrays(n, np.arange(n + 1), np.arange(n), np.ones(n))
    s = capi.Sampler(A, 3, 0)  # test_sampler.cpp:69-75
    assert (s.k, s.m_eff) == (1, 1)
    assert abs(s.factors()[2][0] - 1.0) <= 1e-12


def test_sampler_errors(capi, cuda):
    A = capi.Csr.from_arrays(1, np.array([0, 1]), np.array([0]), np.array([1.0]))
    with pytest.raises(capi.GnpcError, match="EINVAL"):
        capi.Sampler(A, 3, 0)  # n < 2
    B = capi.Csr.from_arrays(2, np.array([0, 1, 2]), np.array([0, 1]), np.array([1.0, 1.0]))
    with pytest.raises(capi.GnpcError, match="EINVAL"):
        capi.Sampler(B, 0, 0)  # m < 1


@pytest.mark.parametrize("grid,m,batch,spectral,skip", [(16, 20, 8, 4, 1), (24, 40, 16, 8, 0), (24, 40, 6, 0, 2)])
def test_device_pairs_match_oracle_sampling(capi, oc, cuda, grid, m, batch, spectral, skip):
    # the training loop's DEVICE pair generator (host MT19937-64 words, device
    # tempering + Box-Muller; spectral x = V (Zsv S^-1 eps) as a device
    # tall-skinny product; b = A x in f64 on the device) against the oracle's
    # assemble_batch (src/sampler.cpp:41-83) on the same factors and stream:
    # 1e-12 (the Gaussian columns differ by libm-vs-device log/cos rounding,
    # the spectral columns by the product's summation order)
    a = oc.prescale(oc.gen_convection_diffusion(grid, 0.5), 8.0).rounded_f32()
    s = capi.Sampler(dev_csr(capi, a), m, 3)
    v, z, sv = s.factors()
    fac = {"v": v, "zsv": z, "s": sv, "k": s.k, "m_eff": s.m_eff}
    xd, bd = capi.device_pairs(s.csr, s if spectral else None, 11, skip, batch, spectral)
    xo, bo = oc.assemble_batch(a, fac, 11, skip, batch, spectral)
    n = a.n
    for c in range(batch):
        xs, xr = xd[c * n:(c + 1) * n], xo[c * n:(c + 1) * n]
        bs, br = bd[c * n:(c + 1) * n], bo[c * n:(c + 1) * n]
        assert np.max(np.abs(xs - xr)) <= 1e-12 * max(1.0, np.max(np.abs(xr))), (c, np.max(np.abs(xs - xr)))
        assert np.max(np.abs(bs - br)) <= 1e-12 * max(1.0, np.max(np.abs(br))), (c, np.max(np.abs(bs - br)))
    # and it is the host assemble_batch of the product up to the same level
    xh, bh = capi.assemble_batch(s.csr, s if spectral else None, 11, skip, batch, spectral)
    assert np.max(np.abs(xd - xh)) <= 1e-12 * np.max(np.abs(xh))


def test_train_preconditioner_spectral_tracks_reference(capi, oc, cuda):
    # reference train_preconditioner with 4 spectral + 4 Gaussian pairs per batch
    g = golden("train_run_spectral.npz")
    a = oc.gen_convection_diffusion(6, 0.5)
    ah = oc.prescale(a, oc.gershgorin_gamma(a))
    best, losses, bl = capi.train_preconditioner(dev_csr(capi, ah), dims=(4, 8, 2), steps=20, batch=8,
                                                 spectral=4, arnoldi_m=10, seed=41, monitor_batch=8)
    want = g["losses"]
    assert np.max(np.abs(losses - want) / want) <= 1e-3
    assert bl == min(losses) and bl < losses[0]
    assert rel_l2(best, g["best"]) <= 1e-3


def test_python_train_default_spectral(gnp, cuda):
    # the reference's Python defaults draw spectral pairs (spectral=8)
    a = gnp.prescale(gnp.gen_convection_diffusion(6, 0.5), 8.0)
    params, losses = gnp.train(a, steps=5, batch=16, d=4, hidden=8, layers=2)
    assert len(losses) == 6 and min(losses) <= losses[0]
