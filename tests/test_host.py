"""Product host layer vs the oracle (CPU only): CSR construction and indexing
bit-exact, transpose, Gershgorin/prescale, content hash, RNG/param init,
GNPCKPT checkpoints, generators, and the reference's error behaviour."""
import os

import numpy as np
import pytest
from conftest import csr_of, golden

from oracle import Csr


def as_csr(a):
    return Csr(a.n, np.array(a.row_ptr, np.int64), np.array(a.col_idx, np.int64),
               np.array(a.values, np.float64))


def test_csr_from_triplets_bit_exact(gnp, oc):
    rng = np.random.default_rng(5)
    n = 300
    r = rng.integers(0, n, 4000)
    c = rng.integers(0, n, 4000)
    v = rng.normal(size=4000)
    # pairs may repeat: exactly-2 duplicates sum order-independently; drop >2
    key = r * n + c
    _, first, counts = np.unique(key, return_index=True, return_counts=True)
    keep = np.isin(key, key[first[counts <= 2]])
    r, c, v = r[keep], c[keep], v[keep]
    a = gnp.csr_from_triplets(n, r.tolist(), c.tolist(), v.tolist())
    o = oc.csr_from_triplets(n, r, c, v)
    assert a.row_ptr == o.row_ptr.tolist()
    assert a.col_idx == o.col_idx.tolist()
    assert a.values == o.values.tolist()


def test_csr_errors_match_reference(gnp):
    with pytest.raises(IndexError):  # std::out_of_range
        gnp.csr_from_triplets(3, [0, 3], [0, 0], [1.0, 1.0])
    with pytest.raises(ValueError):  # std::invalid_argument
        gnp.csr_from_triplets(3, [0, 1], [0], [1.0, 1.0])
    a = gnp.gen_convection_diffusion(4)
    with pytest.raises(ValueError):
        gnp.prescale(a, 0.0)
    with pytest.raises(ValueError):
        gnp.csr_from_arrays(2, [0, 2, 1], [0, 1], [1.0, 1.0])


def test_c1_generator_gamma_hash(gnp):
    g = golden("c1.npz")
    a = gnp.gen_convection_diffusion(64, 0.0)
    assert a.nnz == 20224
    assert gnp.csr_content_hash(a) == int(g["hash"])
    assert gnp.gershgorin_gamma(a) == float(g["gamma"])
    assert gnp.csr_content_hash(gnp.prescale(a, 8.0)) == int(g["ahat_hash"])


def test_random_nonsymmetric_matches_reference(gnp, ref):
    for n, k, dom, seed in [(50, 5, 1.5, 3), (200, 8, 1.3, 11), (12, 4, 1.4, 30)]:
        a = gnp.gen_random_nonsymmetric(n, k, dom, seed)
        b = ref.gen_random_nonsymmetric(n, k, dom, seed)
        assert a.row_ptr == b.row_ptr.tolist()
        assert a.col_idx == b.col_idx.tolist()
        assert a.values == b.values.tolist()


def test_transpose_and_hash(gnp, oc):
    g = golden("nonsym1138.npz")
    a0 = csr_of("a", g)
    a = gnp.csr_from_arrays(a0.n, a0.row_ptr.tolist(), a0.col_idx.tolist(), a0.values.tolist())
    assert gnp.csr_content_hash(a) == int(g["hash"])
    assert gnp.gershgorin_gamma(a) == float(g["gamma"])
    t = gnp.transpose(a)
    o = oc.transpose(a0)
    assert t.row_ptr == o.row_ptr.tolist() and t.col_idx == o.col_idx.tolist()
    assert t.values == o.values.tolist()


def test_matrix_market_parse(gnp, tmp_path):
    g = golden("nonsym1138.npz")
    a0 = csr_of("a", g)
    a = gnp.csr_from_arrays(a0.n, a0.row_ptr.tolist(), a0.col_idx.tolist(), a0.values.tolist())
    path = os.path.join(tmp_path, "m.mtx")
    gnp.write_matrix_market(path, a)
    back = gnp.read_matrix_market(path)
    assert back.values == a.values and back.col_idx == a.col_idx
    assert gnp.csr_content_hash(back) == int(g["hash"])


def test_init_params_bitwise(gnp, oc):
    g = golden("c1.npz")
    p = gnp.init_params(16, 32, 8, 0)
    assert p.total_parameters() == 5265
    assert np.array_equal(np.array(p.flat), g["params"])
    for dims in [(32, 32, 8), (3, 4, 2), (1, 1, 1)]:
        assert np.array_equal(np.array(gnp.init_params(*dims, 7).flat), oc.init_params(*dims, 7))
    assert gnp.init_params(32, 32, 8, 0).total_parameters() == 18593


def test_checkpoint_byte_identical_with_reference(gnp, ref, tmp_path):
    a = gnp.gen_random_nonsymmetric(12, 4, 1.4, 30)
    ra = ref.gen_random_nonsymmetric(12, 4, 1.4, 30)
    p = gnp.init_params(3, 4, 2, 31)
    f1 = os.path.join(tmp_path, "ours.ckpt")
    f2 = os.path.join(tmp_path, "ref.ckpt")
    gnp.save_checkpoint(f1, p, a)
    ref.save_checkpoint(f2, (3, 4, 2), np.array(p.flat), ra)
    assert open(f1, "rb").read() == open(f2, "rb").read()
    back = gnp.load_checkpoint(f2)
    assert back.dims == (3, 4, 2) and back.flat == p.flat
    dims, pp, meta = ref.load_checkpoint(f1)
    assert dims == (3, 4, 2) and np.array_equal(pp, np.array(p.flat))
    assert meta[2] == gnp.csr_content_hash(a)


def test_checkpoint_rejects_garbage_and_truncation(gnp, tmp_path):
    bad = os.path.join(tmp_path, "bad.ckpt")
    open(bad, "w").write("not a checkpoint\n")
    with pytest.raises(RuntimeError):
        gnp.load_checkpoint(bad)
    a = gnp.gen_convection_diffusion(4)
    full = os.path.join(tmp_path, "full.ckpt")
    gnp.save_checkpoint(full, gnp.init_params(3, 4, 2, 33), a)
    data = open(full, "rb").read()
    cut = os.path.join(tmp_path, "cut.ckpt")
    open(cut, "wb").write(data[: len(data) // 2])
    with pytest.raises(RuntimeError):
        gnp.load_checkpoint(cut)


def test_config_generators_shapes(gnp):
    # BASELINE.json configs 2-5 at reduced size: nnz formulas of SURVEY §8(d)
    g = 10
    c2 = gnp.generate("c2_convdiff3d", g, 10.0)
    assert c2.n == g ** 3 and c2.nnz == 7 * g ** 3 - 6 * g ** 2
    c3 = gnp.generate("c3_varcoeff2d", g, 2.0, 0.0, 2)
    assert c3.n == g * g and c3.nnz == 5 * g * g - 4 * g
    c5 = gnp.generate("c5_aniso9pt", g, 1e-3, 30.0)
    assert c5.n == g * g and c5.nnz == (3 * g - 2) ** 2
    c4 = gnp.generate("c4_powerlaw", 4096, 2.2, 0.0, 4)
    rp = np.array(c4.row_ptr)
    lens = np.diff(rp) - 1
    assert lens.min() >= 4 and lens.max() <= 2048
    assert 10 < lens.mean() < 22
    # every generator produces valid CSR identical to the triplet construction
    for a in (c2, c3, c5, c4):
        rows = np.repeat(np.arange(a.n), np.diff(a.row_ptr))
        b = gnp.csr_from_triplets(a.n, rows[::-1].tolist(), a.col_idx[::-1], a.values[::-1])
        assert b.row_ptr == a.row_ptr and b.col_idx == a.col_idx and b.values == a.values


def test_iter_time_auc(gnp):
    # tests/python/test_smoke.py metrics values
    assert gnp.iter_auc([(0, 1.0, 0.0), (1, 1e-4, 0.1), (2, 1e-8, 0.2)], rtol=1e-8) == 12.0
    assert gnp.time_auc([(0, 1.0, 0.0), (1, 1e-4, 1.0)], rtol=1e-8) == 4.0


# ------------------------------------------------------------------ spectral sampler (host half)
def _prod_csr(capi, a):
    return capi.Csr.from_arrays(a.n, a.row_ptr, a.col_idx, a.values)


def test_sampler_host_half_bitwise(capi, oc):
    # the oracle's Arnoldi cycle fed to the product's SVD / rank / sampling
    # (src/sampler.cpp:19-83, src/svd.cpp): bit-identical to the oracle
    a = oc.prescale(oc.gen_convection_diffusion(12, 0.4), 8.0)
    m = 15
    v, h, k, _ = oc.arnoldi_cycle(a, oc.gaussian_vector(4, a.n), m)
    hk = h.reshape(m, m + 1)[:k, : k + 1].copy()  # (k+1) x k col-major
    A = _prod_csr(capi, a)
    s = capi.Sampler.from_arnoldi(A, v, hk.ravel(), k)
    want = oc.spectral_sampler(a, m, 4)
    pv, pz, ps = s.factors()
    assert (s.k, s.m_eff) == (want["k"], want["m_eff"])
    assert np.array_equal(ps, want["s"]) and np.array_equal(pz, want["zsv"])
    assert np.array_equal(pv, want["v"])
    for skip, batch, spec in [(0, 8, 4), (2, 5, 5), (1, 3, 0)]:
        x1, b1 = capi.assemble_batch(A, s, 77, skip, batch, spec)
        x2, b2 = oc.assemble_batch(a, want, 77, skip, batch, spec)
        assert np.array_equal(x1, x2) and np.array_equal(b1, b2)


def test_sampler_host_errors(capi, oc):
    a = oc.prescale(oc.gen_convection_diffusion(4, 0.0), 8.0)
    A = _prod_csr(capi, a)
    with pytest.raises(capi.GnpcError, match="EINVAL"):
        capi.assemble_batch(A, None, 0, 0, 0, 0)  # empty batch
    with pytest.raises(capi.GnpcError, match="EINVAL"):
        capi.assemble_batch(A, None, 0, 0, 2, 3)  # spectral_count > batch
    with pytest.raises(capi.GnpcError, match="EINVAL"):
        capi.assemble_batch(A, None, 0, 0, 4, 2)  # spectral columns without a sampler
    # a numerically zero Hessenberg (src/sampler.cpp:35-36)
    with pytest.raises(capi.GnpcError, match="ERUNTIME"):
        capi.Sampler.from_arnoldi(A, np.zeros(a.n * 2), np.zeros(6), 2)
    # Gaussian-only batches match the oracle's reference stream
    x1, b1 = capi.assemble_batch(A, None, 9, 1, 3, 0)
    x2, b2 = oc.gaussian_batch(a, 9, 1, 3)
    assert np.array_equal(x1, x2) and np.array_equal(b1, b2)
