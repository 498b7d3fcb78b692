"""GPU parity at the BASELINE configs' FULL sizes, through the
C ABI, against the oracle.

The matrices come from the oracle's restatement of the config generators
(oracle/gnp_oracle.c ``oc_gen_named``; pinned to gnpc_csr_generate by content
hash in tests/test_oracle_pins.py).  The checker is the oracle's row-parallel
streaming apply / column-parallel batch gradient, bit-identical to the
sequential restatement (also pinned there), so the f64 reference finishes in
seconds at n = 2^20 .. 2^22 on the GPU box's host cores.

Tolerances (north_star): GNP outputs rel-L2 and max-abs/max-ref <= 1e-4;
gradients per parameter tensor, norm-wise, <= 1e-4; loss <= 1e-5 relative.
"""
import os

import numpy as np
import pytest
from conftest import f32, max_rel, rel_l2

pytestmark = pytest.mark.gpu
TOL = 1e-4


def dev_csr(capi, a):
    return capi.Csr.from_arrays(a.n, a.row_ptr, a.col_idx, a.values)


def scaled(oc, kind, size, p0=0.0, p1=0.0, seed=0):
    a = oc.gen_named(kind, size, p0, p1, seed)
    return oc.prescale(a, oc.gershgorin_gamma(a)).rounded_f32()


def check(y, want, tol=TOL):
    e, m = rel_l2(y, want), max_rel(y, want)
    assert e <= tol and m <= tol, (e, m)
    return e, m


def test_c4_apply_full_size(capi, oc, cuda):
    # C4: power-law rows 4..2048 (long rows take the chunked path), n = 2^20
    ah = scaled(oc, "c4_powerlaw", 1 << 20, 2.2, 0.0, 4)
    assert ah.n == 1 << 20 and ah.nnz == 17069302
    assert np.diff(ah.row_ptr).max() > 1024
    p = f32(oc.init_params(16, 32, 8, 0))
    b = oc.gaussian_vector(4, ah.n)
    y = capi.Model(dev_csr(capi, ah), (16, 32, 8), p).apply(b)
    e, m = check(y, oc.gnn_apply_mt(ah, (16, 32, 8), p, b))
    print(f"C4 full size: rel-L2 {e:.2e}, max-rel {m:.2e}")


def test_c5_apply_full_size(capi, oc, cuda):
    # C5: 9-point anisotropic 2048^2, d = 32, b = A x* with x* ~ N(0, I) from Rng(3)
    ah = scaled(oc, "c5_aniso9pt", 2048, 1e-3, 30.0)
    assert ah.n == 4194304 and ah.nnz == 37724164
    p = f32(oc.init_params(32, 32, 8, 0))
    b = oc.spmv(ah, oc.gaussian_vector(3, ah.n))
    y = capi.Model(dev_csr(capi, ah), (32, 32, 8), p).apply(b)
    e, m = check(y, oc.gnn_apply_mt(ah, (32, 32, 8), p, b))
    print(f"C5 full size: rel-L2 {e:.2e}, max-rel {m:.2e}")


def test_c2_apply_full_size_generated_by_oracle(capi, oc, cuda):
    ah = scaled(oc, "c2_convdiff3d", 64, 10.0)
    assert ah.n == 262144 and ah.nnz == 1810432
    p = f32(oc.init_params(16, 32, 8, 0))
    b = oc.spmv(ah, oc.gaussian_vector(1, ah.n))
    check(capi.Model(dev_csr(capi, ah), (16, 32, 8), p).apply(b), oc.gnn_apply_mt(ah, (16, 32, 8), p, b))


def _slices(d, h, L):
    names, o = [], 0
    for nm, sz in [("enc1", h), ("enc1_b", h), ("enc2", h * d), ("enc2_b", d)]:
        names.append((nm, o, o + sz))
        o += sz
    for l in range(L):
        names.append((f"u{l}", o, o + d * d))
        o += d * d
        names.append((f"w{l}", o, o + d * d))
        o += d * d
    for nm, sz in [("dec1", d * h), ("dec1_b", h), ("dec2", h), ("dec2_b", 1)]:
        names.append((nm, o, o + sz))
        o += sz
    return names


def test_c3_full_size_gradients(capi, oc, cuda):
    # C3 at full size: 512^2 lognormal var-coeff, d = 32, L = 8, B = 32.  The
    # device's weight gradients reduce 8.4M virtual rows with bf16 hi/lo split
    # operands into f64 partials; this checks them per tensor at that size.
    ah = scaled(oc, "c3_varcoeff2d", 512, 2.0, 0.0, 2)
    assert ah.n == 262144 and ah.nnz == 1308672
    dims, B = (32, 32, 8), 32
    p = f32(oc.init_params(*dims, 0))
    x, b = oc.gaussian_batch(ah, 3, 0, B)
    t = capi.Trainer(capi.Model(dev_csr(capi, ah), dims, p), B)
    loss, grads, out = t.forward_backward(x, b)
    want_loss, want, want_out = oc.batch_loss_grads_mt(ah, dims, p, x, b, B, want_out=True)
    assert abs(loss - want_loss) <= 1e-5 * abs(want_loss), (loss, want_loss)
    assert rel_l2(out, want_out) <= TOL
    worst = 0.0
    for nm, lo, hi in _slices(*dims):
        den = np.linalg.norm(want[lo:hi])
        e = np.linalg.norm(grads[lo:hi] - want[lo:hi]) / (den if den > 0 else 1.0)
        worst = max(worst, e)
        assert e <= TOL, (nm, e)
    print(f"C3 full size: loss rel {abs(loss - want_loss) / abs(want_loss):.2e}, worst tensor {worst:.2e}")


# ---------------------------------------------------------------- trained GNP
def _read_gnpckpt(path):
    """Test-side GNPCKPT 1 reader (format: src/gnn.cpp:480-557): text header,
    then per array 'array <name> <count>\\n' + count raw LE f64 + '\\n'."""
    raw = open(path, "rb").read()
    pos = 0

    def line():
        nonlocal pos
        e = raw.index(b"\n", pos)
        s = raw[pos:e].decode()
        pos = e + 1
        return s

    assert line() == "GNPCKPT 1"
    d, h, L = (int(v) for v in line().split()[1:])
    line()  # matrix n nnz hash
    vals = []
    while pos < len(raw):
        tag, _name, cnt = line().split()
        assert tag == "array"
        cnt = int(cnt)
        vals.append(np.frombuffer(raw[pos:pos + 8 * cnt], dtype="<f8").copy())
        pos += 8 * cnt + 1
    return (d, h, L), np.concatenate(vals)


def _trained_fgmres_case(capi, oc, ah, b, dims, steps, rtol, restart, maxiters, tmp_path):
    A = dev_csr(capi, ah)
    best, losses, bl = capi.train_preconditioner(A, dims=dims, steps=steps, batch=16, spectral=8,
                                                 arnoldi_m=40, seed=0)
    assert bl < losses[0]
    path = str(tmp_path / "trained.gnpckpt")
    capi.checkpoint_save(path, dims, best, A)
    dims2, p = _read_gnpckpt(path)
    assert dims2 == dims and np.array_equal(p, best)
    p32 = f32(p)
    m = capi.Model(A, dims, p32)
    dev = capi.fgmres(A, b, model=m, rtol=rtol, maxiters=maxiters, restart=restart)
    # the oracle's f64 FGMRES driven by the device M: isolates the device
    # Krylov machinery from M's precision
    cb = oc.fgmres(ah, b, kind=lambda v: m.apply(v), rtol=rtol, maxiters=maxiters, restart=restart)
    # the oracle end to end: f64 FGMRES with the f64 GNP on the same fp32 params
    oc.set_threads(os.cpu_count() or 1)
    try:
        ref = oc.fgmres(ah, b, kind=1, dims=dims, params=p32, rtol=rtol, maxiters=maxiters, restart=restart)
    finally:
        oc.set_threads(1)
    its = [r["history"][-1][0] for r in (dev, cb, ref)]
    print(f"trained GNP ({steps} steps): iterations device {its[0]}, oracle-FGMRES+device-M {its[1]}, "
          f"oracle {its[2]}")
    assert dev["status"] == cb["status"] == ref["status"] == "converged"
    assert abs(its[0] - its[2]) <= 1 and abs(its[0] - its[1]) <= 1
    for r in (dev, cb, ref):
        assert r["history"][-1][1] <= rtol
    # the device's final true residual, recomputed independently
    assert np.linalg.norm(oc.spmv(ah, dev["x"]) - b) / np.linalg.norm(b) <= rtol * 1.01


def test_trained_gnp_fgmres_iteration_parity_c1(capi, oc, cuda, tmp_path):
    # C1 (64^2 Laplacian, restart 10, rtol 1e-8).  The GPU-trained GNP (2000
    # steps, the reference's train defaults) needs ~114 iterations, so maxiters
    # is raised from C1's 100 to 300 to reach convergence (seed-0 weights stop
    # at maxiters on every config).
    ah = oc.prescale(oc.gen_convection_diffusion(64, 0.0), 8.0)
    b = oc.gaussian_vector(1, ah.n)
    _trained_fgmres_case(capi, oc, ah, b, (16, 32, 8), 2000, 1e-8, 10, 300, tmp_path)


def test_trained_gnp_fgmres_iteration_parity_c2(capi, oc, cuda, tmp_path):
    # C2 at full size (n = 262,144, restart 30, rtol 1e-6, b = A x*)
    ah = scaled(oc, "c2_convdiff3d", 64, 10.0)
    b = oc.spmv(ah, oc.gaussian_vector(1, ah.n))
    _trained_fgmres_case(capi, oc, ah, b, (16, 32, 8), 600, 1e-6, 30, 300, tmp_path)


def test_trained_gnp_fgmres_converges_c5_full_size(capi, oc, cuda):
    # C5 at its full size (n = 4.19M, d = 32, restart 50, rtol 1e-6, b = A x*):
    # a device-trained GNP (300 steps, batch 8) converges where the seed-0
    # weights stall, in fewer iterations than unpreconditioned GMRES, and the
    # oracle's f64 FGMRES driven by the same device M needs the same count
    # (+-1): the Krylov machinery matches at full size.  (The oracle's f64 GNP
    # end to end is ~10 s per apply at this size: profiles/r02_trained_fgmres_c5.json
    # records the run this test repeats.)
    ah = scaled(oc, "c5_aniso9pt", 2048, 1e-3, 30.0)
    A = dev_csr(capi, ah)
    dims, rtol, restart, maxiters = (32, 32, 8), 1e-6, 50, 500
    b = oc.spmv(ah, np.random.default_rng(3).standard_normal(ah.n))
    best, losses, bl = capi.train_preconditioner(A, dims=dims, steps=300, batch=8, spectral=4, arnoldi_m=40,
                                                 seed=0, monitor_batch=8)
    assert bl < 0.1 * losses[0]
    m = capi.Model(A, dims, f32(best))
    dev = capi.fgmres(A, b, model=m, rtol=rtol, maxiters=maxiters, restart=restart)
    plain = capi.fgmres(A, b, rtol=rtol, maxiters=maxiters, restart=restart)
    oc.set_threads(os.cpu_count() or 1)
    try:
        cb = oc.fgmres(ah, b, kind=lambda v: m.apply(v), rtol=rtol, maxiters=maxiters, restart=restart)
    finally:
        oc.set_threads(1)
    its = dev["history"][-1][0]
    print(f"C5 trained GNP: FGMRES {its} iterations (oracle FGMRES + device M {cb['history'][-1][0]}), "
          f"GMRES {plain['history'][-1][0]}")
    assert dev["status"] == "converged" and cb["status"] == "converged"
    assert abs(its - cb["history"][-1][0]) <= 1
    assert plain["status"] == "converged" and its < plain["history"][-1][0]
    assert np.linalg.norm(oc.spmv(ah, dev["x"]) - b) / np.linalg.norm(b) <= rtol * 1.01
