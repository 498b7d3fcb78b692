"""Parity of the sliced-ELL TMA layer pipeline (k_layer_sell) against the
oracle, and against the CSR tensor-core layer on the same inputs.

The device CSR builds its sliced-ELL copy at upload when row lengths are
regular enough (GNPC_NO_SELL=1 suppresses it for one upload), so the same
matrix can be pushed through both kernel paths in one process.  Cases cover
the shapes the pipeline special-cases: staged slices (K <= 24), slices read
straight from HBM (24 < K <= 32), tiles holding long rows (> 32 nonzeros,
chunked path + sliced-ELL padding), a partial last tile, and the projection
epilogue of both widths."""
import os

import numpy as np
import pytest
from conftest import f32, max_rel, rel_l2

from oracle import Csr

pytestmark = pytest.mark.gpu
TOL = 1e-4


def apply_path(capi, a: Csr, dims, p, b, sell):
    # the device copy (and its sliced-ELL slices) is built at the first apply
    if not sell:
        os.environ["GNPC_NO_SELL"] = "1"
    try:
        c = capi.Csr.from_arrays(a.n, a.row_ptr, a.col_idx, a.values)
        y = capi.Model(c, dims, p).apply(b)
        uploaded, sell_built, _ = c.device_layout()
        assert uploaded and sell_built == sell
        return y
    finally:
        os.environ.pop("GNPC_NO_SELL", None)


def apply_both(capi, oc, a, dims, seed):
    p = f32(oc.init_params(*dims, seed))
    b = oc.gaussian_vector(seed + 1, a.n)
    want = oc.gnn_apply(a, dims, p, b)
    y_sell = apply_path(capi, a, dims, p, b, True)
    y_csr = apply_path(capi, a, dims, p, b, False)
    return y_sell, y_csr, want


def check(y, want, tol=TOL):
    assert rel_l2(y, want) <= tol, rel_l2(y, want)
    assert max_rel(y, want) <= tol, max_rel(y, want)


def stencil_plus(oc, grid, extra_rows=(), extra_len=0, seed=0):
    """5-point stencil on grid x grid, optionally with some rows widened to
    extra_len nonzeros (random columns, small values)."""
    a = oc.gen_convection_diffusion(grid, 0.3)
    n = a.n
    rows, cols, vals = [], [], []
    rng = np.random.default_rng(seed)
    for i in range(n):
        s, e = a.row_ptr[i], a.row_ptr[i + 1]
        rows += [i] * (e - s)
        cols += list(a.col_idx[s:e])
        vals += list(a.values[s:e])
        if i in extra_rows:
            have = set(a.col_idx[s:e].tolist())
            c = [int(x) for x in rng.choice(n, size=extra_len + 8, replace=False) if int(x) not in have]
            c = c[: extra_len - (e - s)]
            rows += [i] * len(c)
            cols += c
            vals += list(0.01 * rng.standard_normal(len(c)))
    t = oc.csr_from_triplets(n, rows, cols, vals)
    return oc.prescale(t, oc.gershgorin_gamma(t)).rounded_f32()


@pytest.mark.parametrize("d", [16, 32])
def test_sell_stencil_partial_tile(capi, oc, cuda, d):
    a = stencil_plus(oc, 45)  # n = 2025: last tile holds 105 rows
    y_sell, y_csr, want = apply_both(capi, oc, a, (d, 32, 8), 5)
    check(y_sell, want)
    check(y_csr, want)
    assert rel_l2(y_sell, y_csr) <= 2e-6


@pytest.mark.parametrize("d", [16, 32])
def test_sell_with_long_rows(capi, oc, cuda, d):
    a = stencil_plus(oc, 40, extra_rows={3, 130, 131, 700, 1599}, extra_len=300)
    assert np.diff(a.row_ptr).max() >= 300
    y_sell, y_csr, want = apply_both(capi, oc, a, (d, 32, 4), 7)
    check(y_sell, want)
    check(y_csr, want)


@pytest.mark.parametrize("d", [16, 32])
def test_sell_unstaged_wide_slices(capi, oc, cuda, d):
    # every row of some tiles has 28 entries: K > 24 -> slices read from HBM
    n = 1000
    rng = np.random.default_rng(11)
    rows, cols, vals = [], [], []
    for i in range(n):
        k = 28 if (i // 128) % 2 == 0 else 6
        c = rng.choice(n, size=k, replace=False)
        rows += [i] * k
        cols += c.tolist()
        vals += (rng.standard_normal(k) / k).tolist()
    t = oc.csr_from_triplets(n, rows, cols, vals)
    a = oc.prescale(t, oc.gershgorin_gamma(t)).rounded_f32()
    y_sell, y_csr, want = apply_both(capi, oc, a, (d, 32, 3), 9)
    check(y_sell, want)
    check(y_csr, want)


def test_sell_odd_hidden_projection(capi, oc, cuda):
    # hidden not a multiple of 4: scalar projection loop
    a = stencil_plus(oc, 33)
    y_sell, _, want = apply_both(capi, oc, a, (32, 13, 2), 3)
    check(y_sell, want)


@pytest.mark.parametrize("n_grid", [2, 7, 11])
def test_fused_apply_small_and_partial(capi, oc, cuda, n_grid):
    # d = 16 runs the whole apply as one persistent launch; n = 4, 49, 121
    # (grid smaller than the SM count, a single partial tile)
    a = oc.prescale(oc.gen_convection_diffusion(n_grid, 0.3), 8.6).rounded_f32()
    dims = (16, 32, 8)
    p = f32(oc.init_params(*dims, 1))
    b = oc.gaussian_vector(2, a.n)
    y = apply_path(capi, a, dims, p, b, True)
    check(y, oc.gnn_apply(a, dims, p, b))


def test_fused_apply_zero_and_device_entry(capi, oc, cuda):
    import torch

    a = oc.prescale(oc.gen_convection_diffusion(40, 0.3), 8.6).rounded_f32()
    dims = (16, 32, 8)
    p = f32(oc.init_params(*dims, 1))
    A = capi.Csr.from_arrays(a.n, a.row_ptr, a.col_idx, a.values)
    m = capi.Model(A, dims, p)
    assert np.all(m.apply(np.zeros(a.n)) == 0.0)  # tau = 0 -> M(0) = 0 inside the fused launch
    b = oc.gaussian_vector(6, a.n)
    bt = torch.tensor(b, dtype=torch.float32, device="cuda")
    out = torch.full_like(bt, float("nan"))
    m.apply_device_f32(bt.data_ptr(), out.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    check(out.double().cpu().numpy(), oc.gnn_apply(a, dims, p, b.astype(np.float32).astype(np.float64)))


@pytest.mark.parametrize("rowsort", [False, True])
def test_fused_apply_csr_ragged_rows(capi, oc, cuda, rowsort):
    # ragged rows (1..32 entries, no long rows).  Natural order
    # (GNPC_NO_ROWSORT=1): no sliced-ELL copy, the one-launch apply runs the
    # CSR-staged variant.  Default: the apply renumbers the nodes by row length
    # (flag 32), which makes the sliced-ELL copy applicable; each row keeps
    # its stored order, so both give the same bits.
    n = 3000
    rng = np.random.default_rng(21)
    rows, cols, vals = [], [], []
    for i in range(n):
        k = int(rng.integers(1, 33))
        c = rng.choice(n, size=k, replace=False)
        rows += [i] * k
        cols += c.tolist()
        vals += (rng.standard_normal(k) / k).tolist()
    t = oc.csr_from_triplets(n, rows, cols, vals)
    a = oc.prescale(t, oc.gershgorin_gamma(t)).rounded_f32()
    dims = (16, 32, 8)
    p = f32(oc.init_params(*dims, 4))
    b = oc.gaussian_vector(8, n)

    def run(nosort):
        if nosort:
            os.environ["GNPC_NO_ROWSORT"] = "1"
        try:
            A = capi.Csr.from_arrays(a.n, a.row_ptr, a.col_idx, a.values)
            y = capi.Model(A, dims, p).apply(b)
            return y, A.layout_flags(), A.device_layout()[2]
        finally:
            os.environ.pop("GNPC_NO_ROWSORT", None)

    y, flags, nlong = run(not rowsort)
    assert nlong == 0
    assert (flags & 32 and flags & 1) if rowsort else flags == 0, flags
    check(y, oc.gnn_apply(a, dims, p, b))
    if rowsort:
        assert np.array_equal(y, run(True)[0])


def test_length_sorted_apply_bitwise_with_long_rows(capi, oc, gnp, cuda):
    # power-law rows (long rows up to 2049 entries, the C4 generator at 2^15):
    # the length-sorted apply (default) against the natural order, bit for
    # bit, through the host f64 entry and the device f32 entry
    import torch

    a0 = gnp.generate("c4_powerlaw", 1 << 15, 2.2, 0.0, 4)
    a = Csr(a0.n, np.array(a0.row_ptr), np.array(a0.col_idx), np.array(a0.values))
    ah = oc.prescale(a, oc.gershgorin_gamma(a)).rounded_f32()
    dims = (16, 32, 8)
    p = f32(oc.init_params(*dims, 0))
    b = oc.gaussian_vector(4, a.n)
    bt = torch.tensor(b, dtype=torch.float32, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    res = []
    for nosort in (False, True):
        if nosort:
            os.environ["GNPC_NO_ROWSORT"] = "1"
        try:
            A = capi.Csr.from_arrays(ah.n, ah.row_ptr, ah.col_idx, ah.values)
            m = capi.Model(A, dims, p)
            y = m.apply(b)
            o = torch.full_like(bt, float("nan"))
            m.apply_device_f32(bt.data_ptr(), o.data_ptr(), st)
            torch.cuda.synchronize()
            flags, nlong = A.layout_flags(), A.device_layout()[2]
            assert nlong > 0 and bool(flags & 32) == (not nosort), (flags, nlong)
            res.append((y, o.cpu().numpy()))
        finally:
            os.environ.pop("GNPC_NO_ROWSORT", None)
    assert np.array_equal(res[0][0], res[1][0])
    assert np.array_equal(res[0][1], res[1][1])
    check(res[0][0], oc.gnn_apply(ah, dims, p, b))


def test_fused_apply_zero_copy_pinned_host(capi, oc, cuda):
    # gnpc_apply with page-locked host buffers: the one-launch apply reads b
    # and writes M(b) through their device aliases (no staging copies)
    import ctypes as C

    import torch

    a = oc.prescale(oc.gen_convection_diffusion(40, 0.3), 8.6).rounded_f32()
    dims = (16, 32, 8)
    p = f32(oc.init_params(*dims, 1))
    A = capi.Csr.from_arrays(a.n, a.row_ptr, a.col_idx, a.values)
    m = capi.Model(A, dims, p)
    b = oc.gaussian_vector(6, a.n)
    hb = torch.tensor(b, dtype=torch.float64).pin_memory()
    ho = torch.full((a.n,), float("nan"), dtype=torch.float64).pin_memory()
    for _ in range(2):
        capi.check(capi.lib().gnpc_apply(m.h, C.c_void_p(hb.data_ptr()), C.c_void_p(ho.data_ptr())))
        y = ho.numpy().copy()
        check(y, oc.gnn_apply(a, dims, p, b))
        assert np.array_equal(y, m.apply(b))  # same kernels as the staged path

