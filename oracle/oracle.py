"""oracle/oracle.py — TEST INFRASTRUCTURE ONLY.

ctypes faces over
  * ``liboracle.so``      — the plain-C restatement (oracle/gnp_oracle.c), and
  * ``_ref/libgnpref.so`` — the UNMODIFIED reference library + oracle/ref_shim.cpp.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's ``cpu_baseline`` /
``--impl reference`` legs may import this module; the product package never does.
Both faces expose the same Python signatures so a test can run one case through
either and compare.  Arrays: CSR as (n, row_ptr int64, col_idx int64, values f64);
dense blocks column-major n x k (include/gnp/dense.hpp:20-21); params flat in
the reference's checkpoint order (src/gnn.cpp:40-55).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libgnpref.so")

_d = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_i64 = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_u64p = C.POINTER(C.c_uint64)
_szp = C.POINTER(C.c_size_t)
STATUS = ["converged", "maxiters", "timeout", "solution_failure", "breakdown_exact"]


@dataclass
class Csr:
    n: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    def to_dense(self) -> np.ndarray:
        m = np.zeros((self.n, self.n))
        for i in range(self.n):
            for k in range(self.row_ptr[i], self.row_ptr[i + 1]):
                m[i, self.col_idx[k]] += self.values[k]
        return m

    def rounded_f32(self) -> "Csr":
        """Same pattern with values rounded once to fp32 (the device copy)."""
        return Csr(self.n, self.row_ptr, self.col_idx,
                   self.values.astype(np.float32).astype(np.float64))


def csr_arrays(a: Csr):
    return (a.n, np.ascontiguousarray(a.row_ptr, np.int64),
            np.ascontiguousarray(a.col_idx, np.int64),
            np.ascontiguousarray(a.values, np.float64))


class _CsrBuf(C.Structure):
    _fields_ = [("n", C.c_size_t), ("nnz", C.c_size_t), ("cap", C.c_size_t),
                ("rp", C.POINTER(C.c_int64)), ("ci", C.POINTER(C.c_int64)),
                ("v", C.POINTER(C.c_double))]


_OP_CB_T = C.CFUNCTYPE(None, C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_size_t)


class _OpCb(C.Structure):
    _fields_ = [("fn", _OP_CB_T), ("ctx", C.c_void_p)]


class OracleError(RuntimeError):
    pass


def _load(path):
    if not os.path.exists(path):
        raise FileNotFoundError(f"{path} not built (run: make -C oracle{' ref' if '_ref' in path else ''})")
    return C.CDLL(path)


# --------------------------------------------------------------------------
# plain-C restatement
# --------------------------------------------------------------------------
class Restatement:
    """The plain-C f64 restatement (oracle/gnp_oracle.c)."""

    name = "restatement"

    def __init__(self, path: str = ORACLE_SO):
        L = self.L = _load(path)
        L.oc_last_error.restype = C.c_char_p
        L.oc_gaussian_vector.argtypes = [C.c_uint64, C.c_size_t, _d]
        L.oc_csr_from_triplets.argtypes = [C.c_size_t, C.c_size_t, _i64, _i64, _d, _i64, _i64, _d, _szp]
        L.oc_spmv.argtypes = [C.c_size_t, _i64, _i64, _d, _d, _d]
        L.oc_spmm.argtypes = [C.c_size_t, _i64, _i64, _d, C.c_size_t, _d, _d]
        L.oc_spmv_transpose.argtypes = [C.c_size_t, _i64, _i64, _d, _d, _d]
        L.oc_transpose.argtypes = [C.c_size_t, _i64, _i64, _d, _i64, _i64, _d]
        L.oc_gershgorin_gamma.argtypes = [C.c_size_t, _i64, _i64, _d]
        L.oc_gershgorin_gamma.restype = C.c_double
        L.oc_csr_hash.argtypes = [C.c_size_t, _i64, _i64, _d]
        L.oc_csr_hash.restype = C.c_uint64
        L.oc_gen_convection_diffusion.argtypes = [C.c_size_t, C.c_double, _i64, _i64, _d, _szp]
        L.oc_param_count.argtypes = [C.c_size_t] * 3
        L.oc_param_count.restype = C.c_size_t
        L.oc_init_params.argtypes = [C.c_size_t] * 3 + [C.c_uint64, _d]
        L.oc_gnn_apply.argtypes = [C.c_size_t, _i64, _i64, _d, C.c_size_t, C.c_size_t, C.c_size_t, _d, _d, _d]
        L.oc_gnn_forward_backward.argtypes = [C.c_size_t, _i64, _i64, _d, C.c_size_t, C.c_size_t,
                                              C.c_size_t, _d, _d, _d, _d, _d]
        L.oc_l1_residual_loss.argtypes = [C.c_size_t, _i64, _i64, _d, C.c_size_t, _d, _d,
                                          C.POINTER(C.c_double), _d]
        L.oc_adam_step.argtypes = [C.c_size_t, _d, _d, _d, _d, _szp, C.c_double]
        L.oc_batch_loss_grads.argtypes = [C.c_size_t, _i64, _i64, _d, C.c_size_t, C.c_size_t,
                                          C.c_size_t, _d, C.c_size_t, _d, _d,
                                          C.POINTER(C.c_double), _d, C.c_void_p]
        L.oc_gaussian_batch.argtypes = [C.c_size_t, _i64, _i64, _d, C.c_uint64, C.c_size_t,
                                        C.c_size_t, _d, _d]
        L.oc_hessenberg_lstsq.argtypes = [C.c_size_t, _d, C.c_double, _d, C.POINTER(C.c_double),
                                          C.POINTER(C.c_int)]
        L.oc_fgmres.argtypes = [C.c_size_t, _i64, _i64, _d, _d, C.c_int, C.c_size_t, C.c_size_t,
                                C.c_size_t, C.c_void_p, _d, C.c_double, C.c_size_t, C.c_size_t,
                                C.c_double, _d, C.POINTER(C.c_size_t), _d, _d, C.c_size_t, _szp]
        L.oc_arnoldi_cycle.argtypes = [C.c_size_t, _i64, _i64, _d, _d, C.c_size_t, _d, _d, _szp,
                                       C.POINTER(C.c_int)]
        L.oc_jacobi_svd.argtypes = [C.c_size_t, C.c_size_t, _d, _d, _d, _d]
        L.oc_spectral_sampler.argtypes = [C.c_size_t, _i64, _i64, _d, C.c_size_t, C.c_uint64, _d, _d,
                                          _d, _szp, _szp]
        L.oc_assemble_batch.argtypes = [C.c_size_t, _i64, _i64, _d, C.c_size_t, C.c_size_t, _d, _d,
                                        _d, C.c_uint64, C.c_size_t, C.c_size_t, C.c_size_t, _d, _d]
        L.oc_gen_named.argtypes = [C.c_char_p, C.c_size_t, C.c_double, C.c_double, C.c_uint64,
                                   C.POINTER(_CsrBuf)]
        L.oc_csr_buf_free.argtypes = [C.POINTER(_CsrBuf)]
        L.oc_set_threads.argtypes = [C.c_size_t]
        L.oc_gnn_apply_mt.argtypes = [C.c_size_t, _i64, _i64, _d, C.c_size_t, C.c_size_t, C.c_size_t,
                                      _d, _d, _d, C.c_size_t]
        L.oc_batch_loss_grads_mt.argtypes = [C.c_size_t, _i64, _i64, _d, C.c_size_t, C.c_size_t,
                                             C.c_size_t, _d, C.c_size_t, _d, _d,
                                             C.POINTER(C.c_double), _d, C.c_void_p, C.c_size_t]

    def _check(self, rc):
        if rc != 0:
            raise OracleError(self.L.oc_last_error().decode())

    # ---- full-size parity support (bit-identical threaded restatements)
    def gen_named(self, kind: str, size: int, p0: float = 0.0, p1: float = 0.0, seed: int = 0) -> Csr:
        """BASELINE config matrices C2-C5 (the repo's recipes; see gnp_oracle.c)."""
        buf = _CsrBuf()
        rc = self.L.oc_gen_named(kind.encode(), size, p0, p1, seed, C.byref(buf))
        if rc != 0:
            self.L.oc_csr_buf_free(C.byref(buf))
            raise OracleError(self.L.oc_last_error().decode())
        try:
            n, nnz = buf.n, buf.nnz
            rp = np.ctypeslib.as_array(buf.rp, (n + 1,)).copy()
            ci = np.ctypeslib.as_array(buf.ci, (max(nnz, 1),))[:nnz].copy()
            v = np.ctypeslib.as_array(buf.v, (max(nnz, 1),))[:nnz].copy()
        finally:
            self.L.oc_csr_buf_free(C.byref(buf))
        return Csr(n, rp, ci, v)

    def set_threads(self, t: int) -> None:
        """Threads for oc_fgmres's GNP operator (bit-identical to 1)."""
        self.L.oc_set_threads(max(1, int(t)))

    def gnn_apply_mt(self, a: Csr, dims, params, b, threads=None) -> np.ndarray:
        out = np.empty(a.n)
        self._check(self.L.oc_gnn_apply_mt(*csr_arrays(a), *dims, np.ascontiguousarray(params, np.float64),
                                           np.ascontiguousarray(b, np.float64), out,
                                           threads or (os.cpu_count() or 1)))
        return out

    def batch_loss_grads_mt(self, a: Csr, dims, params, x, b, batch, want_out=False, threads=None):
        loss = C.c_double()
        grads = np.empty(self.param_count(*dims))
        out = np.empty(a.n * batch) if want_out else None
        self._check(self.L.oc_batch_loss_grads_mt(
            *csr_arrays(a), *dims, np.ascontiguousarray(params, np.float64), batch,
            np.ascontiguousarray(x, np.float64), np.ascontiguousarray(b, np.float64),
            C.byref(loss), grads, out.ctypes.data if want_out else None,
            threads or (os.cpu_count() or 1)))
        return (loss.value, grads, out) if want_out else (loss.value, grads)

    # ---- rng
    def gaussian_vector(self, seed: int, n: int) -> np.ndarray:
        out = np.empty(n)
        self.L.oc_gaussian_vector(seed, n, out)
        return out

    # ---- csr
    def csr_from_triplets(self, n, rows, cols, vals) -> Csr:
        rows = np.ascontiguousarray(rows, np.int64)
        cols = np.ascontiguousarray(cols, np.int64)
        vals = np.ascontiguousarray(vals, np.float64)
        m = len(vals)
        if len(rows) != m or len(cols) != m:
            raise OracleError("triplet arrays must have equal length")
        rp = np.zeros(n + 1, np.int64)
        ci = np.zeros(max(m, 1), np.int64)
        v = np.zeros(max(m, 1))
        nnz = C.c_size_t()
        self._check(self.L.oc_csr_from_triplets(n, m, rows, cols, vals, rp, ci, v, C.byref(nnz)))
        return Csr(n, rp, ci[: nnz.value].copy(), v[: nnz.value].copy())

    def gen_convection_diffusion(self, grid: int, conv: float) -> Csr:
        n = grid * grid
        rp = np.zeros(n + 1, np.int64)
        ci = np.zeros(5 * n, np.int64)
        v = np.zeros(5 * n)
        nnz = C.c_size_t()
        self._check(self.L.oc_gen_convection_diffusion(grid, conv, rp, ci, v, C.byref(nnz)))
        return Csr(n, rp, ci[: nnz.value].copy(), v[: nnz.value].copy())

    def spmv(self, a: Csr, x) -> np.ndarray:
        y = np.empty(a.n)
        self.L.oc_spmv(*csr_arrays(a), np.ascontiguousarray(x, np.float64), y)
        return y

    def spmv_transpose(self, a: Csr, x) -> np.ndarray:
        y = np.empty(a.n)
        self.L.oc_spmv_transpose(*csr_arrays(a), np.ascontiguousarray(x, np.float64), y)
        return y

    def spmm(self, a: Csr, x_colmajor: np.ndarray, k: int) -> np.ndarray:
        y = np.empty(a.n * k)
        self.L.oc_spmm(*csr_arrays(a), k, np.ascontiguousarray(x_colmajor, np.float64), y)
        return y

    def transpose(self, a: Csr) -> Csr:
        rp = np.zeros(a.n + 1, np.int64)
        ci = np.zeros(max(a.nnz, 1), np.int64)
        v = np.zeros(max(a.nnz, 1))
        self.L.oc_transpose(*csr_arrays(a), rp, ci, v)
        return Csr(a.n, rp, ci[: a.nnz].copy(), v[: a.nnz].copy())

    def gershgorin_gamma(self, a: Csr) -> float:
        return self.L.oc_gershgorin_gamma(*csr_arrays(a))

    def prescale(self, a: Csr, gamma: float) -> Csr:
        if gamma == 0.0:
            raise OracleError("prescale: gamma must be nonzero")
        return Csr(a.n, a.row_ptr.copy(), a.col_idx.copy(), a.values / gamma)

    def csr_hash(self, a: Csr) -> int:
        return int(self.L.oc_csr_hash(*csr_arrays(a)))

    # ---- gnn
    def param_count(self, d, hidden, layers) -> int:
        return int(self.L.oc_param_count(d, hidden, layers))

    def init_params(self, d, hidden, layers, seed) -> np.ndarray:
        out = np.empty(self.param_count(d, hidden, layers))
        self._check(self.L.oc_init_params(d, hidden, layers, seed, out))
        return out

    def gnn_apply(self, a: Csr, dims, params, b) -> np.ndarray:
        out = np.empty(a.n)
        self._check(self.L.oc_gnn_apply(*csr_arrays(a), *dims, np.ascontiguousarray(params, np.float64),
                                        np.ascontiguousarray(b, np.float64), out))
        return out

    def gnn_forward_backward(self, a: Csr, dims, params, b, gout):
        out = np.empty(a.n)
        grads = np.empty(self.param_count(*dims))
        self._check(self.L.oc_gnn_forward_backward(
            *csr_arrays(a), *dims, np.ascontiguousarray(params, np.float64),
            np.ascontiguousarray(b, np.float64), np.ascontiguousarray(gout, np.float64), out, grads))
        return out, grads

    def l1_residual_loss(self, a: Csr, out, x, batch):
        loss = C.c_double()
        grad = np.empty(a.n * batch)
        self._check(self.L.oc_l1_residual_loss(*csr_arrays(a), batch,
                                               np.ascontiguousarray(out, np.float64),
                                               np.ascontiguousarray(x, np.float64),
                                               C.byref(loss), grad))
        return loss.value, grad

    def adam_step(self, dims, params, grads, m1, m2, t, lr):
        p = np.array(params, np.float64)
        m1 = np.array(m1, np.float64)
        m2 = np.array(m2, np.float64)
        tt = C.c_size_t(t)
        self.L.oc_adam_step(len(p), p, np.ascontiguousarray(grads, np.float64), m1, m2,
                            C.byref(tt), lr)
        return p, m1, m2, tt.value

    def batch_loss_grads(self, a: Csr, dims, params, x, b, batch, want_out=False):
        loss = C.c_double()
        grads = np.empty(self.param_count(*dims))
        out = np.empty(a.n * batch) if want_out else None
        self._check(self.L.oc_batch_loss_grads(
            *csr_arrays(a), *dims, np.ascontiguousarray(params, np.float64), batch,
            np.ascontiguousarray(x, np.float64), np.ascontiguousarray(b, np.float64),
            C.byref(loss), grads, out.ctypes.data if want_out else None))
        return (loss.value, grads, out) if want_out else (loss.value, grads)

    def gaussian_batch(self, a: Csr, seed, skip_batches, batch):
        x = np.empty(a.n * batch)
        b = np.empty(a.n * batch)
        self._check(self.L.oc_gaussian_batch(*csr_arrays(a), seed, skip_batches, batch, x, b))
        return x, b

    # ---- spectral sampler (src/sampler.cpp, src/svd.cpp)
    def arnoldi_cycle(self, a: Csr, r0, m):
        """-> (V n x (m+1) col-major flat, Hbar (m+1) x m col-major flat, steps, breakdown)"""
        v = np.zeros(a.n * (m + 1))
        h = np.zeros((m + 1) * m)
        k = C.c_size_t()
        brk = C.c_int()
        self._check(self.L.oc_arnoldi_cycle(*csr_arrays(a), np.ascontiguousarray(r0, np.float64), m, v, h,
                                            C.byref(k), C.byref(brk)))
        return v, h, k.value, bool(brk.value)

    def jacobi_svd(self, a_colmajor, rows, cols):
        u = np.zeros(rows * cols)
        s = np.zeros(cols)
        v = np.zeros(cols * cols)
        self._check(self.L.oc_jacobi_svd(rows, cols, np.ascontiguousarray(a_colmajor, np.float64), u, s, v))
        return u, s, v

    def spectral_sampler(self, a: Csr, m, seed):
        """-> dict(v n x k flat, zsv k x k flat, s[k], k, m_eff)"""
        v = np.zeros(a.n * m)
        z = np.zeros(m * m)
        s = np.zeros(m)
        k = C.c_size_t()
        me = C.c_size_t()
        self._check(self.L.oc_spectral_sampler(*csr_arrays(a), m, seed, v, z, s, C.byref(k), C.byref(me)))
        k = k.value
        return {"v": v[: a.n * k].copy(), "zsv": z[: k * k].copy(), "s": s[:k].copy(), "k": k,
                "m_eff": me.value}

    def assemble_batch(self, a: Csr, sampler, seed, skip_batches, batch, spectral_count):
        x = np.empty(a.n * batch)
        b = np.empty(a.n * batch)
        if sampler is None:
            sampler = {"v": np.zeros(1), "zsv": np.zeros(1), "s": np.ones(1), "k": 0, "m_eff": 0}
        self._check(self.L.oc_assemble_batch(*csr_arrays(a), sampler["k"], sampler["m_eff"],
                                             np.ascontiguousarray(sampler["v"], np.float64),
                                             np.ascontiguousarray(sampler["zsv"], np.float64),
                                             np.ascontiguousarray(sampler["s"], np.float64), seed,
                                             skip_batches, batch, spectral_count, x, b))
        return x, b

    # ---- krylov
    def hessenberg_lstsq(self, hbar_colmajor, k, beta):
        y = np.zeros(k)
        tr = C.c_double()
        sing = C.c_int()
        self._check(self.L.oc_hessenberg_lstsq(k, np.ascontiguousarray(hbar_colmajor, np.float64),
                                               beta, y, C.byref(tr), C.byref(sing)))
        return y, tr.value, bool(sing.value)

    def fgmres(self, a: Csr, b, kind=0, dims=(0, 0, 0), params=None, x0=None, rtol=1e-8,
               maxiters=100, restart=10, timeout_secs=-1.0):
        n = a.n
        x0 = np.zeros(n) if x0 is None else np.ascontiguousarray(x0, np.float64)
        x = np.empty(n)
        cap = maxiters + 2
        hi = (C.c_size_t * cap)()
        hr = np.empty(cap)
        ht = np.empty(cap)
        hl = C.c_size_t()
        keep = None
        if callable(kind):
            # kind 4: a caller-supplied operator M(v) -> array (e.g. the device GNP)
            fn = kind

            def tramp(ctx, pin, pout, nn):
                vin = np.ctypeslib.as_array(pin, (nn,)).copy()
                np.ctypeslib.as_array(pout, (nn,))[:] = fn(vin)

            keep = _OP_CB_T(tramp)
            cb = _OpCb(keep, None)
            kind, pptr = 4, C.addressof(cb)
        else:
            p = np.ascontiguousarray(params, np.float64) if params is not None else None
            pptr = p.ctypes.data if p is not None else None
        st = self.L.oc_fgmres(*csr_arrays(a), np.ascontiguousarray(b, np.float64), kind, *dims,
                              pptr, x0, rtol, maxiters,
                              restart, timeout_secs, x, hi, hr, ht, cap, C.byref(hl))
        if st < 0:
            raise OracleError(self.L.oc_last_error().decode())
        L = min(hl.value, cap)
        hist = [(int(hi[i]), float(hr[i]), float(ht[i])) for i in range(L)]
        return {"status": STATUS[st], "x": x, "history": hist}


# --------------------------------------------------------------------------
# the unmodified reference (oracle/_ref)
# --------------------------------------------------------------------------
class Reference:
    """The reference library itself, through oracle/ref_shim.cpp."""

    name = "reference"

    def __init__(self, path: str = REF_SO):
        L = self.L = _load(path)
        vp = C.c_void_p
        L.ref_last_error.restype = C.c_char_p
        L.ref_csr_new.restype = vp
        L.ref_csr_new.argtypes = [C.c_size_t, _i64, _i64, _d]
        L.ref_csr_from_triplets.restype = vp
        L.ref_csr_from_triplets.argtypes = [C.c_size_t, C.c_size_t, _i64, _i64, _d]
        L.ref_gen_convection_diffusion.restype = vp
        L.ref_gen_convection_diffusion.argtypes = [C.c_size_t, C.c_double]
        L.ref_gen_random_nonsymmetric.restype = vp
        L.ref_gen_random_nonsymmetric.argtypes = [C.c_size_t, C.c_size_t, C.c_double, C.c_uint64]
        L.ref_read_matrix_market.restype = vp
        L.ref_read_matrix_market.argtypes = [C.c_char_p]
        L.ref_csr_free.argtypes = [vp]
        L.ref_csr_n.argtypes = [vp]
        L.ref_csr_n.restype = C.c_size_t
        L.ref_csr_nnz.argtypes = [vp]
        L.ref_csr_nnz.restype = C.c_size_t
        L.ref_csr_export.argtypes = [vp, _i64, _i64, _d]
        L.ref_gershgorin_gamma.argtypes = [vp]
        L.ref_gershgorin_gamma.restype = C.c_double
        L.ref_prescale.argtypes = [vp, C.c_double]
        L.ref_prescale.restype = vp
        L.ref_transpose.argtypes = [vp]
        L.ref_transpose.restype = vp
        L.ref_csr_hash.argtypes = [vp]
        L.ref_csr_hash.restype = C.c_uint64
        L.ref_spmv.argtypes = [vp, _d, _d]
        L.ref_spmv_transpose.argtypes = [vp, _d, _d]
        L.ref_spmm.argtypes = [vp, C.c_size_t, _d, _d]
        L.ref_gaussian_vector.argtypes = [C.c_uint64, C.c_size_t, _d]
        L.ref_uniform_stream.argtypes = [C.c_uint64, C.c_size_t, _d, _d]
        L.ref_param_count.argtypes = [C.c_size_t] * 3
        L.ref_param_count.restype = C.c_size_t
        L.ref_init_params.argtypes = [C.c_size_t] * 3 + [C.c_uint64, _d]
        L.ref_gnn_apply.argtypes = [vp, C.c_size_t, C.c_size_t, C.c_size_t, _d, _d, _d]
        L.ref_gnn_forward_backward.argtypes = [vp, C.c_size_t, C.c_size_t, C.c_size_t, _d, _d, _d, _d, _d]
        L.ref_l1_residual_loss.argtypes = [vp, C.c_size_t, _d, _d, C.POINTER(C.c_double), _d]
        L.ref_batch_loss_grads.argtypes = [vp, C.c_size_t, C.c_size_t, C.c_size_t, _d, C.c_size_t,
                                           _d, _d, C.POINTER(C.c_double), _d, vp]
        L.ref_adam_step.argtypes = [C.c_size_t] * 3 + [_d, _d, _d, _d, _szp, C.c_double]
        L.ref_train.argtypes = [vp, C.c_size_t, C.c_size_t, C.c_size_t, C.c_double, C.c_size_t,
                                C.c_size_t, C.c_size_t, C.c_size_t, C.c_uint64, C.c_size_t, _d, _d,
                                C.POINTER(C.c_double)]
        L.ref_gaussian_batch.argtypes = [vp, C.c_uint64, C.c_size_t, C.c_size_t, _d, _d]
        L.ref_hessenberg_lstsq.argtypes = [C.c_size_t, _d, C.c_double, _d, C.POINTER(C.c_double),
                                           C.POINTER(C.c_int)]
        L.ref_jacobi_svd.argtypes = [C.c_size_t, C.c_size_t, _d, _d, _d, _d]
        L.ref_spectral_sampler.argtypes = [vp, C.c_size_t, C.c_uint64, _d, _d, _d, _szp, _szp]
        L.ref_assemble_batch.argtypes = [vp, C.c_size_t, C.c_uint64, C.c_uint64, C.c_size_t, C.c_size_t,
                                         C.c_size_t, _d, _d]
        L.ref_arnoldi_cycle.argtypes = [vp, _d, C.c_size_t, C.c_int, C.c_size_t, C.c_size_t,
                                        C.c_size_t, vp, _d, _d, _d, _szp, C.POINTER(C.c_int)]
        L.ref_fgmres.argtypes = [vp, _d, C.c_int, C.c_size_t, C.c_size_t, C.c_size_t, vp, _d,
                                 C.c_double, C.c_size_t, C.c_size_t, C.c_double, _d,
                                 C.POINTER(C.c_size_t), _d, _d, C.c_size_t, _szp]
        L.ref_save_checkpoint.argtypes = [C.c_char_p, C.c_size_t, C.c_size_t, C.c_size_t, _d, vp]
        L.ref_load_checkpoint.argtypes = [C.c_char_p, _szp, _u64p, vp]
        L.ref_time_gnn_apply.argtypes = [vp, C.c_size_t, C.c_size_t, C.c_size_t, _d, _d,
                                         C.c_size_t, vp]
        L.ref_time_gnn_apply.restype = C.c_double

    def _err(self):
        return OracleError(self.L.ref_last_error().decode())

    def _check(self, rc):
        if rc != 0:
            raise self._err()

    # ---- handles
    def _h(self, a: Csr):
        h = self.L.ref_csr_new(*csr_arrays(a))
        return h

    def _export(self, h) -> Csr:
        if not h:
            raise self._err()
        n = self.L.ref_csr_n(h)
        nnz = self.L.ref_csr_nnz(h)
        rp = np.empty(n + 1, np.int64)
        ci = np.empty(max(nnz, 1), np.int64)
        v = np.empty(max(nnz, 1))
        self.L.ref_csr_export(h, rp, ci, v)
        self.L.ref_csr_free(h)
        return Csr(n, rp, ci[:nnz].copy(), v[:nnz].copy())

    def _with(self, a, fn):
        h = self._h(a)
        try:
            return fn(h)
        finally:
            self.L.ref_csr_free(h)

    # ---- rng
    def gaussian_vector(self, seed, n):
        out = np.empty(n)
        self.L.ref_gaussian_vector(seed, n, out)
        return out

    def uniform_stream(self, seed, count):
        u = np.empty(count)
        us = np.empty(count)
        self.L.ref_uniform_stream(seed, count, u, us)
        return u, us

    # ---- csr
    def csr_from_triplets(self, n, rows, cols, vals) -> Csr:
        rows = np.ascontiguousarray(rows, np.int64)
        cols = np.ascontiguousarray(cols, np.int64)
        vals = np.ascontiguousarray(vals, np.float64)
        if not (len(rows) == len(cols) == len(vals)):
            raise OracleError("triplet arrays must have equal length")
        return self._export(self.L.ref_csr_from_triplets(n, len(vals), rows, cols, vals))

    def gen_convection_diffusion(self, grid, conv) -> Csr:
        return self._export(self.L.ref_gen_convection_diffusion(grid, conv))

    def gen_random_nonsymmetric(self, n, k=8, dominance=1.5, seed=0) -> Csr:
        return self._export(self.L.ref_gen_random_nonsymmetric(n, k, dominance, seed))

    def read_matrix_market(self, path) -> Csr:
        return self._export(self.L.ref_read_matrix_market(path.encode()))

    def gershgorin_gamma(self, a):
        return self._with(a, self.L.ref_gershgorin_gamma)

    def prescale(self, a, gamma):
        return self._with(a, lambda h: self._export(self.L.ref_prescale(h, gamma)))

    def transpose(self, a):
        return self._with(a, lambda h: self._export(self.L.ref_transpose(h)))

    def csr_hash(self, a):
        return int(self._with(a, self.L.ref_csr_hash))

    def spmv(self, a, x):
        y = np.empty(a.n)
        self._with(a, lambda h: self._check(self.L.ref_spmv(h, np.ascontiguousarray(x, np.float64), y)))
        return y

    def spmv_transpose(self, a, x):
        y = np.empty(a.n)
        self._with(a, lambda h: self._check(
            self.L.ref_spmv_transpose(h, np.ascontiguousarray(x, np.float64), y)))
        return y

    def spmm(self, a, x_colmajor, k):
        y = np.empty(a.n * k)
        self._with(a, lambda h: self._check(
            self.L.ref_spmm(h, k, np.ascontiguousarray(x_colmajor, np.float64), y)))
        return y

    # ---- gnn
    def param_count(self, d, hidden, layers):
        return int(self.L.ref_param_count(d, hidden, layers))

    def init_params(self, d, hidden, layers, seed):
        out = np.empty(self.param_count(d, hidden, layers))
        self._check(self.L.ref_init_params(d, hidden, layers, seed, out))
        return out

    def gnn_apply(self, a, dims, params, b):
        out = np.empty(a.n)
        self._with(a, lambda h: self._check(self.L.ref_gnn_apply(
            h, *dims, np.ascontiguousarray(params, np.float64), np.ascontiguousarray(b, np.float64), out)))
        return out

    def gnn_forward_backward(self, a, dims, params, b, gout):
        out = np.empty(a.n)
        grads = np.empty(self.param_count(*dims))
        self._with(a, lambda h: self._check(self.L.ref_gnn_forward_backward(
            h, *dims, np.ascontiguousarray(params, np.float64), np.ascontiguousarray(b, np.float64),
            np.ascontiguousarray(gout, np.float64), out, grads)))
        return out, grads

    def l1_residual_loss(self, a, out, x, batch):
        loss = C.c_double()
        grad = np.empty(a.n * batch)
        self._with(a, lambda h: self._check(self.L.ref_l1_residual_loss(
            h, batch, np.ascontiguousarray(out, np.float64), np.ascontiguousarray(x, np.float64),
            C.byref(loss), grad)))
        return loss.value, grad

    def batch_loss_grads(self, a, dims, params, x, b, batch, want_out=False):
        loss = C.c_double()
        grads = np.empty(self.param_count(*dims))
        out = np.empty(a.n * batch) if want_out else None
        self._with(a, lambda h: self._check(self.L.ref_batch_loss_grads(
            h, *dims, np.ascontiguousarray(params, np.float64), batch,
            np.ascontiguousarray(x, np.float64), np.ascontiguousarray(b, np.float64),
            C.byref(loss), grads, out.ctypes.data if want_out else None)))
        return (loss.value, grads, out) if want_out else (loss.value, grads)

    def adam_step(self, dims, params, grads, m1, m2, t, lr):
        p = np.array(params, np.float64)
        m1 = np.array(m1, np.float64)
        m2 = np.array(m2, np.float64)
        tt = C.c_size_t(t)
        self._check(self.L.ref_adam_step(*dims, p, np.ascontiguousarray(grads, np.float64), m1, m2,
                                         C.byref(tt), lr))
        return p, m1, m2, tt.value

    def train(self, a, dims, lr=1e-3, steps=10, batch=8, spectral=0, arnoldi_m=10, seed=0,
              monitor_batch=16):
        best = np.empty(self.param_count(*dims))
        losses = np.empty(steps + 1)
        bl = C.c_double()
        self._with(a, lambda h: self._check(self.L.ref_train(
            h, *dims, lr, steps, batch, spectral, arnoldi_m, seed, monitor_batch, best, losses,
            C.byref(bl))))
        return best, losses, bl.value

    def gaussian_batch(self, a, seed, skip_batches, batch):
        x = np.empty(a.n * batch)
        b = np.empty(a.n * batch)
        self._with(a, lambda h: self._check(self.L.ref_gaussian_batch(h, seed, skip_batches, batch, x, b)))
        return x, b

    # ---- spectral sampler
    def jacobi_svd(self, a_colmajor, rows, cols):
        u = np.zeros(rows * cols)
        s = np.zeros(cols)
        v = np.zeros(cols * cols)
        self._check(self.L.ref_jacobi_svd(rows, cols, np.ascontiguousarray(a_colmajor, np.float64), u, s, v))
        return u, s, v

    def spectral_sampler(self, a, m, seed):
        v = np.zeros(a.n * m)
        z = np.zeros(m * m)
        s = np.zeros(m)
        k = C.c_size_t()
        me = C.c_size_t()
        self._with(a, lambda h: self._check(self.L.ref_spectral_sampler(h, m, seed, v, z, s, C.byref(k),
                                                                         C.byref(me))))
        k = k.value
        return {"v": v[: a.n * k].copy(), "zsv": z[: k * k].copy(), "s": s[:k].copy(), "k": k,
                "m_eff": me.value}

    def assemble_batch(self, a, m, sampler_seed, seed, skip_batches, batch, spectral_count):
        x = np.empty(a.n * batch)
        b = np.empty(a.n * batch)
        self._with(a, lambda h: self._check(self.L.ref_assemble_batch(
            h, m, sampler_seed, seed, skip_batches, batch, spectral_count, x, b)))
        return x, b

    # ---- krylov
    def hessenberg_lstsq(self, hbar_colmajor, k, beta):
        y = np.zeros(k)
        tr = C.c_double()
        sing = C.c_int()
        self._check(self.L.ref_hessenberg_lstsq(k, np.ascontiguousarray(hbar_colmajor, np.float64),
                                                beta, y, C.byref(tr), C.byref(sing)))
        return y, tr.value, bool(sing.value)

    def fgmres(self, a, b, kind=0, dims=(0, 0, 0), params=None, x0=None, rtol=1e-8,
               maxiters=100, restart=10, timeout_secs=-1.0):
        n = a.n
        x0 = np.zeros(n) if x0 is None else np.ascontiguousarray(x0, np.float64)
        x = np.empty(n)
        cap = maxiters + 2
        hi = (C.c_size_t * cap)()
        hr = np.empty(cap)
        ht = np.empty(cap)
        hl = C.c_size_t()
        p = np.ascontiguousarray(params, np.float64) if params is not None else None

        def run(h):
            return self.L.ref_fgmres(h, np.ascontiguousarray(b, np.float64), kind, *dims,
                                     p.ctypes.data if p is not None else None, x0, rtol,
                                     maxiters, restart, timeout_secs, x, hi, hr, ht, cap,
                                     C.byref(hl))
        st = self._with(a, run)
        if st < 0:
            raise self._err()
        L = min(hl.value, cap)
        return {"status": STATUS[st], "x": x,
                "history": [(int(hi[i]), float(hr[i]), float(ht[i])) for i in range(L)]}

    def save_checkpoint(self, path, dims, params, a):
        self._with(a, lambda h: self._check(self.L.ref_save_checkpoint(
            path.encode(), *dims, np.ascontiguousarray(params, np.float64), h)))

    def load_checkpoint(self, path):
        dims = (C.c_size_t * 3)()
        meta = (C.c_uint64 * 3)()
        self._check(self.L.ref_load_checkpoint(path.encode(), dims, meta, None))
        p = np.empty(self.param_count(*dims))
        self._check(self.L.ref_load_checkpoint(path.encode(), dims, meta, p.ctypes.data))
        return (int(dims[0]), int(dims[1]), int(dims[2])), p, (int(meta[0]), int(meta[1]), int(meta[2]))

    def time_gnn_apply(self, a, dims, params, b, reps=1):
        out = np.empty(a.n)
        secs = self._with(a, lambda h: self.L.ref_time_gnn_apply(
            h, *dims, np.ascontiguousarray(params, np.float64), np.ascontiguousarray(b, np.float64),
            reps, out.ctypes.data))
        return secs, out


_cache = {}


def restatement() -> Restatement:
    if "o" not in _cache:
        _cache["o"] = Restatement()
    return _cache["o"]


def reference() -> Reference:
    if "r" not in _cache:
        _cache["r"] = Reference()
    return _cache["r"]


def reference_available() -> bool:
    return os.path.exists(REF_SO)
