"""ctypes face of the C ABI (include/gnpc.h) — the same entry points a cgo /
JNI / ctypes binding of the reference would call.

Used by the parity tests (which must go through the C ABI) and by bench.py for
the device-resident and host-buffer (e2e) timing legs.  Raises GnpcError on any
non-zero gnpc_status; there is no fallback path.
"""
from __future__ import annotations

import ctypes as C
import os
import re

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GNPC_LIB") or os.path.join(HERE, "libgnpc.so")  # GNPC_LIB: a variant build (tuning)
HEADER = os.path.join(os.path.dirname(HERE), "include", "gnpc.h")

STATUS = ["converged", "maxiters", "timeout", "solution_failure", "breakdown_exact"]
ERRORS = {1: "EINVAL", 2: "ERANGE", 3: "ERUNTIME", 4: "ECUDA", 5: "ENOMEM", 6: "EUNSUPPORTED",
          7: "ENODEV"}

_d = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_i64 = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
vp = C.c_void_p


class GnpcError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"gnpc {ERRORS.get(code, code)}: {msg}")
        self.code = code


class SolveConfig(C.Structure):
    _fields_ = [("rtol", C.c_double), ("maxiters", C.c_int64), ("restart", C.c_int64),
                ("timeout_secs", C.c_double)]


class History(C.Structure):
    _fields_ = [("iteration", C.POINTER(C.c_int64)), ("relres", C.POINTER(C.c_double)),
                ("elapsed", C.POINTER(C.c_double)), ("capacity", C.c_int64),
                ("length", C.c_int64), ("reorth", C.c_int64)]


class TrainConfig(C.Structure):
    _fields_ = [("lr", C.c_double), ("steps", C.c_int64), ("batch", C.c_int64),
                ("spectral_count", C.c_int64), ("arnoldi_m", C.c_int64), ("seed", C.c_uint64),
                ("monitor_batch", C.c_int64), ("d", C.c_int64), ("hidden", C.c_int64),
                ("layers", C.c_int64)]


HOST_OP = C.CFUNCTYPE(C.c_int, vp, C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_int64)


def declared_symbols(header: str = HEADER):
    """Every function name declared in include/gnpc.h."""
    txt = open(header).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\**\s+\**(gnpc_\w+)\s*\(", txt, flags=re.M)))


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built; run python -m paper_2406_00809_b200.build")
        L = C.CDLL(LIB_PATH)
        L.gnpc_last_error.restype = C.c_char_p
        _lib = L
    return _lib


def check(rc: int):
    if rc != 0:
        raise GnpcError(rc, lib().gnpc_last_error().decode())


# ------------------------------------------------------------------ handles
class Csr:
    """gnpc_csr handle."""

    def __init__(self, handle):
        self.h = vp(handle) if not isinstance(handle, vp) else handle

    def __del__(self):
        try:
            if self.h and _lib is not None:
                _lib.gnpc_csr_destroy(self.h)
        except Exception:
            pass

    @classmethod
    def from_arrays(cls, n, row_ptr, col_idx, values):
        h = vp()
        check(lib().gnpc_csr_create(C.c_int64(n), np.ascontiguousarray(row_ptr, np.int64).ctypes.data_as(vp),
                                    np.ascontiguousarray(col_idx, np.int64).ctypes.data_as(vp),
                                    np.ascontiguousarray(values, np.float64).ctypes.data_as(vp),
                                    C.byref(h)))
        return cls(h)

    @classmethod
    def from_triplets(cls, n, rows, cols, vals):
        r = np.ascontiguousarray(rows, np.int64)
        c = np.ascontiguousarray(cols, np.int64)
        v = np.ascontiguousarray(vals, np.float64)
        h = vp()
        check(lib().gnpc_csr_from_triplets(C.c_int64(n), C.c_int64(len(v)), r.ctypes.data_as(vp),
                                           c.ctypes.data_as(vp), v.ctypes.data_as(vp), C.byref(h)))
        return cls(h)

    @classmethod
    def generate(cls, kind, size, p0=0.0, p1=0.0, seed=0):
        h = vp()
        check(lib().gnpc_csr_generate(kind.encode(), C.c_int64(size), C.c_double(p0),
                                      C.c_double(p1), C.c_uint64(seed), C.byref(h)))
        return cls(h)

    def info(self):
        n, z = C.c_int64(), C.c_int64()
        check(lib().gnpc_csr_info(self.h, C.byref(n), C.byref(z)))
        return n.value, z.value

    def device_layout(self):
        """(uploaded, sliced_ell, long_rows) of the device copy."""
        u, s, l = C.c_int(), C.c_int(), C.c_int()
        check(lib().gnpc_csr_device_layout(self.h, C.byref(u), C.byref(s), C.byref(l)))
        return bool(u.value), bool(s.value), l.value

    def layout_flags(self):
        """Bit mask of the device layouts built: 1 sliced-ELL, 2 pair-union,
        4 strip-window pair-union (d = 32), 16 training strip windows,
        32 length-sorted node order for the apply (ragged matrices)."""
        u, s, l = C.c_int(), C.c_int(), C.c_int()
        check(lib().gnpc_csr_device_layout(self.h, C.byref(u), C.byref(s), C.byref(l)))
        return s.value

    @property
    def n(self):
        return self.info()[0]

    @property
    def nnz(self):
        return self.info()[1]

    def arrays(self):
        n, z = self.info()
        rp = np.empty(n + 1, np.int64)
        ci = np.empty(max(z, 1), np.int64)
        v = np.empty(max(z, 1))
        check(lib().gnpc_csr_export(self.h, rp.ctypes.data_as(vp), ci.ctypes.data_as(vp),
                                    v.ctypes.data_as(vp)))
        return rp, ci[:z], v[:z]

    def gamma(self):
        g = C.c_double()
        check(lib().gnpc_csr_gershgorin_gamma(self.h, C.byref(g)))
        return g.value

    def prescale(self, gamma):
        h = vp()
        check(lib().gnpc_csr_prescale(self.h, C.c_double(gamma), C.byref(h)))
        return Csr(h)

    def transpose(self):
        h = vp()
        check(lib().gnpc_csr_transpose(self.h, C.byref(h)))
        return Csr(h)

    def hash(self):
        x = C.c_uint64()
        check(lib().gnpc_csr_hash(self.h, C.byref(x)))
        return x.value

    def spmv(self, x):
        x = np.ascontiguousarray(x, np.float64)
        y = np.empty_like(x)
        check(lib().gnpc_spmv(self.h, x.ctypes.data_as(vp), y.ctypes.data_as(vp)))
        return y


def param_count(d, hidden, layers):
    c = C.c_int64()
    check(lib().gnpc_param_count(C.c_int64(d), C.c_int64(hidden), C.c_int64(layers), C.byref(c)))
    return c.value


def init_params(d, hidden, layers, seed):
    p = np.empty(param_count(d, hidden, layers))
    check(lib().gnpc_init_params(C.c_int64(d), C.c_int64(hidden), C.c_int64(layers),
                                 C.c_uint64(seed), p.ctypes.data_as(vp)))
    return p


class Model:
    """gnpc_model handle (GNP bound to Â)."""

    def __init__(self, csr: Csr, dims, params):
        self.csr = csr  # keep the borrowed matrix alive
        self.dims = tuple(dims)
        p = np.ascontiguousarray(params, np.float64)
        h = vp()
        check(lib().gnpc_model_create(csr.h, C.c_int64(dims[0]), C.c_int64(dims[1]),
                                      C.c_int64(dims[2]), p.ctypes.data_as(vp), C.byref(h)))
        self.h = h

    def __del__(self):
        try:
            if self.h and _lib is not None:
                _lib.gnpc_model_destroy(self.h)
        except Exception:
            pass

    def apply(self, b):
        b = np.ascontiguousarray(b, np.float64)
        out = np.empty_like(b)
        check(lib().gnpc_apply(self.h, b.ctypes.data_as(vp), out.ctypes.data_as(vp)))
        return out

    def apply_device_f32(self, b_ptr: int, out_ptr: int, stream: int = 0):
        check(lib().gnpc_apply_device_f32(self.h, vp(b_ptr), vp(out_ptr), vp(stream)))

    def apply_device_f64(self, b_ptr: int, out_ptr: int, stream: int = 0):
        check(lib().gnpc_apply_device_f64(self.h, vp(b_ptr), vp(out_ptr), vp(stream)))

    def apply_profile(self, b_ptr: int, out_ptr: int, stream: int, ms_by_kind: np.ndarray,
                      count_by_kind: np.ndarray):
        """Event-instrumented device apply; accumulates into the 5-slot arrays
        (0 norm, 1 lift, 2 long-row ÂX, 3 fused layer, 4 last layer+projection)."""
        check(lib().gnpc_apply_profile(self.h, vp(b_ptr), vp(out_ptr), vp(stream),
                                       ms_by_kind.ctypes.data_as(vp),
                                       count_by_kind.ctypes.data_as(vp)))

    def set_params(self, params):
        p = np.ascontiguousarray(params, np.float64)
        check(lib().gnpc_model_set_params(self.h, p.ctypes.data_as(vp)))


def _history(cap):
    it = (C.c_int64 * cap)()
    rel = (C.c_double * cap)()
    el = (C.c_double * cap)()
    h = History(C.cast(it, C.POINTER(C.c_int64)), C.cast(rel, C.POINTER(C.c_double)),
                C.cast(el, C.POINTER(C.c_double)), cap, 0, 0)
    return h, (it, rel, el)


def _unpack(h, bufs):
    it, rel, el = bufs
    L = min(h.length, h.capacity)
    return [(int(it[i]), float(rel[i]), float(el[i])) for i in range(L)]


def fgmres(csr: Csr, b, model: Model | None = None, x0=None, rtol=1e-8, maxiters=100,
           restart=10, timeout_secs=-1.0, host_op=None):
    """fgmres_solve through the C ABI; host_op(v) -> z runs on the host per step."""
    b = np.ascontiguousarray(b, np.float64)
    x = np.empty_like(b)
    cfg = SolveConfig(rtol, maxiters, restart, timeout_secs)
    h, bufs = _history(maxiters + 2)
    st = C.c_int()
    x0p = np.ascontiguousarray(x0, np.float64).ctypes.data_as(vp) if x0 is not None else None
    if host_op is None:
        check(lib().gnpc_fgmres(csr.h, model.h if model else None, b.ctypes.data_as(vp), x0p,
                                C.byref(cfg), x.ctypes.data_as(vp), C.byref(h), C.byref(st)))
    else:
        n = len(b)

        def _cb(ctx, pin, pout, nn):
            try:
                vin = np.ctypeslib.as_array(pin, shape=(nn,))
                z = np.asarray(host_op(vin.copy()), np.float64)
                np.ctypeslib.as_array(pout, shape=(nn,))[:] = z
                return 0
            except Exception:
                return 1

        cb = HOST_OP(_cb)
        check(lib().gnpc_fgmres_host_operator(csr.h, cb, None, b.ctypes.data_as(vp), x0p,
                                              C.byref(cfg), x.ctypes.data_as(vp), C.byref(h),
                                              C.byref(st)))
        del n
    return {"status": STATUS[st.value], "x": x, "history": _unpack(h, bufs),
            "reorth_steps": int(h.reorth)}


class Trainer:
    """gnpc_trainer handle: batched forward/backward/Adam on the device.
    Batches cross the ABI as n x B column-major f64 (the reference
    TrainingBatch layout, src/sampler.cpp:68-83)."""

    def __init__(self, model: Model, batch: int, lr: float = 1e-3):
        self.model = model
        self.batch = batch
        h = vp()
        check(lib().gnpc_trainer_create(model.h, C.c_int64(batch), C.c_double(lr), C.byref(h)))
        self.h = h
        self.count = param_count(*model.dims)

    def stream(self) -> int:
        """cudaStream_t (as an int) all of this trainer's kernels run on."""
        p = vp()
        check(lib().gnpc_trainer_stream(self.h, C.byref(p)))
        return p.value or 0

    def __del__(self):
        try:
            if self.h and _lib is not None:
                _lib.gnpc_trainer_destroy(self.h)
        except Exception:
            pass

    @staticmethod
    def _cm(a):
        return np.ascontiguousarray(a, np.float64)

    def forward_backward(self, x, b):
        x, b = self._cm(x), self._cm(b)
        loss = C.c_double()
        grads = np.empty(self.count)
        out = np.empty_like(x)
        check(lib().gnpc_forward_backward(self.h, x.ctypes.data_as(vp), b.ctypes.data_as(vp),
                                          C.byref(loss), grads.ctypes.data_as(vp),
                                          out.ctypes.data_as(vp)))
        return loss.value, grads, out

    def step(self, x, b):
        x, b = self._cm(x), self._cm(b)
        loss = C.c_double()
        check(lib().gnpc_train_step(self.h, x.ctypes.data_as(vp), b.ctypes.data_as(vp),
                                    C.byref(loss)))
        return loss.value

    def step_synthetic(self, seed: int):
        loss = C.c_double()
        check(lib().gnpc_train_step_synthetic(self.h, C.c_uint64(seed), C.byref(loss)))
        return loss.value

    def monitor_loss(self, x, b):
        x, b = self._cm(x), self._cm(b)
        loss = C.c_double()
        check(lib().gnpc_monitor_loss(self.h, x.ctypes.data_as(vp), b.ctypes.data_as(vp),
                                      C.c_int64(self.batch), C.byref(loss)))
        return loss.value

    def backward_only(self, x, b):
        x, b = self._cm(x), self._cm(b)
        loss = C.c_double()
        check(lib().gnpc_train_backward_only(self.h, x.ctypes.data_as(vp), b.ctypes.data_as(vp),
                                             C.byref(loss)))
        return loss.value

    def backward_synthetic(self, seed: int):
        loss = C.c_double()
        check(lib().gnpc_train_backward_synthetic(self.h, C.c_uint64(seed), C.byref(loss)))
        return loss.value

    def apply_grads(self):
        check(lib().gnpc_train_apply_grads(self.h))

    def grad_buffer(self):
        p = C.c_void_p()
        cnt = C.c_int64()
        check(lib().gnpc_trainer_grad_buffer(self.h, C.byref(p), C.byref(cnt)))
        return p.value, cnt.value

    def params(self):
        out = np.empty(self.count)
        check(lib().gnpc_trainer_params(self.h, out.ctypes.data_as(vp)))
        return out

    def adam_state(self):
        m1 = np.empty(self.count)
        m2 = np.empty(self.count)
        t = C.c_int64()
        check(lib().gnpc_trainer_adam_state(self.h, m1.ctypes.data_as(vp), m2.ctypes.data_as(vp),
                                            C.byref(t)))
        return m1, m2, t.value

    def sync_model(self):
        check(lib().gnpc_trainer_sync_model(self.h))


class Sampler:
    """gnpc_sampler: build_spectral_sampler (src/sampler.cpp:10-39), Arnoldi on
    the device, Jacobi SVD on the host."""

    def __init__(self, csr: Csr, m: int = 40, seed: int = 0, _handle=None):
        self.csr = csr
        self.n = csr.info()[0]
        h = _handle
        if h is None:
            h = vp()
            check(lib().gnpc_sampler_create(csr.h, C.c_int64(m), C.c_uint64(seed), C.byref(h)))
        self.h = h
        k, me = C.c_int64(), C.c_int64()
        check(lib().gnpc_sampler_info(self.h, C.byref(k), C.byref(me)))
        self.k, self.m_eff = k.value, me.value

    @classmethod
    def from_arnoldi(cls, csr: Csr, v, hbar, k):
        """Host half only (no device): factor a given cycle's (k+1) x k Hessenberg."""
        n = csr.info()[0]
        v = np.ascontiguousarray(v[: n * k], np.float64)
        hbar = np.ascontiguousarray(hbar, np.float64)
        h = vp()
        check(lib().gnpc_sampler_from_arnoldi(C.c_int64(n), C.c_int64(k), v.ctypes.data_as(vp),
                                              hbar.ctypes.data_as(vp), C.byref(h)))
        return cls(csr, _handle=h)

    def __del__(self):
        try:
            if self.h and _lib is not None:
                _lib.gnpc_sampler_destroy(self.h)
        except Exception:
            pass

    def factors(self):
        """-> (v n x k flat col-major, zsv k x k flat col-major, s[k])"""
        v = np.empty(self.n * self.k)
        z = np.empty(self.k * self.k)
        s = np.empty(self.k)
        check(lib().gnpc_sampler_export(self.h, v.ctypes.data_as(vp), z.ctypes.data_as(vp),
                                        s.ctypes.data_as(vp)))
        return v, z, s


def assemble_batch(csr: Csr, sampler: Sampler | None, seed, skip_batches, batch, spectral_count):
    """assemble_batch (src/sampler.cpp:68-83) from Rng(seed) after skip_batches batches."""
    n = csr.info()[0]
    x = np.empty(n * batch)
    b = np.empty(n * batch)
    check(lib().gnpc_assemble_batch(sampler.h if sampler else None, csr.h, C.c_uint64(seed),
                                    C.c_int64(skip_batches), C.c_int64(batch),
                                    C.c_int64(spectral_count), x.ctypes.data_as(vp),
                                    b.ctypes.data_as(vp)))
    return x, b


def device_pairs(csr: Csr, sampler: Sampler | None, seed, skip_batches, batch, spectral_count):
    """The same batch from the device pair generator of train_preconditioner."""
    n = csr.info()[0]
    x = np.empty(n * batch)
    b = np.empty(n * batch)
    check(lib().gnpc_device_pairs(sampler.h if sampler else None, csr.h, C.c_uint64(seed),
                                  C.c_int64(skip_batches), C.c_int64(batch),
                                  C.c_int64(spectral_count), x.ctypes.data_as(vp),
                                  b.ctypes.data_as(vp)))
    return x, b


def train_preconditioner(csr: Csr, dims=(16, 32, 8), lr=1e-3, steps=2000, batch=16, spectral=8,
                         arnoldi_m=40, seed=0, monitor_batch=16):
    cfg = TrainConfig(lr, steps, batch, spectral, arnoldi_m, seed, monitor_batch, *dims)
    best = np.empty(param_count(*dims))
    losses = np.empty(steps + 1)
    bl = C.c_double()
    check(lib().gnpc_train_preconditioner(csr.h, C.byref(cfg), best.ctypes.data_as(vp),
                                          losses.ctypes.data_as(vp), C.byref(bl)))
    return best, losses, bl.value


def train_run(csr: Csr, dims=(16, 32, 8), lr=1e-3, steps=2000, batch=16, spectral=8, arnoldi_m=40,
              seed=0, monitor_batch=16, timing=False):
    """train_preconditioner with device timings (gnpc_train_preconditioner_timed):
    -> {"best", "losses", "best_loss", "timing": {ms_per_step, pairgen_ms, monitor_ms, host_wait_ms}}"""
    cfg = TrainConfig(lr, steps, batch, spectral, arnoldi_m, seed, monitor_batch, *dims)
    best = np.empty(param_count(*dims))
    losses = np.empty(steps + 1)
    bl = C.c_double()
    tm = np.zeros(4)
    check(lib().gnpc_train_preconditioner_timed(csr.h, C.byref(cfg), best.ctypes.data_as(vp),
                                                losses.ctypes.data_as(vp), C.byref(bl),
                                                tm.ctypes.data_as(vp)))
    s = max(steps, 1)
    return {"best": best, "losses": losses, "best_loss": bl.value,
            "timing": {"ms_per_step": tm[0] / s, "pairgen_ms": tm[1] / s, "monitor_ms": tm[2] / s,
                       "host_wait_ms": tm[3] / s,
                       "how": "CUDA events on the model stream around the whole loop and around each "
                              "step's pair generation and monitoring phases"}}


def fgmres_device(csr: Csr, model: Model | None, b_ptr: int, x_ptr: int, rtol, maxiters, restart,
                  stream: int = 0):
    cfg = SolveConfig(rtol, maxiters, restart, -1.0)
    h, bufs = _history(maxiters + 2)
    st = C.c_int()
    check(lib().gnpc_fgmres_device(csr.h, model.h if model else None, vp(b_ptr), vp(x_ptr),
                                   C.byref(cfg), C.byref(h), C.byref(st), vp(stream)))
    return {"status": STATUS[st.value], "history": _unpack(h, bufs), "reorth_steps": int(h.reorth)}


def checkpoint_save(path: str, dims, params, csr: Csr) -> None:
    """save_checkpoint (src/gnn.cpp:480-531): GNPCKPT 1 file, byte-identical
    to the reference's."""
    p = np.ascontiguousarray(params, np.float64)
    check(lib().gnpc_checkpoint_save(path.encode(), C.c_int64(dims[0]), C.c_int64(dims[1]),
                                     C.c_int64(dims[2]), p.ctypes.data_as(vp), csr.h))


def launch_count() -> int:
    c = C.c_int64()
    check(lib().gnpc_launch_count(C.byref(c)))
    return c.value


def device_count() -> int:
    c = C.c_int()
    check(lib().gnpc_device_count(C.byref(c)))
    return c.value


def gaussian_vector(seed: int, n: int) -> np.ndarray:
    """Reference Rng(seed).gaussian_vector(n) (host, bit-exact)."""
    out = np.empty(n)
    check(lib().gnpc_gaussian_vector(C.c_uint64(seed), C.c_int64(n), out.ctypes.data_as(vp)))
    return out
