"""The C ABI surface (CPU only): libgnpc.so loads, exports every symbol that
include/gnpc.h declares, reports errors through gnpc_last_error, and refuses to
compute without a device instead of falling back to the CPU."""
import ctypes as C

import numpy as np
import pytest


def test_exports_every_declared_symbol(capi):
    syms = capi.declared_symbols()
    assert len(syms) >= 40
    L = capi.lib()
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing
    assert L.gnpc_abi_version() == 1


def test_host_only_entry_points(capi):
    a = capi.Csr.generate("convection_diffusion", 8, 0.3)
    assert a.info() == (64, 288)
    assert a.gamma() == 8.0
    t = a.transpose()
    assert t.info() == (64, 288)
    assert capi.param_count(16, 32, 8) == 5265
    p = capi.init_params(16, 32, 8, 0)
    assert p.shape == (5265,)


def test_errors_are_codes_not_exceptions(capi):
    L = capi.lib()
    h = C.c_void_p()
    r = np.array([0, 5], np.int64)
    rc = L.gnpc_csr_from_triplets(C.c_int64(3), C.c_int64(2), r.ctypes.data_as(C.c_void_p),
                                  r.ctypes.data_as(C.c_void_p),
                                  np.ones(2).ctypes.data_as(C.c_void_p), C.byref(h))
    assert rc == 2  # GNPC_ERANGE
    assert b"out of range" in L.gnpc_last_error()
    with pytest.raises(capi.GnpcError):
        capi.Csr.generate("no_such_generator", 4)


def test_no_cpu_fallback_without_device(capi):
    if capi.device_count() > 0:
        pytest.skip("a CUDA device is present")
    a = capi.Csr.generate("convection_diffusion", 8, 0.3)
    with pytest.raises(capi.GnpcError) as e:
        capi.Model(a, (16, 32, 8), capi.init_params(16, 32, 8, 0))
    assert e.value.code == 7  # GNPC_ENODEV
    with pytest.raises(capi.GnpcError) as e:
        a.spmv(np.ones(64))
    assert e.value.code == 7
