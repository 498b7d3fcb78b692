"""Experiment: GPU-trained GNP, device FGMRES vs oracle FGMRES (f64 M on the
same fp32 params) vs oracle FGMRES driven by the device M, on C1 and C2."""
import sys, time, json
import numpy as np
sys.path.insert(0, "."); sys.path.insert(0, "oracle")
import oracle
from paper_2406_00809_b200 import capi

oc = oracle.restatement()
oc.set_threads(16)
f32 = lambda x: np.asarray(x, np.float64).astype(np.float32).astype(np.float64)
cfg = sys.argv[1]
steps_list = [int(s) for s in sys.argv[2].split(",")]
if cfg == "c1":
    a = oc.prescale(oc.gen_convection_diffusion(64, 0.0), 8.0)
    dims, rtol, restart, maxiters = (16, 32, 8), 1e-8, 10, 100
    b = oc.gaussian_vector(1, a.n)
else:
    a0 = oc.gen_named("c2_convdiff3d", 64, 10.0)
    a = oc.prescale(a0, oc.gershgorin_gamma(a0))
    dims, rtol, restart, maxiters = (16, 32, 8), 1e-6, 30, 100
    b = oc.spmv(a.rounded_f32(), oc.gaussian_vector(1, a.n))
a32 = a.rounded_f32()
A = capi.Csr.from_arrays(a32.n, a32.row_ptr, a32.col_idx, a32.values)
for extra in [int(x) for x in (sys.argv[3].split(",") if len(sys.argv) > 3 else ["100"])]:
  for steps in steps_list:
    t0 = time.time()
    best, losses, bl = capi.train_preconditioner(A, dims=dims, steps=steps, batch=16, spectral=8,
                                                 arnoldi_m=40, seed=0)
    tt = time.time() - t0
    p = f32(best)
    m = capi.Model(A, dims, p)
    mi = maxiters * extra // 100
    t0 = time.time(); dev = capi.fgmres(A, b, model=m, rtol=rtol, maxiters=mi, restart=restart); td = time.time() - t0
    t0 = time.time(); cb = oc.fgmres(a32, b, kind=lambda v: m.apply(v), rtol=rtol, maxiters=mi, restart=restart); tc = time.time() - t0
    t0 = time.time(); o64 = oc.fgmres(a32, b, kind=1, dims=dims, params=p, rtol=rtol, maxiters=mi, restart=restart); to = time.time() - t0
    plain = capi.fgmres(A, b, rtol=rtol, maxiters=mi, restart=restart)
    print(json.dumps({"cfg": cfg, "steps": steps, "maxiters": mi, "train_s": round(tt, 1), "loss0": losses[0], "best": bl,
        "dev": [dev["status"], dev["history"][-1][0], dev["history"][-1][1], round(td, 2)],
        "oracle_fgmres_dev_M": [cb["status"], cb["history"][-1][0], cb["history"][-1][1], round(tc, 2)],
        "oracle_f64": [o64["status"], o64["history"][-1][0], o64["history"][-1][1], round(to, 2)],
        "gmres": [plain["status"], plain["history"][-1][0], plain["history"][-1][1]]}), flush=True)
