"""Trained GNP at the north-star sizes: device training (train_preconditioner),
then device FGMRES with the trained M against (a) the oracle's f64 FGMRES
driven by the same device M (isolates the Krylov machinery: iteration parity)
and (b) unpreconditioned device GMRES.  usage: r2_trained_scale.py c4|c5 steps batch maxiters"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "oracle")
import oracle  # noqa: E402
from paper_2406_00809_b200 import capi  # noqa: E402

cfg, steps, batch, maxiters = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
oc = oracle.restatement()
oc.set_threads(os.cpu_count() or 1)
if cfg == "c4":
    a = capi.Csr.generate("c4_powerlaw", 1 << 20, 2.2, 0.0, 4)
    dims, restart, rtol = (16, 32, 8), 30, 1e-6
elif cfg == "c5":
    a = capi.Csr.generate("c5_aniso9pt", 2048, 1e-3, 30.0, 0)
    dims, restart, rtol = (32, 32, 8), 50, 1e-6
else:
    a = capi.Csr.generate("c2_convdiff3d", 64, 10.0, 0.0, 0)
    dims, restart, rtol = (16, 32, 8), 30, 1e-6
ah = a.prescale(a.gamma())
n, nnz = ah.info()
rp, ci, vv = ah.arrays()
# fp32-rounded values (what the device holds) for the host-side checks
a32 = oracle.Csr(n, rp, ci, vv.astype(np.float32).astype(np.float64))
rng = np.random.default_rng({"c4": 4, "c5": 3}.get(cfg, 1))
if cfg == "c4":
    b = rng.standard_normal(n)
else:
    b = oc.spmv(a32, rng.standard_normal(n))
t0 = time.time()
best, losses, bl = capi.train_preconditioner(ah, dims=dims, steps=steps, batch=batch, spectral=min(8, batch // 2),
                                             arnoldi_m=40, seed=0, monitor_batch=batch)
t_train = time.time() - t0
p32 = np.asarray(best).astype(np.float32).astype(np.float64)
m = capi.Model(ah, dims, p32)
m0 = capi.Model(ah, dims, capi.init_params(*dims, 0))
out = {"cfg": cfg, "n": n, "nnz": nnz, "dims": dims, "train_steps": steps, "batch": batch, "train_s": round(t_train, 1),
       "loss_first": float(losses[0]), "best_loss": bl, "restart": restart, "rtol": rtol, "maxiters": maxiters}
for name, model in (("gnp_trained", m), ("gnp_seed0", m0), ("none", None)):
    t0 = time.time()
    r = capi.fgmres(ah, b, model=model, rtol=rtol, maxiters=maxiters, restart=restart)
    dt = time.time() - t0
    true_rel = float(np.linalg.norm(oc.spmv(a32, r["x"]) - b) / np.linalg.norm(b))
    out[name] = {"status": r["status"], "iterations": r["history"][-1][0], "relres": r["history"][-1][1],
                 "true_relres_host": true_rel, "solve_s": round(dt, 3)}
    print(json.dumps({name: out[name]}), flush=True)
# the oracle's f64 FGMRES driven by the same device M
t0 = time.time()
cb = oc.fgmres(a32, b, kind=lambda v: m.apply(v), rtol=rtol, maxiters=maxiters, restart=restart)
out["oracle_fgmres_device_M"] = {"status": cb["status"], "iterations": cb["history"][-1][0],
                                 "relres": cb["history"][-1][1], "solve_s": round(time.time() - t0, 1)}
out["iteration_gap"] = out["gnp_trained"]["iterations"] - cb["history"][-1][0]
print(json.dumps(out), flush=True)
