"""Train the GNP on a config's matrix on the device, then solve FGMRES with it
(device-resident), printing iterations/time vs the untrained and Jacobi-free
baselines.  Usage: python tools/train_solve.py c2 [steps] [batch]"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2406_00809_b200 import capi  # noqa: E402

import bench  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 300
batch = int(sys.argv[3]) if len(sys.argv) > 3 else 16
kind, size, p0, p1, seed, dims, rhs, fg, desc = bench.CONFIGS[cfg]
a = capi.Csr.generate(kind, size, p0, p1, seed)
ah = a.prescale(a.gamma())
n, _ = ah.info()
b = ah.spmv(capi.gaussian_vector(rhs[1], n)) if rhs[0] == "Ax" else capi.gaussian_vector(rhs[1], n)
restart, rtol, maxiters = fg
t0 = time.perf_counter()
best, losses, bl = capi.train_preconditioner(ah, dims=dims, steps=steps, batch=batch, spectral=0, seed=0,
                                             monitor_batch=batch)
tt = time.perf_counter() - t0
print(f"{cfg}: trained {steps} steps (B={batch}) in {tt:.2f} s; loss {losses[0]:.4g} -> best {bl:.4g}")
for name, params in (("untrained", capi.init_params(*dims, 0)), ("trained", best)):
    m = capi.Model(ah, dims, params)
    capi.fgmres(ah, b, model=m, rtol=rtol, maxiters=3, restart=restart)
    t0 = time.perf_counter()
    s = capi.fgmres(ah, b, model=m, rtol=rtol, maxiters=maxiters, restart=restart)
    el = time.perf_counter() - t0
    print(f"  {name}: {s['status']} after {s['history'][-1][0]} its, relres {s['history'][-1][1]:.3e}, {el*1e3:.1f} ms")
t0 = time.perf_counter()
s = capi.fgmres(ah, b, model=None, rtol=rtol, maxiters=maxiters, restart=restart)
print(f"  no preconditioner: {s['status']} after {s['history'][-1][0]} its, relres {s['history'][-1][1]:.3e}, "
      f"{(time.perf_counter()-t0)*1e3:.1f} ms")
