"""Per-step device time of the C3 training step over a run (is it flat?)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2406_00809_b200 import capi
a = capi.Csr.generate("c3_varcoeff2d", 512, 2.0, 0.0, 2)
ah = a.prescale(a.gamma())
m = capi.Model(ah, (32, 32, 8), capi.init_params(32, 32, 8, 0))
t = capi.Trainer(m, 32, lr=1e-3)
fixed = len(sys.argv) > 1 and sys.argv[1] == "fixed"
out = []
for i in range(int(os.environ.get("STEPS", "24"))):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    e0.record()
    l = t.step_synthetic(1000)
    e1.record()
    torch.cuda.synchronize()
    out.append((round(e0.elapsed_time(e1), 2), round(1e3 * (time.perf_counter() - w0), 2), round(l, 3)))
print(out)
