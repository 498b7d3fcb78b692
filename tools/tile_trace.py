"""Debug (build with GNPC_NVCC_DEFS=-DGNPC_TILE_TRACE=<k>): per-tile clock
stamps of block 0 in the k-th sell_layer call; prints deltas per tile."""
import ctypes as C, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_00809_b200 import capi
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
if cfg == "c2":
    a = capi.Csr.generate("c2_convdiff3d", 64, 10.0); dims = (16, 32, 8)
elif cfg == "c4":
    a = capi.Csr.generate("c4_powerlaw", 1 << 20, 2.2, 0.0, 4); dims = (16, 32, 8)
else:
    a = capi.Csr.generate("c5_aniso9pt", 2048, 1e-3, 30.0); dims = (32, 32, 8)
ah = a.prescale(a.gamma())
m = capi.Model(ah, dims, capi.init_params(*dims, 0))
b = np.random.default_rng(1).standard_normal(ah.n)
m.apply(b)
out = np.zeros(64 * 16, dtype=np.uint64)
rc = capi.lib().gnpc_debug_tile_trace(out.ctypes.data_as(C.c_void_p))
assert rc == 0
t = out.reshape(64, 16).astype(np.int64)
names = ["m:start", "m:full", "m:gathered", "m:mma(t-1)done", "m:epi done", "m:split done", "m:arrived", "", "c:efull", "c:early issued", "c:afull", "c:committed"]
t0 = t[0, 1]
print("cols:", names)
for it in range(18):
    row = t[it]
    print(it, " ".join(f"{(int(v) - int(t0)) if v else -1:7d}" for v in row[:12]))
