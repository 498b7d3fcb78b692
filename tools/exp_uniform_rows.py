"""Experiment: d = 16 layer time on a random-column matrix with UNIFORM row
length (n = 2^20, k off-diagonals per row) — what C4's short rows would cost
if every tile's rows had one length (rows sorted by length)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2406_00809_b200 import capi

n = 1 << 20
for k in (8, 16):
    rng = np.random.default_rng(0)
    cols = rng.integers(0, n, size=(n, k), dtype=np.int64)
    cols = np.concatenate([np.arange(n, dtype=np.int64)[:, None], cols], axis=1)
    cols.sort(axis=1)
    # drop duplicates within a row by nudging (rare); keep it simple: make unique via offsets
    for j in range(1, k + 1):
        dup = cols[:, j] <= cols[:, j - 1]
        cols[dup, j] = cols[dup, j - 1] + 1
    cols = np.minimum(cols, n - 1)
    ok = (np.diff(cols, axis=1) > 0).all(axis=1)
    cols[~ok] = (np.arange(k + 1)[None, :] + np.minimum(np.nonzero(~ok)[0], n - k - 2)[:, None])
    rp = np.arange(n + 1, dtype=np.int64) * (k + 1)
    vals = rng.standard_normal(n * (k + 1)) / (k + 1)
    a = capi.Csr.from_arrays(n, rp, cols.reshape(-1), vals)
    dims = (16, 32, 8)
    m = capi.Model(a, dims, capi.init_params(*dims, 0))
    b = torch.randn(n, device="cuda", dtype=torch.float32)
    o = torch.empty_like(b)
    st = torch.cuda.current_stream().cuda_stream
    ms, cnt = np.zeros(5), np.zeros(5, np.int64)
    for i in range(3):
        m.apply_profile(b.data_ptr(), o.data_ptr(), st, ms, cnt)
    ms[:] = 0; cnt[:] = 0
    for i in range(10):
        m.apply_profile(b.data_ptr(), o.data_ptr(), st, ms, cnt)
    torch.cuda.synchronize()
    print(f"k={k}: nnz {n*(k+1)} flags {a.layout_flags()} layer {1e3*ms[3]/cnt[3]:.1f} us last {1e3*ms[4]/cnt[4]:.1f} us; per M nnz {1e3*ms[3]/cnt[3]/(n*(k+1)/1e6):.2f} us")
