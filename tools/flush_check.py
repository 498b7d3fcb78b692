"""Weight-gradient fp32 fold interval check at C3 size: gradients from the
library in GNPC_LIB on one fixed batch, written to argv[1] (compare builds)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_00809_b200 import capi
a = capi.Csr.generate("c3_varcoeff2d", 512, 2.0, 0.0, 2)
ah = a.prescale(a.gamma())
n, _ = ah.info()
B = 32
m = capi.Model(ah, (32, 32, 8), capi.init_params(32, 32, 8, 0))
t = capi.Trainer(m, B)
rng = np.random.default_rng(3)
x = rng.standard_normal((B, n))
b = np.stack([ah.spmv(x[k]) for k in range(B)])
loss, g, _ = t.forward_backward(x.reshape(-1), b.reshape(-1))
np.save(sys.argv[1], g)
print("loss", loss)
