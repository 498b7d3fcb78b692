import sys, numpy as np
sys.path.insert(0,'.'); sys.path.insert(0,'oracle')
from paper_2406_00809_b200 import capi
import oracle
oc=oracle.restatement()
a=oc.prescale(oc.gen_convection_diffusion(64,0.0),8.0)
p=oc.init_params(16,32,8,0); b=oc.gaussian_vector(1,a.n)
A=capi.Csr.from_arrays(a.n,a.row_ptr,a.col_idx,a.values)
m=capi.Model(A,(16,32,8),p)
y=m.apply(b); print('ok', np.linalg.norm(y))
