import os, sys, numpy as np
sys.path.insert(0, '.')
from paper_2406_00809_b200 import capi
cfg = sys.argv[1]
import bench
w = bench.build_workload(capi, cfg)
for _ in range(3):
    w['model'].apply(w['b'])
