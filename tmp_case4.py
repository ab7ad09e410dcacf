import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_1802_06466_b200 as rbe
from oracle.oracle import gen_queries
from tests.test_gpu_parity import gpu_search
N, dim, kp, qp, P, geo, n, rw, Q = (20000, 200, 1, 6, 1, (1, 384, 64, 1), 50, True, 2)
dix = rbe.DeviceIndex.synthetic(dim, kp, rw, N, P, 0xD0C5)
qs = gen_queries(0x0E1, Q, dim, qp)
t = time.time()
r = gpu_search(rbe, dix, qs, geo, n, "tensor")
print("ok", time.time() - t, r[3], flush=True)
