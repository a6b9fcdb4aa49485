"""XMGN_DYN_FWD=1 (dynamic tile queue in the edge-forward kernel) vs 0: bitwise identical results."""
import os, sys
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
from xmgn_inputs import configs
from gpu_util import run_gpu
b = configs.custom((3000, 40000), k=6, P=4, halo=3)
for prec in (2, 0):
    os.environ["XMGN_DYN_FWD"] = "0"; r0 = run_gpu(b, 512, 3, prec)
    os.environ["XMGN_DYN_FWD"] = "1"; r1 = run_gpu(b, 512, 3, prec)
    print(prec, {k: bool(np.array_equal(r0[k], r1[k])) for k in ("h", "params", "h0", "e0")}, flush=True)
