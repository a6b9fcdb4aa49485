"""XMGN_LN_STATS=1 (forward's LayerNorm statistics reused by the backward) vs 0 (recomputed):
outputs and gradients must be bitwise identical in the FP16 mode (the recompute is bit-identical)."""
import os, sys
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
from xmgn_inputs import configs
from gpu_util import run_gpu
b = configs.custom((300, 1500), k=6, P=4, halo=3)
for H, prec in ((512, 2), (128, 2), (512, 0)):
    os.environ["XMGN_LN_STATS"] = "0"; r0 = run_gpu(b, H, 3, prec)
    os.environ["XMGN_LN_STATS"] = "1"; r1 = run_gpu(b, H, 3, prec)
    print(H, prec, {k: (bool(np.array_equal(r0[k], r1[k])), float(np.abs(r0[k] - r1[k]).max())) for k in ("h", "params", "h0", "e0")}, flush=True)
