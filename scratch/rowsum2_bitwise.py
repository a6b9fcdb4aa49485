"""XMGN_ROWSUM2 (one exchange for the LN-backward row sums) vs two exchanges: bitwise identical.
Run twice: with the default library and with XMGN_LIB_OVERRIDE=.../libxmgn_rs1.so; compares dumps."""
import os, sys
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
from xmgn_inputs import configs
from gpu_util import run_gpu
b = configs.custom((300, 1500), k=6, P=4, halo=3)
out = {}
for H in (512, 128):
    r = run_gpu(b, H, 3, 2)
    for k in ("h", "params", "h0", "e0"):
        out[f"{H}_{k}"] = r[k]
np.savez(sys.argv[1], **out)
print("saved", sys.argv[1])
