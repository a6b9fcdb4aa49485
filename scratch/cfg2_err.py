"""Print CFG2 full-size FP16 forward max|dh|/RMS and a probe-gradient error vs the oracle (the lib
under test via XMGN_LIB_OVERRIDE)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from xmgn_inputs import configs, tensors
from gpu_util import max_over_rms, run_gpu, oracle_probe, per_tensor_rel
import oracle
b = configs.load("cfg2")
res = run_gpu(b, 128, 15, 2, want_inputs=False)
off, src = b["offsets"], b["sources"]
N, E = len(off) - 1, len(src)
f = oracle.forward(off, src, tensors.params(128, 15).double().numpy(),
                   tensors.node_features(np.arange(N), 128).double().numpy(),
                   tensors.edge_features(np.arange(E), 128).double().numpy(), 128, 15)
print("cfg2 fp16 fwd max/RMS", max_over_rms(res["h"], f["h"][-1]), flush=True)
probes = np.random.default_rng(0).choice(N, 6, replace=False)
mask = np.zeros(N); mask[probes] = 1.0
res = run_gpu(b, 128, 15, 2, g_rows=mask)
Gp = None
for pnode in probes:
    o = oracle_probe(b, int(pnode), 128, 15)
    Gp = o["params"] if Gp is None else Gp + o["params"]
print("cfg2 fp16 probe grad worst rel Frobenius", per_tensor_rel(res["params"], Gp, 128, 15), flush=True)
