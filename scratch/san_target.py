"""Small end-to-end target for compute-sanitizer: the processor fwd+bwd (PIPE edge kernels at
H = 512, the generic kernel at H = 128), the full model fwd+bwd, and the GPU graph build."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
from xmgn_inputs import configs
from paper_2411_17164_b200 import xmgn
from paper_2411_17164_b200.processor import Processor

b = configs.custom((300, 1200), k=6, P=2, halo=2)
st = torch.cat([torch.zeros(28), torch.ones(28)]).cuda()
import os
PREC = xmgn.PREC_BF16 if os.environ.get("SAN_PREC") == "bf16" else xmgn.PREC_FP16
for H in (int(a) for a in sys.argv[1:] or ["128", "512"]):
    pr = Processor(b, H, 2, precision=PREC)
    params, io = pr.make_params(), pr.make_io_params()
    gp, gio = torch.zeros(pr.n_params, device="cuda"), torch.zeros_like(io)
    loss = torch.zeros(1, device="cuda")
    for p in pr.parts:
        h0, e0, g = pr.make_inputs(p)
        pr.forward(p, params, h0, e0)
        pr.backward(p, params, g, gp, want_inputs=True)
        pos, nrm, t = pr.make_model_inputs(p, b)
        pr.model_forward(p, params, io, pos, nrm, st, t, 1500, loss)
        pr.model_backward(p, params, io, gp, gio)
    torch.cuda.synchronize()
    pr.close()
    print("H", H, "ok", float(loss.item()))
out = xmgn.build_graph(torch.as_tensor(b["positions"], device="cuda"), (300, 1200), 6, 2, 2)
assert np.array_equal(out["sources"], b["sources"])
print("build ok")
