"""A/B timing of chain-kernel variants (XMGN_LIB_OVERRIDE selects the library).
usage: XMGN_LIB_OVERRIDE=... python scratch/ab.py <tag> [n_points] [H] [L]"""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from xmgn_inputs import configs
from paper_2411_17164_b200 import xmgn
from paper_2411_17164_b200.processor import Processor
tag = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 400000
H = int(sys.argv[3]) if len(sys.argv) > 3 else 512
L = int(sys.argv[4]) if len(sys.argv) > 4 else 3
cache = f"/tmp/ab_graph_{n}.npz"
if os.path.exists(cache):
    b = dict(np.load(cache))
else:
    b = configs.custom((n,), k=6, P=1, halo=L, shape="car")
    np.savez(cache, **b)
pr = Processor(b, H, L, precision=xmgn.PREC_FP16, halo_depth=L)
params = pr.make_params()
h0, e0, g = pr.make_inputs(0)
gp = torch.zeros(pr.n_params, device="cuda")
for _ in range(2):
    gp.zero_()
    out = pr.forward(0, params, h0, e0)
    pr.backward(0, params, g, gp)
torch.cuda.synchronize()
dbgs = os.environ.get("AB_DBG", "0").split(",")
for dbg in dbgs:
    os.environ["XMGN_DBG"] = dbg
    for _ in range(1):
        gp.zero_(); out = pr.forward(0, params, h0, e0); pr.backward(0, params, g, gp)
    torch.cuda.synchronize()
    xmgn.profile_enable(True); xmgn.profile_collect()
    K = 3
    t = time.time()
    for _ in range(K):
        gp.zero_()
        out = pr.forward(0, params, h0, e0)
        pr.backward(0, params, g, gp)
    torch.cuda.synchronize()
    wall = (time.time() - t) / K
    prof = xmgn.profile_collect()
    res = {"tag": tag, "dbg": dbg, "wall_ms": round(wall * 1e3, 2), "E": int(pr.info[0]["e_local"]),
           "scopes": {k: round(v[0] / K, 3) for k, v in sorted(prof.items(), key=lambda kv: -kv[1][0])}}
    ref = f"/tmp/ab_ref_{n}_{H}_{L}.pt"
    if not os.path.exists(ref):
        torch.save({"out": out.cpu(), "gp": gp.cpu()}, ref)
    else:
        r = torch.load(ref)
        res["d_out"] = float((out.cpu() - r["out"]).abs().max() / r["out"].pow(2).mean().sqrt())
        res["d_gp"] = float((gp.cpu() - r["gp"]).norm() / r["gp"].norm())
    print(json.dumps(res), flush=True)
