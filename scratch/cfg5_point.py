"""CFG5 (BASELINE.json configs[4]: 2.5M/5M/10M-point car cloud, k=6, H=512, L=15, 32 halo
partitions on 8 B200) sized against one GPU's HBM and timed for one rank's share.

The graph is built on the GPU by xmgn_build_graph (NEXT-4).  Rank 0 of 8 owns partitions 0-3
(contiguous blocks); their processor fwd+bwd (inputs generated per partition
outside the timed region) is timed with CUDA events.  Prints one JSON line."""
import json, sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
from xmgn_inputs import configs, geometry
from paper_2411_17164_b200 import xmgn
from paper_2411_17164_b200.processor import Processor

c = configs.CONFIGS["cfg5"]
t0 = time.time()
pos, nrm = geometry.nested_levels(c["levels"], shape="car", seed=0)
t_geo = time.time() - t0
pt = torch.as_tensor(pos, device="cuda")
torch.cuda.synchronize()
t0 = time.time()
b = xmgn.build_graph(pt, c["levels"], c["k"], c["P"], c["L"])
torch.cuda.synchronize()
t_build = time.time() - t0
del pt
b["positions"], b["normals"] = pos, nrm
E = len(b["sources"])
world, rank = 8, 0
parts = list(range(rank * c["P"] // world, (rank + 1) * c["P"] // world))
pr = Processor(b, c["H"], c["L"], precision=xmgn.PREC_FP16, parts=parts)
ws_bytes = pr.ws.nbytes()
params = pr.make_params()
gp = torch.zeros(pr.n_params, device="cuda")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ms, rows = 0.0, 0
for rep in range(2):            # rep 0 warms up
    tot = 0.0
    for p in parts:
        h0, e0, g = pr.make_inputs(p)
        torch.cuda.synchronize()
        ev[0].record()
        pr.forward(p, params, h0, e0)
        pr.backward(p, params, g, gp)
        ev[1].record()
        torch.cuda.synchronize()
        tot += ev[0].elapsed_time(ev[1])
        if rep == 1:
            rows += pr.info[p]["e_local"]
        del h0, e0, g
    ms = tot
peak = torch.cuda.max_memory_allocated() + ws_bytes
e_loc = [int(b["halo_offsets"][p + 1] - b["halo_offsets"][p]) for p in range(c["P"])]
print(json.dumps({"config": "cfg5", "levels": c["levels"], "E_global": E, "partitions": c["P"],
                  "rank0_parts": parts, "geometry_s": round(t_geo, 1), "gpu_graph_build_s": round(t_build, 2),
                  "workspace_GB": round(ws_bytes / 1e9, 1), "peak_GB_incl_torch": round(peak / 1e9, 1),
                  "rank0_ms_fwd_bwd": round(ms, 1), "rank0_local_edges": rows,
                  "est_8gpu_edges_per_s_if_balanced": round(E / (ms / 1e3)),
                  "halo_nodes_per_part_max": max(e_loc)}), flush=True)
