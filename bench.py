"""Benchmark: partitioned X-MeshGraphNet processor fwd+bwd (15 layers) on B200.

Metric (BASELINE.json): processor edges/s fwd+bwd (15 layers) at 1/2/4/8 B200,
with the dominant kernel's roofline fraction.  Workload: CFG4 -- the 2M-point
3-level (500k/1M/2M) car-proxy cloud, k=6, H=512, L=15, m=2,
8 RCB partitions with halo 15, spread over the ranks in contiguous blocks.

One step = fwd + bwd of every partition of this rank (gradients summed in
partition order) + one NCCL all-reduce of the flat FP32 gradient
(xmgn_grad_reduce) when N > 1.  value = global unique directed edges x ranks'
steps / max-over-ranks device time.  Inputs (h0, e0, g per partition) are
generated on the device before the timed region; every per-partition tensor is
far larger than L2 (e0 alone is ~6.6 GB), so no explicit flush is needed.

--impl reference: the FP64 CPU oracle (oracle/, the tier's reference arm) on a
bounded sample of the same workload, rank 0 only.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

H, L, M_HID = 512, 15, 2
METRIC = "processor edges/s fwd+bwd (15 layers)"


def assign_parts(P, world, rank):
    """Contiguous blocks of partitions per rank (RCB order), SURVEY §8(e)."""
    return list(range(rank * P // world, (rank + 1) * P // world))


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return None


# ---------------------------------------------------------------- CPU oracle sample
def oracle_sample(bundle, target_edges, H_=H, L_=L, m=M_HID):
    """A connected subgraph of the workload (BFS ball around node 0 grown until it
    holds >= target_edges local edges) as a single owned set: returns its CSR."""
    import oracle
    off, src = bundle["offsets"], bundle["sources"]
    seed = np.array([int(bundle["owned"][0])])
    for depth in range(1, 40):
        lg = oracle.local_graph(off, src, seed, depth)
        if len(lg["sources"]) >= target_edges:
            break
    return lg


def time_oracle(lg, H_=H, L_=L, m=M_HID, reps=1):
    import oracle
    from xmgn_inputs import tensors
    P = tensors.params(H_, L_, m).double().numpy()
    h0 = tensors.node_features(lg["gid"], H_).double().numpy()
    e0 = tensors.edge_features(lg["edge_gid"], H_).double().numpy()
    g = tensors.upstream_grad(lg["gid"], H_).double().numpy()
    ts = []
    for _ in range(reps):
        t = time.perf_counter()
        f = oracle.forward(lg["offsets"], lg["sources"], P, h0, e0, H_, L_, m)
        oracle.backward(lg["offsets"], lg["sources"], P, f, g, H_, L_, m)
        ts.append(time.perf_counter() - t)
    return ts


def cpu_cores():
    return int(os.environ.get("OMP_NUM_THREADS", os.cpu_count()))


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


# ---------------------------------------------------------------- clocks
class Clocks:
    def __init__(self, device):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None
        self.device = device

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={self.device}", f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        if self.p:
            self.p.terminate()
            self.p.wait()

    def summary(self):
        self.f.flush()
        rows = []
        for line in open(self.f.name):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 9:
                rows.append(parts)
        os.unlink(self.f.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ---------------------------------------------------------------- algorithmic work per scope
def scope_work(info, H_=H, L_=L, m=M_HID):
    """Algorithmic FLOPs (MMA work the method needs; recompute excluded) and
    executed FLOPs per launch scope for one fwd+bwd of one partition, plus the
    aggregation's algorithmic bytes.  Rows per layer follow halo shrinking."""
    rn, re_ = info["ring_nodes"], info["ring_edges"]
    n_at = lambda l: rn[L_ - l + 1]  # noqa: E731
    e_at = lambda l: re_[L_ - l + 1]  # noqa: E731
    H2 = H_ * H_
    w = {}

    def add(k, alg, exe=None):
        a, e = w.get(k, (0.0, 0.0))
        w[k] = (a + alg, e + (alg if exe is None else exe))
    add("chain_proj", 2 * 2 * H2 * n_at(0))                       # fwd P for layer 1
    for l in range(1, L_ + 1):
        nl, el, npv = n_at(l), e_at(l), n_at(l - 1)
        add("chain_edge_fwd", 2 * (1 + m) * H2 * el)
        add("chain_node_fwd", 2 * ((2 + m) * H2 + (2 * H2 if l < L_ else 0)) * nl)
        add("aggregate", 0)
        fw_e, fw_n = 2 * (1 + m) * H2 * el, 2 * (2 + m) * H2 * nl
        add("chain_node_bwd", 2 * (m + 2) * H2 * nl, fw_n + 2 * (m + 2) * H2 * nl)
        add("chain_edge_bwd", 2 * (m + 1) * H2 * el, fw_e + 2 * (m + 1) * H2 * el)
        add("chain_projbwd", 2 * 2 * H2 * npv)
        add("wgrad", 2 * ((2 + m) * H2 * nl + (1 + m) * H2 * el + 2 * H2 * npv))
    agg_bytes = sum(2 * H_ * e_at(l) + 2 * H_ * n_at(l) for l in range(1, L_ + 1))   # 16-bit edge rows in, 16-bit a out
    rows = {"chain_edge_bwd": sum(e_at(l) for l in range(1, L_ + 1)),
            "chain_edge_fwd": sum(e_at(l) for l in range(1, L_ + 1)),
            "chain_node_bwd": sum(n_at(l) for l in range(1, L_ + 1)),
            "chain_node_fwd": sum(n_at(l) for l in range(1, L_ + 1))}
    return w, agg_bytes, rows


def relaunch(n):
    """`bench.py --gpus N` outside torchrun: start N ranks (one process per GPU,
    NCCL) on this node with torch.distributed.run and pass rank 0's output through."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="xmgn", choices=["xmgn", "reference"])
    ap.add_argument("--config", default="cfg4")
    ap.add_argument("--precision", default="fp16", choices=["fp16", "bf16"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-model", action="store_true")
    ap.add_argument("--no-bf16-leg", action="store_true")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "xmgn":
        return relaunch(args.gpus)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return reference(args, world, rank)

    import torch
    import torch.distributed as dist
    from xmgn_inputs import configs
    from paper_2411_17164_b200 import xmgn
    from paper_2411_17164_b200.processor import Processor

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    cfg = configs.CONFIGS[args.config]
    Hc, Lc = cfg["H"], cfg["L"]
    # rank 0 builds (and caches) the graph, the others read the cache
    if world > 1 and rank != 0:
        dist.barrier()
    t_gen = time.time()
    bundle = configs.load(args.config)
    t_gen = time.time() - t_gen
    if world > 1 and rank == 0:
        dist.barrier()
    P = len(bundle["owned_offsets"]) - 1
    parts = assign_parts(P, world, rank)
    prec = xmgn.PREC_FP16 if args.precision == "fp16" else xmgn.PREC_BF16
    pr = Processor(bundle, Hc, Lc, m=M_HID, precision=prec, device=local, parts=parts, halo_depth=Lc)
    E_global = int(len(bundle["sources"]))
    params = pr.make_params()
    grad = torch.zeros(pr.n_params, device=dev)
    inputs = {p: pr.make_inputs(p) for p in parts}
    comm = None
    if world > 1:
        uid = [xmgn.Comm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = xmgn.Comm(uid[0], world, rank, local)
    stream = torch.cuda.current_stream()

    def step():
        grad.zero_()
        pr.step(params, grad, inputs, stream)
        if comm is not None:
            comm.grad_reduce(grad, stream)

    def sync_all():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
            torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    sync_all()
    xmgn.profile_enable(True)
    xmgn.profile_collect()
    l0 = xmgn.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    with Clocks(local) as clk:
        ev0.record(stream)
        evs[0].record(stream)
        for i in range(args.steps):
            step()
            evs[i + 1].record(stream)
        ev1.record(stream)
        sync_all()
    step_ms = [evs[i].elapsed_time(evs[i + 1]) for i in range(args.steps)]
    launches = xmgn.launch_count() - l0
    xmgn.profile_enable(False)
    prof = xmgn.profile_collect()
    ms = ev0.elapsed_time(ev1) / args.steps
    t = torch.tensor([ms], device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    value = E_global / (ms / 1e3)
    clocks = clk.summary()
    xmgn.check_finite(grad)

    # ---- roofline of the dominant kernel scope (this rank's live CUDA-event timings)
    work = {}
    agg_bytes = 0
    scope_rows = {}
    for p in parts:
        w, ab, rws = scope_work(pr.info[p], Hc, Lc, M_HID)
        agg_bytes += ab
        for k, v in rws.items():
            scope_rows[k] = scope_rows.get(k, 0) + v
        for k, (a, e) in w.items():
            A, Ee = work.get(k, (0.0, 0.0))
            work[k] = (A + a, Ee + e)
    pk = peaks() or {}
    dom = max(prof, key=lambda k: prof[k][0]) if prof else None
    roof = None
    if dom:
        tot_ms, n_launch = prof[dom]
        per_launch_s = tot_ms / 1e3 / n_launch
        if dom == "aggregate":
            achieved = agg_bytes * args.steps / n_launch / per_launch_s / 1e9
            peak, unit, bound, src = pk.get("hbm_gbs", 6650.0), "GB/s", "hbm", "measured" if pk else "fallback"
        else:
            alg = work.get(dom, (0.0, 0.0))[0] * args.steps / n_launch
            achieved = alg / per_launch_s / 1e12
            peak = pk.get("bf16_tflops_sustained", 1400.0)
            unit, bound, src = "TFLOP/s", "tensor", "measured sustained bf16 (fp16 same nominal rate)"
        # DRAM traffic per launch: dram__bytes_read.sum + dram__bytes_write.sum of one ncu --set
        # full capture of this scope (profiles/ncu_traffic.json, bytes per row of that launch),
        # scaled to this run's average rows per launch
        traffic = None
        tf = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(tf):
            ent = json.load(open(tf)).get(dom)
            rows = scope_rows.get(dom)
            if ent and rows and ent.get("config", args.config) == args.config:
                traffic = round(ent["bytes_per_row"] * rows * args.steps / n_launch)
        roof = {"bound": bound, "achieved": round(achieved, 2), "peak": peak, "unit": unit,
                "frac": round(achieved / peak, 4), "traffic": traffic, "kernel": dom, "peak_source": src,
                "launches": n_launch, "avg_launch_ms": round(tot_ms / n_launch, 4),
                "share_of_step": round(tot_ms / (ms * args.steps), 4)}
        exe = work.get(dom, (0.0, 0.0))[1] * args.steps / n_launch
        if exe and dom != "aggregate":
            roof["executed_tflops"] = round(exe / per_launch_s / 1e12, 2)
    scopes = {k: {"ms_per_step": round(v[0] / args.steps, 3), "launches_per_step": v[1] / args.steps}
              for k, v in sorted(prof.items(), key=lambda kv: -kv[1][0])}
    total_alg = sum(a for a, _ in work.values())
    t2 = torch.tensor([total_alg], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t2)

    # ---- e2e through the public API with host buffers (H2D inputs, D2H result)
    e2e = None
    if not args.no_e2e:
        host = {}
        for p in parts:
            host[p] = [x.cpu().pin_memory() for x in inputs[p]]
        grad_host = torch.empty(pr.n_params, dtype=torch.float32).pin_memory()
        bi = sum(x.numel() * 4 for p in parts for x in host[p])
        bo = grad_host.numel() * 4
        # two device staging sets (sized for the largest partition of this rank): partition
        # i+1's inputs are copied host->device on a copy stream while partition i computes
        del inputs
        torch.cuda.empty_cache()
        shapes = [max(host[p][j].shape[0] for p in parts) for j in range(3)]
        stage = [[torch.empty((shapes[j], Hc), dtype=torch.float32, device=dev) for j in range(3)] for _ in range(2)]
        cstream = torch.cuda.Stream(device=dev)
        ready = [torch.cuda.Event() for _ in range(2)]
        free = [torch.cuda.Event() for _ in range(2)]
        for f in free:
            f.record(stream)

        # staging sets are used round-robin over a running partition counter, and the last
        # partition of a step prefetches the NEXT step's first partition, so with one partition
        # per rank (CFG2) or at a step boundary the H2D copy overlaps compute too (a data-loader
        # style input pipeline: every step still copies every one of its inputs once)
        cnt = [0]

        def h2d(gi, p):
            b = gi % 2
            cstream.wait_event(free[b])
            with torch.cuda.stream(cstream):
                for j in range(3):
                    stage[b][j][:host[p][j].shape[0]].copy_(host[p][j], non_blocking=True)
            ready[b].record(cstream)

        def e2e_step(first=False):
            grad.zero_()
            if first:
                h2d(cnt[0], parts[0])
            for i, p in enumerate(parts):
                gi = cnt[0] + i
                b = gi % 2
                h2d(gi + 1, parts[i + 1] if i + 1 < len(parts) else parts[0])
                stream.wait_event(ready[b])
                h0, e0, g = (stage[b][j][:host[p][j].shape[0]] for j in range(3))
                pr.forward(p, params, h0, e0, stream)
                pr.backward(p, params, g, grad, stream=stream)
                free[b].record(stream)
            cnt[0] += len(parts)
            if comm is not None:
                comm.grad_reduce(grad, stream)
            grad_host.copy_(grad, non_blocking=True)

        e2e_step(first=True)
        sync_all()
        k2 = max(1, min(args.steps, 2))
        # the first timed step's first partition was prefetched (and landed) before ev0; the last
        # timed step prefetches the next one, which ev1 waits for: exactly K x P copies inside
        ev0.record(stream)
        for _ in range(k2):
            e2e_step()
        stream.wait_event(ready[cnt[0] % 2])
        ev1.record(stream)
        sync_all()
        ms2 = ev0.elapsed_time(ev1) / k2
        t3 = torch.tensor([ms2], device=dev)
        if world > 1:
            dist.all_reduce(t3, op=dist.ReduceOp.MAX)
        e2e = {"value": E_global / (float(t3.item()) / 1e3), "unit": "edges/s", "h2d_bytes_per_step": bi,
               "d2h_bytes_per_step": bo, "steps": k2,
               "note": "pinned host inputs copied on a second stream into two staging sets, each partition's "
                       "copy overlapping the previous partition's compute (across step boundaries too)"}
        del host, stage
        torch.cuda.empty_cache()

    # ---- the full training step of the paper's model (NEXT-1 + NEXT-2) through the public API:
    # encoders -> processor -> decoder -> owned-row MSE -> backward (every partition of this rank,
    # gradients summed) -> all-reduce -> global-norm clip + Adam + cosine LR over all parameters.
    # Inputs per step are positions / normals / targets (H2D from pinned host memory), the
    # result read back is the loss.  Feature stats: identity (the bench does not normalise).
    model = None
    if not args.no_model:
        if e2e is None:
            del inputs
            torch.cuda.empty_cache()
        n_io = xmgn.io_param_count(pr.cfg)
        allp = torch.empty(pr.n_params + n_io, device=dev)
        allp[:pr.n_params] = params
        allp[pr.n_params:] = pr.make_io_params()
        mparams, mio = allp[:pr.n_params], allp[pr.n_params:]
        allg = torch.zeros_like(allp)
        mgrad, mgio = allg[:pr.n_params], allg[pr.n_params:]
        opt = xmgn.Adam(allp.numel(), 2000, device=local)
        stats = torch.cat([torch.zeros(28), torch.ones(28)]).to(dev)
        N_global = len(bundle["offsets"]) - 1
        mhost = {}
        for p in parts:
            mhost[p] = [x.cpu().pin_memory() for x in pr.make_model_inputs(p, bundle)]
        mdev = {p: [torch.empty_like(x, device=dev) for x in mhost[p]] for p in parts}
        loss = torch.zeros(1, device=dev)
        loss_host = torch.empty(1).pin_memory()
        mbi = sum(x.numel() * 4 for p in parts for x in mhost[p])

        def model_step():
            allg.zero_()
            loss.zero_()
            for p in parts:
                for d, h in zip(mdev[p], mhost[p]):
                    d.copy_(h, non_blocking=True)
                pos, nrm, tg = mdev[p]
                pr.model_forward(p, mparams, mio, pos, nrm, stats, tg, N_global, loss, stream)
                pr.model_backward(p, mparams, mio, mgrad, mgio, stream)
            if comm is not None:
                comm.grad_reduce(allg, stream)
            opt.step(allp, allg, stream=stream)
            loss_host.copy_(loss, non_blocking=True)

        model_step()
        sync_all()
        k3 = max(1, min(args.steps, 2))
        ev0.record(stream)
        for _ in range(k3):
            model_step()
        ev1.record(stream)
        sync_all()
        t4 = torch.tensor([ev0.elapsed_time(ev1) / k3], device=dev)
        if world > 1:
            dist.all_reduce(t4, op=dist.ReduceOp.MAX)
        mms = float(t4.item())
        model = {"what": "encoders + processor + decoder + owned-row MSE, fwd+bwd of every partition, "
                         "gradient all-reduce, global-norm clip + Adam + cosine LR (xmgn_model_fwd/bwd, "
                         "xmgn_adam_step)",
                 "value": E_global / (mms / 1e3), "unit": "edges/s", "ms_per_step": mms, "steps": k3,
                 "h2d_bytes_per_step": mbi, "d2h_bytes_per_step": 4, "loss": float(loss_host.item()),
                 "processor_share": round(ms / mms, 4)}

    # ---- the same processor step with BF16 operands (north_star's precision; the FP16 headline
    # runs the same tcgen05 kind::f16 datapath): a fresh BF16 workspace, 1 warm-up + 2 timed steps
    bf16_leg = None
    if args.precision == "fp16" and not args.no_bf16_leg:
        if e2e is None and model is None:
            del inputs
        pr.close()
        torch.cuda.empty_cache()
        pr = Processor(bundle, Hc, Lc, m=M_HID, precision=xmgn.PREC_BF16, device=local, parts=parts,
                       halo_depth=Lc)
        inputs = {p: pr.make_inputs(p) for p in parts}
        step()
        sync_all()
        k5 = max(1, min(args.steps, 2))
        ev0.record(stream)
        for _ in range(k5):
            step()
        ev1.record(stream)
        sync_all()
        t5 = torch.tensor([ev0.elapsed_time(ev1) / k5], device=dev)
        if world > 1:
            dist.all_reduce(t5, op=dist.ReduceOp.MAX)
        bms = float(t5.item())
        bf16_leg = {"dtype": "bf16", "value": E_global / (bms / 1e3), "unit": "edges/s", "ms_per_step": bms,
                    "steps": k5, "note": "BF16 operands (FP32 edge stream, FP16 P, 2 x BF16 node first-GEMM "
                                         "and pre-projection operands): max|dh|/RMS 1.6e-2 <= 2e-2 at L = 15 "
                                         "(DESIGN.md section 3)"}
        del inputs

    # ---- CPU baseline: the oracle on a bounded sample (rank 0, N = 1)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        lg = oracle_sample(bundle, 2500)
        ts = time_oracle(lg, Hc, Lc)
        cpu = {"value": len(lg["sources"]) / ts[0], "unit": "edges/s", "cores": cpu_cores(), "cpu_model": cpu_model(), "kind": "oracle",
               "sample": f"FP64 oracle fwd+bwd, {Lc} layers, H={Hc}, on a {len(lg['sources'])}-edge "
                         f"{len(lg['gid'])}-node BFS ball of the {args.config} graph ({ts[0]:.1f} s)"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "edges/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "ms_per_step_median_rank0": statistics.median(step_ms),
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None, "dtype": args.precision, "data": "synthetic",
            "config": {"workload": f"{args.config}: {cfg['levels']} points, k={cfg['k']}, H={Hc}, L={Lc}, "
                                   f"m={M_HID}, {P} halo partitions (depth {Lc})",
                       "edges_global": E_global, "partitions": P, "partitions_per_gpu": len(parts),
                       "parallelism": f"halo-partition dp{world}", "l2": "inputs larger than L2 (no flush)",
                       "graph_build_s": round(t_gen, 1)},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "model_step": model, "bf16_step": bf16_leg,
            "clocks": clocks,
            "gpu_launches": launches,
            "alg_tflops_per_s": round(float(t2.item()) * args.steps / (ms * args.steps / 1e3) / 1e12, 2),
            "scopes": scopes,
        }
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
    pr.close()
    if world > 1:
        dist.destroy_process_group()


def reference(args, world, rank):
    """Reference arm: the FP64 oracle as it stands, on host cores, bounded samples."""
    if rank != 0:
        return
    from xmgn_inputs import configs
    cfg = configs.CONFIGS[args.config]
    bundle = configs.load(args.config)
    lg = oracle_sample(bundle, 600)
    for _ in range(args.warmup):
        time_oracle(lg, cfg["H"], cfg["L"])
    ts = time_oracle(lg, cfg["H"], cfg["L"], reps=args.steps)
    s = sum(ts) / len(ts)
    v = len(lg["sources"]) / s
    sample = (f"FP64 oracle fwd+bwd, {cfg['L']} layers, H={cfg['H']}, on a {len(lg['sources'])}-edge "
              f"{len(lg['gid'])}-node BFS ball of the {args.config} graph per step")
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "edges/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": s * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.config} (bounded sample)", "parallelism": "host cores"},
            "cpu_baseline": {"value": v, "unit": "edges/s", "cores": cpu_cores(), "cpu_model": cpu_model(), "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": v, "unit": "edges/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    sys.exit(main() or 0)
