import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import oracle
from xmgn_inputs import configs, tensors
from paper_2411_17164_b200 import xmgn
from paper_2411_17164_b200.processor import Processor

def run(bundle, H, L, prec, P_label):
    t = time.time()
    pr = Processor(bundle, H, L, precision=prec)
    params = pr.make_params()
    N = len(bundle['offsets']) - 1; E = len(bundle['sources'])
    gp = torch.zeros(pr.n_params, device='cuda')
    hout = {}; gh = np.zeros((N, H)); ge = np.zeros((E, H))
    for p in pr.parts:
        h0, e0, g = pr.make_inputs(p)
        hout[p] = pr.forward(p, params, h0, e0)
        a, b = pr.backward(p, params, g, gp, want_inputs=True)
        inf = pr.info[p]
        np.add.at(gh, inf['gid'], a.double().cpu().numpy())
        np.add.at(ge, inf['edge_gid'], b.double().cpu().numpy())
    torch.cuda.synchronize()
    hfull = np.zeros((N, H))
    for p in pr.parts:
        inf = pr.info[p]
        hfull[inf['gid'][:inf['n_owned']]] = hout[p].double().cpu().numpy()
    print(P_label, 'gpu time', time.time() - t, flush=True)
    return hfull, gp.double().cpu().numpy(), gh, ge

def main():
    b = configs.custom((2000,), k=6, P=1, halo=2)
    b4 = configs.custom((2000,), k=6, P=4, halo=2)
    H, L = 128, 2
    off, src = b['offsets'], b['sources']
    N, E = len(off)-1, len(src)
    params = tensors.params(H, L).double().numpy()
    h0 = tensors.node_features(np.arange(N), H).double().numpy()
    e0 = tensors.edge_features(np.arange(E), H).double().numpy()
    g = tensors.upstream_grad(np.arange(N), H).double().numpy()
    f = oracle.forward(off, src, params, h0, e0, H, L)
    bk = oracle.backward(off, src, params, f, g, H, L)
    ref = f['h'][-1]; rms = np.sqrt((ref**2).mean())
    for prec, name in [(1, 'fp32check'), (0, 'bf16')]:
        for bb, lab in [(b, 'P1'), (b4, 'P4')]:
            try:
                h, gp, gh, ge = run(bb, H, L, prec, name + lab)
            except Exception as ex:
                print(name, lab, 'ERROR', ex, flush=True); continue
            err = np.abs(h - ref).max() / rms
            gerr = np.linalg.norm(gp - bk['params']) / np.linalg.norm(bk['params'])
            gherr = np.linalg.norm(gh - bk['h0']) / np.linalg.norm(bk['h0'])
            geerr = np.linalg.norm(ge - bk['e0']) / np.linalg.norm(bk['e0'])
            # per-tensor
            lay, _ = tensors.param_layout(H, L)
            worst = (0, '')
            for nm, l, blk, slot, o, shape, fan in lay:
                n = int(np.prod(shape)); r = bk['params'][o:o+n]; d = gp[o:o+n]
                e_ = np.linalg.norm(d - r) / max(np.linalg.norm(r), 1e-30)
                if e_ > worst[0]: worst = (e_, f'{nm} l{l} b{blk}')
            print(name, lab, 'fwd max/rms', err, 'grad rel', gerr, 'worst tensor', worst, 'gh0', gherr, 'ge0', geerr, flush=True)

main()
