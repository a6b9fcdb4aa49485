import sys, time, os, numpy as np, torch
sys.path.insert(0, '.')
import oracle
from xmgn_inputs import configs, tensors
from paper_2411_17164_b200 import xmgn
from paper_2411_17164_b200.processor import Processor

precs = [int(x) for x in sys.argv[1].split(',')] if len(sys.argv) > 1 else [0]
cfg = sys.argv[2] if len(sys.argv) > 2 else 'cfg2'
b = configs.load(cfg)
H, L = 128, 15
outs = {}
for prec in precs:
    pr = Processor(b, H, L, precision=prec)
    params = pr.make_params()
    h0, e0, g = pr.make_inputs(0)
    gp = torch.zeros(pr.n_params, device='cuda')
    for it in range(3):
        out = pr.forward(0, params, h0, e0); pr.backward(0, params, g, gp)
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    for it in range(5):
        out = pr.forward(0, params, h0, e0); pr.backward(0, params, g, gp)
    t1.record(); torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / 5
    E = len(b['sources'])
    print(f'{cfg} prec={prec} step {ms:.2f} ms, {E/ms*1e3/1e6:.2f} M edges/s, ws {pr.ws.nbytes()/1e9:.2f} GB', flush=True)
    t0.record(); out = pr.forward(0, params, h0, e0); t1.record(); torch.cuda.synchronize()
    print('fwd ms', t0.elapsed_time(t1), flush=True)
    outs[prec] = out.double().cpu().numpy()
    P = params.double().cpu().numpy(); hh = h0.double().cpu().numpy(); ee = e0.double().cpu().numpy()
    pr.close()
t = time.time()
off, src = b['offsets'], b['sources']
f = oracle.forward(off, src, P, hh, ee, H, L)
print('oracle fwd s', time.time() - t, 'threads', os.cpu_count(), flush=True)
ref = f['h'][-1]
rms = np.sqrt((ref ** 2).mean())
for prec, out in outs.items():
    err = np.abs(out - ref)
    print('prec', prec, 'max/rms', err.max() / rms, 'p99.99/rms', np.quantile(err, 0.9999) / rms, 'rms', rms, flush=True)
