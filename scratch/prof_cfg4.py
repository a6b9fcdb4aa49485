"""One fwd+bwd of CFG4 partition 0 (H=512, L=15, FP16) -- a target for ncu/sanitizer captures."""
import sys, torch
sys.path.insert(0, '.')
from xmgn_inputs import configs
from paper_2411_17164_b200.processor import Processor
cfgname = sys.argv[1] if len(sys.argv) > 1 else 'cfg4'
b = configs.load(cfgname)
c = configs.CONFIGS[cfgname]
pr = Processor(b, c['H'], c['L'], precision=2, parts=[0])
params = pr.make_params()
h0, e0, g = pr.make_inputs(0)
gp = torch.zeros(pr.n_params, device='cuda')
pr.forward(0, params, h0, e0); pr.backward(0, params, g, gp)
torch.cuda.synchronize()
print('done')
