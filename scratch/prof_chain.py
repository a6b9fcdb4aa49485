import sys, torch
sys.path.insert(0, '.')
from xmgn_inputs import configs
from paper_2411_17164_b200.processor import Processor
H = int(sys.argv[1]) if len(sys.argv) > 1 else 512
n = int(sys.argv[2]) if len(sys.argv) > 2 else 100000
b = configs.load('cfg2') if n == 100000 else configs.custom((n,), k=6, P=1, halo=2, shape='car')
pr = Processor(b, H, 2, precision=2, halo_depth=15 if n == 100000 else 2)
params = pr.make_params()
h0, e0, g = pr.make_inputs(0)
gp = torch.zeros(pr.n_params, device='cuda')
for it in range(2):
    pr.forward(0, params, h0, e0); pr.backward(0, params, g, gp)
torch.cuda.synchronize()
print('done')
