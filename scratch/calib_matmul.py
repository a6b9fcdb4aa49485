"""Tensor-counter calibration: a dense bf16 8192^3 torch.matmul (cuBLAS) whose
ncu sm__pipe_tensor_cycles_active % is the scale the chain kernels' counter is read against."""
import torch
a = torch.randn(8192, 8192, device='cuda', dtype=torch.bfloat16)
b = torch.randn(8192, 8192, device='cuda', dtype=torch.bfloat16)
for _ in range(3):
    c = a @ b
torch.cuda.synchronize()
print('done')
