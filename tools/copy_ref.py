"""Reference memory-bound kernels of the window kernel's traffic shape (for ncu): fp32 -> fp16 conversion of
23.04M floats (92 MB read, 46 MB write, = 1024 beds x 3 leads x 7500) and a same-size fp32 copy."""
import torch
n = 1024 * 3 * 7500
x = torch.randn(n, device="cuda")
y = torch.empty(n, device="cuda", dtype=torch.float16)
z = torch.empty(n, device="cuda")
big = torch.empty(64 * 1024 * 1024, device="cuda")
for _ in range(4):
    big.zero_()
    y.copy_(x)
    big.zero_()
    z.copy_(x)
torch.cuda.synchronize()
print("ok")
