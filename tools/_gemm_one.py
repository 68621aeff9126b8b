import sys, torch
sys.path.insert(0, '.')
from paper_2507_11507_b200 import _lib
N, K = 5120, 5120
w = torch.randn((N, K), device="cuda").to(torch.bfloat16)
for B in (64, 128):
    x = torch.randn((B, K), device="cuda").to(torch.bfloat16)
    for _ in range(3):
        _lib.decode_gemm(w, x)
torch.cuda.synchronize()
