"""Probe: does TMA zero-fill (OOB boxes) slow the conv kernels?  Run under ncu."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1912_12675_b200 import ops
for (N, C, H, k, pad) in [(128, 16, 32, 3, 1), (128, 16, 34, 3, 0), (128, 16, 32, 1, 0)]:
    x = torch.randn(N, C, H, H, device="cuda")
    w = torch.randn(C, C, k, k, device="cuda")
    Ho = H + 2 * pad - k + 1
    gy = torch.randn(N, C, Ho, Ho, device="cuda")
    ops.conv2d_fwd(x, w, 1, pad)
    ops.conv2d_wgrad(x, gy, k, 1, pad)
    torch.cuda.synchronize()
    print("case", N, C, H, k, pad, flush=True)
