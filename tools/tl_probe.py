import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["PST_DBG_TL"] = "1"
import torch
from paper_1912_12675_b200 import ops
# warm the GPU clocks first
a = torch.randn(8192, 8192, device="cuda")
for _ in range(20): a @ a
for (N, C, H, k, pad) in [(128, 16, 32, 3, 1), (128, 32, 16, 3, 1), (128, 64, 8, 3, 1)]:
    x = torch.randn(N, C, H, H, device="cuda"); w = torch.randn(C, C, k, k, device="cuda")
    gy = torch.randn(N, C, H, H, device="cuda")
    for _ in range(3): a @ a
    ops.conv2d_fwd(x, w, 1, pad); torch.cuda.synchronize()
    for _ in range(3): a @ a
    ops.conv2d_wgrad(x, gy, k, 1, pad); torch.cuda.synchronize()
    print("^^ case", N, C, H, k, pad, flush=True)
