import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
from paper_1912_12675_b200 import ops
from oracle import layers as Lx
for (N, Cin, H, W, Cout, k, S, p) in [(128, 64, 1, 1, 10, 1, 1, 0), (128, 16, 32, 32, 16, 3, 1, 1)]:
    x = torch.randn(N, Cin, H, W); gy = torch.randn(N, Cout, (H+2*p-k)//S+1, (W+2*p-k)//S+1)
    gw = ops.conv2d_wgrad(x.cuda(), gy.cuda(), k, S, p).cpu().numpy()
    _, ref, _ = Lx.conv2d_backward(x.double().numpy(), np.zeros((Cout, Cin, k, k)), gy.double().numpy(), S, p, need_gx=False)
    print("wgrad", (N, Cin, H, W, Cout, k), float(np.abs(gw-ref).max()/np.abs(ref).max()))
