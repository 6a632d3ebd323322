"""Timeline of CTA 0 of one TS forward conv (PST_DBG_TL): per event the clock64 stamps (kcycles since
kernel start) -- band TMA issue, converter group start/done, MMA group issue, epilogue start/done.
usage: PST_DBG_TL=1 python tools/tl_probe.py g1|g2|g3"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1912_12675_b200 import ops
shapes = {"g1": (128, 16, 32, 16), "g2": (128, 32, 16, 32), "g3": (128, 64, 8, 64)}
N, C, H, Co = shapes[sys.argv[1] if len(sys.argv) > 1 else "g1"]
x = torch.randn((N, C, H, H), device="cuda")
w = torch.randn((Co, C, 3, 3), device="cuda")
for _ in range(3):
    ops.conv2d_fwd(x, w, 1, 1)
if len(sys.argv) > 2 and sys.argv[2] == "wgrad":
    gy = torch.randn((N, Co, H, H), device="cuda")
    for _ in range(2):
        ops.conv2d_wgrad(x, gy, 3, 1, 1)
