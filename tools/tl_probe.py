"""Timeline of CTA 0 of one conv launch (PST_DBG_TL): us since kernel start per event.
usage: python tools/tl_probe.py [g1|g2|g3] [fwd|wgrad]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["PST_DBG_TL"] = "1"
import torch
from paper_1912_12675_b200 import ops
shapes = {"g1": (128, 16, 32), "g2": (128, 32, 16), "g3": (128, 64, 8)}
which = sys.argv[1] if len(sys.argv) > 1 else "g1"
kind = sys.argv[2] if len(sys.argv) > 2 else "fwd"
a = torch.randn(8192, 8192, device="cuda")
for _ in range(20): a @ a
N, C, H = shapes[which]
x = torch.randn(N, C, H, H, device="cuda"); w = torch.randn(C, C, 3, 3, device="cuda")
for _ in range(3): a @ a
if kind == "fwd": ops.conv2d_fwd(x, w, 1, 1)
else: ops.conv2d_wgrad(x, x, 3, 1, 1)
torch.cuda.synchronize()
print("^^", which, kind, os.environ.get("PST_TS_KNOB", "0"), flush=True)
