"""Per-launch device time of the conv kernels at the ResNet-CIFAR shapes (B=128), graph replay
on resident buffers.  usage: python tools/conv_lab.py [iters]   (env knobs pass through)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1912_12675_b200 import ops
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 50
shapes = [("g1", 128, 16, 32, 16), ("g2", 128, 32, 16, 32), ("g3", 128, 64, 8, 64)]
tag = os.environ.get("LAB_TAG", "")
for name, N, C, H, Co in shapes:
    t = [ops.time_conv(w, N, C, H, H, Co, 3, 1, 1, iters) for w in (0, 1, 2)]
    print(f"{tag} {name} fwd {t[0]:7.2f} us  dgrad {t[1]:7.2f} us  wgrad {t[2]:7.2f} us", flush=True)
