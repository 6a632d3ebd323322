"""Kernel-level parity (GPU): the tcgen05 implicit-GEMM convolution passes against
the float64 oracle (oracle/layers.py) on the same compute-dtype-rounded inputs.

Inputs are rounded to the library's compute dtype first, so both sides see
identical operands; products of two 8-bit-mantissa values are exact in float32,
leaving only float32 summation order (fwd, wgrad: float32 outputs) and the
final output rounding (dgrad: compute-dtype output, |err| <= 2^-8 relative).
Shapes span several 128-pixel tiles, ragged tails (W=28, 10x10, 5x5, N not a
multiple of the tile), padded channels (3, 6, 10, 84, 120), stride 2 and FC.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import layers as Lx

pytestmark = pytest.mark.gpu

CASES = [
    # N, Cin, H, W, Cout, k, stride, pad
    (4, 16, 32, 32, 16, 3, 1, 1),     # ResNet group 1
    (3, 16, 32, 32, 32, 3, 2, 1),     # ResNet downsample 16->32 (stride 2)
    (2, 32, 16, 16, 64, 3, 2, 1),     # ResNet downsample 32->64
    (5, 64, 8, 8, 64, 3, 1, 1),       # ResNet group 3, two images per tile, ragged N
    (3, 3, 32, 32, 16, 3, 1, 1),      # conv1: 3 input channels (padded to 16)
    (2, 1, 28, 28, 6, 5, 1, 2),       # LeNet conv1: W=28 ragged tile, Cout 6
    (3, 6, 14, 14, 16, 5, 1, 0),      # LeNet conv2: no padding, 10x10 output
    (2, 64, 16, 16, 192, 5, 1, 2),    # AlexNet conv2 (Cout 192)
    (2, 192, 8, 8, 384, 3, 1, 1),     # AlexNet conv3 (Cout 384 -> 3 N tiles)
    (2, 512, 2, 2, 512, 3, 1, 1),     # VGG late layer (Cout 512)
    (37, 400, 1, 1, 120, 1, 1, 0),    # LeNet FC1 as 1x1 (ragged batch)
    (130, 84, 1, 1, 10, 1, 1, 0),     # FC -> logits, batch > one tile
]


def rnd(t):
    """Round to the library's storage dtype (identity for the float32 build)."""
    from paper_1912_12675_b200 import build_info
    info = build_info()
    if "act=f16" in info:
        return t.to(torch.float16).to(torch.float32)
    if "act=bf16" in info:
        return t.to(torch.bfloat16).to(torch.float32)
    return t


def tol(kind):
    """float32-storage 3xTF32 build: ~1e-6 relative; 16-bit builds: summation order /
    output rounding only (inputs pre-rounded)."""
    from paper_1912_12675_b200 import build_info
    f32 = "f32" in build_info()
    return {"fwd": 1e-4 if f32 else 2e-5, "dgrad": 1e-4 if f32 else 8e-3, "wgrad": 1e-4 if f32 else 2e-5}[kind]


@pytest.fixture(scope="module")
def ops():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1912_12675_b200 import ops as o
    return o


def _rel(a, b):
    return float(np.abs(a - b).max() / max(1e-12, np.abs(b).max()))


@pytest.mark.parametrize("case", CASES, ids=[str(c) for c in CASES])
def test_conv_fwd(ops, case):
    N, Cin, H, W, Cout, k, S, p = case
    g = torch.Generator().manual_seed(1)
    x = rnd(torch.randn(N, Cin, H, W, generator=g))
    w = rnd(torch.randn(Cout, Cin, k, k, generator=g) / np.sqrt(Cin * k * k))
    y = ops.conv2d_fwd(x.cuda(), w.cuda(), S, p).cpu().numpy()
    ref = Lx.conv2d_forward(x.double().numpy(), w.double().numpy(), None, S, p)
    assert y.shape == ref.shape
    assert _rel(y, ref) < tol("fwd"), _rel(y, ref)


@pytest.mark.parametrize("case", CASES, ids=[str(c) for c in CASES])
def test_conv_dgrad(ops, case):
    N, Cin, H, W, Cout, k, S, p = case
    g = torch.Generator().manual_seed(2)
    Ho, Wo = (H + 2 * p - k) // S + 1, (W + 2 * p - k) // S + 1
    gy = rnd(torch.randn(N, Cout, Ho, Wo, generator=g))
    w = rnd(torch.randn(Cout, Cin, k, k, generator=g) / np.sqrt(Cout * k * k))
    gx = ops.conv2d_dgrad(gy.cuda(), w.cuda(), (H, W), S, p).cpu().numpy()
    x0 = np.zeros((N, Cin, H, W))
    ref, _, _ = Lx.conv2d_backward(x0, w.double().numpy(), gy.double().numpy(), S, p)
    assert _rel(gx, ref) < tol("dgrad"), _rel(gx, ref)


@pytest.mark.parametrize("case", CASES, ids=[str(c) for c in CASES])
def test_conv_wgrad(ops, case):
    N, Cin, H, W, Cout, k, S, p = case
    g = torch.Generator().manual_seed(3)
    Ho, Wo = (H + 2 * p - k) // S + 1, (W + 2 * p - k) // S + 1
    x = rnd(torch.randn(N, Cin, H, W, generator=g))
    gy = rnd(torch.randn(N, Cout, Ho, Wo, generator=g))
    gw = ops.conv2d_wgrad(x.cuda(), gy.cuda(), k, S, p).cpu().numpy()
    _, ref, _ = Lx.conv2d_backward(x.double().numpy(), np.zeros((Cout, Cin, k, k)), gy.double().numpy(), S, p,
                                   need_gx=False)
    assert _rel(gw, ref) < tol("wgrad"), _rel(gw, ref)
