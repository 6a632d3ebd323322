"""CPU oracle for pipelined backpropagation with stale weights (arXiv 1912.12675).

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import anything
from this package.  The product path (`paper_1912_12675_b200`, `libpst.so`)
never imports, links or executes it, and this package never imports the
product path; the two share no code.  The only common inputs come from
`pst_workloads` (seeded nets/init/data, no arithmetic).

Plain, slow, obviously-correct NumPy in float64 (the paper does not fix the
precision; GTX1060 FP32 is presumed, reading AMB-20), following the paper in
its order and notation:

  layers.py    per-op forward/backward definitions (§2)
  network.py   a stage = contiguous weighted layers; forward x^(l) and
               backward delta^(l) through a stage
  pipeline.py  Oracle A (mini-batch order + weight-version history, the
               definition) and Oracle B (the step-clocked schedule
               P:L61/L67/L183), hybrid training, staleness metrics.

Parity pins (tests/test_oracle_*.py): finite differences for every VJP,
PyTorch-CPU fp64 functional ops, K=1 == textbook SGD (torch autograd +
torch.optim.SGD), Oracle A == Oracle B bitwise, version log == closed form
max(0, i - 2(K-1-s)), the hand-derived scalar worked example
(tests/golden/scalar_pipeline_k2.json), Table 6 parameter counts.
Parity unpinned: nothing in the oracle beyond the readings listed in
DESIGN.md (the paper prints no numeric worked example of its own; the
scalar example is derived from P:L61-75).
"""
from . import layers, network, pipeline  # noqa: F401
