"""The five BASELINE.json configs as data (nets, batch, partitions, hparams).

PPVs: paper values where the paper gives them (Table 1 PAPER.md L91-98,
Table 5), otherwise the roofline-balanced block-boundary PPVs of
SURVEY.md Appendix A -- except ResNet-110/362, whose PPVs come from the
profile-driven balancer (balance.py) on the per-layer costs
measured on the B200 (b200_costs.json, round 2), over every layer boundary including the
mid-block ones (SURVEY f-2), with the per-group costs fitted to the per-stage step times measured
inside the pipeline: ResNet-110 K=2 (45), K=4 (22,45,75), K=8 (10,21,32,45,60,75,92) allow 1.00 /
0.98 / 0.97 of the ideal speedup by the cost model (the paper's hand placement (37): 0.85);
`paper_ppv` keeps the paper's.  Hyperparameters: Appendix A/B of the paper
(PAPER.md L282-306): momentum 0.9; weight decay 5e-4 (LeNet, VGG), 4e-3
(AlexNet), 1e-4 (ResNet); base lr 0.01 (LeNet), 0.001 (AlexNet), 0.1 (VGG,
ResNet); the pipelined ResNet's stale stages use the Table 7 BKS_2 rate
(0.001 for ResNet-110/362), the last stage the base rate (reading AMB-9).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, Tuple

from .nets import NetSpec, by_name


@dataclass(frozen=True)
class Config:
    name: str
    net: str
    batch: int
    ppv: Dict[int, Tuple[int, ...]]       # K -> PPV (K-1 weighted-layer numbers)
    base_lr: float
    stale_lr: float                         # lr of every non-last stage when K > 1
    momentum: float
    weight_decay: float
    steps: int
    milestones: Tuple[int, ...] = ()
    gamma: float = 0.1
    steps_per_epoch: int = 390
    hybrid_epoch: int = -1
    paper_ppv: Dict[int, Tuple[int, ...]] = field(default_factory=dict)   # the paper's own (Table 1/5)

    def netspec(self) -> NetSpec:
        return by_name(self.net)

    def lr_vector(self, K: int):
        if K == 1:
            return [self.base_lr]
        return [self.stale_lr] * (K - 1) + [self.base_lr]


CONFIGS = {
    "lenet5": Config("lenet5", "lenet5", 64, {1: (), 2: (1,), 3: (1, 2), 4: (1, 2, 3)},
                     0.01, 0.01, 0.9, 5e-4, 20),
    "alexnet": Config("alexnet", "alexnet", 128, {1: (), 2: (1,), 4: (1, 2, 3)},
                      0.001, 0.001, 0.9, 4e-3, 100),
    "vgg16": Config("vgg16", "vgg16", 128,
                    {1: (), 2: (2,), 4: (2, 4, 7), 8: (1, 2, 4, 6, 7, 9, 10)},
                    0.1, 0.1, 0.9, 5e-4, 100),
    "resnet110": Config("resnet110", "resnet110", 128,
                        {1: (), 2: (45,), 4: (22, 45, 75), 8: (10, 21, 32, 45, 60, 75, 92)},
                        0.1, 0.001, 0.9, 1e-4, 100, milestones=(100, 150), paper_ppv={2: (37,)}),
    "resnet362": Config("resnet362", "resnet362", 128,
                        {1: (), 2: (148,), 4: (70, 148, 248), 8: (35, 70, 105, 148, 197, 247, 304)},
                        0.1, 0.001, 0.9, 1e-4, 20, milestones=(100, 150),
                        steps_per_epoch=5, hybrid_epoch=2, paper_ppv={2: (121,)}),
}
