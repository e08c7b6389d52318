"""Fixed CNN drivers on synthetic data (BASELINE.json configs C2-C5).

These are the forward/backward workloads Poseidon synchronises; they are not
the optimisation target (north_star).  Shapes follow the BVLC Caffe models the
paper trains, without LRN / dropout so that a
training step is deterministic (reading Z15).  Random init, synthetic data.
"""
from __future__ import annotations

import torch
import torch.nn as nn
import torch.nn.functional as F


class CifarQuick(nn.Module):
    """Caffe cifar10_quick: 3 conv + ip1 + ip2, 145,578 parameters."""

    def __init__(self, n_classes: int = 10):
        super().__init__()
        self.conv1 = nn.Conv2d(3, 32, 5, padding=2)
        self.conv2 = nn.Conv2d(32, 32, 5, padding=2)
        self.conv3 = nn.Conv2d(32, 64, 5, padding=2)
        self.ip1 = nn.Linear(64 * 4 * 4, 64)
        self.ip2 = nn.Linear(64, n_classes)

    def forward(self, x):
        x = F.relu(F.max_pool2d(self.conv1(x), 3, 2, ceil_mode=True))
        x = F.avg_pool2d(F.relu(self.conv2(x)), 3, 2, ceil_mode=True)
        x = F.avg_pool2d(F.relu(self.conv3(x)), 3, 2, ceil_mode=True)
        x = self.ip1(torch.flatten(x, 1))
        return self.ip2(x)


class AlexNet(nn.Module):
    """bvlc_alexnet (groups=2 on conv2/4/5), 227x227 input; fc8 width configurable
    (1000 for ILSVRC12 / C3, 21841 for the ImageNet-22K net of C5)."""

    def __init__(self, n_classes: int = 1000, fc_width: int = 4096):
        super().__init__()
        self.conv1 = nn.Conv2d(3, 96, 11, stride=4)
        self.conv2 = nn.Conv2d(96, 256, 5, padding=2, groups=2)
        self.conv3 = nn.Conv2d(256, 384, 3, padding=1)
        self.conv4 = nn.Conv2d(384, 384, 3, padding=1, groups=2)
        self.conv5 = nn.Conv2d(384, 256, 3, padding=1, groups=2)
        self.fc6 = nn.Linear(256 * 6 * 6, fc_width)
        self.fc7 = nn.Linear(fc_width, fc_width)
        self.fc8 = nn.Linear(fc_width, n_classes)

    def forward(self, x):
        x = F.max_pool2d(F.relu(self.conv1(x)), 3, 2)
        x = F.max_pool2d(F.relu(self.conv2(x)), 3, 2)
        x = F.relu(self.conv3(x))
        x = F.relu(self.conv4(x))
        x = F.max_pool2d(F.relu(self.conv5(x)), 3, 2)
        x = torch.flatten(x, 1)
        x = F.relu(self.fc6(x))
        x = F.relu(self.fc7(x))
        return self.fc8(x)


class _BasicConv(nn.Module):
    def __init__(self, cin, cout, k, stride=1, padding=0):
        super().__init__()
        self.conv = nn.Conv2d(cin, cout, k, stride=stride, padding=padding)

    def forward(self, x):
        return F.relu(self.conv(x))


class _Inception(nn.Module):
    def __init__(self, cin, c1, c3r, c3, c5r, c5, pp):
        super().__init__()
        self.b1 = _BasicConv(cin, c1, 1)
        self.b2r = _BasicConv(cin, c3r, 1)
        self.b2 = _BasicConv(c3r, c3, 3, padding=1)
        self.b3r = _BasicConv(cin, c5r, 1)
        self.b3 = _BasicConv(c5r, c5, 5, padding=2)
        self.b4 = _BasicConv(cin, pp, 1)

    def forward(self, x):
        return torch.cat([self.b1(x), self.b2(self.b2r(x)), self.b3(self.b3r(x)),
                          self.b4(F.max_pool2d(x, 3, 1, padding=1))], 1)


class GoogLeNet(nn.Module):
    """bvlc_googlenet without the auxiliary heads: 57 conv layers + one
    1024x1000 FC, 6,998,552 parameters (reading Z15)."""

    def __init__(self, n_classes: int = 1000):
        super().__init__()
        self.conv1 = _BasicConv(3, 64, 7, stride=2, padding=3)
        self.conv2r = _BasicConv(64, 64, 1)
        self.conv2 = _BasicConv(64, 192, 3, padding=1)
        self.i3a = _Inception(192, 64, 96, 128, 16, 32, 32)
        self.i3b = _Inception(256, 128, 128, 192, 32, 96, 64)
        self.i4a = _Inception(480, 192, 96, 208, 16, 48, 64)
        self.i4b = _Inception(512, 160, 112, 224, 24, 64, 64)
        self.i4c = _Inception(512, 128, 128, 256, 24, 64, 64)
        self.i4d = _Inception(512, 112, 144, 288, 32, 64, 64)
        self.i4e = _Inception(528, 256, 160, 320, 32, 128, 128)
        self.i5a = _Inception(832, 256, 160, 320, 32, 128, 128)
        self.i5b = _Inception(832, 384, 192, 384, 48, 128, 128)
        self.fc = nn.Linear(1024, n_classes)

    def forward(self, x):
        x = F.max_pool2d(self.conv1(x), 3, 2, ceil_mode=True)
        x = F.max_pool2d(self.conv2(self.conv2r(x)), 3, 2, ceil_mode=True)
        x = self.i3b(self.i3a(x))
        x = F.max_pool2d(x, 3, 2, ceil_mode=True)
        x = self.i4e(self.i4d(self.i4c(self.i4b(self.i4a(x)))))
        x = F.max_pool2d(x, 3, 2, ceil_mode=True)
        x = self.i5b(self.i5a(x))
        x = F.adaptive_avg_pool2d(x, 1)
        return self.fc(torch.flatten(x, 1))


# name -> (constructor, per-GPU batch K, input hw, classes)   (BASELINE.json configs)
CONFIGS = {
    "C2": dict(model=lambda: CifarQuick(), batch=100, hw=32, classes=10, scheme="ps",
               name="cifar10_quick"),
    "C3": dict(model=lambda: AlexNet(), batch=256, hw=227, classes=1000, scheme="auto",
               name="bvlc_alexnet"),
    "C4": dict(model=lambda: GoogLeNet(), batch=128, hw=224, classes=1000, scheme="auto",
               name="bvlc_googlenet"),
    "C5": dict(model=lambda: AlexNet(n_classes=21841), batch=256, hw=227, classes=21841, scheme="auto",
               name="alexnet_i22k"),
}


def param_split(model: nn.Module):
    """(conv params, fc params) of a model."""
    conv = sum(p.numel() for m in model.modules() if isinstance(m, nn.Conv2d) for p in m.parameters())
    fc = sum(p.numel() for m in model.modules() if isinstance(m, nn.Linear) for p in m.parameters())
    return conv, fc
