"""CPU checks of the CNN drivers against the paper's printed parameter counts."""
import json
import os

import torch

from drivers.cnn import AlexNet, CifarQuick, GoogLeNet, param_split

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "driver_param_counts.json")


def _g():
    with open(GOLDEN) as f:
        return json.load(f)


def test_cifar_quick_param_count_and_shapes():
    m = CifarQuick()
    assert sum(p.numel() for p in m.parameters()) == _g()["cifar10_quick"]["total_params"]
    y = m(torch.zeros(2, 3, 32, 32))
    assert y.shape == (2, 10)


def test_alexnet_param_split_matches_table():
    m = AlexNet()
    conv, fc = param_split(m)
    g = _g()["alexnet"]
    assert round(conv / 1e6, 1) == g["conv_params_millions_1dp"]
    assert round(fc / 1e6) == g["fc_params_millions_0dp"]
    assert conv == 2_334_080 and fc == 58_631_144
    with torch.device("meta"):
        y = AlexNet()(torch.empty(2, 3, 227, 227))
    assert y.shape == (2, 1000)


def test_googlenet_structure():
    m = GoogLeNet()
    convs = [x for x in m.modules() if isinstance(x, torch.nn.Conv2d)]
    fcs = [x for x in m.modules() if isinstance(x, torch.nn.Linear)]
    assert len(convs) == 57 and len(fcs) == 1
    assert sum(p.numel() for p in m.parameters()) == 6_998_552
    with torch.device("meta"):
        y = GoogLeNet()(torch.empty(2, 3, 224, 224))
    assert y.shape == (2, 1000)
