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


def test_alexnet_flop_split_matches_table():
    """Forward FLOPs per image (2 x multiply-adds of every conv / FC, from the layers' own output shapes)
    against Table tb:distribution."""
    g = _g()["alexnet_flops"]
    flops = {"conv": 0, "fc": 0}

    def hook(mod, inp, out):
        if isinstance(mod, torch.nn.Conv2d):
            k = mod.in_channels // mod.groups * mod.kernel_size[0] * mod.kernel_size[1]
            flops["conv"] += 2 * out[0].numel() * k
        else:
            flops["fc"] += 2 * mod.in_features * mod.out_features

    with torch.device("meta"):
        m = AlexNet()
        for x in m.modules():
            if isinstance(x, (torch.nn.Conv2d, torch.nn.Linear)):
                x.register_forward_hook(hook)
        m(torch.empty(1, 3, 227, 227))
    assert round(flops["fc"] / 1e6) == g["fc_mflops"]
    assert abs(flops["conv"] / 1e6 / g["conv_mflops"] - 1) < 0.02
    assert abs(100 * flops["conv"] / (flops["conv"] + flops["fc"]) - g["conv_pct"]) < 0.2
