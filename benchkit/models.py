"""Benchmark workloads (BASELINE.json configs) built from torchvision /
hand-written modules with random init, synthetic data, and the trainable
subset each config names.  The memsave arm is the same model passed through
``convert_to_memory_saving``; the stock arm is left untouched.
"""

from __future__ import annotations

import dataclasses

import torch
from torch import nn


@dataclasses.dataclass
class Workload:
    name: str
    model: nn.Module
    make_batch: callable          # (batch, device) -> (inputs tuple on device)
    loss_fn: callable             # (model, *inputs) -> scalar loss
    batch: int
    input_requires_grad: bool
    dtype: torch.dtype
    config: dict


def randomize_bn_stats(model: nn.Module, seed: int = 0) -> None:
    """BN running stats randomised (mu ~ N(0, 0.1^2), var ~ U(0.5, 2)) so eval BN is
    not the identity."""
    g = torch.Generator().manual_seed(seed)
    for m in model.modules():
        if isinstance(m, nn.BatchNorm2d) and m.running_mean is not None:
            m.running_mean.copy_(torch.randn(m.num_features, generator=g) * 0.1)
            m.running_var.copy_(torch.rand(m.num_features, generator=g) * 1.5 + 0.5)


def resnet18_input_only(batch: int = 256, dtype=torch.bfloat16, device="cuda") -> Workload:
    """configs[1]: ResNet-18, frozen weights, input-only gradient (adversarial-example
    mode), batch 256x3x224x224 bf16, model.eval() (BN uses running stats)."""
    import torchvision
    torch.manual_seed(0)
    m = torchvision.models.resnet18()
    randomize_bn_stats(m)
    m = m.to(device=device, dtype=dtype).to(memory_format=torch.channels_last).eval()
    for p in m.parameters():
        p.requires_grad_(False)

    def make_batch(b, dev):
        gen = torch.Generator(device=dev).manual_seed(1)
        x = torch.randn((b, 3, 224, 224), generator=gen, device=dev, dtype=dtype)
        x = x.contiguous(memory_format=torch.channels_last)
        y = torch.randint(0, 1000, (b,), generator=gen, device=dev)
        return x, y

    def loss_fn(model, x, y):
        return nn.functional.cross_entropy(model(x).float(), y)

    return Workload("resnet18_input_only", m, make_batch, loss_fn, batch, True, dtype,
                    {"workload": "ResNet-18 frozen weights, input-only gradient "
                                 "(adversarial-example mode), eval-mode BN",
                     "model": "resnet18", "global_batch": batch, "image": [3, 224, 224],
                     "layout": "channels_last", "trainable": "input only"})


class DeepCNN(nn.Sequential):
    """Fig. 1 network: L size-preserving Conv2d(C->C, 3x3, pad 1, no bias)
    (SPEC.md:500-504)."""

    def __init__(self, depth: int = 8, channels: int = 8):
        super().__init__(*[nn.Conv2d(channels, channels, 3, padding=1, bias=False)
                           for _ in range(depth)])


def fig1_cnn(batch: int = 32, dtype=torch.float32, device="cuda", depth: int = 8) -> Workload:
    """configs[0]: 8 size-preserving conv layers, only layer 1's weight trainable,
    input (32, 8, 256, 256) fp32."""
    torch.manual_seed(0)
    m = DeepCNN(depth).to(device=device, dtype=dtype)
    for i, p in enumerate(m.parameters()):
        p.requires_grad_(i == 0)

    def make_batch(b, dev):
        gen = torch.Generator(device=dev).manual_seed(1)
        return (torch.randn((b, 8, 256, 256), generator=gen, device=dev, dtype=dtype),)

    def loss_fn(model, x):
        return model(x).sum()

    return Workload("fig1_cnn", m, make_batch, loss_fn, batch, False, dtype,
                    {"workload": "Fig.1 deep CNN: 8x Conv2d(8->8, 3x3, p1), only layer-1 "
                                 "weight trainable", "model": "deepcnn8", "global_batch": batch,
                     "image": [8, 256, 256], "layout": "NCHW", "trainable": "0.weight"})


WORKLOADS = {"resnet18": resnet18_input_only, "fig1": fig1_cnn}


def resnet18_conv_shapes(batch: int):
    """(n, c, h, w, k, r, stride, pad, count) for every conv launch of one
    ResNet-18 forward (torchvision layout)."""
    shapes = [(batch, 3, 224, 224, 64, 7, 2, 3, 1)]
    h = 56
    cin = 64
    for li, cout in enumerate((64, 128, 256, 512)):
        stride = 1 if li == 0 else 2
        ho = h // stride
        shapes.append((batch, cin, h, h, cout, 3, stride, 1, 1))      # block0 conv1
        shapes.append((batch, cout, ho, ho, cout, 3, 1, 1, 3))        # b0 conv2, b1 conv1+conv2
        if stride != 1 or cin != cout:
            shapes.append((batch, cin, h, h, cout, 1, stride, 0, 1))  # downsample
        cin, h = cout, ho
    return shapes
