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


def _image_batch(dtype, requires_grad=False, classes=1000):
    def make_batch(b, dev):
        gen = torch.Generator(device=dev).manual_seed(1)
        x = torch.randn((b, 3, 224, 224), generator=gen, device=dev, dtype=dtype)
        x = x.contiguous(memory_format=torch.channels_last)
        y = torch.randint(0, classes, (b,), generator=gen, device=dev)
        return x, y
    return make_batch


def _ce_loss(model, x, y):
    return nn.functional.cross_entropy(model(x).float(), y)


def resnet101_finetune(batch: int = 128, dtype=torch.bfloat16, device="cuda") -> Workload:
    """configs[2] (ResNet-101 reading): last 2 Bottlenecks (layer4.1, layer4.2) + fc + all
    BN affine params trainable, BN in eval mode, input without grad."""
    import torchvision
    torch.manual_seed(0)
    m = torchvision.models.resnet101()
    randomize_bn_stats(m)
    m = m.to(device=device, dtype=dtype).to(memory_format=torch.channels_last).eval()
    for name, p in m.named_parameters():
        p.requires_grad_(name.startswith(("layer4.1.", "layer4.2.", "fc.")) or ".bn" in name
                         or "downsample.1" in name or name.startswith("bn1"))
    ntrain = sum(p.numel() for p in m.parameters() if p.requires_grad)
    return Workload("resnet101_finetune", m, _image_batch(dtype), _ce_loss, batch, False, dtype,
                    {"workload": "ResNet-101 fine-tuning: layer4.1, layer4.2, fc and all BN "
                                 "affine parameters trainable, BN eval", "model": "resnet101",
                     "global_batch": batch, "image": [3, 224, 224], "layout": "channels_last",
                     "trainable_params": ntrain})


def vgg16_finetune(batch: int = 128, dtype=torch.bfloat16, device="cuda") -> Workload:
    """configs[2] (VGG-16 reading): conv blocks 4-5 (features[17:]) + classifier trainable,
    eval mode (dropout off), input without grad."""
    import torchvision
    torch.manual_seed(0)
    m = torchvision.models.vgg16()
    m = m.to(device=device, dtype=dtype).to(memory_format=torch.channels_last).eval()
    for name, p in m.named_parameters():
        layer = name.split(".")
        trainable = name.startswith("classifier.") or (layer[0] == "features" and
                                                       int(layer[1]) >= 17)
        p.requires_grad_(trainable)
    ntrain = sum(p.numel() for p in m.parameters() if p.requires_grad)
    return Workload("vgg16_finetune", m, _image_batch(dtype), _ce_loss, batch, False, dtype,
                    {"workload": "VGG-16 fine-tuning: conv blocks 4-5 (features[17:]) and the "
                                 "classifier trainable", "model": "vgg16", "global_batch": batch,
                     "image": [3, 224, 224], "layout": "channels_last",
                     "trainable_params": ntrain})


def bert_base_biases(batch: int = 64, seq: int = 512, dtype=torch.bfloat16,
                     device="cuda") -> Workload:
    """configs[3]: BERT-base random init, only the attention Linear biases and the
    classifier trainable, train mode (dropout 0.1), seq 512, batch 64."""
    from transformers import BertConfig, BertForSequenceClassification
    torch.manual_seed(0)
    cfg = BertConfig(num_labels=2, attn_implementation="sdpa")
    m = BertForSequenceClassification(cfg).to(device=device, dtype=dtype).train()
    for name, p in m.named_parameters():
        p.requires_grad_(name.startswith("classifier.") or (
            ".attention." in name and name.endswith(".bias") and "LayerNorm" not in name))
    ntrain = sum(p.numel() for p in m.parameters() if p.requires_grad)

    def make_batch(b, dev):
        gen = torch.Generator(device=dev).manual_seed(1)
        ids = torch.randint(0, cfg.vocab_size, (b, seq), generator=gen, device=dev)
        y = torch.randint(0, 2, (b,), generator=gen, device=dev)
        return ids, y

    def loss_fn(model, ids, y):
        return nn.functional.cross_entropy(model(input_ids=ids).logits.float(), y)

    return Workload("bert_base_biases", m, make_batch, loss_fn, batch, False, dtype,
                    {"workload": "BERT-base random init, attention Linear biases + classifier "
                                 "trainable, train mode", "model": "bert-base", "global_batch": batch,
                     "seq_len": seq, "trainable_params": ntrain})


def llama3_8b_last4(batch: int = 2, seq: int = 2048, dtype=torch.bfloat16, device="cuda",
                    layers: int = 32) -> Workload:
    """configs[4]: Llama-3-8B architecture, random init, frozen except the last 4 decoder
    layers, seq 2048, batch 2 per GPU."""
    from transformers import LlamaConfig, LlamaForCausalLM
    torch.manual_seed(0)
    cfg = LlamaConfig(vocab_size=128256, hidden_size=4096, intermediate_size=14336,
                      num_hidden_layers=layers, num_attention_heads=32, num_key_value_heads=8,
                      max_position_embeddings=8192, rope_theta=500000.0,
                      attn_implementation="sdpa", torch_dtype=dtype)
    with torch.device(device):
        m = LlamaForCausalLM(cfg).to(dtype)
    m.train()
    for name, p in m.named_parameters():
        parts = name.split(".")
        trainable = len(parts) > 3 and parts[1] == "layers" and int(parts[2]) >= layers - 4
        p.requires_grad_(trainable)
    ntrain = sum(p.numel() for p in m.parameters() if p.requires_grad)

    def make_batch(b, dev):
        gen = torch.Generator(device=dev).manual_seed(1)
        return (torch.randint(0, cfg.vocab_size, (b, seq), generator=gen, device=dev),)

    def loss_fn(model, ids):
        return model(input_ids=ids, labels=ids).loss

    return Workload("llama3_8b_last4", m, make_batch, loss_fn, batch, False, dtype,
                    {"workload": "Llama-3-8B architecture random init, last 4 decoder layers "
                                 "trainable", "model": "llama3-8b-arch", "global_batch": batch,
                     "seq_len": seq, "trainable_params": ntrain})


WORKLOADS = {"resnet18": resnet18_input_only, "fig1": fig1_cnn,
             "resnet101": resnet101_finetune, "vgg16": vgg16_finetune,
             "bert": bert_base_biases, "llama": llama3_8b_last4}


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
