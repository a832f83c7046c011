import copy, sys, torch, torchvision
sys.path.insert(0, '/root/repo')
from paper_2404_12406_b200.nn import convert_to_memory_saving
from benchkit.models import randomize_bn_stats
DEV = 'cuda'
torch.manual_seed(0)
base = torchvision.models.resnet18().eval()
randomize_bn_stats(base)
for p in base.parameters(): p.requires_grad_(False)
ref = copy.deepcopy(base).to(DEV).to(memory_format=torch.channels_last)
m1 = convert_to_memory_saving(copy.deepcopy(base)).to(DEV, torch.bfloat16).to(memory_format=torch.channels_last)
m2 = convert_to_memory_saving(copy.deepcopy(base), fuse=True).to(DEV, torch.bfloat16).to(memory_format=torch.channels_last)
stock = copy.deepcopy(base).to(DEV, torch.bfloat16).to(memory_format=torch.channels_last)
x = torch.randn(4, 3, 224, 224, device=DEV).contiguous(memory_format=torch.channels_last)
outs = {}
for name, m, dt in (("fp32", ref, torch.float32), ("stock_bf16", stock, torch.bfloat16), ("memsave", m1, torch.bfloat16), ("fused", m2, torch.bfloat16)):
    xi = x.to(dt).clone().requires_grad_(True)
    y = m(xi)
    y.float().sum().backward()
    outs[name] = (y.float(), xi.grad.float())
r = outs["fp32"]
for k, (y, g) in outs.items():
    print(k, "y rel", ((y - r[0]).norm() / r[0].norm()).item(), "grad rel", ((g - r[1]).norm() / r[1].norm()).item())
