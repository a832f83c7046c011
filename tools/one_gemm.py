"""One bf16 Linear forward at a given (M, N, K), for ncu captures:
python tools/one_gemm.py M N K [reps]"""
import sys
import torch
sys.path.insert(0, ".")
from paper_2404_12406_b200._ops import ops  # noqa: E402

M, N, K = (int(v) for v in sys.argv[1:4])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
dev = torch.device("cuda", 0)
x = torch.randn(M, K, device=dev, dtype=torch.bfloat16)
w = torch.randn(N, K, device=dev, dtype=torch.bfloat16) / K ** 0.5
for _ in range(reps):
    y = ops().linear_fwd(x, w, None)
torch.cuda.synchronize()
print("ok", tuple(y.shape))
