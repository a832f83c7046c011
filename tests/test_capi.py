"""The C-ABI library loads and exports every symbol include/memsave_b200.h
declares (no compute calls — this runs without a GPU)."""

import ctypes
import os
import re

from paper_2404_12406_b200 import _lib

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include",
                      "memsave_b200.h")


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"MS_API\s+[\w\s\*]+?\b(ms_\w+)\s*\(", src)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("ms_conv2d_fwd", "ms_conv2d_dx", "ms_conv2d_dw", "ms_linear_fwd", "ms_linear_dx",
              "ms_linear_dw", "ms_bn_eval_fwd", "ms_bn_eval_bwd", "ms_bias_grad"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    for s in declared_symbols():
        assert hasattr(L, s), s
        assert s in _lib.SIGNATURES, f"{s} has no ctypes signature"


def test_host_only_queries():
    L = _lib.lib()
    assert L.ms_version() >= 1
    assert L.ms_status_string(0) == b"MS_OK"
    assert L.ms_status_string(4) == b"MS_ERR_UNSUPPORTED"
    d = _lib.ConvDesc(256, 3, 224, 224, 64, 7, 7, 2, 2, 3, 3, _lib.MS_NHWC, _lib.MS_NHWC,
                      _lib.MS_BF16)
    assert L.ms_conv2d_out_h(ctypes.byref(d)) == 112
    assert L.ms_conv2d_out_w(ctypes.byref(d)) == 112
    # stem: 3 channels -> padded activation copy + repacked weight in the workspace
    assert L.ms_conv2d_workspace(ctypes.byref(d), _lib.MS_CONV_FWD) > 0
    # fp32 dW | db accumulators + the finalize ticket of the NHWC backward
    assert L.ms_bn_eval_workspace(2, 64, 49, _lib.MS_NHWC) == 2 * 64 * 4 + 16


def test_fp32_linear_workspace_is_the_tf32_split():
    """float32 Linear (3xTF32) keeps hi / lo planes of both operands, K-major with
    a 16-byte pitch, in the caller's workspace; small products stay on the SIMT
    kernel and need none (csrc/linear.cu plan_linear)."""
    L = _lib.lib()
    al = lambda b: (b + 255) // 256 * 256  # noqa: E731
    M, N, K = 4096, 1000, 130
    ld = (K + 3) // 4 * 4
    assert L.ms_linear_workspace(M, N, K, _lib.MS_F32, 0) == 2 * al(4 * M * ld) + 2 * al(4 * N * ld)
    # dX: out M x K, reduction N; dW: out N x K, reduction M
    ldn, ldm = (N + 3) // 4 * 4, (M + 3) // 4 * 4
    assert L.ms_linear_workspace(M, N, K, _lib.MS_F32, 1) == 2 * al(4 * M * ldn) + 2 * al(4 * K * ldn)
    assert L.ms_linear_workspace(M, N, K, _lib.MS_F32, 2) == 2 * al(4 * N * ldm) + 2 * al(4 * K * ldm)
    assert L.ms_linear_workspace(64, 2, 768, _lib.MS_F32, 0) == 0  # classifier head: SIMT


def test_invalid_descriptor_rejected_without_gpu():
    L = _lib.lib()
    d = _lib.ConvDesc(1, 0, 8, 8, 4, 3, 3, 1, 1, 1, 1, _lib.MS_NHWC, _lib.MS_NHWC, _lib.MS_BF16)
    st = L.ms_conv2d_fwd(ctypes.byref(d), None, None, None, None, None, 0, None)
    assert st == 1  # MS_ERR_SHAPE
    assert b"non-positive" in L.ms_last_error()


# ------------------------------------------------------------------ torch.ops.memsave
OPS = ["linear_fwd", "linear_dx", "linear_dw", "bias_grad", "conv2d_fwd", "conv2d_dx",
       "conv2d_dw", "conv2d_db", "conv_transpose2d_fwd", "bn_eval_fwd", "bn_eval_bwd",
       "bn_relu_fwd", "bn_add_relu_bwd", "bn_relu_bwd", "relu_fwd", "relu_fwd_", "relu_bwd",
       "add_relu_fwd", "maxpool2d_fwd", "maxpool2d_bwd", "maxpool2d_relu_bwd", "dropout_fwd",
       "dropout_fwd_", "dropout_bwd", "layernorm_fwd", "layernorm_bwd", "conv2d_bn_fwd",
       "conv2d_bn_dx"]


def test_torch_op_library_registers_every_op():
    import torch

    from paper_2404_12406_b200._ops import ops
    O = ops()
    for name in OPS:
        op = getattr(O, name)  # the .default OpOverload
        # a CUDA kernel and a Meta kernel, no CPU kernel (no CPU path)
        assert torch._C._dispatch_has_kernel_for_dispatch_key(op.name(), "CUDA")
        assert torch._C._dispatch_has_kernel_for_dispatch_key(op.name(), "Meta")
        assert not torch._C._dispatch_has_kernel_for_dispatch_key(op.name(), "CPU")


def test_torch_ops_meta_shapes_and_fake_tensors():
    import torch
    from torch._subclasses.fake_tensor import FakeTensorMode

    from paper_2404_12406_b200._ops import ops
    O = ops()
    cl = torch.channels_last
    x = torch.empty(4, 64, 9, 9, device="meta", dtype=torch.bfloat16).contiguous(memory_format=cl)
    w = torch.empty(32, 64, 3, 3, device="meta", dtype=torch.bfloat16).contiguous(memory_format=cl)
    y = O.conv2d_fwd(x, w, None, [2, 2], [1, 1], 1, 1)
    assert y.shape == (4, 32, 5, 5) and y.is_contiguous(memory_format=cl)
    dx = O.conv2d_dx(y, w, [4, 64, 9, 9], [2, 2], [1, 1], 1, 1)
    assert dx.shape == x.shape and dx.is_contiguous(memory_format=cl)
    y2, mask = O.conv2d_bn_fwd(x, w, None, None, None, None, None, 0.0, None, True, True,
                               [1, 1], [1, 1], 1, 1)
    assert mask.numel() == (4 * 32 * 9 * 9 + 7) // 8 and mask.dtype == torch.uint8
    with FakeTensorMode():
        xf = torch.empty(8, 512, 768, device="cuda", dtype=torch.bfloat16)
        wf = torch.empty(3072, 768, device="cuda", dtype=torch.bfloat16)
        yf = O.linear_fwd(xf, wf, None)
        assert yf.shape == (8, 512, 3072) and yf.device.type == "cuda"
        ln = O.layernorm_fwd(yf, None, None, 1e-5, 3072, True)
        assert ln[1].shape == (8 * 512,) and ln[1].dtype == torch.float32


def test_cpu_tensors_have_no_kernel():
    import pytest
    import torch

    from paper_2404_12406_b200._ops import ops
    with pytest.raises(NotImplementedError):
        ops().relu_fwd(torch.randn(8), True)


def test_gemm_kernels_keep_their_epilogue_in_registers():
    """ptxas report of the last build: no tcgen05 GEMM instantiation spills or
    keeps an array on the stack (a dynamically indexed epilogue array costs
    ~40 % of the 768-wide BERT GEMMs' time)."""
    import re
    log = os.path.join(os.path.dirname(__file__), "..", "paper_2404_12406_b200", "csrc", "build",
                       "host.ptxas.log")
    if not os.path.exists(log):
        pytest.skip("no ptxas log (library not built here)")
    fn, bad = None, []
    for line in open(log):
        m = re.search(r"Function properties for (\S+)", line)
        if m:
            fn = m.group(1)
            continue
        m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores", line)
        if m and fn and "umma_gemm_kernel" in fn and (int(m.group(1)) > 64 or int(m.group(2))):
            bad.append((fn, line.strip()))
    assert not bad, bad
