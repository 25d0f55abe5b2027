"""Child process for tests/test_gpu_parity.py::test_launch_switches_bit_identical: one
layer forward + backward at a small-m and a multi-wave shape, outputs saved to an
.npz (the library's launch switches are read once per process, from the env)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch

from paper_2309_16119_b200 import modulora as M
from tests.gpu_util import random_quantized

out = {}
for d_out, d_in, m in ((1024, 2048, 300), (4096, 4096, 2048)):
    q, *_ = random_quantized(d_out, d_in, 3, 128, seed=d_out + m)
    a = (torch.randn(d_out, 16, generator=torch.Generator().manual_seed(1)) * 0.02).cuda()
    b = (torch.randn(d_in, 16, generator=torch.Generator().manual_seed(2)) * 0.02).cuda()
    layer = M.ModuLoraLayer("sw", M.DeviceQuantizedMatrix(q), M.LoraAdapter(a, b, 16, 32.0),
                            bias=torch.zeros(d_out).cuda(), bias_trainable=True)
    x = torch.randn(m, d_in, generator=torch.Generator().manual_seed(3)).to(torch.bfloat16).cuda()
    dy = torch.randn(m, d_out, generator=torch.Generator().manual_seed(4)).to(torch.bfloat16).cuda()
    y, xb = M.layer_forward(layer, x)
    dx = M.layer_backward(layer, x, xb, dy)
    da, db = M.grads_of_adapter(layer)
    for k, t in (("y", y), ("xb", xb), ("dx", dx), ("da", da), ("db", db), ("dbias", layer.grad_bias)):
        out[f"{k}_{m}"] = t.float().cpu().numpy()
np.savez(sys.argv[1], **out)
