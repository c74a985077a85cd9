"""Runs torch SDPA (cuDNN backend) once at the Hunyuan 720p shape, for an ncu look at the library's
dense kernel (launch configuration and pipe utilisation; context for K4's design, not used by it)."""
import torch
import torch.nn.functional as F
from torch.nn.attention import SDPBackend, sdpa_kernel
B, H, N, D = 1, 24, 118800, 128
q, k, v = (torch.randn((B, H, N, D), device="cuda", dtype=torch.bfloat16) for _ in range(3))
with sdpa_kernel(SDPBackend.CUDNN_ATTENTION):
    for _ in range(2):
        F.scaled_dot_product_attention(q, k, v)
torch.cuda.synchronize()
