"""Test helpers: NG8 activation layout <-> [P, C, L] (see csrc/hb_kernels.cuh)."""
import numpy as np
import torch


def lp(length: int) -> int:
    return (length + 7) // 8 * 8


def to_ng8(x: torch.Tensor) -> torch.Tensor:
    """[P, C, L] -> contiguous [P, C/8, Lp, 8] fp16 on x.device, padding rows zero."""
    P, C, L = x.shape
    out = torch.zeros(P, C // 8, lp(L), 8, dtype=torch.float16, device=x.device)
    out[:, :, :L, :] = x.reshape(P, C // 8, 8, L).permute(0, 1, 3, 2).to(torch.float16)
    return out.contiguous()


def from_ng8(a: torch.Tensor, C: int, L: int) -> torch.Tensor:
    P = a.shape[0]
    return a[:, :, :L, :].permute(0, 1, 3, 2).reshape(P, C, L)
