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


def lh(length: int) -> int:
    return ((length + 1) // 2 + 7) // 8 * 8


def to_split(x: torch.Tensor) -> torch.Tensor:
    """[P, C, L] -> parity-split S layout [P, C/8, 2, Lh, 8] fp16 (even / odd positions), zero padded."""
    P, C, L = x.shape
    h = lh(L)
    out = torch.zeros(P, C // 8, 2, h, 8, dtype=torch.float16, device=x.device)
    g = x.reshape(P, C // 8, 8, L).permute(0, 1, 3, 2).to(torch.float16)  # [P, G, L, 8]
    out[:, :, 0, : (L + 1) // 2, :] = g[:, :, 0::2, :]
    out[:, :, 1, : L // 2, :] = g[:, :, 1::2, :]
    return out.contiguous()


def from_split(a: torch.Tensor, C: int, L: int) -> torch.Tensor:
    P = a.shape[0]
    g = torch.empty(P, C // 8, L, 8, dtype=a.dtype, device=a.device)
    g[:, :, 0::2, :] = a[:, :, 0, : (L + 1) // 2, :]
    g[:, :, 1::2, :] = a[:, :, 1, : L // 2, :]
    return g.permute(0, 1, 3, 2).reshape(P, C, L)


def lq(length: int, q: int) -> int:
    return (-(-length // q) + 7) // 8 * 8


def to_q(x: torch.Tensor, q: int) -> torch.Tensor:
    """[P, C, L] -> Q-phase layout [P, C/8, Q, lq, 8] fp16 (position l at phase l % Q, row l // Q), zero padded."""
    P, C, L = x.shape
    rows = lq(L, q)
    out = torch.zeros(P, C // 8, q, rows, 8, dtype=torch.float16, device=x.device)
    g = x.reshape(P, C // 8, 8, L).permute(0, 1, 3, 2).to(torch.float16)  # [P, G, L, 8]
    for ph in range(q):
        n = len(range(ph, L, q))
        out[:, :, ph, :n, :] = g[:, :, ph::q, :]
    return out.contiguous()


def from_q(a: torch.Tensor, C: int, L: int, q: int) -> torch.Tensor:
    P = a.shape[0]
    g = torch.empty(P, C // 8, L, 8, dtype=a.dtype, device=a.device)
    for ph in range(q):
        n = len(range(ph, L, q))
        g[:, :, ph::q, :] = a[:, :, ph, :n, :]
    return g.permute(0, 1, 3, 2).reshape(P, C, L)


def q_padding_zero(a: torch.Tensor, L: int, q: int) -> bool:
    """Every slot of the Q-phase planes past position L holds zero."""
    for ph in range(q):
        n = len(range(ph, L, q))
        if not bool((a[:, :, ph, n:, :] == 0).all()):
            return False
    return True
