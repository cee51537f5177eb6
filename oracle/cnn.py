"""ORACLE (test infrastructure only) — CPU fp32 restatement of the member forward.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU legs may import
this module, and only as the checker / CPU baseline.  The product path never
routes through it.

Parity status: **unpinned against the reference** — the reference has no CNN
(its per-window scores are binormal draws, `pkg/src/zooserve/runtime.py:118-136`).
This restates the architecture frozen in `paper_2008_04063_b200/arch.py`
(paper grid `PAPER.md:384-386`) in plain PyTorch fp32 on CPU, and the
aggregation conventions the reference does pin:
  * mean of member latents, normalised by popcount (`cohort.py:89-97`),
  * sigmoid on the latent for probabilities (`cohort.py:105-108`),
  * plus the north-star mean of member sigmoids.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.nn.functional as F

from paper_2008_04063_b200.arch import member_layers


def znorm(windows: np.ndarray) -> np.ndarray:
    """Per-window z-normalisation (population std; zero variance -> zeros)."""
    w = np.asarray(windows, dtype=np.float64)
    mean = w.mean(axis=-1, keepdims=True)
    std = w.std(axis=-1, keepdims=True)
    return ((w - mean) / np.maximum(std, 1e-6)).astype(np.float32)


def member_forward(x: np.ndarray, params: dict, width: int, depth: int,
                   round_fp16: bool = False) -> np.ndarray:
    """x: [P, L] normalised windows -> logits [P] (fp32).

    round_fp16 rounds every stored activation to fp16 (what the device stores
    between layers) — used only to separate rounding error from logic error.
    """
    layers = member_layers(width, depth, x.shape[-1])
    h = torch.from_numpy(np.ascontiguousarray(x, np.float32))[:, None, :]
    rnd = (lambda t: t.half().float()) if round_fp16 else (lambda t: t)
    h = rnd(h)
    block_in = None
    for spec in layers:
        w, b = params[spec.name]
        wt, bt = torch.from_numpy(w), torch.from_numpy(b)
        total = max(0, (spec.lout - 1) * spec.stride + 16 - spec.lin)
        padded = F.pad(h, (spec.pad, total - spec.pad))
        y = F.conv1d(padded, wt, bt, stride=spec.stride)
        if spec.name == "stem" or spec.name.endswith("conv1"):
            if spec.name.endswith("conv1"):
                block_in = h
            h = rnd(torch.relu(y))
            continue
        sc = block_in
        if spec.res == "maxpool":
            if sc.shape[-1] % 2:
                sc = F.pad(sc, (0, 1))          # post-ReLU input: pad value 0 == ignore
            sc = F.max_pool1d(sc, 2, 2)
        if spec.cout > spec.res_c:
            sc = F.pad(sc, (0, 0, 0, spec.cout - spec.res_c))
        y = torch.relu(y + sc)
        h = y if spec.head else rnd(y)
    fc_w, fc_b = params["fc"]
    pooled = h.mean(dim=-1)                     # [P, C]
    logit = pooled @ torch.from_numpy(fc_w) + float(fc_b[0])
    return logit.numpy().astype(np.float32)


def sigmoid(x):
    return 1.0 / (1.0 + np.exp(-np.asarray(x, np.float64)))


def ensemble(member_logits: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """member_logits [P, M] -> (mean of sigmoids [P], mean latent [P]), fixed member order."""
    ml = np.asarray(member_logits, np.float64)
    return sigmoid(ml).mean(axis=1), ml.mean(axis=1)
