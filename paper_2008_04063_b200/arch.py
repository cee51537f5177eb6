"""The frozen member architecture: a 1-D ResNet per zoo profile.

The reference has no network at all (its scores are binormal draws,
`pkg/src/zooserve/runtime.py:118-136`); the paper trains "ResNeXt with 1-D
stripe kernels", first-conv filters {8..128} x residual blocks {2..16}
(`PAPER.md:384-386`).  This module freezes one concrete member per
`ModelProfile(width, depth)` — the 1-D ResNet family of the paper's authors
(kernel 16, stride 2 every 2nd block, channels x2 every 4th block) — in a
post-activation form so every op fuses into a conv epilogue:

    stem   : conv(1 -> w, k16, s1) + BN + ReLU
    block i: s = 2 if i % 2 == 1 else 1
             c_in = w * 2**((i-1)//4) (block 0: w), c_out = 2*c_in if i%4==0 and i>0
             h = ReLU(BN(conv(x, c_in -> c_out, k16, s)))
             y = ReLU(BN(conv(h, c_out -> c_out, k16, 1)) + shortcut(x))
             shortcut = maxpool(k=s, s) then zero channels [c_in, c_out)
    head   : mean over positions -> FC(c_last -> 1) = logit; prob = sigmoid(logit)

"same" padding: L_out = ceil(L_in/s), pad_left = max(0,(L_out-1)s+16-L_in)//2.
BN is folded into (weight, bias) at generation time and the folded weights are
rounded to fp16-representable values, so the CPU oracle (fp32 math) and the
tensor-core path (fp16 operands, fp32 accumulate) use the same parameters.

Parameters are flattened in one documented order (`pack_order`) that the C-ABI
`hb_add_member` consumes (`include/holmes_b200.h`).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .seeds import derive_seed

TAPS = 16
WINDOW = 7500


@dataclass(frozen=True)
class ConvSpec:
    name: str
    cin: int
    cout: int
    stride: int
    lin: int
    lout: int
    pad: int
    res: str          # "none" | "identity" | "maxpool"
    res_c: int        # channels of the shortcut source (0 when res == "none")
    head: bool        # last conv: fuse mean-pool + FC into the epilogue

    @property
    def flops(self) -> int:
        """Algorithmic FLOPs per window: 2 * C_in * C_out * taps * L_out."""
        return 2 * self.cin * self.cout * TAPS * self.lout


def same_pad(lin: int, stride: int, k: int = TAPS) -> tuple[int, int]:
    lout = -(-lin // stride)
    return lout, max(0, (lout - 1) * stride + k - lin) // 2


def member_layers(width: int, depth: int, window: int = WINDOW) -> list[ConvSpec]:
    """Conv layers of member (width, depth), in execution order."""
    if width % 8 or width < 8:
        raise ValueError("width must be a positive multiple of 8")
    if depth < 1:
        raise ValueError("depth must be >= 1")
    lout, pad = same_pad(window, 1)
    layers = [ConvSpec("stem", 1, width, 1, window, lout, pad, "none", 0, False)]
    length = window
    for i in range(depth):
        stride = 2 if i % 2 == 1 else 1
        cin = width if i == 0 else width * 2 ** ((i - 1) // 4)
        cout = 2 * cin if (i % 4 == 0 and i > 0) else cin
        l1, p1 = same_pad(length, stride)
        l2, p2 = same_pad(l1, 1)
        layers.append(ConvSpec(f"b{i}.conv1", cin, cout, stride, length, l1, p1, "none", 0, False))
        layers.append(ConvSpec(f"b{i}.conv2", cout, cout, 1, l1, l2, p2,
                               "maxpool" if stride == 2 else "identity", cin, i == depth - 1))
        length = l2
    return layers


def member_flops(width: int, depth: int, window: int = WINDOW) -> int:
    return sum(l.flops for l in member_layers(width, depth, window))


def member_act_bytes(width: int, depth: int, window: int = WINDOW) -> int:
    """fp16 activation bytes written + read once per window (HBM/L2 traffic floor)."""
    tot = window * 2
    for l in member_layers(width, depth, window):
        tot += (l.cin * l.lin + (0 if l.head else l.cout * l.lout)) * 2
    return tot


def _fp16_round(a: np.ndarray) -> np.ndarray:
    return a.astype(np.float16).astype(np.float32)


def _calibration_windows(n: int = 8, length: int = 1500) -> np.ndarray:
    """Fixed z-normalised synthetic ECG used only to set BN statistics."""
    from .synth import ecg_samples
    x = np.stack([ecg_samples(12345, p, p % 3, 0, length) for p in range(n)]).astype(np.float64)
    x = (x - x.mean(1, keepdims=True)) / np.maximum(x.std(1, keepdims=True), 1e-6)
    return x.astype(np.float32)


def member_params(width: int, depth: int, seed: int, member_id: str,
                  window: int = WINDOW) -> dict:
    """Deterministic synthetic parameters (random init; no checkpoints exist).

    Conv weights are He-normal.  BN running statistics are *measured* the way a
    trained BN's would be: one forward pass of a fixed 4-window calibration
    batch (CPU, at parameter-synthesis time only — never on the scoring path)
    sets each channel's mean/var, then (gamma, beta) are drawn and folded into
    (W, b); folded W is rounded to fp16-representable values.  The residual
    branch gain is 0.5.  The FC is the top principal direction of the pooled
    calibration features, scaled/centred so logits are O(1) and input
    dependent (sigmoid unsaturated) without amplifying rounding noise.
    Returns {layer name: (W[cout, cin, 16] fp32, b[cout] fp32)} + "fc": (w, b[1]).
    """
    import torch
    import torch.nn.functional as F

    rng = np.random.default_rng(derive_seed(seed, "weights", member_id))
    xc = _calibration_windows()
    specs = member_layers(width, depth, xc.shape[1])
    out = {}
    with torch.no_grad():
        h = torch.from_numpy(xc)[:, None, :]
        block_in = None
        for spec in specs:
            w = rng.standard_normal((spec.cout, spec.cin, TAPS)).astype(np.float32)
            w *= math.sqrt(2.0 / (spec.cin * TAPS))
            gamma = rng.uniform(0.8, 1.2, spec.cout).astype(np.float32)
            if spec.name.endswith("conv2"):
                gamma *= 0.5
            beta = rng.uniform(-0.1, 0.1, spec.cout).astype(np.float32)
            total = max(0, (spec.lout - 1) * spec.stride + TAPS - spec.lin)
            hp = F.pad(h, (spec.pad, total - spec.pad))
            y = F.conv1d(hp, torch.from_numpy(w), stride=spec.stride)
            mean = y.mean(dim=(0, 2)).numpy()
            var = y.var(dim=(0, 2), unbiased=False).numpy()
            scale = gamma / np.sqrt(var + 1e-5)
            wf = _fp16_round(w * scale[:, None, None])
            bf = (beta - mean * scale).astype(np.float32)
            out[spec.name] = (wf, bf)
            y = F.conv1d(hp, torch.from_numpy(wf), torch.from_numpy(bf), stride=spec.stride)
            if spec.name.endswith("conv2"):
                sc = block_in
                if spec.res == "maxpool":
                    if sc.shape[-1] % 2:
                        sc = F.pad(sc, (0, 1))
                    sc = F.max_pool1d(sc, 2, 2)
                if spec.cout > spec.res_c:
                    sc = F.pad(sc, (0, 0, 0, spec.cout - spec.res_c))
                y = y + sc
            elif spec.name.endswith("conv1"):
                block_in = h
            h = torch.relu(y)
        pooled = h.mean(dim=-1).numpy().astype(np.float64)
    # Head direction: the top principal component of the pooled features over
    # the calibration batch (random sign), scaled so logits have std ~1.5.  A
    # random direction would only see ~1/C of the input-dependent variance and
    # the rescale would amplify fp16 rounding noise by ~sqrt(C).
    centred = pooled - pooled.mean(axis=0, keepdims=True)
    _, _, vt = np.linalg.svd(centred, full_matrices=False)
    fc_w = vt[0] * (1.0 if rng.uniform() < 0.5 else -1.0)
    raw = pooled @ fc_w
    fc_w = fc_w * (1.5 / max(raw.std(), 1e-6))
    fc_b = -(pooled @ fc_w).mean() + rng.uniform(-0.5, 0.5)
    out["fc"] = (fc_w.astype(np.float32), np.array([fc_b], dtype=np.float32))
    return out


def pack_order(width: int, depth: int, window: int = WINDOW) -> list[str]:
    return [l.name for l in member_layers(width, depth, window)] + ["fc"]


def flatten_params(params: dict, width: int, depth: int, window: int = WINDOW) -> np.ndarray:
    """Flat fp32 blob for `hb_add_member`: per conv layer W[cout][cin][16] then
    b[cout], in execution order, then fc_w[c_last], fc_b[1]."""
    parts = []
    for name in pack_order(width, depth, window):
        w, b = params[name]
        parts += [np.ascontiguousarray(w, dtype=np.float32).ravel(),
                  np.ascontiguousarray(b, dtype=np.float32).ravel()]
    return np.concatenate(parts)


def flat_param_count(width: int, depth: int, window: int = WINDOW) -> int:
    layers = member_layers(width, depth, window)
    return sum(l.cout * l.cin * TAPS + l.cout for l in layers) + layers[-1].cout + 1
