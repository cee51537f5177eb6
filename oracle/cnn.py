"""ORACLE (test infrastructure only) — CPU fp32 restatement of the member forward.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU legs may import
this module, and only as the checker / CPU baseline.  The product path never
routes through it.

Parity status: **unpinned against the reference** — the reference has no CNN
(its per-window scores are binormal draws, `pkg/src/zooserve/runtime.py:118-136`).
The network is the builder's frozen 1-D ResNet (paper grid `PAPER.md:384-386`);
this module restates it INDEPENDENTLY of the product:

  * `layers()` is this module's own restatement of the layer table (the
    product has two more: `arch.member_layers` in Python and `member_layers`
    in `csrc/hb_api.cu`; `tests/test_oracle_cnn.py` checks all three agree, so
    a wrong-but-consistent product table cannot pass by construction);
  * `unflatten()` decodes the exact fp32 parameter blob the product hands to
    `hb_add_member` (`include/holmes_b200.h`), with this module's table, so the
    oracle and the device consume the same bytes;
  * the forward is plain PyTorch fp32 `conv1d`/`max_pool1d` on the CPU.

The aggregation conventions are the ones the reference does pin:
  * mean of member latents, normalised by popcount (`cohort.py:89-97`),
  * sigmoid on the latent for probabilities (`cohort.py:105-108`),
  * plus the north-star mean of member sigmoids.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.nn.functional as F

TAPS = 16


@dataclass(frozen=True)
class Layer:
    name: str
    cin: int
    cout: int
    stride: int
    lin: int
    lout: int
    pad_left: int
    shortcut: str     # "none" | "identity" | "maxpool"


def layers(width: int, depth: int, window: int) -> list[Layer]:
    """The frozen architecture, restated:

    stem: conv(1 -> w, k16, s1); block i: stride 2 on odd i, channels double on
    every 4th block (i = 4, 8, 12), conv1 (stride s) then conv2 (stride 1) with
    a shortcut (maxpool by 2 after a stride-2 conv1, identity otherwise, zero
    channel padding when the block widens).  "Same" padding: L_out = ceil(L/s),
    the total pad (L_out-1)*s + 16 - L split with the smaller half on the left.
    """
    def conv(name, cin, cout, s, lin, shortcut):
        lout = (lin + s - 1) // s
        total = max(0, (lout - 1) * s + TAPS - lin)
        return Layer(name, cin, cout, s, lin, lout, total // 2, shortcut)

    out = [conv("stem", 1, width, 1, window, "none")]
    c, length = width, window
    for i in range(depth):
        s = 1 if i % 2 == 0 else 2
        c_out = 2 * c if (i > 0 and i % 4 == 0) else c
        c1 = conv(f"b{i}.conv1", c, c_out, s, length, "none")
        c2 = conv(f"b{i}.conv2", c_out, c_out, 1, c1.lout, "maxpool" if s == 2 else "identity")
        out += [c1, c2]
        c, length = c_out, c2.lout
    return out


def unflatten(blob: np.ndarray, width: int, depth: int, window: int) -> dict:
    """The `hb_add_member` blob -> {layer name: (W[cout, cin, 16], b[cout])} + "fc": (w, b[1]).
    Blob order (include/holmes_b200.h): per conv layer W then b, then fc_w[c_last], fc_b."""
    blob = np.asarray(blob, np.float32)
    out, o = {}, 0
    ls = layers(width, depth, window)
    for L in ls:
        n = L.cout * L.cin * TAPS
        out[L.name] = (blob[o:o + n].reshape(L.cout, L.cin, TAPS), blob[o + n:o + n + L.cout])
        o += n + L.cout
    c = ls[-1].cout
    out["fc"] = (blob[o:o + c], blob[o + c:o + c + 1])
    if o + c + 1 != blob.size:
        raise ValueError(f"parameter blob has {blob.size} floats, the oracle's table needs {o + c + 1}")
    return out


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
    h = torch.from_numpy(np.ascontiguousarray(x, np.float32))[:, None, :]
    rnd = (lambda t: t.half().float()) if round_fp16 else (lambda t: t)
    h = rnd(h)
    block_in = None
    with torch.no_grad():
        for L in layers(width, depth, x.shape[-1]):
            w, b = params[L.name]
            total = max(0, (L.lout - 1) * L.stride + TAPS - L.lin)
            y = F.conv1d(F.pad(h, (L.pad_left, total - L.pad_left)), torch.from_numpy(np.ascontiguousarray(w)),
                         torch.from_numpy(np.ascontiguousarray(b)), stride=L.stride)
            if L.shortcut == "none":
                if L.name != "stem":
                    block_in = h
                h = rnd(torch.relu(y))
                continue
            sc = block_in
            if L.shortcut == "maxpool":
                if sc.shape[-1] % 2:
                    sc = F.pad(sc, (0, 1))          # post-ReLU input: a zero pad never wins the max
                sc = F.max_pool1d(sc, 2, 2)
            if L.cout > sc.shape[1]:
                sc = F.pad(sc, (0, 0, 0, L.cout - sc.shape[1]))
            h = torch.relu(y + sc)
            last = L.name == f"b{depth - 1}.conv2"
            h = h if last else rnd(h)
        fc_w, fc_b = params["fc"]
        logit = h.mean(dim=-1) @ torch.from_numpy(np.ascontiguousarray(fc_w)) + float(fc_b[0])
    return logit.numpy().astype(np.float32)


def sigmoid(x):
    return 1.0 / (1.0 + np.exp(-np.asarray(x, np.float64)))


def ensemble(member_logits: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """member_logits [P, M] -> (mean of sigmoids [P], mean latent [P]), fixed member order."""
    ml = np.asarray(member_logits, np.float64)
    return sigmoid(ml).mean(axis=1), ml.mean(axis=1)
