"""Per-layer parity of the tcgen05 implicit-GEMM conv (K4) and the stem (K3)
against a plain PyTorch fp32 reference of the same op.

Tolerance: outputs are stored as fp16, accumulation is fp32 on both sides, so
the device result must match the fp32 reference to within one fp16 rounding:
|dev - ref| <= 2e-3 * |ref| + 2e-3.
"""
import ctypes as C

import numpy as np
import pytest
import torch
import torch.nn.functional as F

from _ng8 import from_ng8, from_split, lh, lp, to_ng8, to_split

pytestmark = pytest.mark.gpu


def _lib():
    from paper_2008_04063_b200 import _lib
    return _lib


def ref_conv(x, w, b, stride, res=None, res_mode=0, relu=True):
    """x [P,Cin,L] fp32 (fp16-exact), w [Cout,Cin,16] fp32 (fp16-exact)."""
    P, cin, L = x.shape
    lout = -(-L // stride)
    tot = max(0, (lout - 1) * stride + 16 - L)
    y = F.conv1d(F.pad(x, (tot // 2, tot - tot // 2)), w, b, stride=stride)
    if res_mode:
        sc = res
        if res_mode == 2:
            if sc.shape[-1] % 2:
                sc = F.pad(sc, (0, 1))
            sc = F.max_pool1d(sc, 2, 2)
        if w.shape[0] > sc.shape[1]:
            sc = F.pad(sc, (0, 0, 0, w.shape[0] - sc.shape[1]))
        y = y + sc
    return torch.relu(y) if relu else y


def run_conv(x, w, b, stride, res=None, res_mode=0, fc_w=None, out_split=0):
    """Device conv through the C-ABI; layouts: stride-2 input and maxpool shortcut
    in the parity-split layout, everything else interleaved."""
    L = _lib()
    P, cin, lin = x.shape
    cout = w.shape[0]
    lout = -(-lin // stride)
    dev = torch.device("cuda")
    xin = to_split(x.to(dev)) if stride == 2 else to_ng8(x.to(dev))
    if out_split:
        out = torch.full((P, cout // 8, 2, lh(lout), 8), 7.0, dtype=torch.float16, device=dev)
    else:
        out = torch.full((P, cout // 8, lp(lout), 8), 7.0, dtype=torch.float16, device=dev)
    rin = None
    if res is not None:
        rin = to_split(res.to(dev)) if res_mode == 2 else to_ng8(res.to(dev))
    mt = L.lib().hb_conv_mt(cin, cout, lin, stride, 1)       # [N tiles x M tiles] head partials
    head = torch.zeros(P, mt, dtype=torch.float32, device=dev) if fc_w is not None else None
    wn = np.ascontiguousarray(w.numpy(), np.float32)
    bn = np.ascontiguousarray(b.numpy(), np.float32)
    fcn = np.ascontiguousarray(fc_w.numpy(), np.float32) if fc_w is not None else None
    rc = L.lib().hb_op_conv1d(
        C.c_void_p(xin.data_ptr()), P, cin, lin, stride, L.fptr(wn), L.fptr(bn), cout,
        C.c_void_p(rin.data_ptr()) if rin is not None else None, res_mode,
        res.shape[1] if res is not None else 0, res.shape[2] if res is not None else 0,
        C.c_void_p(out.data_ptr()), int(out_split), L.fptr(fcn),
        C.c_void_p(head.data_ptr()) if head is not None else None,
        C.c_void_p(torch.cuda.current_stream().cuda_stream))
    L.check(rc)
    torch.cuda.synchronize()
    return out, head, lout


def _rand(shape, g, scale=1.0):
    return (torch.randn(shape, generator=g) * scale).half().float()


CASES = [
    # cin, cout, lin, stride, res_mode, P
    (32, 32, 7500, 1, 0, 2),
    (32, 32, 7500, 2, 0, 2),
    (64, 64, 1875, 2, 0, 3),
    (64, 64, 938, 1, 1, 2),
    (32, 64, 1875, 1, 1, 2),   # channel-increase conv2 with zero-padded shortcut
    (8, 8, 7500, 1, 0, 2),     # cout < 16: N padded to 16
    (8, 8, 7500, 2, 0, 2),     # 8-channel K-steps pair taps (t, t+2)
    (16, 16, 469, 2, 0, 2),
    (128, 128, 300, 1, 1, 2),  # B streamed (does not fit resident)
    (256, 256, 120, 1, 0, 2),
    (256, 512, 60, 1, 0, 1),   # N split across two tiles
]


@pytest.mark.parametrize("out_split", [0, 1])
@pytest.mark.parametrize("cin,cout,lin,stride,res_mode,P", CASES)
def test_conv_matches_fp32(cin, cout, lin, stride, res_mode, P, out_split):
    g = torch.Generator().manual_seed(cin * 7 + cout + lin + stride)
    x = torch.relu(_rand((P, cin, lin), g))
    w = _rand((cout, cin, 16), g, (2.0 / (cin * 16)) ** 0.5)
    b = _rand((cout,), g, 0.1)
    res = None
    if res_mode == 1:
        res = torch.relu(_rand((P, min(cin, cout), -(-lin // stride)), g))
    out, _, lout = run_conv(x, w, b, stride, res, res_mode, out_split=out_split)
    ref = ref_conv(x, w, b, stride, res, res_mode)
    got = (from_split(out, cout, lout) if out_split else from_ng8(out, cout, lout)).float().cpu()
    err = (got - ref).abs()
    tol = 2e-3 * ref.abs() + 2e-3
    assert bool((err <= tol).all()), f"max err {err.max().item():.3e} at {torch.nonzero(err > tol)[:4].tolist()}"
    # padding positions >= lout must be written as zero (the next layer's TMA reads them)
    if out_split:
        assert bool((out[:, :, 0, (lout + 1) // 2:, :] == 0).all())
        assert bool((out[:, :, 1, lout // 2:, :] == 0).all())
    else:
        assert bool((out[:, :, lout:, :] == 0).all())


@pytest.mark.parametrize("lin,res_len", [(3750, 7500), (938, 1875)])
def test_conv_maxpool_shortcut(lin, res_len):
    """conv2 of a downsampling block: shortcut = maxpool(block input), odd lengths included."""
    g = torch.Generator().manual_seed(lin)
    P, c = 2, 32
    x = torch.relu(_rand((P, c, lin), g))
    blk = torch.relu(_rand((P, c, res_len), g))
    w = _rand((c, c, 16), g, (2.0 / (c * 16)) ** 0.5)
    b = _rand((c,), g, 0.1)
    out, _, lout = run_conv(x, w, b, 1, blk, 2)
    ref = ref_conv(x, w, b, 1, blk, 2)
    got = from_ng8(out, c, lout).float().cpu()
    assert torch.allclose(got, ref, rtol=2e-3, atol=2e-3), (got - ref).abs().max()


@pytest.mark.parametrize("L", [128, 1024, 937, 7500])
def test_layout_padding_edges(L):
    """Lengths at / just off tile and 8-row boundaries, both output layouts."""
    g = torch.Generator().manual_seed(L)
    P, c = 2, 16
    x = torch.relu(_rand((P, c, L), g))
    w = _rand((c, c, 16), g, (2.0 / (c * 16)) ** 0.5)
    b = _rand((c,), g, 0.1)
    for split in (0, 1):
        out, _, lout = run_conv(x, w, b, 1, out_split=split)
        got = (from_split(out, c, lout) if split else from_ng8(out, c, lout)).float().cpu()
        assert torch.allclose(got, ref_conv(x, w, b, 1), rtol=2e-3, atol=2e-3)
        x2 = torch.relu(_rand((P, c, L), g))
        out2, _, l2 = run_conv(x2, w, b, 2)
        assert torch.allclose(from_ng8(out2, c, l2).float().cpu(), ref_conv(x2, w, b, 2), rtol=2e-3, atol=2e-3)


@pytest.mark.parametrize("c", [64, 512])
def test_conv_fused_head(c):
    """Last conv + mean-pool + FC in the epilogue; 512 channels = two N tiles of partials."""
    g = torch.Generator().manual_seed(5)
    P, lin = 3, 469
    x = torch.relu(_rand((P, c, lin), g))
    blk = torch.relu(_rand((P, c, 938), g))
    w = _rand((c, c, 16), g, (2.0 / (c * 16)) ** 0.5)
    b = _rand((c,), g, 0.1)
    fc = torch.randn(c, generator=g) / c ** 0.5
    _, head, lout = run_conv(x, w, b, 1, blk, 2, fc_w=fc)
    ref = ref_conv(x, w, b, 1, blk, 2)          # [P, c, lout] fp32
    ref_sum = (ref * fc[None, :, None]).sum(dim=(1, 2))
    got = head.cpu().sum(dim=1)
    assert torch.allclose(got, ref_sum, rtol=1e-4, atol=1e-2), (got, ref_sum)


@pytest.mark.parametrize("cout", [8, 32, 128])
def test_stem_matches_fp32(cout):
    L = _lib()
    g = torch.Generator().manual_seed(cout)
    P, n = 3, 7500
    x = _rand((P, n), g)
    w = _rand((cout, 1, 16), g, 0.25)
    b = _rand((cout,), g, 0.1)
    dev = torch.device("cuda")
    xd = x.half().to(dev).contiguous()
    out = torch.zeros(P, cout // 8, lp(n), 8, dtype=torch.float16, device=dev)
    wn = np.ascontiguousarray(w.numpy().reshape(cout, 16), np.float32)
    bn = np.ascontiguousarray(b.numpy(), np.float32)
    L.check(L.lib().hb_op_stem(C.c_void_p(xd.data_ptr()), P, n, L.fptr(wn), L.fptr(bn), cout,
                               C.c_void_p(out.data_ptr()), C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    torch.cuda.synchronize()
    ref = ref_conv(x[:, None, :], w, b, 1)
    got = from_ng8(out, cout, n).float().cpu()
    assert torch.allclose(got, ref, rtol=2e-3, atol=2e-3), (got - ref).abs().max()
