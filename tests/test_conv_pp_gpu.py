"""Per-layer parity of the polyphase tcgen05 conv (K4b, csrc/conv_pp.cu) and
of the Q-phase activation layouts every producer now writes, against a plain
PyTorch fp32 reference of the same op (the op is the builder's own network:
the reference, zooserve, has no model -- see DESIGN.md section 2).

Tolerance as for K4: fp16 output of an fp32 accumulation,
|dev - ref| <= 2e-3 * |ref| + 2e-3.
"""
import ctypes as C

import numpy as np
import pytest
import torch

from _ng8 import from_q, lq, q_padding_zero, to_q
from test_conv_gpu import _rand, ref_conv

pytestmark = pytest.mark.gpu

K_TC, K_PP = 0, 1


def _lib():
    from paper_2008_04063_b200 import _lib
    return _lib


def run_q(x, w, b, stride, kind, res=None, res_mode=0, res_q=1, out_q=1):
    L = _lib()
    P, cin, lin = x.shape
    cout = w.shape[0]
    lout = -(-lin // stride)
    dev = torch.device("cuda")
    in_q = stride * (128 // cout) if kind == K_PP else stride
    xin = to_q(x.to(dev), in_q)
    out = torch.full((P, cout // 8, out_q, lq(lout, out_q), 8), 7.0, dtype=torch.float16,
                     device=dev)
    rin = to_q(res.to(dev), res_q) if res is not None else None
    wn = np.ascontiguousarray(w.numpy(), np.float32)
    bn = np.ascontiguousarray(b.numpy(), np.float32)
    rc = L.lib().hb_op_conv1d_q(
        C.c_void_p(xin.data_ptr()), P, cin, lin, stride, L.fptr(wn), L.fptr(bn), cout,
        C.c_void_p(rin.data_ptr()) if rin is not None else None, res_mode,
        res.shape[1] if res is not None else 0, res.shape[2] if res is not None else 0, res_q,
        C.c_void_p(out.data_ptr()), out_q, None, None, kind,
        C.c_void_p(torch.cuda.current_stream().cuda_stream))
    L.check(rc)
    torch.cuda.synchronize()
    return out, lout


PP_CASES = [
    # cin, cout, lin, stride, res_mode, P, out_q
    (32, 32, 7500, 1, 0, 2, 4),
    (32, 32, 7500, 1, 0, 2, 1),
    (32, 32, 7500, 2, 0, 2, 4),
    (32, 32, 3750, 1, 1, 2, 8),
    (32, 64, 1875, 1, 1, 2, 2),   # channel doubling: shortcut zero-padded to 64
    (64, 64, 938, 1, 1, 3, 2),
    (64, 64, 1875, 2, 0, 2, 4),
    (64, 64, 469, 1, 1, 2, 1),
    (16, 16, 469, 2, 0, 2, 8),
    (16, 16, 937, 1, 1, 2, 16),
    (16, 32, 1875, 1, 1, 2, 4),
    (64, 32, 300, 1, 0, 1, 2),
    (32, 16, 129, 1, 0, 2, 32),
]


@pytest.mark.parametrize("res_layout", ["native", "other"])
@pytest.mark.parametrize("cin,cout,lin,stride,res_mode,P,out_q", PP_CASES)
def test_pp_conv_matches_fp32(cin, cout, lin, stride, res_mode, P, out_q, res_layout):
    """res_layout "native": the identity shortcut is in this conv's own Q-phase
    layout (Q = 128/cout) and runs as selection MMAs on the tensor core;
    "other": a different Q, read by the epilogue."""
    if res_mode == 0 and res_layout == "other":
        pytest.skip("no shortcut")
    g = torch.Generator().manual_seed(cin * 5 + cout + lin + stride + out_q)
    x = torch.relu(_rand((P, cin, lin), g))
    w = _rand((cout, cin, 16), g, (2.0 / (cin * 16)) ** 0.5)
    b = _rand((cout,), g, 0.1)
    res = None
    if res_mode == 1:
        res = torch.relu(_rand((P, min(cin, cout), -(-lin // stride)), g))
    rq = (128 // cout if res_layout == "native" else (2 if 128 // cout != 2 else 4)) if res is not None else 1
    out, lout = run_q(x, w, b, stride, K_PP, res, res_mode, res_q=rq, out_q=out_q)
    ref = ref_conv(x, w, b, stride, res, res_mode)
    got = from_q(out, cout, lout, out_q).float().cpu()
    err = (got - ref).abs()
    tol = 2e-3 * ref.abs() + 2e-3
    assert bool((err <= tol).all()), f"max err {err.max().item():.3e} at {torch.nonzero(err > tol)[:4].tolist()}"
    assert q_padding_zero(out, lout, out_q), "padding slots must be written as zero"


@pytest.mark.parametrize("c,lin,res_len,res_q", [(32, 3750, 7500, 8), (32, 938, 1875, 2), (64, 1875, 3750, 4),
                                                 (16, 469, 937, 16)])
def test_pp_maxpool_shortcut(c, lin, res_len, res_q):
    """conv2 of a downsampling block on K4b: shortcut = maxpool(block input) read from its Q-phase layout."""
    g = torch.Generator().manual_seed(lin + c)
    P = 2
    x = torch.relu(_rand((P, c, lin), g))
    blk = torch.relu(_rand((P, c, res_len), g))
    w = _rand((c, c, 16), g, (2.0 / (c * 16)) ** 0.5)
    b = _rand((c,), g, 0.1)
    out, lout = run_q(x, w, b, 1, K_PP, blk, 2, res_q=res_q, out_q=1)
    ref = ref_conv(x, w, b, 1, blk, 2)
    got = from_q(out, c, lout, 1).float().cpu()
    assert torch.allclose(got, ref, rtol=2e-3, atol=2e-3), (got - ref).abs().max()


@pytest.mark.parametrize("out_q,res_q", [(4, 8), (8, 1), (16, 2)])
def test_tc_conv_q_layouts(out_q, res_q):
    """K4 writes and reads the shortcut in any Q-phase layout (it still reads I / S input)."""
    g = torch.Generator().manual_seed(out_q * 3 + res_q)
    P, c, lin = 2, 128, 938
    x = torch.relu(_rand((P, c, lin), g))
    blk = torch.relu(_rand((P, c, 2 * lin), g))
    w = _rand((c, c, 16), g, (2.0 / (c * 16)) ** 0.5)
    b = _rand((c,), g, 0.1)
    out, lout = run_q(x, w, b, 1, K_TC, blk, 2, res_q=res_q, out_q=out_q)
    ref = ref_conv(x, w, b, 1, blk, 2)
    got = from_q(out, c, lout, out_q).float().cpu()
    assert torch.allclose(got, ref, rtol=2e-3, atol=2e-3), (got - ref).abs().max()
    assert q_padding_zero(out, lout, out_q)


@pytest.mark.parametrize("cout,out_q,n", [(32, 4, 7500), (64, 2, 7500), (16, 8, 7500), (8, 1, 7500), (128, 1, 7500),
                                          (32, 1, 1001), (32, 2, 999), (64, 4, 1250), (16, 16, 777), (24, 4, 600), (48, 2, 1500), (128, 2, 500)])
def test_stem_q_layout(cout, out_q, n):
    L = _lib()
    g = torch.Generator().manual_seed(cout + out_q + n)
    P = 2
    x = _rand((P, n), g)
    w = _rand((cout, 1, 16), g, 0.25)
    b = _rand((cout,), g, 0.1)
    dev = torch.device("cuda")
    xd = x.half().to(dev).contiguous()
    out = torch.full((P, cout // 8, out_q, lq(n, out_q), 8), 7.0, dtype=torch.float16, device=dev)
    wn = np.ascontiguousarray(w.numpy().reshape(cout, 16), np.float32)
    bn = np.ascontiguousarray(b.numpy(), np.float32)
    L.check(L.lib().hb_op_stem_q(C.c_void_p(xd.data_ptr()), P, n, L.fptr(wn), L.fptr(bn), cout,
                                 C.c_void_p(out.data_ptr()), out_q, C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    torch.cuda.synchronize()
    ref = ref_conv(x[:, None, :], w, b, 1)
    got = from_q(out, cout, n, out_q).float().cpu()
    assert torch.allclose(got, ref, rtol=2e-3, atol=2e-3), (got - ref).abs().max()
    assert q_padding_zero(out, n, out_q)


def test_planner_routes_narrow_layers_to_pp():
    L = _lib()
    assert L.lib().hb_conv_kind(32, 32, 1, 0) == K_PP
    assert L.lib().hb_conv_kind(32, 32, 2, 0) == K_PP
    assert L.lib().hb_conv_kind(128, 128, 1, 0) == K_TC
    assert L.lib().hb_conv_kind(32, 32, 1, 1) == K_PP   # fused head on K4b too
    assert L.lib().hb_conv_kind(128, 128, 1, 1) == K_TC
    assert L.lib().hb_conv_kind(8, 8, 1, 0) == K_TC


@pytest.mark.parametrize("c,lin,P", [(64, 469, 3), (64, 1875, 2), (32, 938, 2), (16, 235, 4)])
def test_pp_fused_head(c, lin, P):
    """Last conv of a member on K4b: maxpool shortcut + ReLU + mean-pool.FC fused into the epilogue;
    the per-(tile, warp) partials sum to the fp32 reference (fp16 activations inside the dot)."""
    L = _lib()
    g = torch.Generator().manual_seed(c + lin + 11)
    x = torch.relu(_rand((P, c, lin), g))
    blk = torch.relu(_rand((P, c, 2 * lin), g))
    w = _rand((c, c, 16), g, (2.0 / (c * 16)) ** 0.5)
    b = _rand((c,), g, 0.1)
    fc = torch.randn(c, generator=g) / c ** 0.5
    dev = torch.device("cuda")
    in_q = 128 // c
    res_q = 2
    xin = to_q(x.to(dev), in_q)
    rin = to_q(blk.to(dev), res_q)
    mt = L.lib().hb_conv_head_mt(P, c, c, lin, 1, 2, K_PP)
    assert mt > 0
    head = torch.full((P, mt), 123.0, dtype=torch.float32, device=dev)
    wn = np.ascontiguousarray(w.numpy(), np.float32)
    bn = np.ascontiguousarray(b.numpy(), np.float32)
    fcn = np.ascontiguousarray(fc.numpy(), np.float32)
    L.check(L.lib().hb_op_conv1d_q(
        C.c_void_p(xin.data_ptr()), P, c, lin, 1, L.fptr(wn), L.fptr(bn), c, C.c_void_p(rin.data_ptr()), 2, c,
        2 * lin, res_q, None, 1, L.fptr(fcn), C.c_void_p(head.data_ptr()), K_PP,
        C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    torch.cuda.synchronize()
    ref = ref_conv(x, w, b, 1, blk, 2)
    ref_sum = (ref * fc[None, :, None]).sum(dim=(1, 2))
    got = head.cpu().sum(dim=1)
    assert torch.allclose(got, ref_sum, rtol=2e-3, atol=2e-2), (got, ref_sum)
