"""The CNN oracle is independent of the product's architecture code.

Three restatements of the frozen layer table exist: the oracle's own
(`oracle/cnn.layers`), the Python product's (`arch.member_layers`) and the one
the C-ABI library serves (`hb_member_layers`, csrc/hb_api.cu).  They must agree
on every zoo member, and the oracle decodes the exact parameter blob the
library consumes with its own table.  CPU only (the table query touches no
device)."""
import ctypes as C

import numpy as np
import pytest

from oracle import cnn, cpu_path
from paper_2008_04063_b200 import _lib, arch
from paper_2008_04063_b200.zoo import holmes_zoo

SHORTCUT = {"none": 0, "identity": 1, "maxpool": 2}


def _lib_table(width, depth, window):
    out = (C.c_int * (9 * 64))()
    n = _lib.lib().hb_member_layers(width, depth, window, out, 64)
    assert n > 0
    return np.array(out[:9 * n]).reshape(n, 9)


@pytest.mark.parametrize("window", [7500, 1000, 257])
def test_three_layer_tables_agree(window):
    shapes = sorted({(p.width, p.depth) for p in holmes_zoo().profiles})
    assert len(shapes) == 20
    for width, depth in shapes:
        mine = cnn.layers(width, depth, window)
        prod = arch.member_layers(width, depth, window)
        lib = _lib_table(width, depth, window)
        assert len(mine) == len(prod) == len(lib) == 1 + 2 * depth
        for k, (o, a, row) in enumerate(zip(mine, prod, lib)):
            assert o.name == a.name
            assert (o.cin, o.cout, o.stride, o.lin, o.lout, o.pad_left) == (a.cin, a.cout, a.stride, a.lin, a.lout, a.pad)
            assert o.shortcut == a.res
            want = [o.cin, o.cout, o.stride, o.lin, o.lout, o.pad_left, SHORTCUT[o.shortcut]]
            assert list(row[:7]) == want, (width, depth, k, row, want)
            assert row[8] == int(k == 2 * depth)          # the head is the last conv
            if o.shortcut != "none":
                assert row[7] == mine[k - 1].cin == a.res_c


def test_oracle_decodes_the_library_blob():
    zoo = holmes_zoo()
    for i in (0, 10, 13, 57):
        prof = zoo.profiles[i]
        params = arch.member_params(prof.width, prof.depth, 0, prof.id)
        blob = arch.flatten_params(params, prof.width, prof.depth)
        assert blob.size == arch.flat_param_count(prof.width, prof.depth)
        dec = cnn.unflatten(blob, prof.width, prof.depth, 7500)
        assert set(dec) == set(params)
        for k, (w, b) in params.items():
            assert np.array_equal(dec[k][0], w) and np.array_equal(dec[k][1], b), k
    with pytest.raises(ValueError):
        cnn.unflatten(np.zeros(10, np.float32), 8, 2, 7500)


def test_oracle_forward_small_cases():
    """Sanity of the oracle forward itself: finite O(1) logits, batch-independent per bed,
    and fp16 activation rounding moves logits by far less than the parity bar."""
    zoo = holmes_zoo()
    prof = zoo.profiles[0]            # ecg-i-w8-d2
    from paper_2008_04063_b200 import synth
    x = cnn.znorm(synth.ecg_block(0, 3, 1, 0, 7500)[:, 0])
    p = cpu_path.params_for(prof)
    a = cnn.member_forward(x, p, prof.width, prof.depth)
    b = np.concatenate([cnn.member_forward(x[i:i + 1], p, prof.width, prof.depth) for i in range(3)])
    assert np.all(np.isfinite(a)) and np.abs(a).max() < 20
    assert np.allclose(a, b, atol=1e-5)
    r = cnn.member_forward(x, p, prof.width, prof.depth, round_fp16=True)
    assert np.abs(r - a).max() < 2e-2
