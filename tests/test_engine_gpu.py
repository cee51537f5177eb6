"""End-to-end tick parity: ring ingest -> window -> z-norm -> every member's
forward -> aggregation, on the device through the C-ABI, against the CPU oracle
on identical synthetic streams.

Bars (BASELINE.json north_star):
  * window contents / indices: bit-exact (raw fp32 samples);
  * member and ensemble probabilities: |dev - oracle| <= 1e-3 absolute;
  * logits are compared too (sigmoid saturation cannot hide errors): <= 2e-2.
"""
import numpy as np
import pytest

from oracle import cnn, cpu_path, windows
from paper_2008_04063_b200 import synth
from paper_2008_04063_b200.zoo import Selector, holmes_zoo

pytestmark = pytest.mark.gpu

PROB_TOL = 1e-3
LOGIT_TOL = 2e-2
C2 = [10, 13, 30, 50]   # ecg-i-w32-d8, ecg-i-w64-d4, ecg-ii-w32-d8, ecg-iii-w32-d8


def _streams(P, n, seed=0, zero_patient=None):
    s = synth.ecg_block(seed, P, 3, 0, n)
    if zero_patient is not None:
        s[zero_patient] = 0.0
    return s


def _oracle_tick(zoo, sel, streams, end, W=7500, seed=0):
    return cpu_path.cpu_tick(zoo, sel, streams, end, W, seed)


def _compare(res, ml, prob, mean_logit):
    assert np.abs(res.member_logits - ml).max() <= LOGIT_TOL, np.abs(res.member_logits - ml).max()
    assert np.abs(cnn.sigmoid(res.member_logits) - cnn.sigmoid(ml)).max() <= PROB_TOL
    assert np.abs(res.ens_prob - prob).max() <= PROB_TOL
    assert np.abs(res.ens_mean_logit - mean_logit).max() <= LOGIT_TOL


def test_sliding_ticks_match_oracle():
    from paper_2008_04063_b200.engine import EnsembleEngine
    zoo = holmes_zoo()
    sel = Selector.from_indices(60, C2)
    P, W, hop = 5, 7500, 250
    streams = _streams(P, W + 2 * hop, zero_patient=3)
    with EnsembleEngine(zoo, sel, P, hop=hop, keep_windows=True) as eng:
        eng.ingest(streams[:, :, : W - hop])
        for k in range(3):
            end = W + k * hop
            res = eng.tick(streams[:, :, end - hop:end])
            raw, stats = eng.last_windows()
            for p in range(P):
                for lead in range(3):
                    exp = windows.sliding_window(streams[p, lead], end, W)
                    assert np.array_equal(raw[p, lead], exp), (k, p, lead)
            assert np.all(stats[3, :, 1] == 0.0)          # constant stream: zero-variance guard
            _compare(res, *_oracle_tick(zoo, sel, streams, end))


def test_tumbling_mode_equals_aggregator_windows():
    """hop == window: tick k scores exactly reference window k = samples [kW, (k+1)W)."""
    from paper_2008_04063_b200.engine import EnsembleEngine
    zoo = holmes_zoo()
    sel = Selector.from_indices(60, [10])
    P, W = 2, 7500
    streams = _streams(P, 2 * W, seed=3)
    with EnsembleEngine(zoo, sel, P, hop=W, keep_windows=True) as eng:
        for k in range(2):
            res = eng.tick(streams[:, :, k * W:(k + 1) * W])
            raw, _ = eng.last_windows()
            for p in range(P):
                for lead in range(3):
                    tumbling = windows.tumbling_windows(streams[p, lead], W)
                    assert np.array_equal(raw[p, lead], tumbling[k][1])
            _compare(res, *_oracle_tick(zoo, sel, streams, (k + 1) * W))


def test_selector_change_and_single_member():
    from paper_2008_04063_b200.engine import EnsembleEngine
    zoo = holmes_zoo()
    P, W, hop = 3, 7500, 250
    streams = _streams(P, W, seed=7)
    sel_a = Selector.from_indices(60, [0, 21])      # w8-d2 lead I, w8-d4 lead II
    with EnsembleEngine(zoo, sel_a, P, hop=hop) as eng:
        eng.ingest(streams[:, :, : W - hop])
        res = eng.tick(streams[:, :, W - hop:])
        _compare(res, *_oracle_tick(zoo, sel_a, streams, W))
        sel_b = Selector.from_indices(60, [6])       # ecg-i-w16-d16 (deep, 8 downsamples)
        eng.set_selector(sel_b)
        eng.ingest(np.zeros((P, 3, 0), np.float32))
        # re-score the same window: rewind is not supported, so compare the next tick
        more = synth.ecg_block(7, P, 3, W, hop)
        full = np.concatenate([streams, more], axis=2)
        res = eng.tick(more)
        _compare(res, *_oracle_tick(zoo, sel_b, full, W + hop))


def test_empty_selector_rejected():
    from paper_2008_04063_b200.engine import EnsembleEngine
    from paper_2008_04063_b200.errors import EmptyEnsembleError
    with pytest.raises(EmptyEnsembleError):
        EnsembleEngine(holmes_zoo(), Selector.zeros(60), 2)


def test_full_zoo_c3_matches_oracle():
    """Config c3's ensemble: all 60 members (every width 8..128 x depth 2..16 x lead),
    incl. streamed weights and multi-N-tile layers (w128-d16 reaches 1024 channels)."""
    from paper_2008_04063_b200.engine import EnsembleEngine
    zoo = holmes_zoo()
    sel = Selector.ones(60)
    P, W = 2, 7500
    streams = _streams(P, W, seed=11)
    with EnsembleEngine(zoo, sel, P, hop=W) as eng:
        res = eng.tick(streams)
    _compare(res, *_oracle_tick(zoo, sel, streams, W))


def test_patient_chunking_is_bit_identical(monkeypatch):
    """Member chains over patient chunks (activation budget) give bit-identical results."""
    from paper_2008_04063_b200.engine import EnsembleEngine
    zoo = holmes_zoo()
    sel = Selector.from_indices(60, C2)
    P, W, hop = 7, 7500, 250
    streams = _streams(P, W + hop, seed=12)
    outs = []
    for budget in (None, "0.05"):          # 50 MB forces chunks of 1-2 beds
        if budget:
            monkeypatch.setenv("HB_ACT_BUDGET_GB", budget)
        with EnsembleEngine(zoo, sel, P, hop=hop) as eng:
            eng.ingest(streams[:, :, :W - hop])
            eng.tick(streams[:, :, W - hop:W])
            outs.append(eng.tick(streams[:, :, W:W + hop]))
    assert np.array_equal(outs[0].member_logits, outs[1].member_logits)
    assert np.array_equal(outs[0].ens_prob, outs[1].ens_prob)


@pytest.mark.parametrize("knob", [("HB_STEM_GMAX", "1"), ("HB_STEM", "0")])
def test_stem_launch_variants_are_bit_identical(monkeypatch, knob):
    """The stem split into one launch per member (HB_STEM_GMAX=1) gives bit-identical outputs; the
    builder stem kernel (HB_STEM=0) agrees within fp32 summation order."""
    from paper_2008_04063_b200.engine import EnsembleEngine
    zoo = holmes_zoo()
    sel = Selector.from_indices(60, C2)
    P, W, hop = 5, 7500, 250
    streams = _streams(P, W + hop, seed=21)
    outs = []
    for env in (None, knob):
        if env:
            monkeypatch.setenv(*env)
        with EnsembleEngine(zoo, sel, P, hop=hop) as eng:
            eng.ingest(streams[:, :, :W - hop])
            eng.tick(streams[:, :, W - hop:W])
            outs.append(eng.tick(streams[:, :, W:W + hop]))
    if knob[0] == "HB_STEM_GMAX":
        assert np.array_equal(outs[0].member_logits, outs[1].member_logits)
        assert np.array_equal(outs[0].ens_prob, outs[1].ens_prob)
    else:
        assert np.allclose(outs[0].member_logits, outs[1].member_logits, rtol=0, atol=2e-2)
        assert np.allclose(outs[0].ens_prob, outs[1].ens_prob, rtol=0, atol=1e-3)


def test_pipelined_submit_collect_matches_blocking_ticks():
    """submit(t+1) before collect(t): same outputs, bit for bit, as one blocking tick per step;
    a third submit while both slots hold uncollected ticks is refused."""
    from paper_2008_04063_b200.engine import EnsembleEngine
    zoo = holmes_zoo()
    sel = Selector.from_indices(60, [0, 21])
    P, W, hop, n = 4, 7500, 250, 6
    streams = _streams(P, W + n * hop, seed=3)
    blocks = [np.ascontiguousarray(streams[:, :, W - hop + k * hop: W + k * hop]) for k in range(n)]
    ref = []
    with EnsembleEngine(zoo, sel, P, hop=hop) as eng:
        eng.ingest(streams[:, :, : W - hop])
        for b in blocks:
            r = eng.tick(b)
            ref.append((r.member_logits.copy(), r.ens_prob.copy(), r.ens_mean_logit.copy()))
    got = []
    with EnsembleEngine(zoo, sel, P, hop=hop) as eng:
        eng.ingest(streams[:, :, : W - hop])
        slot = eng.submit(blocks[0])
        for k in range(n):
            nxt = eng.submit(blocks[k + 1]) if k + 1 < n else None
            if k == 0:
                with pytest.raises(RuntimeError):
                    eng.submit(blocks[0])   # both slots busy (HB_E_STATE)
            r = eng.collect(slot)
            got.append((r.member_logits.copy(), r.ens_prob.copy(), r.ens_mean_logit.copy()))
            slot = nxt
    for (a, b, c), (x, y, z) in zip(ref, got):
        assert np.array_equal(a, x) and np.array_equal(b, y) and np.array_equal(c, z)


def test_many_ticks_across_ring_wraps():
    """70 sliding ticks: the ring (R = roundup(W + hop, 256)) wraps twice; every tick's gathered
    window stays bit-exact (the mirrored ring tail keeps each window one contiguous run) and the
    last tick's scores match the oracle."""
    from paper_2008_04063_b200.engine import EnsembleEngine
    zoo = holmes_zoo()
    sel = Selector.from_indices(60, [0])
    P, W, hop, n = 2, 7500, 250, 70
    streams = _streams(P, W + n * hop, seed=7)
    with EnsembleEngine(zoo, sel, P, hop=hop, keep_windows=True) as eng:
        eng.ingest(streams[:, :, : W - hop])
        for k in range(n):
            end = W + k * hop
            res = eng.tick(streams[:, :, end - hop:end])
            if k % 7 == 0 or k == n - 1:
                raw, _ = eng.last_windows()
                for p in range(P):
                    for lead in range(3):
                        assert np.array_equal(raw[p, lead], windows.sliding_window(streams[p, lead], end, W)), k
        _compare(res, *_oracle_tick(zoo, sel, streams, end))


def test_selector_change_refused_while_a_tick_is_uncollected():
    """a submitted tick keeps its own member layout.  Changing the selector (or
    registering a member) while a slot holds an uncollected tick is refused (HB_E_STATE ->
    RuntimeError) instead of freeing that slot's pinned outputs; after collect it works."""
    from paper_2008_04063_b200.engine import EnsembleEngine
    zoo = holmes_zoo()
    P, W, hop = 3, 7500, 250
    streams = _streams(P, W + hop, seed=9)
    sel_a = Selector.from_indices(60, [0])
    sel_b = Selector.from_indices(60, [0, 21, 40])
    with EnsembleEngine(zoo, sel_a, P, hop=hop) as eng:
        eng.ingest(streams[:, :, : W - hop])
        slot = eng.submit(np.ascontiguousarray(streams[:, :, W - hop:W]))
        with pytest.raises(RuntimeError, match="uncollected"):
            eng.set_selector(sel_b)
        res = eng.collect(slot)
        assert res.member_ids == ("ecg-i-w8-d2",) and res.member_logits.shape == (P, 1)
        _compare(res, *_oracle_tick(zoo, sel_a, streams, W))
        eng.set_selector(sel_b)
        res = eng.tick(np.ascontiguousarray(streams[:, :, W:W + hop]))
        assert res.member_logits.shape == (P, 3)
        _compare(res, *_oracle_tick(zoo, sel_b, streams, W + hop))


@pytest.mark.parametrize("chain", ["0", "1"])
def test_nonfinite_samples_stay_in_their_bed(monkeypatch, chain):
    """Fault isolation: a NaN sample (bed 3, lead I) and an Inf sample (bed 8, lead III) make
    exactly the members reading those leads non-finite for those beds -- z-normalisation, the
    convs (NaN-propagating ReLU / max-pool, as the fp32 oracle), the head and the aggregate are
    per bed and per lead -- and so the beds' ensemble scores; every other bed, and those beds'
    other members, are bit-identical to a run on clean streams, on both tick paths."""
    from paper_2008_04063_b200.engine import EnsembleEngine
    monkeypatch.setenv("HB_CHAIN", chain)
    zoo = holmes_zoo()
    sel = Selector.from_indices(60, C2)
    P, W, hop = 12, 7500, 250
    clean = _streams(P, W + hop, seed=21)
    dirty = clean.copy()
    dirty[3, 0, W - 40] = np.nan      # bed 3, lead I (read by two members)
    dirty[8, 2, W + 10] = np.inf      # bed 8, lead III, in the newest hop
    outs = []
    for s in (clean, dirty):
        with EnsembleEngine(zoo, sel, P, hop=hop) as eng:
            eng.ingest(s[:, :, :W - hop])
            eng.tick(s[:, :, W - hop:W])
            outs.append(eng.tick(s[:, :, W:W + hop]))
    ok = [p for p in range(P) if p not in (3, 8)]
    assert np.array_equal(outs[0].member_logits[ok], outs[1].member_logits[ok])
    assert np.array_equal(outs[0].ens_prob[ok], outs[1].ens_prob[ok])
    assert np.isfinite(outs[0].member_logits).all() and np.isfinite(outs[0].ens_prob).all()
    ml = outs[1].member_logits    # columns: ecg-i-w32-d8, ecg-i-w64-d4 (lead I), ecg-ii-w32-d8, ecg-iii-w32-d8
    assert np.isnan(ml[3, :2]).all() and np.array_equal(ml[3, 2:], outs[0].member_logits[3, 2:])
    assert np.isnan(ml[8, 3]) and np.array_equal(ml[8, :3], outs[0].member_logits[8, :3])
    assert np.isnan(outs[1].ens_prob[[3, 8]]).all() and np.isnan(outs[1].ens_mean_logit[[3, 8]]).all()
