"""Oracle parity at the configurations the benchmark times (VERDICT r1 lead item).

The benchmark's c2 tick (4 members, 64 beds) and the north-star 1024-bed tick
run K4b's multi-wave paths — persistent CTAs looping over several tiles, the
second TMEM accumulator and its epilogue warpgroups, member-partitioned CTAs,
mid-CTA weight reloads, 160/240-wide column tiles — that small-P tests never
reach.  Every test here compares the device tick through the C-ABI with the
CPU fp32 oracle (`oracle/cpu_path.cpu_tick`, PyTorch fp32, the oracle's own
layer table) on identical synthetic streams:

  * raw window samples: bit-exact (`Aggregator` semantics, runtime.py:98-115);
  * z-normalised fp16 windows: within 1 fp16 ulp of the fp64 oracle value;
  * member / ensemble probabilities: |dev - oracle| <= 1e-3 (north star);
  * logits: <= 2e-2 (sigmoid saturation cannot hide an error).

Configs: BASELINE.json configs c1 (1 member, 1 bed), c2 (4 members, 64 beds,
every bed, 3 sliding ticks), north-star scale (1024 beds, 64 sampled beds),
c3 (60-member zoo, 100 beds, sampled beds), plus the multi-tile K4b paths
forced at small P through the planner's knobs.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle import cnn, cpu_path, windows
from paper_2008_04063_b200 import synth
from paper_2008_04063_b200.zoo import Selector, holmes_zoo

pytestmark = pytest.mark.gpu

PROB_TOL = 1e-3
LOGIT_TOL = 2e-2
W = 7500
C2 = [10, 13, 30, 50]   # ecg-i-w32-d8, ecg-i-w64-d4, ecg-ii-w32-d8, ecg-iii-w32-d8
HERE = os.path.dirname(os.path.abspath(__file__))


def _compare(got_ml, got_prob, got_ml_mean, ml, prob, mean_logit):
    d_logit = float(np.abs(got_ml - ml).max())
    d_mprob = float(np.abs(cnn.sigmoid(got_ml) - cnn.sigmoid(ml)).max())
    d_prob = float(np.abs(got_prob - prob).max())
    d_mean = float(np.abs(got_ml_mean - mean_logit).max())
    assert d_logit <= LOGIT_TOL and d_mprob <= PROB_TOL and d_prob <= PROB_TOL and d_mean <= LOGIT_TOL, \
        (d_logit, d_mprob, d_prob, d_mean)
    return d_logit, d_prob


XN_FLOOR = 1e-6


def _check_xn(xn, streams, end, beds, zoo_leads=3):
    """Device z-normalised windows vs the fp64 oracle: within one fp16 ulp at the oracle value's
    magnitude, or XN_FLOOR absolute where that ulp is smaller (|z| < ~1e-3: the device's fp32
    mean/std carry ~1e-7 of rounding that a subnormal-range fp16 ulp cannot absorb)."""
    for lead in range(zoo_leads):
        win = np.stack([windows.sliding_window(streams[p, lead], end, W) for p in beds]).astype(np.float64)
        mean = win.mean(axis=-1, keepdims=True)
        ref = (win - mean) / np.maximum(win.std(axis=-1, keepdims=True), 1e-6)
        dev = xn[lead, beds].astype(np.float64)
        ulp = np.maximum(np.spacing(np.abs(ref).astype(np.float16)).astype(np.float64), XN_FLOOR)
        bad = np.abs(dev - ref) > ulp
        assert not bad.any(), (lead, int(bad.sum()), float(np.abs(dev - ref).max()))


def _run(sel, P, hop, ticks, seed, check_beds, zero_bed=None, check_every_tick=True, xn_check=True):
    from paper_2008_04063_b200.engine import EnsembleEngine
    zoo = holmes_zoo()
    streams = synth.ecg_block(seed, P, 3, 0, W + ticks * hop)
    if zero_bed is not None:
        streams[zero_bed] = 0.0          # the reference's own wall-clock signal (runtime.py:358)
    worst = (0.0, 0.0)
    with EnsembleEngine(zoo, sel, P, hop=hop, keep_windows=True) as eng:
        eng.ingest(streams[:, :, :W - hop])
        for k in range(ticks):
            end = W + k * hop
            res = eng.tick(streams[:, :, end - hop:end])
            if not check_every_tick and k != ticks - 1:
                continue
            raw, stats = eng.last_windows()
            for p in check_beds:
                for lead in range(3):
                    assert np.array_equal(raw[p, lead], windows.sliding_window(streams[p, lead], end, W)), (k, p)
            if zero_bed is not None:
                assert np.all(stats[zero_bed, :, 1] == 0.0)
            if xn_check:
                _check_xn(eng.last_normalized(), streams, end, check_beds)
            ml, prob, mlog = cpu_path.cpu_tick(zoo, sel, streams, end, beds=check_beds)
            d = _compare(res.member_logits[check_beds], res.ens_prob[check_beds], res.ens_mean_logit[check_beds],
                         ml, prob, mlog)
            worst = tuple(max(a, b) for a, b in zip(worst, d))
    return worst


def test_c1_one_member_one_bed():
    """BASELINE c1: ecg-i-w32-d8, 1 bed, 1 s sliding ticks (the config the CPU reference runs)."""
    _run(Selector.from_indices(60, [10]), 1, 250, 4, 0, [0])


def test_c2_64_beds_every_bed_three_ticks():
    """BASELINE c2 exactly as bench.py times it: 4 members, 64 beds, hop 250, every bed, 3 ticks."""
    _run(Selector.from_indices(60, C2), 64, 250, 3, 0, list(range(64)), zero_bed=17)


@pytest.mark.parametrize("chain", ["auto", "one_launch", "chunks"])
def test_north_star_1024_beds_sampled(monkeypatch, chain):
    """The north-star scale: 1024 beds; 64 beds spread over the range (first, last, and
    the chunk/tile boundaries in between) against the oracle, 2 ticks -- on the default path
    (per-layer launches at this bed count), the K4c chain as ONE launch over every bed, and the
    chain over 64-bed chunks (HB_CHAIN_CHUNK_P=64, one launch each)."""
    if chain == "one_launch":
        monkeypatch.setenv("HB_CHAIN", "1")
    elif chain == "chunks":
        monkeypatch.setenv("HB_CHAIN_CHUNK_P", "64")
    beds = sorted(set(np.linspace(0, 1023, 62).astype(int).tolist()) | {511, 512})
    _run(Selector.from_indices(60, C2), 1024, 250, 2, 1, beds, zero_bed=511, check_every_tick=False)


def test_c3_full_zoo_100_beds_sampled():
    """BASELINE c3: the whole 60-member zoo over 100 beds (K4 wide layers, streamed weights,
    multi-N-tile heads), 5 sampled beds against the oracle."""
    _run(Selector.ones(60), 100, 250, 1, 2, [0, 33, 50, 71, 99], xn_check=True)


@pytest.mark.parametrize("hop", [249, 251, 7500])
def test_window_alignment_and_warmup(hop):
    """The vectorised window kernel reads 16-B aligned float4s and shifts by the window start's
    misalignment (start mod 4, uniform per tick).  An odd hop walks the start through all four
    residues; ticks from an EMPTY ring put the window start before the stream's first sample
    (zeros, `oracle.windows.sliding_window`).  Raw samples bit-exact, fp16 z-norm within 1 ulp,
    and the tick's scores against the oracle at the last tick."""
    from paper_2008_04063_b200.engine import EnsembleEngine
    zoo = holmes_zoo()
    sel = Selector.from_indices(60, [10])
    P, ticks = 3, 5 if hop < W else 2
    streams = synth.ecg_block(21, P, 3, 0, ticks * hop)
    residues = set()
    with EnsembleEngine(zoo, sel, P, hop=hop, keep_windows=True) as eng:
        for k in range(ticks):
            end = (k + 1) * hop
            res = eng.tick(streams[:, :, end - hop:end])
            residues.add((end - W) % 4)
            raw, _ = eng.last_windows()
            for p in range(P):
                for lead in range(3):
                    assert np.array_equal(raw[p, lead], windows.sliding_window(streams[p, lead], end, W)), (k, p)
            _check_xn(eng.last_normalized(), streams, end, list(range(P)))
    ml, prob, mlog = cpu_path.cpu_tick(zoo, sel, streams, end, beds=list(range(P)))
    _compare(res.member_logits, res.ens_prob, res.ens_mean_logit, ml, prob, mlog)
    if hop < W:
        assert residues == {0, 1, 2, 3}


@pytest.mark.parametrize("lane_sms", ["3", "4", "6", "9"])
def test_k4b_multi_tile_paths_forced(monkeypatch, lane_sms):
    """Per-layer K4b launches (HB_CHAIN=0) with every conv grid capped at a few CTAs
    (HB_LANE_SMS) so that at 5 beds each persistent CTA loops over many tiles: both TMEM
    accumulators and all four epilogue warpgroups, and either member-partitioned CTAs (6, 9: the
    grid splits evenly over the 3-member group) or round-robin CTAs that reload a different
    member's weight image mid-layer (3, 4)."""
    monkeypatch.setenv("HB_CHAIN", "0")
    monkeypatch.setenv("HB_LANE_SMS", ",".join([lane_sms] * 4))
    _run(Selector.from_indices(60, C2), 5, 250, 2, 3, list(range(5)), xn_check=False)


@pytest.mark.parametrize("chain_sms", ["1", "3", "5", "13"])
def test_k4c_chain_capped_grid(monkeypatch, chain_sms):
    """The K4c chain launch on a capped grid (HB_CHAIN_SMS): with fewer CTAs than queues every
    queue but the home ones is drained by stealing (1, 3), and with a few CTAs per queue each CTA
    walks many layers, weight images and dependency waits (5, 13) -- 7 beds, 2 sliding ticks,
    every bed against the oracle."""
    monkeypatch.setenv("HB_CHAIN", "1")
    monkeypatch.setenv("HB_CHAIN_SMS", chain_sms)
    _run(Selector.from_indices(60, C2), 7, 250, 2, 6, list(range(7)), xn_check=False)


def test_k4c_chain_is_the_c2_tick():
    """The benchmark's c2 selection runs as the window kernel, ONE stem launch for both member
    groups and ONE chain launch (kind 6) with the ensemble aggregation fused in: three launches per
    tick (HB_CHAIN_AGG=0 adds the separate aggregate kernel, kind 3)."""
    from paper_2008_04063_b200.engine import EnsembleEngine
    zoo = holmes_zoo()
    with EnsembleEngine(zoo, Selector.from_indices(60, C2), 8, hop=250) as eng:
        eng.ingest(synth.ecg_block(0, 8, 3, 0, W))
        kinds = eng.profile_tick()[0].tolist()
    assert kinds == [0, 1, 6], kinds


@pytest.mark.parametrize("P,extra", [(64, {}), (16, {"HB_CHAIN_SMS": "5"}), (9, {"HB_CHAIN_SMS": "2"})])
def test_chain_fused_aggregation_bit_identical(tmp_path, P, extra):
    """Aggregation fused into the K4c launch (warp 3 of CTA p mod grid sums bed p's head partials
    once the bed's per-launch head-tile count is reached; the last CTA out advances the ring
    cursor) against the separate aggregate kernel (HB_CHAIN_AGG=0): bit-identical over three
    sliding ticks (the cursor and the epoch-relative counters carry across ticks), with capped
    grids where one CTA aggregates several beds; both match the oracle."""
    hop, ticks, seed = 250, 3, 15
    outs = {}
    for agg in ("0", "1"):
        out = tmp_path / f"tick{agg}.npz"
        e = dict(os.environ, HB_CHAIN="1", HB_CHAIN_AGG=agg, **extra)
        subprocess.run([sys.executable, os.path.join(HERE, "_tick_worker.py"), str(out), str(P), str(hop),
                        str(ticks), str(seed), ",".join(map(str, C2))], check=True, env=e, timeout=600)
        outs[agg] = np.load(out)
    for k in ("member_logits", "ens_prob", "ens_mean_logit"):
        assert np.array_equal(outs["1"][k], outs["0"][k]), k
    got = outs["1"]
    streams = synth.ecg_block(seed, P, 3, 0, W + ticks * hop)
    beds = sorted({0, P // 2, P - 1})
    ml, prob, mlog = cpu_path.cpu_tick(holmes_zoo(), Selector.from_indices(60, C2), streams, int(got["end"]),
                                       beds=beds)
    _compare(got["member_logits"][beds], got["ens_prob"][beds], got["ens_mean_logit"][beds], ml, prob, mlog)


def test_k4b_group_caps(monkeypatch):
    """HB_MAX_GROUP=2: the three w32 members split into a 2-group and a 1-group (other lanes,
    other tile plans)."""
    monkeypatch.setenv("HB_MAX_GROUP", "2")
    _run(Selector.from_indices(60, C2), 7, 250, 1, 4, list(range(7)), xn_check=False)


STATIC_KNOBS = [
    {"HB_PP_NB": "64"},                       # narrowest column tiles: most tiles per CTA
    {"HB_PP_NB": "256"},                      # widest tiles
    {"HB_PP_NB": "160", "HB_PP_SPLIT": "0"},  # 160-wide tiles, round-robin CTAs
    {"HB_PP_SPLIT": "0", "HB_LANE_SMS": "5,5,5,5"},
    {"HB_PP_STAGES": "2"},                    # shallowest B pipeline
    {"HB_PP_RES_EPI": "1"},                   # identity shortcut in the epilogue instead of MMAs
    {"HB_WIN": "1"},                          # shared-memory window kernel
    {"HB_WIN": "2"},                          # scalar register window kernel (pre-vectorisation)
    {"HB_WIN_NB": "3"},                       # TMA window kernel, 3 buffers (two streams of look-ahead)
    {"HB_WIN_NB": "1"},                       # TMA window kernel, 1 buffer (no look-ahead, 6 CTAs/SM)
    {"HB_CHAIN": "0"},                        # per-layer K4b launches (lanes), no chain
    {"HB_CHAIN": "0", "HB_PP_NB": "160"},     # per-layer, 160-wide tiles
    {"HB_PP_STAGES": "6"},                    # chain: producer up to three items ahead of the MMA
]


@pytest.mark.parametrize("env", STATIC_KNOBS, ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items()))
def test_k4b_planner_variants_match_oracle(tmp_path, env):
    """Planner knobs read once per process: run the tick in a subprocess and check its outputs
    against the oracle (64 beds, c2 — the benchmark's shape; the K4c chain unless HB_CHAIN=0)."""
    P, hop, ticks, seed = 64, 250, 2, 5
    out = tmp_path / "tick.npz"
    e = dict(os.environ, **env)
    subprocess.run([sys.executable, os.path.join(HERE, "_tick_worker.py"), str(out), str(P), str(hop), str(ticks),
                    str(seed), ",".join(map(str, C2))], check=True, env=e, timeout=600)
    got = np.load(out)
    streams = synth.ecg_block(seed, P, 3, 0, W + ticks * hop)
    beds = list(range(0, 64, 3))
    ml, prob, mlog = cpu_path.cpu_tick(holmes_zoo(), Selector.from_indices(60, C2), streams, int(got["end"]),
                                       beds=beds)
    _compare(got["member_logits"][beds], got["ens_prob"][beds], got["ens_mean_logit"][beds], ml, prob, mlog)


def test_k4c_timeline_is_complete_and_causal(monkeypatch):
    """The chain launch's per-item timeline (HB_CHAIN_PROF=1, `hb_chain_trace`): every queue item of
    every layer was pulled, got its weight image, had its dependencies met and published both column
    halves, in that order; and within each member chain no layer's item had its dependencies met
    before the first tile of the layer it reads was published."""
    import ctypes as C

    from paper_2008_04063_b200 import _lib
    from paper_2008_04063_b200.engine import EnsembleEngine
    monkeypatch.setenv("HB_CHAIN", "1")
    monkeypatch.setenv("HB_CHAIN_PROF", "1")
    P = 16
    with EnsembleEngine(holmes_zoo(), Selector.from_indices(60, C2), P, hop=250) as eng:
        eng.ingest(synth.ecg_block(3, P, 3, 0, W))
        eng.time_tick(2)
        cap = 1 << 18
        tr = np.zeros((cap, 5), np.uint64)
        items = np.zeros(cap, np.int32)
        n = _lib.lib().hb_chain_trace(eng._h, tr.ctypes.data_as(C.c_void_p), items.ctypes.data_as(C.c_void_p), cap)
    assert n > 0
    tr, items = tr[:n].astype(np.int64), items[:n]
    assert (tr > 0).all(), "an item was never pulled, readied or published"
    assert (tr[:, 0] <= tr[:, 1]).all() and (tr[:, 1] <= tr[:, 2]).all()
    assert (tr[:, 2] <= tr[:, 3]).all() and (tr[:, 2] <= tr[:, 4]).all()
    layer = items >> 22
    done = np.maximum(tr[:, 3], tr[:, 4])
    # chain layers in order: w32 group (16 conv layers), then w64 (8): layer j > first of its group reads j - 1
    firsts = {0, 16}
    for j in sorted(set(layer.tolist())):
        if j in firsts:
            continue
        assert tr[layer == j, 2].min() >= done[layer == j - 1].min(), j


WIDE = [15, 16, 17, 36]   # w64-d16 (up to 512 channels), w128-d2 (x2, grouped), w128-d4: K4 with streamed weights


def test_k4_streamed_weight_slots_bit_identical(tmp_path):
    """K4's streamed-weight ring depth (HB_K4_BSLOTS: 2 = double buffer, default up to 4 images in
    flight) changes only when weight images arrive, never the MMA order: the ticks are bit-identical
    across depths, and both match the oracle."""
    P, hop, ticks, seed = 4, 250, 1, 11
    outs = {}
    for slots in ("2", "3", "4"):
        out = tmp_path / f"tick{slots}.npz"
        e = dict(os.environ, HB_K4_BSLOTS=slots)
        subprocess.run([sys.executable, os.path.join(HERE, "_tick_worker.py"), str(out), str(P), str(hop),
                        str(ticks), str(seed), ",".join(map(str, WIDE))], check=True, env=e, timeout=600)
        outs[slots] = np.load(out)
    for slots in ("3", "4"):
        for k in ("member_logits", "ens_prob", "ens_mean_logit"):
            assert np.array_equal(outs[slots][k], outs["2"][k]), (slots, k)
    got = outs["4"]
    streams = synth.ecg_block(seed, P, 3, 0, W + ticks * hop)
    beds = list(range(P))
    ml, prob, mlog = cpu_path.cpu_tick(holmes_zoo(), Selector.from_indices(60, WIDE), streams, int(got["end"]),
                                       beds=beds)
    _compare(got["member_logits"][beds], got["ens_prob"][beds], got["ens_mean_logit"][beds], ml, prob, mlog)


def test_k4_cta_pairs_bit_identical(tmp_path):
    """K4 on CTA pairs (HB_K4_PAIR=1: cta_group::2, M = 256 over two CTAs, weights split along N
    and streamed through the leader's barriers) against single-CTA tiles: each output element sees
    the same MMA sequence, so the ticks are bit-identical; both match the oracle.  Odd tile counts
    (the last pair's second tile past the layer) and the head layers' partials are covered by the
    w64-d16 member's short deep layers."""
    P, hop, ticks, seed = 5, 250, 1, 12
    outs = {}
    for pair in ("0", "1"):
        out = tmp_path / f"tick{pair}.npz"
        e = dict(os.environ, HB_K4_PAIR=pair)
        subprocess.run([sys.executable, os.path.join(HERE, "_tick_worker.py"), str(out), str(P), str(hop),
                        str(ticks), str(seed), ",".join(map(str, WIDE))], check=True, env=e, timeout=600)
        outs[pair] = np.load(out)
    for k in ("member_logits", "ens_prob", "ens_mean_logit"):
        assert np.array_equal(outs["1"][k], outs["0"][k]), k
    got = outs["1"]
    streams = synth.ecg_block(seed, P, 3, 0, W + ticks * hop)
    beds = list(range(P))
    ml, prob, mlog = cpu_path.cpu_tick(holmes_zoo(), Selector.from_indices(60, WIDE), streams, int(got["end"]),
                                       beds=beds)
    _compare(got["member_logits"][beds], got["ens_prob"][beds], got["ens_mean_logit"][beds], ml, prob, mlog)


DEEP = [15, 19]   # w64-d16 (512-channel L = 59 / 30 layers), w128-d16 (1024-channel L = 59 / 30 layers)


@pytest.mark.parametrize("agg", ["1", "0"])
def test_chain_bed_chunks_bit_identical(tmp_path, agg):
    """HB_CHAIN_CHUNK_P=64: above HB_CHAIN_MAX_P beds the chain runs one launch per bed chunk
    (buffers reused, head partials and the fused aggregation per chunk, the ring cursor advanced
    by the last chunk; opt-in, measured slower than the per-layer launches).  200 beds in chunks of 64 (the last one 8 beds + 56 padding rows) against
    the per-layer launches and against one chain launch over every bed: bit-identical over two
    sliding ticks, with the fused aggregation and with K5; sampled beds against the oracle."""
    P, hop, ticks, seed = 200, 250, 2, 16
    outs = {}
    for name, env in (("chunks", {"HB_CHAIN_CHUNK_P": "64"}), ("layers", {"HB_CHAIN": "0"}),
                      ("one", {"HB_CHAIN": "1", "HB_CHAIN_CHUNK_P": "0"})):
        out = tmp_path / f"tick_{name}.npz"
        e = dict(os.environ, HB_CHAIN_AGG=agg, **env)
        subprocess.run([sys.executable, os.path.join(HERE, "_tick_worker.py"), str(out), str(P), str(hop),
                        str(ticks), str(seed), ",".join(map(str, C2))], check=True, env=e, timeout=600)
        outs[name] = np.load(out)
    for other in ("layers", "one"):
        for k in ("member_logits", "ens_prob", "ens_mean_logit"):
            assert np.array_equal(outs["chunks"][k], outs[other][k]), (other, k)
    got = outs["chunks"]
    streams = synth.ecg_block(seed, P, 3, 0, W + ticks * hop)
    beds = [0, 63, 64, 127, 128, 191, 192, 199]
    ml, prob, mlog = cpu_path.cpu_tick(holmes_zoo(), Selector.from_indices(60, C2), streams, int(got["end"]),
                                       beds=beds)
    _compare(got["member_logits"][beds], got["ens_prob"][beds], got["ens_mean_logit"][beds], ml, prob, mlog)


def test_k4_half_pairs_bit_identical(tmp_path):
    """K4 half pairs (HB_K4_HALF=1: M = 128 over the CTA pair, 64 output rows per CTA, two beds per
    pair) on the deep layers whose output fits 64 rows per bed, against full 256-row pairs: every
    output element sees the same MMA sequence, so the ticks are bit-identical; both match the
    oracle.  An odd bed count leaves the last pair's second half past the layer."""
    P, hop, ticks, seed = 3, 250, 1, 14
    outs = {}
    for half in ("0", "1"):
        out = tmp_path / f"tick{half}.npz"
        e = dict(os.environ, HB_K4_HALF=half)
        subprocess.run([sys.executable, os.path.join(HERE, "_tick_worker.py"), str(out), str(P), str(hop),
                        str(ticks), str(seed), ",".join(map(str, DEEP))], check=True, env=e, timeout=600)
        outs[half] = np.load(out)
    for k in ("member_logits", "ens_prob", "ens_mean_logit"):
        assert np.array_equal(outs["1"][k], outs["0"][k]), k
    got = outs["1"]
    streams = synth.ecg_block(seed, P, 3, 0, W + ticks * hop)
    beds = list(range(P))
    ml, prob, mlog = cpu_path.cpu_tick(holmes_zoo(), Selector.from_indices(60, DEEP), streams, int(got["end"]),
                                       beds=beds)
    _compare(got["member_logits"][beds], got["ens_prob"][beds], got["ens_mean_logit"][beds], ml, prob, mlog)


def test_k4_cta_pairs_under_lane_caps(tmp_path):
    """CTA-pair K4 launches inside SM-capped lanes (HB_LANE_SMS=1,2,3,5: a lane below two SMs still
    gets one cluster; odd caps round down to whole pairs): bit-identical to the uncapped tick."""
    P, hop, ticks, seed = 3, 250, 1, 13
    outs = {}
    for name, env in (("free", {}), ("capped", {"HB_LANE_SMS": "1,2,3,5"})):
        out = tmp_path / f"tick_{name}.npz"
        subprocess.run([sys.executable, os.path.join(HERE, "_tick_worker.py"), str(out), str(P), str(hop),
                        str(ticks), str(seed), ",".join(map(str, WIDE))], check=True, env=dict(os.environ, **env),
                       timeout=600)
        outs[name] = np.load(out)
    for k in ("member_logits", "ens_prob", "ens_mean_logit"):
        assert np.array_equal(outs["capped"][k], outs["free"][k]), k
