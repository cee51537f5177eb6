"""The K4c chain launch against the per-layer path on random selections (seeded): any mix of the
K4b-eligible members (widths 16-64: one to four groups, 1-3 members each, depth 2-16), random bed
counts and chain grid caps.  The two paths must agree bit for bit (every output element
accumulates its MMAs in the same order whatever the tile plan, and the head partials use the same
grouping), so this exercises the chain's planner, queues, stealing and dependency ranges on shapes
the fixed-configuration tests do not reach; one case per seed is also checked against the CPU
oracle."""
import numpy as np
import pytest

from oracle import cpu_path
from paper_2008_04063_b200 import synth
from paper_2008_04063_b200.zoo import Selector, holmes_zoo

pytestmark = pytest.mark.gpu
W = 7500


def _eligible(zoo):
    from paper_2008_04063_b200 import arch
    out = []
    for i, p in enumerate(zoo.profiles):
        L = arch.member_layers(p.width, p.depth)
        if all(16 <= l.cin <= 64 and 16 <= l.cout <= 64 for l in L[1:]):
            out.append(i)
    return out


def _tick(monkeypatch, zoo, sel, P, streams, hop, env):
    from paper_2008_04063_b200.engine import EnsembleEngine
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    with EnsembleEngine(zoo, sel, P, hop=hop) as eng:
        eng.ingest(streams[:, :, :W - hop])
        eng.tick(streams[:, :, W - hop:W])
        res = eng.tick(streams[:, :, W:W + hop])
        kinds = eng.profile_tick()[0].tolist()
    for k in env:
        monkeypatch.delenv(k)
    return res, kinds


@pytest.mark.parametrize("seed", range(12))
def test_chain_matches_per_layer_path_on_random_selections(monkeypatch, seed):
    zoo = holmes_zoo()
    rng = np.random.default_rng(100 + seed)
    elig = _eligible(zoo)
    k = int(rng.integers(1, 7))
    idx = sorted(rng.choice(elig, size=k, replace=False).tolist())
    sel = Selector.from_indices(60, idx)
    P = int(rng.integers(1, 24))
    hop = 250
    streams = synth.ecg_block(seed, P, 3, 0, W + hop)
    cap = str(int(rng.choice([0, 3, 17, 148])))
    chain, kinds_c = _tick(monkeypatch, zoo, sel, P, streams, hop, {"HB_CHAIN": "1", "HB_CHAIN_SMS": cap} if cap != "0"
                           else {"HB_CHAIN": "1"})
    layer, kinds_l = _tick(monkeypatch, zoo, sel, P, streams, hop, {"HB_CHAIN": "0"})
    assert 6 in kinds_c and 6 not in kinds_l, (kinds_c, kinds_l)
    assert np.array_equal(chain.member_logits, layer.member_logits), (idx, P, cap)
    assert np.array_equal(chain.ens_prob, layer.ens_prob)
    assert np.array_equal(chain.ens_mean_logit, layer.ens_mean_logit)
    bed = [int(rng.integers(0, P))]
    ml, prob, _ = cpu_path.cpu_tick(zoo, sel, streams, W + hop, beds=bed)
    assert np.abs(chain.member_logits[bed] - ml).max() <= 2e-2
    assert np.abs(chain.ens_prob[bed] - prob).max() <= 1e-3
