"""Stem share of the c2 tick (eager profile, kind 1) on the chain and per-layer paths; HB_STEM_DBG
variants give its floors (timing only).  usage: python tools/stemtick.py [P]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2008_04063_b200.engine import EnsembleEngine  # noqa: E402
from paper_2008_04063_b200.zoo import Selector, holmes_zoo  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 64
zoo = holmes_zoo()
with EnsembleEngine(zoo, Selector.from_indices(60, [10, 13, 30, 50]), P, hop=250) as eng:
    eng.ingest(np.random.default_rng(0).standard_normal((P, 3, 7500)).astype(np.float32))
    rows = []
    for _ in range(7):
        kinds, ms = eng.profile_tick()[:2]
        rows.append([float(ms[kinds == k].sum()) for k in (0, 1, 6, 5, 3)])
    med = np.median(np.array(rows), axis=0) * 1e3
    print(f"P={P} {os.environ.get('HB_CHAIN', 'auto')} DBG={os.environ.get('HB_STEM_DBG', '0')}: window {med[0]:.1f} us, "
          f"stem {med[1]:.1f} us, chain {med[2]:.1f} us, k4b {med[3]:.1f} us, agg {med[4]:.1f} us")
