"""In-process A/B of tick configurations: one engine per env setting (the
settings must be read per build, e.g. HB_CHAIN, HB_CHAIN_OPTS, HB_CHAIN_SMS),
graph ticks timed back to back with CUDA events, configurations interleaved so
they share the box's power/thermal state.  Unflushed L2 (relative numbers).
usage: python tools/abtick.py "HB_CHAIN=1" "HB_CHAIN=0" ..."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2008_04063_b200.engine import EnsembleEngine  # noqa: E402
from paper_2008_04063_b200.zoo import Selector, holmes_zoo  # noqa: E402

P = int(os.environ.get("AB_P", "64"))
SEL = os.environ.get("AB_SEL", "c2")  # "c2" (the benchmark's 4 members) or "all" (the 60-member zoo, c3)
zoo = holmes_zoo()
engs = []
base = dict(os.environ)
for cfg in sys.argv[1:]:
    env = dict(base)
    for kv in cfg.split():
        k, v = kv.split("=")
        env[k] = v
    os.environ.clear()
    os.environ.update(env)
    sel = Selector.ones(60) if SEL == "all" else Selector.from_indices(60, [10, 13, 30, 50])
    e = EnsembleEngine(zoo, sel, P, hop=250)
    e.ingest(np.random.default_rng(0).standard_normal((P, 3, 7500)).astype(np.float32))
    e.prepare()
    engs.append((cfg, e))
os.environ.clear()
os.environ.update(base)
res = {c: [] for c, _ in engs}
for r in range(int(os.environ.get("AB_ROUNDS", "8"))):
    for c, e in engs:
        res[c].append(e.time_tick(int(os.environ.get("AB_TICKS", "25"))) * 1e3)
for c, v in res.items():
    print(f"{c:40s} median {np.median(v):.4f} ms  min {min(v):.4f}  max {max(v):.4f}")
