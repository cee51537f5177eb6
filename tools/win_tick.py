"""Run a few eager ticks at P beds (for ncu captures of the window kernel)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2008_04063_b200.engine import EnsembleEngine  # noqa: E402
from paper_2008_04063_b200.zoo import Selector, holmes_zoo  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
HOP = int(sys.argv[2]) if len(sys.argv) > 2 else 250
N = int(sys.argv[3]) if len(sys.argv) > 3 else 4
eng = EnsembleEngine(holmes_zoo(), Selector.from_indices(60, [10, 13, 30, 50]), P, hop=HOP)
eng.ingest(np.random.default_rng(0).standard_normal((P, 3, 7500)).astype(np.float32))
blk = np.random.default_rng(1).standard_normal((P, 3, HOP)).astype(np.float32)
for _ in range(N):
    eng.tick(blk)
print("ok")
