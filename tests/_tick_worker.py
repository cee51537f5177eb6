"""Subprocess worker for parity tests whose planner knobs are read once per
process (HB_PP_NB, HB_PP_SPLIT, HB_PP_STAGES, HB_WIN, ... are `static` in the
library): runs `ticks` sliding ticks of an ensemble on cuda:0 and saves the
last tick's outputs.  Usage: python _tick_worker.py OUT.npz P HOP TICKS SEED IDX[,IDX...]
Test infrastructure only."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2008_04063_b200 import synth  # noqa: E402
from paper_2008_04063_b200.engine import EnsembleEngine  # noqa: E402
from paper_2008_04063_b200.zoo import Selector, holmes_zoo  # noqa: E402


def main():
    out, P, hop, ticks, seed, idx = sys.argv[1], *map(int, sys.argv[2:6]), sys.argv[6]
    W = 7500
    sel = Selector.from_indices(60, [int(i) for i in idx.split(",")])
    streams = synth.ecg_block(seed, P, 3, 0, W + ticks * hop)
    with EnsembleEngine(holmes_zoo(), sel, P, hop=hop) as eng:
        eng.ingest(streams[:, :, :W - hop])
        for k in range(ticks):
            end = W + k * hop
            res = eng.tick(streams[:, :, end - hop:end])
    np.savez(out, member_logits=res.member_logits, ens_prob=res.ens_prob, ens_mean_logit=res.ens_mean_logit,
             end=end)


if __name__ == "__main__":
    main()
