"""Where the pipelined end-to-end tick loses time against the device-timed graph (c2, 64 beds)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2008_04063_b200.engine import EnsembleEngine, TickResult  # noqa: E402
from paper_2008_04063_b200.zoo import Selector, holmes_zoo  # noqa: E402

P, hop, K = 64, 250, 300
eng = EnsembleEngine(holmes_zoo(), Selector.from_indices(60, [10, 13, 30, 50]), P, hop=hop)
rng = np.random.default_rng(0)
eng.ingest(rng.standard_normal((P, 3, 7500)).astype(np.float32))
host_in = torch.empty((K + 2, P, 3, hop), dtype=torch.float32, pin_memory=True)
host_in.numpy()[:] = rng.standard_normal((K + 2, P, 3, hop)).astype(np.float32)
hin = host_in.numpy()
M = 4
out = TickResult(eng.member_ids, torch.empty((P, M), pin_memory=True).numpy(), torch.empty(P, pin_memory=True).numpy(),
                 torch.empty(P, pin_memory=True).numpy())
for i in range(10):
    eng.tick(hin[i], out=out)
print("graph only (time_tick, warm L2): %.1f us" % (eng.time_tick(50) * 1e6))
t0 = time.perf_counter()
slot = eng.submit(hin[0])
gio = []
for i in range(K):
    nxt = eng.submit(hin[i + 1]) if i + 1 < K else None
    eng.collect(slot, out=out)
    slot = nxt
dt = (time.perf_counter() - t0) / K
print("pipelined submit/collect: %.1f us per tick" % (dt * 1e6))
eng.tick(hin[0], out=out)
print("graph_io duration (last tick events): %.1f us" % (eng.last_tick_seconds() * 1e6))
t0 = time.perf_counter()
for i in range(K):
    eng.tick(hin[i], out=out)
print("blocking tick: %.1f us per tick" % ((time.perf_counter() - t0) / K * 1e6))
# host cost of the API calls alone
t0 = time.perf_counter()
for i in range(200):
    s = eng.submit(hin[i])
    eng.collect(s, out=out)
print("submit+collect back to back (incl. device): %.1f us" % ((time.perf_counter() - t0) / 200 * 1e6))
print("graph only again, after the loops (same thermal state): %.1f us" % (eng.time_tick(50) * 1e6))
