import sys, numpy as np, torch
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
from paper_2008_04063_b200.engine import EnsembleEngine
from paper_2008_04063_b200.zoo import Selector, holmes_zoo
from paper_2008_04063_b200 import arch
zoo = holmes_zoo()
P = int(sys.argv[1]) if len(sys.argv) > 1 else 64
idx = [int(x) for x in sys.argv[2].split(',')] if len(sys.argv) > 2 else [10, 13]
sel = Selector.from_indices(60, idx)
eng = EnsembleEngine(zoo, sel, P, hop=250)
eng.ingest(np.random.default_rng(0).standard_normal((P, 3, 7500)).astype(np.float32))
s = torch.cuda.Stream()
for _ in range(3): eng.profile_tick(s.cuda_stream)
res = [eng.profile_tick(s.cuda_stream) for _ in range(5)]
k = res[0][0]; ms = np.median([r[1] for r in res], axis=0); fl = res[0][2]; by = res[0][3]
specs = []
for i in idx:
    pr = zoo.profiles[i]
    specs += [("ingest",)] if not specs else []
    for L in arch.member_layers(pr.width, pr.depth):
        specs.append((pr.id, L.name, L.cin, L.cout, L.stride, L.lout))
j = 0
names = [s for s in specs]
ci = 1
for n in range(len(k)):
    tag = names[ci] if (k[n] in (1, 2) and ci < len(names)) else (k[n],)
    if k[n] in (1, 2): ci += 1
    print(f"{n:3d} kind={k[n]} {ms[n]*1e3:8.1f} us  {fl[n]/ms[n]/1e9 if ms[n]>0 else 0:7.1f} TF/s  {by[n]/ms[n]/1e6 if ms[n]>0 else 0:7.1f} GB/s  {tag}")
print("total ms", ms.sum())
