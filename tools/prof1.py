import sys, numpy as np, torch
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
from paper_2008_04063_b200.engine import EnsembleEngine
from paper_2008_04063_b200.zoo import Selector, holmes_zoo
zoo = holmes_zoo()
idx = [int(x) for x in sys.argv[1].split(',')]
eng = EnsembleEngine(zoo, Selector.from_indices(60, idx), 64, hop=250)
eng.ingest(np.random.default_rng(0).standard_normal((64, 3, 7500)).astype(np.float32))
s = torch.cuda.Stream()
eng.profile_tick(s.cuda_stream)
torch.cuda.synchronize()
