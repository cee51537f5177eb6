"""One K6 launch over the c4 cohort (n=10, N=20000) for ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2008_04063_b200 import cohort, composer
from paper_2008_04063_b200.zoo import generate_zoo
z = generate_zoo(1, [8, 16, 32, 64, 128], [2, 4], seed=3)
print(composer.sweep_aucs(cohort.synthesize_cohort(z, 10000, 10000, 0.5, 0))[:3])
