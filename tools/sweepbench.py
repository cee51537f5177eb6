"""K6 sweep timing: n=10 and n=16 exhaustive over N=20000 (device time via wall around a synchronous call)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2008_04063_b200 import cohort, composer
from paper_2008_04063_b200.zoo import generate_zoo
for n, grid in ((10, ([8, 16, 32, 64, 128], [2, 4])), (16, ([8, 16, 32, 64], [2, 4, 8, 16]))):
    coh = cohort.synthesize_cohort(generate_zoo(1, grid[0], grid[1], seed=3), 10000, 10000, 0.5, 0)
    coh.device().auc_range(1, 64)
    t0 = time.perf_counter(); a = composer.sweep_aucs(coh); dt = time.perf_counter() - t0
    print(f"n={n}: {len(a)} candidates in {dt*1e3:.2f} ms -> {len(a)/dt:,.0f}/s; sorted keys/s {len(a)*10000/dt:.3e}")
