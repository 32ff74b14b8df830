"""1024 x 1024 x K dense GEMMs for fixed-cost / per-k-cost separation under ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import tools.bench_variants as bv  # noqa: E402

bv.timeit = lambda fn, reps=3, warm=2: [fn() for _ in range(warm + reps)] and 1.0
n = int(os.environ.get("N", "1024"))
for k in (320, 1024, 4096):
    bv.dense(n, m=n, k=k)
