"""A few launches of dense fp16 GEMMs at the given sizes (for ncu launch-time lists)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import tools.bench_variants as bv  # noqa: E402

bv.timeit = lambda fn, reps=3, warm=2: [fn() for _ in range(warm + reps)] and 1.0
for n in [int(x) for x in (sys.argv[1:] or ["1024", "2048", "4096"])]:
    bv.dense(n)
