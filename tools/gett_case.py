"""A few launches of the GETT benchmark cases (for ncu launch lists)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import tools.bench_variants as bv  # noqa: E402

bv.timeit = lambda fn, reps=2, warm=1: [fn() for _ in range(warm + reps)] and 1.0
bv.gett_case("abcd-aebf-dfce", dict(a=128, b=64, c=128, d=64, e=128, f=64))
bv.gett_case("abc-acd-db", dict(a=128, b=8192, c=64, d=8192))
bv.gett_case("abc-bda-dc", dict(a=64, b=128, c=8192, d=8192))
