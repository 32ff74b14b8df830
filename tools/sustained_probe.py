"""Sustained (power-capped) throughput: graph-replayed back-to-back GEMMs for ~0.5 s, per
kernel variant (env knobs) -- the regime where energy per flop sets the clock."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["GRAPH"] = "1"
import tools.bench_variants as bv  # noqa: E402

n = int(os.environ.get("N", "16384"))
reps = int(os.environ.get("REPS", "6"))
orig = bv.timeit
bv.timeit = lambda fn, reps=reps, warm=2: orig(fn, reps=reps, warm=warm)
for env in [e for e in os.environ.get("VARIANTS", ",TK_PAIR_NSUB=2").split(",")]:
    for kv in ("TK_PAIR_NSUB", "TK_SERPENTINE", "TK_GROUP_M"):
        os.environ.pop(kv, None)
    for kv in [x for x in env.split("+") if x]:
        k, v = kv.split("=")
        os.environ[k] = v
    bv.dense(n, name=f"sustained {n}^3 x{10 * reps} {env or 'default'}")
if os.environ.get("CUBLAS", "1") == "1":
    bv.cublas_ref(n)
