"""Small single-wave shapes: tile width x split-K sweep (graph-replayed device time)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["GRAPH"] = "1"
import tools.bench_variants as bv  # noqa: E402

for n in [int(x) for x in os.environ.get("NS", "1024,2048").split(",")]:
    for bni in os.environ.get("BNIS", "64,128,256").split(","):
        for minkb in os.environ.get("MINKBS", "64,4,2").split(","):
            os.environ["TK_PAIR_BNI"] = bni
            os.environ["TK_SPLITK_MINKB"] = minkb
            bv.dense(n, name=f"{n}^3 bni={bni} splitk_minkb={minkb}")
