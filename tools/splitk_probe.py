"""Split-K on/off timing on partial-last-wave shapes (graph-replayed device time)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["GRAPH"] = "1"
import tools.bench_variants as bv  # noqa: E402

for (m, n, k) in [(4096, 4096, 4096), (4096, 4096, 16384), (2560, 2560, 8192), (1536, 4096, 16384),
                  (6144, 6144, 8192)]:
    for sk in ("0", "1"):
        os.environ["TK_SPLITK"] = sk
        bv.dense(n, m=m, k=k, name=f"{m}x{n}x{k} splitk={sk}")
