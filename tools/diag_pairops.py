"""Complex / dual CTA-pair kernel: full vs mainloop-only throughput and in-kernel clock."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import tools.bench_variants as bv  # noqa: E402

for kind in ("complex", "dual"):
    for skip in ("0", "1"):
        os.environ["TK_DBG_SKIP_EPI"] = skip
        bv.pair_op(kind, int(os.environ.get("N", "8192")), True)
        bv.results[-1]["case"] += f" skip_epi={skip}"
        print(bv.results[-1]["case"], flush=True)
