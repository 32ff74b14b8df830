"""Run one named GEMM case a few times (for ncu captures): dense8192, c3_8192, fused8192,
complex8192, dual8192, diag16384, skinny128, tc_large, tc_paper, gett2, splitk, dense1024,
complex8192i (interleaved), simt2048 (exact lane), dense1024k8192."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("COOLDOWN", "0")
import tools.bench_variants as bv  # noqa: E402

case = sys.argv[1]
bv.timeit = lambda fn, reps=3, warm=2: [fn() for _ in range(warm + reps)] and 1.0
{
    "dense8192": lambda: bv.dense(8192),
    "c3_8192": lambda: bv.fused_c3(8192),
    "fused8192": lambda: bv.fused_builder(8192),
    "complex8192": lambda: bv.pair_op("complex", 8192, True),
    "dual8192": lambda: bv.pair_op("dual", 8192, True),
    "diag16384": lambda: bv.diagonal(16384),
    "skinny128": lambda: bv.skinny(8192, 128),
    "tc_large": lambda: bv.contraction(64, 128, 8192, 8192),
    "tc_paper": lambda: bv.contraction(64, 32, 2048, 2048),
    "gett2": lambda: bv.gett_case("abcd-aebf-dfce", dict(a=128, b=64, c=128, d=64, e=128, f=64)),
    "splitk": lambda: bv.dense(4096, m=1536, k=16384),
    "dense1024": lambda: bv.dense(1024),
    "dense1024k8192": lambda: bv.dense(1024, k=8192),
    "complex8192i": lambda: bv.pair_op("complex", 8192, False),
    "simt2048": lambda: bv.simt_f32(2048),
}[case]()
