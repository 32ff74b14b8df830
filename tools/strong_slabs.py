"""Per-GPU column slabs of the 16384^3 strong-scaling problem, one GPU."""
import os, sys
sys.path.insert(0, ".")
os.environ["GRAPH"] = "1"
import tools.bench_variants as bv
for n in (16384, 8192, 4096, 2048):
    bv.dense(n, m=16384, k=16384, name=f"strong-scaling slab 16384x{n}x16384 (G={16384 // n})")
