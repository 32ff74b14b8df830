import os, sys
sys.path.insert(0, os.getcwd())
os.environ.setdefault("X", "1")
import tools.bench_variants as bv
bv.fused_c3(8192)
