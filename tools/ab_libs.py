"""A/B the default build against build/var_*/libtk_sm100.so variants, interleaved (tuning only).
CASES: comma list of bench_variants expressions, e.g. "dense(8192),pair_op('complex',8192,True)"."""
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASES = os.environ.get("CASES", "dense(8192);dense(2048);dense(1024);dense(4096);"
                       "pair_op('complex',8192,True);pair_op('dual',8192,True)").split(";")
libs = [("default", None)] + [(os.path.basename(os.path.dirname(p)), p) for p in
                              sorted(glob.glob(os.path.join(ROOT, "build", "var_*", "libtk_sm100.so")))]
code = ("import os,sys; sys.path.insert(0, %r); os.environ.setdefault('GRAPH','1'); "
        "os.environ.setdefault('COOLDOWN','0.5'); import tools.bench_variants as bv; " % ROOT) + \
    "; ".join(f"bv.{c}" for c in CASES)
for rnd in range(int(os.environ.get("ROUNDS", "2"))):
    for name, lib in libs:
        env = dict(os.environ)
        if lib:
            env["TK_SM100_LIB"] = lib
        out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                             timeout=900)
        for line in (out.stdout + out.stderr).splitlines():
            if "TFLOPS" in line or "GB/s" in line or "rror" in line:
                print(f"r{rnd} {name:12s} {line}", flush=True)
