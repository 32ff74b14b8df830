"""Run tools/diag_dense.py-style cases against every build/var_*/libtk_sm100.so (tuning)."""
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
cases = sys.argv[1] if len(sys.argv) > 1 else "default,mainloop"
for lib in sorted(glob.glob(os.path.join(ROOT, "build", "var_*", "libtk_sm100.so"))):
    name = os.path.basename(os.path.dirname(lib))
    env = dict(os.environ, TK_SM100_LIB=lib, CASES=cases)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "diag_dense.py")], env=env,
                         capture_output=True, text=True, timeout=600)
    for line in (out.stdout + out.stderr).splitlines():
        if "TFLOPS" in line or "Error" in line or "error" in line:
            print(f"{name:14s} {line}", flush=True)
