"""e2e (host buffers through tk_gemm_ex_raw) vs the number of pipelined column slabs (tuning)."""
import os, sys, time, subprocess
sys.path.insert(0, ".")
for sl in ("8", "16", "4", "32"):
    out = subprocess.run([sys.executable, "-c", f"""
import os, sys, time, json
os.environ['TK_EX_SLABS'] = '{sl}'
sys.path.insert(0, '.')
import torch, argparse
import bench
import paper_2009_12263_b200 as tk
from paper_2009_12263_b200 import api
a = argparse.Namespace(dtype='fp16', steps=5, e2e_steps=5)
r = bench.run_e2e(a, tk, api, torch, torch.device('cuda', 0), 8192, 8192, 8192, 1)
print('slabs {sl}', round(r['value'], 1), 'TF', round(r['ms_per_step'], 2), 'ms')
"""], capture_output=True, text=True)
    print(out.stdout.strip(), out.stderr.strip()[-300:])
