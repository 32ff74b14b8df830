"""Quick first-light diagnostics of the tcgen05 lane (prints errors instead of asserting)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2009_12263_b200 as tk
from oracle import oracle as O

def dev(x):
    return torch.from_numpy(np.ascontiguousarray(np.asarray(x).ravel(order="F"))).cuda()

for (m, n, k, ta, tb) in [(128, 256, 64, 0, 0), (128, 256, 128, 0, 0), (256, 512, 256, 0, 0),
                          (256, 512, 256, 1, 0), (256, 512, 256, 0, 1), (256, 512, 256, 1, 1)]:
    rng = np.random.default_rng(0)
    a = rng.integers(-4, 5, (m, k)).astype(np.float16)
    b = rng.integers(-4, 5, (k, n)).astype(np.float16)
    c = np.zeros((m, n), np.float32)
    cfg = tk.build_dense_config(m, n, k, np.float16, trans_a=bool(ta), trans_b=bool(tb))
    d = torch.zeros(m * n, dtype=torch.float32, device="cuda")
    t0 = time.time()
    tk.matmul(cfg, dev(a.T if ta else a), dev(b.T if tb else b), dev(c), d)
    got = d.cpu().numpy().reshape((m, n), order="F")
    want = a.astype(np.float32) @ b.astype(np.float32)
    bad = np.argwhere(got != want)
    print(f"{m}x{n}x{k} t{ta}{tb}: lane={tk.last_run()['lane']} mismatches={len(bad)} "
          f"maxdiff={np.max(np.abs(got-want)):.3g} t={time.time()-t0:.2f}s", flush=True)
    if len(bad):
        print("  first bad", bad[:5].tolist(), got[tuple(bad[0])], want[tuple(bad[0])])
