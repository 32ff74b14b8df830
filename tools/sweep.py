"""Tuning sweep: TFLOPS of the dense 8192^3 fp16 GEMM under env-var knobs (CUDA events)."""
import os, subprocess, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
extra = os.environ.get("SWEEP_ARGS", "").split()
knobs = [dict(kv.split("=") for kv in arg.split(",")) if arg != "default" else {} for arg in sys.argv[1:]]
for env in knobs:
    e = dict(os.environ, **env)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--no-cpu", "--e2e-steps", "1",
                          "--steps", "40", *extra], env=e, capture_output=True, text=True)
    try:
        d = json.loads(out.stdout.strip().splitlines()[-1])
        print(env, extra, f"{d['value']:.1f} TFLOPS ms={d['ms_per_step']:.4f} clocks={d['clocks']}", flush=True)
    except Exception:
        print(env, "FAILED", out.stdout[-500:], out.stderr[-2000:], flush=True)
