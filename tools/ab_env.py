"""A/B of environment switches on the bench workload (tool): runs bench.py
once per setting (no modes / e2e / cpu baseline) and prints the sweep split.
Usage: python tools/ab_env.py 'PRGPU_COLD_ALLOC=0' 'PRGPU_COLD_ALLOC=1' ..."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for spec in sys.argv[1:]:
    env = dict(os.environ)
    for kv in spec.split(","):
        if kv:
            k, v = kv.split("=")
            env[k] = v
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "5", "--warmup", "3",
                          "--no-modes", "--no-e2e", "--no-cpu-baseline"], env=env, capture_output=True, text=True)
    try:
        d = json.loads(out.stdout.strip().splitlines()[-1])
    except Exception:
        print(spec, "FAILED", out.stderr[-2000:])
        continue
    r, ps = d["roofline"], d.get("plain_sweep", {})
    print(f"{spec:40s} value {d['value']:.1f} GTEPS  step {d['ms_per_step']:.2f} ms  converge {d['run']['time_to_converge_ms']:.2f} ms "
          f"create {d['run']['create_ms']:.2f}  gather {r['launch_ms']:.4f} finalize {r['sweep']['finalize_ms']:.4f} ms  "
          f"plain gather {ps.get('gather_ms')} finalize {ps.get('finalize_ms')}  t_iter {d.get('t_iter_difference', {}).get('ms')}",
          flush=True)
