"""A/B one environment switch on bench.py lines.

usage: python tools/bench_ab.py VAR=VALUE -- <bench.py args...>
Runs bench.py with and without VAR, prints ms/step, roofline frac and e2e ms.
"""
import json
import os
import subprocess
import sys

sep = sys.argv.index("--")
env_kv = sys.argv[1]
args = sys.argv[sep + 1:]
name, val = env_kv.split("=", 1)
for label, set_it in (("base", False), (env_kv, True)):
    env = dict(os.environ)
    env.pop(name, None)
    if set_it:
        env[name] = val
    out = subprocess.run([sys.executable, "bench.py"] + args, env=env, capture_output=True, text=True).stdout
    d = json.loads(out.strip().splitlines()[-1])
    e2e = (d.get("e2e") or {}).get("ms_per_step")
    print(f"{label:>24}: step {d['ms_per_step']:.3f} ms  frac {(d.get('roofline') or {}).get('frac', 0):.3f}  "
          f"e2e {e2e if e2e is None else round(e2e, 3)} ms")
