"""Config-3 simulate time per register budget (ASC_SIM_MINB forces 4..8 resident CTAs per SM)."""
import os, sys, subprocess
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for m in sys.argv[1:] or ["4", "5", "6", "7", "8"]:
    env = dict(os.environ, ASC_SIM_MINB=m)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "time_sim.py")], env=env,
                       capture_output=True, text=True)
    print(f"minb {m}:", r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-300:], flush=True)
