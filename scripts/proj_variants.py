"""Time the projection-tile variants (RBRP_PROJ_VARIANT) on c2 in separate processes."""
import os, subprocess, sys
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for v in range(4):
    env = dict(os.environ, RBRP_PROJ_VARIANT=str(v))
    out = subprocess.run([sys.executable, os.path.join(root, "scripts", "quick.py"), "c2"], env=env,
                         capture_output=True, text=True)
    print(f"variant {v}:", out.stdout.strip().splitlines()[0] if out.stdout else out.stderr[-500:], flush=True)
