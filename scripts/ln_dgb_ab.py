"""LayerNorm backward timing at configs[2]'s shape (graph-replayed) for the dgain/dbias split size."""
import os, subprocess, sys
for rows_per in (64, 128, 256, 512):
    out = subprocess.run([sys.executable, os.path.join(os.path.dirname(__file__), "ln_time.py")], capture_output=True,
                         text=True, env={**os.environ, "SWARM_LN_DGB_ROWS": str(rows_per)})
    print(f"SWARM_LN_DGB_ROWS={rows_per}:", " | ".join(out.stdout.strip().splitlines()), out.stderr[-300:], flush=True)
