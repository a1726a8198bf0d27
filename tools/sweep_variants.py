"""Times every build_variants/*.so (or the given ones) on config-1 sweeps,
each in its own process.  python tools/sweep_variants.py [--nx 2048] [libs...]"""
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
args = [a for a in sys.argv[1:] if a.endswith(".so")]
extra = [a for a in sys.argv[1:] if not a.endswith(".so")]
libs = args or sorted(glob.glob(os.path.join(ROOT, "build_variants", "*.so")))
for lib in libs:
    env = dict(os.environ, HYDRO_B200_LIB=lib)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "profile_step.py"),
                          "--steps", "10", *extra], env=env, capture_output=True, text=True)
    line = (out.stdout.strip().splitlines() or ["?"])[-1]
    print(f"{os.path.basename(lib):24s} {line} {out.stderr.strip()[-200:] if out.returncode else ''}",
          flush=True)
