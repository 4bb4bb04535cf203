"""Max co-resident clusters of the AG+GEMM kernel per cluster size (prints
what the split-K chooser sees)."""
import os, sys, subprocess
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for M in (128, 256, 512):
    env = dict(os.environ, TFB_KSPLIT_VERBOSE="1")
    subprocess.run([sys.executable, os.path.join(ROOT, "tools", "probe_gemm.py"), str(M), "8192", "8192"], env=env)
