"""Iteration counts of schwarz2 PCG when the local-solve operands are rounded
to k mantissa bits (TSV_AS_ROUND_BITS), to size a low-precision local solve."""
import os, subprocess, sys, json
cfgs = sys.argv[1] if len(sys.argv) > 1 else "2 3"
for bits in [0, 23, 10, 7]:
    env = dict(os.environ, TSV_AS_ROUND_BITS=str(bits))
    out = subprocess.run([sys.executable, os.path.join(os.path.dirname(__file__), "schwarz_perf.py")] + cfgs.split() + ["--jacobi"] * 0,
                         env=env, capture_output=True, text=True).stdout
    for line in out.splitlines():
        if line.startswith("cfg"):
            print("bits", bits, line, flush=True)
