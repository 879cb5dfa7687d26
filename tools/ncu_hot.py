"""Hottest source lines (CUDA-C, with the SASS instruction count per line)
of one kernel in an ncu report captured with --import-source on.

    python tools/ncu_hot.py gpurun_out/x.ncu-rep <kernel-regex> [n_lines] [sass]
"""
import csv
import io
import os
import subprocess
import sys

path, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
view = sys.argv[4] if len(sys.argv) > 4 else "cuda"
raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--kernel-name",
                      f"regex:{kern}", "--launch-count", "1", "--launch-skip", os.environ.get("SKIP", "0"), "--print-source", view],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hi = next((i for i, r in enumerate(rows) if r and "Warp Stall Sampling (All Samples)" in r), None)
if hi is None:
    sys.exit("no metric columns in the source view (try the sass view)")
h = rows[hi]
ci = h.index("Warp Stall Sampling (All Samples)")
ie = h.index("Instructions Executed") if "Instructions Executed" in h else None
src = 1
body = [r for r in rows[hi + 1:] if len(r) > ci and r[ci].replace(".", "", 1).isdigit()]
tot = sum(float(r[ci]) for r in body)
ti = sum(float(r[ie]) for r in body if ie is not None and r[ie].replace(".", "", 1).isdigit())
print(f"stall samples {tot:.0f}, warp instructions {ti:.0f}")
for r in sorted(body, key=lambda r: -float(r[ci]))[:n]:
    inst = r[ie] if ie is not None else ""
    print(f"{float(r[ci]) / tot * 100:5.1f}%  inst {inst:>10}  {r[0][:6]:>6} {r[src].strip()[:110]}")
