"""Per CUDA source line: warp instructions executed and stall samples of one
kernel (ncu --page source --print-source cuda,sass; the report must have
been captured with --import-source on).

    python tools/ncu_lines2.py <report> <kernel-regex> [n] [skip]
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

path, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 40
skip = sys.argv[4] if len(sys.argv) > 4 else "0"
raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--kernel-name",
                      f"regex:{kern}", "--launch-skip", skip, "--launch-count", "1",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
inst = defaultdict(float)
stall = defaultdict(float)
text = {}
fname = ""
for row in csv.reader(io.StringIO(raw)):
    if not row:
        continue
    if row[0] == "File Path":
        fname = row[1].split("/")[-1]
        continue
    if row[0] in ("Function Name", "Line No"):
        if row[0] == "Line No":
            hdr = row
        continue
    if len(row) < 8 or not row[0].isdigit():
        continue
    key = (fname, int(row[0]))
    text[key] = row[1]
    try:
        stall[key] += float(row[hdr.index("Warp Stall Sampling (All Samples)")])
        inst[key] += float(row[hdr.index("Instructions Executed")])
    except ValueError:
        pass
ti, ts = sum(inst.values()), sum(stall.values())
print(f"warp instructions {ti:.0f}, stall samples {ts:.0f}")
for k in sorted(inst, key=lambda k: -inst[k])[:n]:
    print(f"{inst[k] / ti * 100:5.1f}% inst {stall[k] / max(ts, 1) * 100:5.1f}% stall  "
          f"{k[0]}:{k[1]:<5d} {text[k].strip()[:90]}")
