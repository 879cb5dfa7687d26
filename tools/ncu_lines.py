"""Per-CUDA-source-line instruction / stall totals from an ncu report.

    python tools/ncu_lines.py report.ncu-rep [top] [kernel-base-name[:skip]]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
want = sys.argv[3] if len(sys.argv) > 3 else ""
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
if want:  # kernel base name[:n-th match] (import mode honours -k / --launch-skip)
    name, _, skip = want.partition(":")
    cmd[3:3] = ["-k", name] + (["--launch-skip", skip] if skip else [])
out = subprocess.run(cmd, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
agg = []
fname = ""
hdr = None
func_ok = True
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) == 2 and r[0] == "Function Name":
        func_ok = True
        continue
    if not func_ok:
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    if r[0] != "":  # a source line row (aggregated over its SASS)
        ie = hdr.index("Instructions Executed")
        st = hdr.index("Warp Stall Sampling (All Samples)")
        try:
            agg.append((int(r[ie]), int(r[st]), fname, r[0], r[1]))
        except ValueError:
            pass
tot = sum(a[0] for a in agg)
stot = sum(a[1] for a in agg)
print(f"total warp instructions {tot}, stall samples {stot}")
for ie, st, f, ln, src in sorted(agg, key=lambda a: -a[0])[:top]:
    print(f"{f:>12}:{ln:<5} {ie:10d} {100 * ie / tot:5.1f}%  stall {100 * st / max(stot, 1):5.1f}%  {src.strip()[:80]}")
print("-- by stall")
for ie, st, f, ln, src in sorted(agg, key=lambda a: -a[1])[:15]:
    print(f"{f:>12}:{ln:<5} {ie:10d} {100 * ie / tot:5.1f}%  stall {100 * st / max(stot, 1):5.1f}%  {src.strip()[:80]}")
