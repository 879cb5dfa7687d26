"""Summarise ncu captures into the markdown/CSV kept under profiles/.

    python tools/ncu_summary.py full  gpurun_out/prof.ncu-rep  > profiles/x.md
    python tools/ncu_summary.py launches gpurun_out/launches.csv > profiles/x_launches.md
    python tools/ncu_summary.py traffic gpurun_out/prof.ncu-rep "source" > profiles/traffic.json
"""

from __future__ import annotations

import csv
import io
import subprocess
import sys
from collections import OrderedDict, defaultdict

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram % peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % peak"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe % active"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64 pipe %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("sm__inst_executed.avg.per_cycle_active", "IPC (per SM)"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
]


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units = rows[0], rows[1]
    idx = {m: head.index(m) for m, _ in METRICS if m in head}
    kn = head.index("Kernel Name")
    seen = OrderedDict()
    for r in rows[2:]:
        name = r[kn]
        short = name.split("(")[0].replace("void ", "").replace("nif::<unnamed>::", "")
        seen.setdefault(short, []).append(r)
    out = ["| kernel | " + " | ".join(lbl for m, lbl in METRICS if m in idx) + " |",
           "|---" * (1 + len(idx)) + "|"]
    for short, rs in seen.items():
        r = rs[-1]
        cells = []
        for m, _ in METRICS:
            if m not in idx:
                continue
            cells.append(f"{r[idx[m]]} {units[idx[m]]}".strip())
        out.append(f"| `{short}` | " + " | ".join(cells) + " |")
    print("\n".join(out))


def traffic(path, source="ncu --set full"):
    """DRAM bytes per launch of each kernel (last launch captured), keyed by
    the short kernel name bench.py uses for roofline.traffic."""
    import json
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units = rows[0], rows[1]
    kn = head.index("Kernel Name")
    rd, wr = head.index("dram__bytes_read.sum"), head.index("dram__bytes_write.sum")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    out = {"_source": source}
    for r in rows[2:]:
        short = r[kn].split("(")[0].replace("void ", "").split("::")[-1]
        out[short] = {"dram_bytes_read": int(float(r[rd].replace(",", "")) * scale[units[rd]]),
                      "dram_bytes_write": int(float(r[wr].replace(",", "")) * scale[units[wr]])}
    print(json.dumps(out, indent=1))


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = defaultdict(list)
    unit = rows[hi + 1][ui]
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        short = r[ki].split("(")[0].replace("void ", "").replace("nif::<unnamed>::", "")
        agg[short].append(float(r[vi].replace(",", "")))
    total = sum(sum(v) for v in agg.values())
    print(f"| kernel | launches | mean ({unit}) | total ({unit}) | share |")
    print("|---|---|---|---|---|")
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        print(f"| `{k[:70]}` | {len(v)} | {sum(v) / len(v):.1f} | {sum(v):.1f} | "
              f"{100 * sum(v) / total:.1f}% |")


if __name__ == "__main__":
    {"full": full, "launches": launches, "traffic": traffic}[sys.argv[1]](*sys.argv[2:])
