"""bench.py --impl reference runs the reference CPU path from oracle/ alone
(the arm loaded the package's .so and timed 20k rays). CPU."""

import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]

PROBE = """
import runpy, sys
sys.argv = ['bench.py', '--impl', 'reference', '--config', 'c1', '--steps', '1', '--warmup', '0']
runpy.run_path('bench.py', run_name='__main__')
bad = sorted(m for m in sys.modules if m.startswith('paper_2306_07191_b200'))
so = [l for l in open('/proc/self/maps') if 'libnif_b200' in l]
print('MODULES', bad, 'SO', len(so))
"""


def test_reference_arm_is_oracle_only():
    r = subprocess.run([sys.executable, "-c", PROBE], cwd=ROOT, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = r.stdout.strip().splitlines()
    line = json.loads(lines[-2])
    assert lines[-1] == "MODULES [] SO 0", lines[-1]
    assert line["impl"] == "reference" and line["value"] > 0
    # the whole C1 frame, with the record counts SURVEY.md §8(a) a9 quotes
    assert line["config"]["rays_per_frame"] == 50411
    assert (line["config"]["outer_records"], line["config"]["inner_records"]) == (4781, 31836)
    assert line["e2e"]["h2d_bytes_per_step"] == 0
