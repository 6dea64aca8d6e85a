"""bench.py's contract pieces that run on CPU: the reference arm (--impl
reference) maps no library of this package -- only oracle/_ref (or the port) --
prints exactly one JSON line on stdout, and carries the same `config` object as
our arm (same workload and sets per step), so the driver's ratio is valid."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

PROBE = r"""
import sys
sys.argv = ['bench.py', '--impl', 'reference', '--sets', '1024', '--steps', '1', '--warmup', '1',
            '--workload', 'cfg1']
import bench
bench.main()
maps = open('/proc/self/maps').read()
libs = sorted(set(l.split()[-1] for l in maps.splitlines() if l.split()[-1].endswith('.so')
                  and '/repo/' in l.split()[-1] or 'librrgpu' in l))
sys.stderr.write('LIBS ' + repr(libs) + '\n')
"""


def test_reference_arm_maps_only_the_reference_and_prints_one_line():
    p = subprocess.run([sys.executable, "-c", PROBE], cwd=ROOT, capture_output=True, text=True,
                       timeout=300)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [l for l in p.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, p.stdout
    line = json.loads(lines[0])
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["config"]["sets_per_step"] == 1024
    libs = [l for l in p.stderr.splitlines() if l.startswith("LIBS ")][-1]
    assert "librrgpu" not in libs, libs
    assert "oracle" in libs, libs


def test_both_arms_share_the_config_builder():
    sys.path.insert(0, ROOT)
    import bench
    g = bench.graphs_module()
    cfg = g.CONFIGS["cfg4"]
    a = bench.bench_config(cfg, 10, 20, 1 << 20, 1)
    b = bench.bench_config(cfg, 10, 20, 1 << 20, 1)
    assert a == b and a["sets_per_step"] == 1 << 20
