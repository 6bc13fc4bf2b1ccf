"""bench.py contract checks that run on CPU: the reference arm runs the
unmodified reference without mapping this repository's product library,
and both arms name the same config keys."""

from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

from oracle import ref as R

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(not R.available(), reason="oracle/_ref not built")
def test_reference_arm_does_not_load_the_product_library():
    code = (
        "import sys, json; sys.argv = ['bench.py', '--impl', 'reference', '--rows', '20000', '--steps', '1', "
        "'--warmup', '1', '--ref-queries', '4']\n"
        "import bench; bench.main()\n"
        "maps = open('/proc/self/maps').read()\n"
        "print(json.dumps({'product_mapped': 'libhyre_b200' in maps, 'ref_mapped': 'libhyre_ref' in maps}))\n")
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    line, maps = lines[0], lines[-1]
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "reference"
    assert maps == {"product_mapped": False, "ref_mapped": True}
    import argparse
    import dataclasses

    import bench
    from paper_2402_13435_b200.workloads import WORKLOADS
    cfg = bench.workload_config(dataclasses.replace(WORKLOADS["c3"], n=20000), argparse.Namespace(batch=64, k=100))
    assert line["config"] == cfg  # our arm prints workload_config(w, args) too
