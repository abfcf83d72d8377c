"""bench.py --impl reference: runs the reference's own code (oracle/_ref) on a
tiny config-4 sample, prints the contract's JSON line, and never loads the
product library (libme_b200.so) — the reference arm must be clean."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_is_clean():
    import oracle

    if not oracle.available("reference"):
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    code = (
        "import sys, json, io, contextlib\n"
        f"sys.path.insert(0, {ROOT!r})\n"
        "sys.argv = ['bench.py', '--impl', 'reference', '--steps', '1', '--warmup', '0', '--n-seq', '2', '--frames', '4']\n"
        "import bench\n"
        "rc = bench.main()\n"
        "maps = open('/proc/self/maps').read()\n"
        "print('LOADED_B200', 'libme_b200' in maps)\n"
        "sys.exit(rc)\n"
    )
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert lines, r.stdout
    line = json.loads(lines[-1])
    assert line["impl"] == "reference" and line["value"] > 0 and line["unit"] == "MB/s"
    assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0
    assert "LOADED_B200 False" in r.stdout
