"""The INTEGRATION.md C++ binding, compiled and run: oracle/_ref/dropin_driver
links the reference's own sources (built here from /root/reference by
oracle/build_dropin.sh) and libminimod_b200.so, runs one SimConfig through the
reference's run() (driver.cpp:83-144) and through the drop-in engine
(driver.cpp:116-121 replaced as INTEGRATION.md shows) and mm_run(), and
compares the receiver trace matrices bit for bit."""
import json
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

BIN = ROOT / "oracle" / "_ref" / "dropin_driver"


@pytest.mark.parametrize("n,nsteps,fs", [(64, 200, 0), (80, 150, 1), (240, 100, 0)])
def test_cpp_dropin_equals_reference_run(n, nsteps, fs):
    if not BIN.exists():
        pytest.skip("oracle/_ref/dropin_driver not built (needs /root/reference)")
    r = subprocess.run([str(BIN), str(n), str(nsteps), str(fs)], capture_output=True, text=True,
                       timeout=600)
    line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else ""
    assert r.returncode == 0, (r.returncode, line, r.stderr[-2000:])
    out = json.loads(line)
    assert out["ok"] and out["dropin"]["bitwise"] and out["mm_run"]["bitwise"], out
    assert out["dropin"]["max_abs"] == 0.0 and out["mm_run"]["rel_l2"] == 0.0
