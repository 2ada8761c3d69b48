"""Drop-in proof: the reference's own acceptance driver (proj/tests/acceptance.cpp), compiled
unchanged against include/spde2d_b200.hpp and linked with the B200 library (tests/cpp/Makefile,
built by __graft_entry__.build() where /root/reference exists), passes the same criteria as
the reference does on CPU: 1-9 PASS; 10 (a CPU timing comparison) fails for the reference too."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "build", "dropin", "acceptance_b200")

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not os.path.exists(BIN), reason="drop-in acceptance binary not built")
def test_reference_acceptance_driver_on_b200():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=900)
    lines = [l for l in r.stdout.splitlines() if l.startswith("[")]
    status = {int(l.split("criterion")[1].split(":")[0]): l.startswith("[PASS]") for l in lines}
    assert sorted(status) == list(range(1, 11)), r.stdout[-2000:]
    for c in range(1, 10):
        assert status[c], [l for l in lines if f"criterion {c:2d}" in l]
