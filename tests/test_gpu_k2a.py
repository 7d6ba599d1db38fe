"""GPU parity of K2a (W rows resident in tensor memory, spmm_tca.cu) against
the C oracle, both activation layouts.  Selected with SI_K2_VARIANT=tmemw,
which the library reads once per process, so the cases run in a subprocess
(tests/k2a_quick.py)."""

import os
import subprocess
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.gpu
def test_k2a_bit_exact_against_oracle():
    env = dict(os.environ, SI_K2_VARIANT="tmemw")
    r = subprocess.run([sys.executable, os.path.join(HERE, "k2a_quick.py"), "parity"], env=env,
                       capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out
    ran = [l for l in out.splitlines() if "mismatches" in l]
    assert len(ran) >= 12, out
    assert all(l.split("mismatches")[1].split()[0] == "0" for l in ran), out
