"""GPU parity of K2t (the X-stationary 2:4 kernel, spmm_tcx.cu) against the C
oracle.  K2t is selected with SI_K2_VARIANT=xsparse, which the library reads
once per process, so the cases run in a subprocess (tests/k2t_quick.py)."""

import os
import subprocess
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.gpu
def test_k2t_bit_exact_against_oracle():
    env = dict(os.environ, SI_K2_VARIANT="xsparse")
    r = subprocess.run([sys.executable, os.path.join(HERE, "k2t_quick.py"), "parity"], env=env,
                       capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out
    ran = [l for l in out.splitlines() if "mismatches" in l]
    assert len(ran) >= 7, out
    assert all(l.split("mismatches")[1].split()[0] == "0" for l in ran), out
