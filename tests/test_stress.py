"""Randomised stress (GPU): scripts/stress_check.py over 120 seeded cases --
sizes 1..3M, adversarial and skewed distributions, single arrays, repeated
calls (graph replay), host buffers, ragged batches and 4 concurrent threads --
every output bytewise equal to torch.sort.  The committed long run against the
self-checking build is profiles/r02_stress_check.log."""
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_randomised_stress_120_cases():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "stress_check.py"), "--cases", "120"],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "0 failures, 0 concurrent failures" in r.stdout
