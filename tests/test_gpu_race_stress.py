"""Race stress (SURVEY.md §5 race detection; compute-sanitizer is closed on this GPU pool):
tools/race_stress.py runs the cluster exchange, the split schedule and the 16-warp n > 32
build under seeded timing perturbation with device-side protocol asserts (libsfb_checks.so)
and requires bitwise-equal results. Marked `gpu`."""

import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_protocols_are_race_free_under_perturbation():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not os.path.exists(os.path.join(ROOT, "paper_2510_09204_b200", "libsfb_checks.so")):
        pytest.skip("libsfb_checks.so not built (__graft_entry__.build builds it)")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "race_stress.py"), "2"],
                       capture_output=True, text=True, timeout=1800)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-2000:]
