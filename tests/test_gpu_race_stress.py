"""GPU: run-to-run determinism stress of every kernel family with concurrent hand-offs
(tools/race_stress.py --quick): identical bytes over repetitions, oracle-exact indices, both
all-sparse merge kernels bit-identical.  compute-sanitizer is closed on this GPU pool; this is
the round's race check (profiles/r02_race_stress.md holds the full 50-repetition run)."""

import json
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_race_stress_quick(cuda):
    r = subprocess.run([sys.executable, str(ROOT / "tools" / "race_stress.py"), "--quick"], capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    rep = json.loads(r.stdout.strip().splitlines()[-1])
    assert rep["ok"], rep
