"""The compute-sanitizer substitute for this GPU pool (where compute-sanitizer is closed): build
the library with -DSG_CHECKS (device-side bounds checks on every computed address of the hot
path: candidate slots, boundary lists, output slots, merge offsets, staged merge entries,
sample slots, sampler pool rows; a failed check prints its site and traps) into
gpurun_out/diag/, then run the given command with SG_LIB_PATH pointing at it.

    python tools/checked_run.py python -m pytest tests -m gpu -x -q
    python tools/checked_run.py python tools/race_stress.py --reps 3

Exit status is the command's; a trapped check fails the command loudly.
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2301_08897_b200 import build  # noqa: E402


def main():
    out = ROOT / "gpurun_out" / "diag" / "libscadles_b200_checked.so"
    out.parent.mkdir(parents=True, exist_ok=True)
    build.build_variant(out, ["-DSG_CHECKS"])
    env = dict(os.environ, SG_LIB_PATH=str(out))
    sys.exit(subprocess.run(sys.argv[1:], env=env, cwd=ROOT).returncode)


if __name__ == "__main__":
    main()
