#!/usr/bin/env python3
"""Install the unmodified reference package (`streamsgd`) into the git-ignored baseline/_ref/.

baseline/_ref/ is not gpurun-ignored, so it travels with every gpurun snapshot: the live
drop-in test (tests/test_gpu_dropin.py), the per-rank runner's byte-identity test and
`bench.py --impl reference` import the reference from there on the GPU box, where
/root/reference does not exist.  Run this before every GPU call (idempotent).

Install route (recorded in DESIGN.md §5): the documented offline pip install of the package
(`pip install --no-index --no-build-isolation --find-links /opt/wheelhouse --target ...`) from
a /tmp copy of /root/reference/pkg (the build writes into its source tree); dependency
resolution needs numpy from an index, so `--no-deps` (numpy is already in the image).  If pip
fails, the package sources are copied verbatim (it is pure Python).
"""

from __future__ import annotations

import shutil
import subprocess
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
DEST = ROOT / "baseline" / "_ref"
SRC = Path("/root/reference/pkg")


def installed() -> bool:
    return (DEST / "streamsgd" / "comm.py").exists()


def install(force: bool = False, quiet: bool = False) -> str:
    if installed() and not force:
        return "present"
    if not SRC.exists():
        raise SystemExit(f"{SRC} not found (run this in the build container)")
    if DEST.exists():
        shutil.rmtree(DEST)
    DEST.mkdir(parents=True)
    with tempfile.TemporaryDirectory() as tmp:
        pkg = Path(tmp) / "pkg"
        shutil.copytree(SRC, pkg, ignore=shutil.ignore_patterns("frontend", "node_modules", ".hypothesis"))
        cmd = [sys.executable, "-m", "pip", "install", "--no-index", "--no-build-isolation", "--find-links",
               "/opt/wheelhouse", "--no-deps", "--target", str(DEST), str(pkg)]
        r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode == 0 and installed():
        how = "pip --no-deps"
    else:
        shutil.copytree(SRC / "src" / "streamsgd", DEST / "streamsgd")
        how = "copied sources (pip failed: " + (r.stderr.strip().splitlines() or ["?"])[-1] + ")"
    if not quiet:
        print(f"reference installed into {DEST} ({how})")
    return how


if __name__ == "__main__":
    install(force="--force" in sys.argv)
