"""BASELINE config 5: synthetic flat-gradient sweep (1M..1B fp32 elements per worker) of the
weighted Top-k aggregation, plus the cr sweep of config 3 (0.1 / 0.01 / 0.001) at ResNet-152
size.  Each point is one `bench.py` run (device-resident leg only: `--no-e2e
--no-cpu-baseline`), so every number keeps bench.py's timing rules; the table collects
value, ms/step, the Top-k roofline fraction and the whole-step HBM fraction.

    python tools/sweep.py [--gpus N] [--out gpurun_out/sweep_n1.json]

With --gpus N > 1 every point is launched under torchrun (127.0.0.1).  Points whose
per-GPU bucket (W/N * D * 4 B) is below the 126 MB L2 are marked l2_resident: they measure
the launch chain, not HBM.
"""

from __future__ import annotations

import argparse
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
DIMS = [1 << 20, 1 << 24, 60_192_808, 143_667_240, 1 << 28, 1 << 30]
CRS = [0.1, 0.01, 0.001]
R_DIM = 60_192_808


def point(gpus, dim, cr, steps, warmup, workload="topk"):
    cmd = [sys.executable, str(ROOT / "bench.py"), "--gpus", str(gpus), "--steps", str(steps), "--warmup",
           str(warmup), "--dim", str(dim), "--cr", str(cr), "--workload", workload, "--no-e2e",
           "--no-cpu-baseline"]
    if gpus > 1:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
               "--master-addr", "127.0.0.1", "--master-port", "29533"] + cmd[1:]
    r = subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT, timeout=900)
    line = next((ln for ln in reversed(r.stdout.splitlines()) if ln.startswith("{")), None)
    if r.returncode != 0 or line is None:
        return {"dim": dim, "cr": cr, "workload": workload, "error": (r.stderr or r.stdout)[-600:]}
    j = json.loads(line)
    roof = j.get("roofline") or {}
    step = j.get("step_roofline") or {}
    return {"dim": dim, "cr": cr, "workload": workload, "value": j["value"], "ms_per_step": j["ms_per_step"],
            "topk_frac": roof.get("frac"), "topk_us": roof.get("avg_launch_us"), "step_frac": step.get("frac"),
            "paths": j["config"].get("paths"), "l2": j["config"].get("l2")}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--dims", type=str, default=",".join(map(str, DIMS)))
    ap.add_argument("--out", type=str, default=str(ROOT / "gpurun_out" / "sweep.json"))
    args = ap.parse_args()
    rows = []
    for d in map(int, args.dims.split(",")):
        rows.append(point(args.gpus, d, 0.01, args.steps, args.warmup))
        print(json.dumps(rows[-1]), flush=True)
    for cr in CRS:
        if cr != 0.01:
            rows.append(point(args.gpus, R_DIM, cr, args.steps, args.warmup))
            print(json.dumps(rows[-1]), flush=True)
    rows.append(point(args.gpus, R_DIM, 0.01, args.steps, args.warmup, workload="dense"))
    print(json.dumps(rows[-1]), flush=True)
    Path(args.out).parent.mkdir(parents=True, exist_ok=True)
    Path(args.out).write_text(json.dumps({"gpus": args.gpus, "rows": rows}, indent=1))


if __name__ == "__main__":
    main()
