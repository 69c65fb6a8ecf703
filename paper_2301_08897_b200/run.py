"""``python -m paper_2301_08897_b200.run CONFIG.json --out DIR`` -- the reference's ``run``
subcommand (cli.py:78-105) on the B200 path: one process per GPU (launch with torchrun for
P > 1), devices sharded over the ranks, metrics.csv + summary.json written by rank 0 in the
reference's exact format.

The reference package supplies what is out of scope here: its strict config parser
(config.parse_config) and the gradient producer (datagen.generate_dataset, the MLP).  It is
imported from ``--ref`` (default: the git-ignored baseline/_ref that tools/install_ref.py
fills) or from the Python path.  Exit codes follow cli.py:23-25 (0 ok, 1 config error,
2 divergence).
"""

from __future__ import annotations

import argparse
import os
import sys
from pathlib import Path

import torch
import torch.distributed as dist

EXIT_OK, EXIT_CONFIG, EXIT_DIVERGED = 0, 1, 2


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="paper_2301_08897_b200.run")
    ap.add_argument("config")
    ap.add_argument("--out", required=True)
    ap.add_argument("--seed", type=int, default=None)
    ap.add_argument("--ref", default=str(Path(__file__).resolve().parent.parent / "baseline" / "_ref"))
    ap.add_argument("--dtype", choices=["f64", "f32"], default="f64",
                    help="f64: bit-identical to the reference; f32: the throughput kernels")
    args = ap.parse_args(argv)
    if args.ref and Path(args.ref).exists() and args.ref not in sys.path:
        sys.path.insert(0, args.ref)
    import streamsgd.config as config

    from . import build, runner

    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    group = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        group = dist.group.WORLD
    build.build()
    try:
        cfg = config.load_config(args.config)
        if args.seed is not None:
            cfg.seed = args.seed
    except (config.ConfigError, OSError) as exc:
        print(f"config error: {exc}", file=sys.stderr)
        return EXIT_CONFIG
    dtype = torch.float64 if args.dtype == "f64" else torch.float32
    try:
        r = runner.RankRunner(cfg, runner.ReferenceProducer.from_package(), group=group, device=dev, dtype=dtype)
        res = r.run()
    except runner.DivergenceError as exc:
        print(f"run diverged: {exc}", file=sys.stderr)
        return EXIT_DIVERGED
    if group is None or dist.get_rank() == 0:
        runner.write_outputs(args.out, res, cfg.n_devices)
        s = res.summary
        acc = "n/a" if s.final_accuracy is None else f"{s.final_accuracy:.4f}"
        print(f"{args.out}: {s.iterations} iterations, {s.epochs_completed} epochs, "
              f"sim time {s.sim_time_s:.2f}s, accuracy {acc}")
    if group is not None:
        dist.destroy_process_group()
    return EXIT_OK


if __name__ == "__main__":
    sys.exit(main())
