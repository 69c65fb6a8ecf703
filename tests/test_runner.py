"""The per-rank loop (runner.RankRunner) writes the reference's metrics wire format
(cli.py:27-75: metrics.csv + summary.json), byte-identical to the reference's own run of the
same config -- at P = 1 and with the devices sharded over 2 gloo ranks (CPU, the kernels
replaced by their oracle-backed stand-ins; the GPU twin is tests/test_gpu_runner.py).

Configs: the golden config 1 (4 devices, S-weighted, cr 0.1 / delta 0.5, mixed decisions) and a
non-IID + injection + truncation + rate-jitter variant (config 4's data side) whose reference
output is produced live from the installed reference (baseline/_ref)."""

import json
import os
import socket
import sys

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import GOLDEN, ROOT
from host_ops import NumpySamplerOps, OracleOps

REF = ROOT / "baseline" / "_ref"


def _ref():
    if not (REF / "streamsgd" / "engine.py").exists():
        pytest.skip("reference not installed in baseline/_ref (tools/install_ref.py)")
    if str(REF) not in sys.path:
        sys.path.insert(0, str(REF))
    import streamsgd.cli as cli
    import streamsgd.config as config
    import streamsgd.engine as engine

    return cli, config, engine


def variant_config():
    cfg = json.loads((GOLDEN / "config1.json").read_text())
    cfg["partition"] = {"mode": "noniid", "labels_per_device": 5}
    cfg["injection"] = {"enabled": True, "alpha": 0.5, "beta": 0.5}
    cfg["retention"] = "truncation"
    cfg["rate_jitter"] = True
    cfg["max_epochs"] = 4
    cfg["optimizer"] = {"base_lr": 0.2, "momentum": 0.9, "weight_decay": 1e-4, "schedule": [[2, 0.5]]}
    cfg["compression"] = {"enabled": True, "cr": 0.05, "delta": 0.6}
    return cfg


def reference_outputs(cfg_dict):
    cli, config, engine = _ref()
    import dataclasses
    import io
    import csv

    cfg = config.parse_config(json.dumps(cfg_dict))
    result = engine.run_experiment(cfg)
    buf = io.StringIO()
    w = csv.writer(buf, lineterminator="\n")
    w.writerow(cli.metrics_columns(cfg.n_devices))
    for row in result.metrics:
        w.writerow(cli.metrics_row(row))
    return buf.getvalue(), json.dumps(dataclasses.asdict(result.summary), indent=2) + "\n"


def run_rank(rank, world, port, cfg_dict, result):
    sys.path.insert(0, str(REF))
    import streamsgd.config as config

    from paper_2301_08897_b200 import runner

    group = None
    if world > 1:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        group = dist.group.WORLD
    cfg = config.parse_config(json.dumps(cfg_dict))
    c = cfg.compression
    r = runner.RankRunner(cfg, runner.ReferenceProducer.from_package(), group=group, device=torch.device("cpu"),
                          ops=OracleOps(c.cr, c.delta), sampler_ops=NumpySamplerOps())
    res = r.run()
    result[rank] = (runner.metrics_csv(res, cfg.n_devices), runner.summary_json(res), r.param_checksum())
    if group is not None:
        dist.barrier()
        dist.destroy_process_group()


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_runner_config1_single_rank_matches_golden():
    _ref()
    cfg = json.loads((GOLDEN / "config1.json").read_text())
    res = {}
    run_rank(0, 1, 0, cfg, res)
    csv_text, summary, _ = res[0]
    assert csv_text == (GOLDEN / "config1_metrics.csv").read_text()
    assert summary == reference_outputs(cfg)[1]


@pytest.mark.parametrize("which", ["config1", "variant"])
def test_runner_two_ranks_byte_identical(which):
    _ref()
    cfg = json.loads((GOLDEN / "config1.json").read_text()) if which == "config1" else variant_config()
    want_csv, want_summary = reference_outputs(cfg)
    ctx = mp.get_context("spawn")
    with ctx.Manager() as mgr:
        res = mgr.dict()
        port = free_port()
        procs = [ctx.Process(target=run_rank, args=(r, 2, port, cfg, res)) for r in range(2)]
        for p in procs:
            p.start()
        for p in procs:
            p.join(timeout=300)
            assert p.exitcode == 0
        res = dict(res)
    for rank in range(2):
        csv_text, summary, checksum = res[rank]
        assert csv_text == want_csv, rank
        assert summary == want_summary, rank
    assert res[0][2] == res[1][2]  # replicas identical (engine.py:284-286)
