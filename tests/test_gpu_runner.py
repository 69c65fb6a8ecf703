"""GPU: the per-rank loop on the sm_100a float64 kernels writes metrics.csv / summary.json
byte-identical to the reference's own run (cli.py:27-75) -- config 1
(golden) and the non-IID + injection + truncation + rate-jitter variant, at P = 1 in-process
and at P = 2/4 under torchrun through ``python -m paper_2301_08897_b200.run``."""

import json
import os
import subprocess
import sys

import pytest
import torch

from conftest import GOLDEN, ROOT
from test_runner import REF, _ref, reference_outputs, variant_config

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("which", ["config1", "variant"])
def test_gpu_runner_single_gpu_byte_identical(cuda, which):
    assert (REF / "streamsgd" / "engine.py").exists(), "run tools/install_ref.py before the GPU call"
    _ref()
    import streamsgd.config as config

    from paper_2301_08897_b200 import runner

    cfg_dict = json.loads((GOLDEN / "config1.json").read_text()) if which == "config1" else variant_config()
    want_csv, want_summary = reference_outputs(cfg_dict)
    if which == "config1":
        assert want_csv == (GOLDEN / "config1_metrics.csv").read_text()
    cfg = config.parse_config(json.dumps(cfg_dict))
    r = runner.RankRunner(cfg, runner.ReferenceProducer.from_package(), device=cuda)
    res = r.run()
    assert runner.metrics_csv(res, cfg.n_devices) == want_csv
    assert runner.summary_json(res) == want_summary


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("which", ["config1", "variant"])
def test_gpu_runner_multi_gpu_byte_identical(cuda, which, tmp_path):
    _ref()
    n = 4 if torch.cuda.device_count() >= 4 else 2
    cfg_dict = json.loads((GOLDEN / "config1.json").read_text()) if which == "config1" else variant_config()
    (tmp_path / "cfg.json").write_text(json.dumps(cfg_dict))
    want_csv, want_summary = reference_outputs(cfg_dict)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}", "--master-addr",
           "127.0.0.1", "--master-port", "29547", "-m", "paper_2301_08897_b200.run", str(tmp_path / "cfg.json"),
           "--out", str(tmp_path / "out")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=str(ROOT), env=dict(os.environ))
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert (tmp_path / "out" / "metrics.csv").read_text() == want_csv
    assert (tmp_path / "out" / "summary.json").read_text() == want_summary
