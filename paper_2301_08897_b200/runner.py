"""Per-rank training loop over the B200 hot path, writing the reference's metrics wire format.

This is ``Simulation`` (reference engine.py:102-380) restated for one process per GPU, so a
multi-GPU run produces the same ``metrics.csv`` / ``summary.json`` (cli.py:27-75) as the
reference's in-process simulation:

* host planning, identical on every rank (same numpy RNG calls and labelled seeds): stream
  rates (streams.py:58-69), the contiguous-range ``StreamBuffer`` s, the barrier wait
  (engine.py:213-221), injection plans and picks (engine.py:229-242), per-epoch rate jitter
  and augmentation tables (engine.py:180-199);
* device sampler (item 5): this rank's devices' batches are resolved and gathered on the GPU
  (``streams.DeviceSampler``; at P > 1 the pool-sharded ``streams.ShardedSampler``, injected
  samples crossing GPUs in one all-gather);
* the gradient *producer* (the reference MLP's ``loss_and_grad``; out of scope)
  fills this rank's rows of the gradient bucket;
* gate, exchange, weighted aggregation and momentum SGD: :class:`exchange.GradientExchange`
  (one launch sequence per step; float64 kernels in "exact" mode, so the aggregate and the
  post-step weights are bit-identical to numpy's at any P);
* accounting from the device: floats/bytes sent and CNC come from the device gate counters
  (``GradientExchange.volume`` / ``gate_counters``, summed over ranks), the per-device
  decisions that size the simulated all-reduce (engine.py:288-290) from the gathered decision
  bytes.

The simulated clock, the cost model and the metrics rows are host scalars, computed in the
reference's operation order so every float prints identically.
"""

from __future__ import annotations

import dataclasses
import json
import math
from dataclasses import dataclass, field

import numpy as np
import torch
import torch.distributed as dist

from . import comm, exchange, nn, streams


class DivergenceError(RuntimeError):
    """Training produced a non-finite loss (engine.py:28-29)."""


@dataclass
class IterationMetrics:
    """One metrics.csv row (engine.py:44-64)."""

    iteration: int
    sim_time_s: float
    epoch: int
    global_batch: int
    lr_used: float
    train_loss: float
    test_accuracy: float | None
    wait_time_s: float
    buffer_occupancy: list[int]
    buffer_bytes: int
    floats_sent_cum: int
    bytes_sent_cum: int
    cnc_cum: float | None
    injection_bytes: int
    injection_bytes_cum: int

    @property
    def buffer_samples_total(self) -> int:
        return sum(self.buffer_occupancy)


@dataclass
class RunSummary:
    """summary.json (engine.py:67-84)."""

    final_accuracy: float | None
    best_accuracy: float | None
    final_train_loss: float
    iterations: int
    epochs_completed: int
    sim_time_s: float
    target_accuracy: float | None
    reached_target: bool
    time_to_target_s: float | None
    floats_sent_total: int
    bytes_sent_total: int
    cnc: float | None
    injection_bytes_total: int
    final_buffer_samples: int
    final_buffer_bytes: int
    seed: int


@dataclass
class RunResult:
    summary: RunSummary
    metrics: list[IterationMetrics] = field(default_factory=list)


# -- the wire format (cli.py:27-75) ---------------------------------------------------------

BASE_COLUMNS = [
    "iteration", "sim_time_s", "epoch", "global_batch", "lr_used", "train_loss", "test_accuracy",
    "wait_time_s", "buffer_samples_total", "buffer_bytes", "floats_sent_cum", "bytes_sent_cum",
    "cnc_cum", "injection_bytes", "injection_bytes_cum",
]


def metrics_columns(n_devices: int) -> list[str]:
    return BASE_COLUMNS + [f"buffer_len_dev{d}" for d in range(n_devices)]


def _cell(value) -> str:
    return "" if value is None else repr(value) if isinstance(value, float) else str(value)


def metrics_row(m: IterationMetrics) -> list[str]:
    values = [
        m.iteration, m.sim_time_s, m.epoch, m.global_batch, m.lr_used, m.train_loss, m.test_accuracy,
        m.wait_time_s, m.buffer_samples_total, m.buffer_bytes, m.floats_sent_cum, m.bytes_sent_cum,
        m.cnc_cum, m.injection_bytes, m.injection_bytes_cum,
    ]
    return [_cell(v) for v in values] + [str(o) for o in m.buffer_occupancy]


def metrics_csv(result: RunResult, n_devices: int) -> str:
    import csv
    import io

    buf = io.StringIO()
    w = csv.writer(buf, lineterminator="\n")
    w.writerow(metrics_columns(n_devices))
    for row in result.metrics:
        w.writerow(metrics_row(row))
    return buf.getvalue()


def summary_json(result: RunResult) -> str:
    return json.dumps(dataclasses.asdict(result.summary), indent=2) + "\n"


def write_outputs(out_dir, result: RunResult, n_devices: int) -> None:
    """metrics.csv + summary.json exactly as ``cli._execute_run`` writes them."""
    from pathlib import Path

    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    with open(out / "metrics.csv", "w", encoding="utf-8", newline="\n") as fh:
        fh.write(metrics_csv(result, n_devices))
    with open(out / "summary.json", "w", encoding="utf-8") as fh:
        fh.write(summary_json(result))


# -- the gradient producer ------------------------------------------------------------------


class ReferenceProducer:
    """The reference's dataset generator and MLP (datagen.generate_dataset, nn.init_model /
    loss_and_grad / evaluate): the step *before* and the evaluation *after* the hot path,
    out of scope here and taken from the reference package unchanged."""

    def __init__(self, datagen_module, nn_module):
        self.datagen, self.nn = datagen_module, nn_module

    @classmethod
    def from_package(cls, pkg: str = "streamsgd"):
        import importlib

        return cls(importlib.import_module(f"{pkg}.datagen"), importlib.import_module(f"{pkg}.nn"))

    def generate_dataset(self, spec):
        return self.datagen.generate_dataset(spec)

    def init_model(self, sizes, seed):
        return self.nn.init_model(sizes, seed)

    def loss_and_grad(self, model, x, y):
        return self.nn.loss_and_grad(model, x, y)

    def evaluate(self, model, x, y) -> float:
        return self.nn.evaluate(model, x, y)


# -- the loop -------------------------------------------------------------------------------


class RankRunner:
    """One rank of a P-process run of the reference's ``Simulation`` over the B200 hot path.

    ``config`` is a reference ``SimConfig`` (validated by the caller, e.g.
    ``streamsgd.config.parse_config``); devices are sharded contiguously over the ranks of
    ``group`` (rank r owns [r*k, (r+1)*k), the exchange's worker sharding).  ``ops`` and
    ``sampler_ops`` are test-only stand-ins for the kernels (CPU gloo tests).
    """

    def __init__(self, config, producer, *, group=None, device=None, dtype=torch.float64, ops=None,
                 sampler_ops=None):
        cfg = self.config = config
        n = cfg.n_devices
        self.group = group
        self.world = dist.get_world_size(group) if group is not None else 1
        self.rank = dist.get_rank(group) if group is not None else 0
        if n % self.world:
            raise ValueError("n_devices must divide evenly over ranks")
        self.k = n // self.world
        self.lo = self.rank * self.k
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device())
        self.device = device
        self.producer = producer
        seed = cfg.seed
        rd = cfg.rate_dist
        self.rate_dist = streams.RateDistribution(rd.kind, rd.mean, rd.std)
        self.rates = streams.sample_rates(self.rate_dist, n, streams.derive_seed(seed, "rates"))
        self.dataset = producer.generate_dataset(cfg.dataset)
        self.pools = streams.partition(self.dataset.train_y, n, cfg.partition.mode, cfg.partition.labels_per_device,
                                       streams.derive_seed(seed, "partition"))
        self.buffers = [streams.StreamBuffer(rate=r, policy=cfg.retention) for r in self.rates]
        if cfg.prefill_seconds > 0:
            for buf in self.buffers:
                buf.enqueue_arrivals(cfg.prefill_seconds)
        sizes = (cfg.dataset.feature_dim, *cfg.model.hidden, cfg.dataset.n_classes)
        self.model = producer.init_model(sizes, streams.derive_seed(seed, "model_init"))
        self.dim = int(self.model.flat.size)
        c = cfg.compression
        self.ex = exchange.GradientExchange(
            self.dim, n, cr=c.cr, delta=c.delta, ewma_factor=c.ewma_factor, raw_gate=c.raw_gate,
            compression=c.enabled, momentum=cfg.optimizer.momentum, weight_decay=cfg.optimizer.weight_decay,
            group=group, ops=ops, device=device, dtype=dtype)
        self.ex.params.copy_(torch.from_numpy(np.asarray(self.model.flat, dtype=np.float64)).to(device, dtype=dtype))
        x, y = self.dataset.train_x, self.dataset.train_y
        if self.world > 1:
            self.sampler = streams.ShardedSampler(x, y, self.pools, self.lo, self.k, group=group, device=device,
                                                  ops=sampler_ops)
        else:
            self.sampler = streams.DeviceSampler(x, y, self.pools, device=device, ops=sampler_ops)
        self.link = comm.LinkModel(cfg.cost.link_latency, cfg.cost.link_bandwidth)
        self.base_global_batch = (cfg.optimizer.base_global_batch if cfg.optimizer.base_global_batch is not None
                                  else n * 64)
        self.now = 0.0
        self.iteration = 0
        self.injection_bytes_cum = 0
        self.epoch = 0
        self.iter_in_epoch = 0
        self._refresh_epoch_layout()
        self._set_augmentation(0)

    # -- per-epoch scaffolding (engine.py:171-199) ----------------------------------------------

    def _refresh_epoch_layout(self) -> None:
        cfg = self.config
        self.batch_sizes = [streams.compute_batch_size(cfg.mode, r, cfg.b_min, cfg.b_max, cfg.fixed_batch)
                            for r in self.rates]
        self.iters_per_epoch = max(1, math.ceil(self.dataset.n_train / sum(self.batch_sizes)))

    def _set_augmentation(self, epoch: int) -> None:
        std = self.config.model.augment_std
        if std <= 0:
            self.sampler.set_augmentation(None)
            return
        rng = np.random.default_rng(streams.derive_seed(self.config.seed, f"augment:{epoch}"))
        self.sampler.set_augmentation(rng.normal(0.0, std, self.dataset.train_x.shape))

    def _start_epoch(self, epoch: int) -> None:
        cfg = self.config
        self.epoch = epoch
        self.iter_in_epoch = 0
        self._set_augmentation(epoch)
        if cfg.rate_jitter and epoch > 0:
            self.rates = streams.sample_rates(self.rate_dist, cfg.n_devices,
                                              streams.derive_seed(cfg.seed, f"rates:{epoch}"))
            for buf, rate in zip(self.buffers, self.rates):
                buf.rate = rate
            self._refresh_epoch_layout()

    # -- the global step (engine.py:208-322) ----------------------------------------------------

    def _gather_floats(self, local: np.ndarray) -> np.ndarray:
        if self.world == 1:
            return local
        t = torch.from_numpy(np.ascontiguousarray(local, dtype=np.float64)).to(self.ex.device)
        out = torch.empty(self.world * t.numel(), dtype=torch.float64, device=self.ex.device)
        dist.all_gather_into_tensor(out, t, group=self.group)
        return out.cpu().numpy()

    def _sum_ints(self, vals) -> list[int]:
        if self.world == 1:
            return [int(v) for v in vals]
        t = torch.tensor([int(v) for v in vals], dtype=torch.int64, device=self.ex.device)
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        return [int(v) for v in t.cpu().tolist()]

    def run_iteration(self) -> IterationMetrics:
        cfg = self.config
        n = cfg.n_devices
        b = self.batch_sizes
        waits = [streams.streaming_wait(len(buf), b[d], self.rates[d]) for d, buf in enumerate(self.buffers)]
        global_wait = max(waits)
        if global_wait > 0:
            for buf in self.buffers:
                buf.enqueue_arrivals(global_wait)
        draws = [buf.draw_batch(b[d]) for d, buf in enumerate(self.buffers)]
        plan = picks = None
        injection_bytes = 0
        sizes = list(b)
        if cfg.injection.enabled and cfg.injection.alpha > 0:
            it = self.iteration
            plan = streams.injection_plan(n, cfg.injection.alpha, cfg.injection.beta, b,
                                          streams.derive_seed(cfg.seed, f"inject-plan:{it}"))
            draw_rng = np.random.default_rng(streams.derive_seed(cfg.seed, f"inject-draw:{it}"))
            picks = streams.injection_picks(plan, b, draw_rng)
            injection_bytes = streams.injection_bytes(plan, n, cfg.sample_bytes)
            self.injection_bytes_cum += injection_bytes
            for s, c in plan:
                for d in range(n):
                    if d != s:
                        sizes[d] += c
        # this rank's devices' batches, staged on the device
        x, y, ptr = self.sampler.stage(draws, plan, picks)
        xh, yh = x.cpu().numpy(), y.cpu().numpy()
        losses_local = np.empty(self.k)
        for i in range(self.k):
            xs, ys = xh[ptr[i]:ptr[i + 1]], yh[ptr[i]:ptr[i + 1]]
            loss, grad = self.producer.loss_and_grad(self.model, xs, ys)
            losses_local[i] = loss
            self.ex.bucket[i, :self.dim].copy_(torch.from_numpy(np.asarray(grad, dtype=np.float64)))
        losses = self._gather_floats(losses_local)
        if cfg.mode == streams.MODE_RATE_MATCHED:
            weights = comm.weights_from_rates(self.rates)
        else:
            weights = np.full(n, 1.0 / n)
        train_loss = float(weights @ losses)
        if not np.isfinite(train_loss):
            raise DivergenceError(f"non-finite loss at iteration {self.iteration + 1}")
        lr = nn.lr_at_epoch(cfg.optimizer.base_lr, cfg.optimizer.schedule, self.epoch)
        if cfg.mode == streams.MODE_RATE_MATCHED:
            lr = nn.scale_lr(lr, sum(self.rates), self.base_global_batch)
        # gate -> exchange -> weighted aggregate -> momentum SGD (engine.py:253-283)
        self.ex.step(weights, lr)
        self.model.flat[...] = self.ex.params.cpu().numpy()
        # accounting from the device: decisions of every device, gate counters of every rank
        if cfg.compression.enabled:
            dec = self._all_decisions()
            payload_sizes = [comm.payload_bytes(bool(dec[d]), self.dim, cfg.compression.cr) for d in range(n)]
        else:
            payload_sizes = [comm.payload_bytes(False, self.dim, 1.0)] * n
        floats, nbytes = self._sum_ints(self.ex.volume())
        compute_time = max(cfg.cost.c0 + cfg.cost.c1 * sizes[d] for d in range(n))
        comm_t = comm.comm_time(max(payload_sizes), self.link, n)
        busy = compute_time + comm_t
        for buf in self.buffers:
            buf.enqueue_arrivals(busy)
        for buf in self.buffers:
            buf.apply_retention()
        self.now += global_wait + busy
        self.iteration += 1
        self.iter_in_epoch += 1
        occupancy = [len(buf) for buf in self.buffers]
        cnc = None
        if cfg.compression.enabled:
            rec = self.ex.gate_counters()
            n_comp, n_unc = self._sum_ints([int(rec["n_compressed"].sum()), int(rec["n_uncompressed"].sum())])
            cnc = n_comp / (n_comp + n_unc)
        return IterationMetrics(
            iteration=self.iteration, sim_time_s=self.now, epoch=self.epoch, global_batch=sum(b), lr_used=lr,
            train_loss=train_loss, test_accuracy=None, wait_time_s=global_wait, buffer_occupancy=occupancy,
            buffer_bytes=sum(occupancy) * cfg.sample_bytes, floats_sent_cum=floats, bytes_sent_cum=nbytes,
            cnc_cum=cnc, injection_bytes=injection_bytes, injection_bytes_cum=self.injection_bytes_cum)

    def _all_decisions(self) -> np.ndarray:
        ex = self.ex
        if self.world == 1:
            return ex.decision.cpu().numpy()
        if getattr(ex, "dec_all", None) is not None:
            return ex.dec_all.cpu().numpy()
        out = torch.empty(ex.W, dtype=torch.uint8, device=ex.device)
        dist.all_gather_into_tensor(out, ex.decision.contiguous(), group=self.group)
        return out.cpu().numpy()

    def evaluate(self) -> float:
        return self.producer.evaluate(self.model, self.dataset.test_x, self.dataset.test_y)

    def param_checksum(self) -> float:
        """Replica check (engine.py:284-286): identical on every rank by construction."""
        return self.ex.param_checksum()

    def run(self, sink=None) -> RunResult:
        """Run until target accuracy or max_epochs (engine.py:327-380)."""
        cfg = self.config
        rows: list[IterationMetrics] = []
        best_acc = final_acc = time_to_target = None
        reached = False
        while True:
            row = self.run_iteration()
            epoch_done = self.iter_in_epoch >= self.iters_per_epoch
            if epoch_done:
                acc = self.evaluate()
                row.test_accuracy = acc
                final_acc = acc
                best_acc = acc if best_acc is None else max(best_acc, acc)
                if cfg.target_accuracy is not None and acc >= cfg.target_accuracy and not reached:
                    reached = True
                    time_to_target = row.sim_time_s
            rows.append(row)
            if sink is not None:
                sink(row)
            if epoch_done:
                completed = self.epoch + 1
                if reached:
                    break
                if cfg.max_epochs is not None and completed >= cfg.max_epochs:
                    break
                self._start_epoch(completed)
        floats, nbytes = rows[-1].floats_sent_cum, rows[-1].bytes_sent_cum
        summary = RunSummary(
            final_accuracy=final_acc, best_accuracy=best_acc, final_train_loss=rows[-1].train_loss,
            iterations=len(rows), epochs_completed=self.epoch + 1, sim_time_s=self.now,
            target_accuracy=cfg.target_accuracy, reached_target=reached, time_to_target_s=time_to_target,
            floats_sent_total=floats, bytes_sent_total=nbytes, cnc=rows[-1].cnc_cum,
            injection_bytes_total=self.injection_bytes_cum, final_buffer_samples=rows[-1].buffer_samples_total,
            final_buffer_bytes=rows[-1].buffer_bytes, seed=cfg.seed)
        return RunResult(summary, rows)
