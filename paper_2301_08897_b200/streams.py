"""Streaming-rate-driven variable-batch sampler and non-IID injection, staged on the device
(item 5).  Mirrors ``streamsgd.streams`` / ``streamsgd.datagen`` (reference
pkg/src/streamsgd/streams.py, datagen.py) and the sampler section of
``Simulation.run_iteration`` (engine.py:213-242, _materialize 201-204).

Host side (identical numpy calls and seeds, so every random draw matches the reference):
  ``derive_seed``, ``RateDistribution``/``sample_rates``, ``compute_batch_size``,
  ``streaming_wait``, ``StreamBuffer`` (the FIFO of pending sample ids is always one
  contiguous id range, so it is kept as (head, next_id, credit) instead of a deque),
  ``injection_plan`` / ``injection_picks``, ``partition``.
Device side (sm_100a kernels via the C-ABI): :class:`DeviceSampler` resolves drawn id
ranges to train rows (pools[d][a % len]), builds the injected batches, and gathers
x = train_x[rows] + augment[rows] (binary64 add, bit-exact) into one batch tensor.
"""

from __future__ import annotations

import hashlib
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import kernels

FLOOR_EPS = 1e-9  # streams.py:19
PERSISTENCE = "persistence"
TRUNCATION = "truncation"
RETENTION_POLICIES = (PERSISTENCE, TRUNCATION)
RATE_KINDS = ("uniform", "normal")
MODE_FIXED_BATCH = "fixed_batch"
MODE_RATE_MATCHED = "rate_matched"


def derive_seed(master: int, label: str) -> int:
    """Labelled sha256 seed (config.py:235-238)."""
    digest = hashlib.sha256(f"{master}:{label}".encode()).digest()
    return int.from_bytes(digest[:8], "little")


class WouldBlock(Exception):
    """A batch draw needs more samples than the buffer holds (streams.py:28-33)."""

    def __init__(self, shortfall: int):
        super().__init__(f"buffer short by {shortfall} samples")
        self.shortfall = shortfall


@dataclass
class RateDistribution:
    """streams.py:36-55: uniform with the given mean/std, or normal."""

    kind: str
    mean: float
    std: float = 0.0

    def __post_init__(self):
        if self.kind not in RATE_KINDS:
            raise ValueError(f"unknown rate distribution kind: {self.kind!r}")
        if self.mean <= 0:
            raise ValueError("rate distribution mean must be positive")
        if self.std < 0:
            raise ValueError("rate distribution std must be non-negative")


def sample_rates(dist: RateDistribution, n: int, seed: int) -> list[int]:
    """Integer rates, rounded to nearest and clamped >= 1 (streams.py:58-69)."""
    if n < 1:
        raise ValueError("need at least one device rate")
    rng = np.random.default_rng(seed)
    if dist.kind == "uniform":
        half = dist.std * math.sqrt(3.0)
        raw = rng.uniform(dist.mean - half, dist.mean + half, n)
    else:
        raw = rng.normal(dist.mean, dist.std, n)
    return [int(r) for r in np.maximum(1, np.rint(raw).astype(int))]


def compute_batch_size(mode: str, rate: int, b_min: int, b_max: int, fixed_batch: int) -> int:
    """engine.py:93-99: fixed batch, or the rate clamped to [b_min, b_max]."""
    if mode == MODE_FIXED_BATCH:
        return fixed_batch
    if mode == MODE_RATE_MATCHED:
        return min(max(rate, b_min), b_max)
    raise ValueError(f"unknown mode: {mode!r}")


def streaming_wait(buffer_len: int, b: int, rate: int) -> float:
    """Seconds until b samples are available (streams.py:130-134)."""
    if rate < 1:
        raise ValueError("rate must be >= 1")
    return max(0.0, (b - buffer_len) / rate)


class StreamBuffer:
    """FIFO of pending sample ids fed at a fixed rate (streams.py:72-127).

    Ids are issued consecutively and drawn/retained from the front, so the pending set is
    always the contiguous range [head, next_id); a draw returns ``range(head, head + b)``.
    """

    def __init__(self, rate: int, policy: str = PERSISTENCE):
        if rate < 1:
            raise ValueError("stream rate must be >= 1")
        if policy not in RETENTION_POLICIES:
            raise ValueError(f"unknown retention policy: {policy!r}")
        self.rate = rate
        self.policy = policy
        self.head = 0
        self.next_id = 0
        self.fractional_credit = 0.0

    def __len__(self) -> int:
        return self.next_id - self.head

    @property
    def pending(self) -> range:
        return range(self.head, self.next_id)

    def enqueue_arrivals(self, elapsed: float) -> int:
        if elapsed < 0:
            raise ValueError("elapsed time must be non-negative")
        exact = self.rate * elapsed + self.fractional_credit
        added = int(math.floor(exact + FLOOR_EPS))
        self.fractional_credit = min(max(exact - added, 0.0), math.nextafter(1.0, 0.0))
        self.next_id += added
        return added

    def draw_batch(self, b: int) -> range:
        if b < 1:
            raise ValueError("batch size must be >= 1")
        if len(self) < b:
            raise WouldBlock(b - len(self))
        ids = range(self.head, self.head + b)
        self.head += b
        return ids

    def apply_retention(self) -> int:
        if self.policy == PERSISTENCE:
            return 0
        discard = max(0, len(self) - self.rate)
        self.head += discard
        return discard


def partition(train_y: np.ndarray, n_devices: int, mode: str, labels_per_device: int, seed: int) -> list[np.ndarray]:
    """Train-index pools per device (datagen.py:110-144), same RNG calls as the reference."""
    if mode not in ("iid", "noniid"):
        raise ValueError(f"unknown partition mode: {mode!r}")
    rng = np.random.default_rng(seed)
    n = n_devices
    if mode == "iid":
        perm = rng.permutation(len(train_y))
        return [np.sort(p) for p in np.array_split(perm, n)]
    labels = np.unique(train_y)
    k = len(labels)
    lpd = labels_per_device
    if k % lpd != 0:
        raise ValueError(f"{k} labels cannot be split into groups of {lpd}")
    groups = k // lpd
    if n * lpd < k or n < groups:
        raise ValueError(f"{n} devices cannot cover {k} labels at {lpd} labels/device")
    order = rng.permutation(labels)
    members: list[list[int]] = [[] for _ in range(groups)]
    for d in range(n):
        members[d % groups].append(d)
    pools: list[np.ndarray] = [np.empty(0, dtype=np.int64)] * n
    for g in range(groups):
        idx = rng.permutation(np.flatnonzero(np.isin(train_y, order[g * lpd:(g + 1) * lpd])))
        for d, part in zip(members[g], np.array_split(idx, len(members[g]))):
            pools[d] = np.sort(part)
    return pools


def injection_plan(n_devices: int, alpha: float, beta: float, batch_sizes, seed: int) -> list[tuple[int, int]]:
    """ceil(alpha*n) senders (sorted choice), each sharing ceil(beta*b_i) (datagen.py:162-179)."""
    if n_devices < 2:
        raise ValueError("injection needs at least two devices")
    if len(batch_sizes) != n_devices:
        raise ValueError("one batch size per device required")
    n_senders = math.ceil(alpha * n_devices)
    if n_senders == 0:
        return []
    rng = np.random.default_rng(seed)
    senders = np.sort(rng.choice(n_devices, size=n_senders, replace=False))
    return [(int(i), math.ceil(beta * batch_sizes[i])) for i in senders]


def injection_picks(plan, batch_sizes, rng: np.random.Generator) -> list[np.ndarray]:
    """Positions each sender shares, drawn exactly as datagen.inject does (datagen.py:200-203)."""
    picks = []
    for sender, count in plan:
        if count == 0:
            picks.append(np.zeros(0, dtype=np.int64))
            continue
        picks.append(np.asarray(rng.choice(batch_sizes[sender], size=count, replace=False), dtype=np.int64))
    return picks


def injection_bytes(plan, n_devices: int, sample_bytes: int) -> int:
    """Bytes moved by one injection step: every (sender, recipient) copy (datagen.py:208)."""
    return sum(c * (n_devices - 1) * sample_bytes for _, c in plan if c)


class _Done:
    """Event stand-in for host-memory staging (test ops): copies are synchronous."""

    def record(self):
        pass

    def synchronize(self):
        pass


class DeviceSampler:
    """Per-iteration batch staging on the GPU.

    ``train_x`` (float64 or float32), ``train_y`` and the pools live on the device; the
    per-epoch augmentation table is generated on the host with the reference's RNG
    (engine.py:180-185) and uploaded once per epoch.
    """

    def __init__(self, train_x: np.ndarray, train_y: np.ndarray, pools: list[np.ndarray], *,
                 device: torch.device | None = None, dtype: torch.dtype = torch.float64, ops=None):
        # ``ops`` (tests only): a stand-in for the three kernels with the same contract, so the
        # multi-rank protocol of ShardedSampler can run on CPU over gloo; the product path is
        # always the sm_100a kernels
        self.ops = ops if ops is not None else kernels
        if ops is None:
            kernels.require_cuda()
            self.device = device or torch.device("cuda", torch.cuda.current_device())
        else:
            self.device = device or torch.device("cpu")
        self.dtype = dtype
        self.pool_lens = [len(p) for p in pools]
        self.train_x = torch.from_numpy(np.ascontiguousarray(train_x)).to(self.device, dtype=dtype)
        self.train_y = torch.from_numpy(np.asarray(train_y, dtype=np.int64)).to(self.device)
        lens = [len(p) for p in pools]
        self.pool_ptr = torch.tensor(np.concatenate([[0], np.cumsum(lens)]), dtype=torch.int64, device=self.device)
        self.pool_rows = torch.from_numpy(np.concatenate([np.asarray(p, dtype=np.int64) for p in pools])).to(self.device)
        self.n_dev = len(pools)
        self.augment = None

    def set_augmentation(self, table: np.ndarray | None) -> None:
        self.augment = None if table is None else torch.from_numpy(np.ascontiguousarray(table)).to(self.device, dtype=self.dtype)

    def _upload(self, parts):
        """One pinned host buffer and one H2D copy for every small index array of a step;
        returns device views (int64, or int32 for parts given as int32)."""
        sizes = [(a.size * a.itemsize + 7) // 8 for a in parts]
        total = max(sum(sizes), 1)
        if getattr(self, "_host", None) is None or self._host.numel() < total:
            self._host = torch.empty(max(total, 1024), dtype=torch.int64, pin_memory=self.device.type == "cuda")
            self._dev = torch.empty(max(total, 1024), dtype=torch.int64, device=self.device)
        else:
            # the previous step's copy must have left the pinned buffer before it is refilled
            self._copied.synchronize()
        h = self._host.numpy()
        off, spans = 0, []
        for a, n in zip(parts, sizes):
            if a.dtype == np.int32:
                h[off:off + n].view(np.int32)[:a.size] = a
            else:
                h[off:off + n] = a
            spans.append((off, n, a.dtype, a.size))
            off += n
        self._dev[:total].copy_(self._host[:total], non_blocking=True)
        self._copied = torch.cuda.Event() if self.device.type == "cuda" else _Done()
        self._copied.record()
        out = []
        for o, n, dt, size in spans:
            v = self._dev[o:o + n]
            out.append(v.view(torch.int32)[:size] if dt == np.int32 else v[:size])
        return out

    def stage(self, draws: list[range], plan=None, picks=None):
        """Rows of every device's batch (CSR) and the gathered batch.

        ``draws[d]`` is the id range drawn from device d's StreamBuffer; ``plan``/``picks``
        come from :func:`injection_plan` / :func:`injection_picks`.  Returns
        (x [rows, F], y [rows], ptr [n_dev + 1] host int64) with device d's batch in
        rows ptr[d]:ptr[d+1] in the reference's order (own samples, then injected ones).
        All the step's small index arrays go to the device in one pinned copy.
        """
        dev = self.device
        b = np.array([len(r) for r in draws], dtype=np.int64)
        for d, n in enumerate(b):
            if n and not self.pool_lens[d]:  # the reference fails at `a % len(pool)` (engine.py:224-227)
                raise ZeroDivisionError(f"integer modulo by zero (device {d} draws from an empty pool)")
        head = np.array([r.start for r in draws], dtype=np.int64)
        base_ptr = np.concatenate([[0], np.cumsum(b)]).astype(np.int64)
        total = int(base_ptr[-1])
        ptr = base_ptr
        parts = [head, b, base_ptr]
        if plan:
            counts = np.array([c for _, c in plan], dtype=np.int64)
            sizes = b.copy()
            for (s, c) in plan:
                sizes += c
                sizes[s] -= c
            ptr = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
            pick_ptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
            all_picks = np.concatenate(picks).astype(np.int64) if len(picks) else np.zeros(0, dtype=np.int64)
            senders = np.array([s for s, _ in plan], dtype=np.int32)
            parts += [senders, pick_ptr, all_picks if all_picks.size else np.zeros(1, dtype=np.int64), ptr]
        views = self._upload(parts)
        rows = torch.empty(max(total, 1), dtype=torch.int64, device=dev)
        self.ops.resolve_stream_rows(views[0], views[1], views[2], self.pool_ptr, self.pool_rows, total, rows)
        if plan:
            d_senders, d_pick_ptr, d_picks, d_ptr = views[3:]
            out_rows = torch.empty(max(int(ptr[-1]), 1), dtype=torch.int64, device=dev)
            self.ops.inject_rows(views[2], rows, d_senders, d_pick_ptr, d_picks, d_ptr, out_rows)
            rows = out_rows
        n = int(ptr[-1])
        x = torch.empty((n, self.train_x.shape[1]), dtype=self.dtype, device=dev)
        y = torch.empty(n, dtype=torch.int64, device=dev)
        self.ops.gather_batch(self.train_x, self.augment, self.train_y, rows[:n], x, y)
        return x, y, ptr


class ShardedSampler:
    """the pool-sharded dataset, with injected samples moved between GPUs
    instead of a replicated train set.

    One process per GPU; rank r owns the contiguous devices [lo, lo + k) (the exchange's worker
    sharding) and holds only the train rows of their pools.  Every rank runs the same host
    planning (stream buffers, ``injection_plan`` / ``injection_picks`` with the shared seeds), so
    each knows every sender's share count and the layout of the exchanged buffer without a
    size exchange.  Per step:
      1. the local devices' own batches: ``DeviceSampler.stage`` on the shard (rows resolved,
         x = train_x[rows] + augment[rows] gathered on the device);
      2. each local sender's shared samples (its pre-injection batch at the picked positions)
         are materialised rows of step 1, so they are gathered into a send buffer;
      3. one ``all_gather_into_tensor`` (NCCL over NVLink) of the padded send buffers -- the
         allgatherv of datagen.inject's wire format (datagen.py:182-210);
      4. each local device's batch = its own rows, then every other sender's shared rows in plan
         order (datagen.py:204-207), assembled by one device gather.
    Bit-identical to ``DeviceSampler`` over the replicated set (tools/multi_sampler_check.py).
    """

    def __init__(self, train_x: np.ndarray, train_y: np.ndarray, pools: list[np.ndarray], lo: int, k: int, *,
                 group=None, device: torch.device | None = None, dtype: torch.dtype = torch.float64, ops=None):
        self.n_dev, self.lo, self.k, self.group = len(pools), lo, k, group
        local = [np.asarray(pools[d], dtype=np.int64) for d in range(lo, lo + k)]
        self._rows = np.concatenate(local) if local else np.zeros(0, dtype=np.int64)
        offs = np.concatenate([[0], np.cumsum([len(p) for p in local])])
        local_pools = [np.arange(offs[i], offs[i + 1], dtype=np.int64) for i in range(k)]
        self.inner = DeviceSampler(np.asarray(train_x)[self._rows], np.asarray(train_y)[self._rows], local_pools,
                                   device=device, dtype=dtype, ops=ops)
        self.ops = self.inner.ops
        self.device = self.inner.device
        self.F = self.inner.train_x.shape[1]

    def set_augmentation(self, table: np.ndarray | None) -> None:
        self.inner.set_augmentation(None if table is None else np.asarray(table)[self._rows])

    def stage(self, draws: list[range], plan=None, picks=None):
        """``draws``: all n_dev id ranges (identical on every rank).  Returns (x, y, ptr) for the
        LOCAL devices: device lo + i's batch in rows ptr[i]:ptr[i + 1]."""
        import torch.distributed as dist

        lo, k, dev = self.lo, self.k, self.device
        x_own, y_own, ptr_own = self.inner.stage(draws[lo:lo + k])
        if not plan:
            return x_own, y_own, ptr_own
        world = dist.get_world_size(self.group)
        kk = [self.n_dev // world] * world  # devices per rank (the exchange's even sharding)
        owner = np.repeat(np.arange(world), kk)
        per_rank = np.zeros(world, dtype=np.int64)
        for s, c in plan:
            per_rank[owner[s]] += c
        smax = max(int(per_rank.max()), 1)
        rank = dist.get_rank(self.group)
        # 2. send buffer: this rank's senders' shares in plan order (positions in x_own)
        send_pos = [ptr_own[s - lo] + np.asarray(p, dtype=np.int64)
                    for (s, c), p in zip(plan, picks) if owner[s] == rank and c]
        send_pos = np.concatenate(send_pos) if send_pos else np.zeros(0, dtype=np.int64)
        sx = torch.zeros((smax, self.F), dtype=x_own.dtype, device=dev)
        sy = torch.zeros(smax, dtype=torch.int64, device=dev)
        if send_pos.size:
            d_pos = self.inner._upload([send_pos])[0]
            self.ops.gather_batch(x_own, None, y_own, d_pos, sx[:send_pos.size], sy[:send_pos.size])
        # 3. allgatherv as one padded all-gather
        gx = torch.empty((world * smax, self.F), dtype=x_own.dtype, device=dev)
        gy = torch.empty(world * smax, dtype=torch.int64, device=dev)
        dist.all_gather_into_tensor(gx, sx, group=self.group)
        dist.all_gather_into_tensor(gy, sy, group=self.group)
        # 4. source = [x_own ; gathered]; sender s's shares start at n_own + owner(s)*smax + (its
        # offset among its rank's senders)
        n_own = int(ptr_own[-1])
        start = np.zeros(len(plan), dtype=np.int64)
        fill = np.zeros(world, dtype=np.int64)
        for i, (s, c) in enumerate(plan):
            start[i] = n_own + owner[s] * smax + fill[owner[s]]
            fill[owner[s]] += c
        rows, ptr = [], [0]
        for i in range(k):
            d = lo + i
            mine = [np.arange(ptr_own[i], ptr_own[i + 1], dtype=np.int64)]
            mine += [np.arange(start[j], start[j] + c, dtype=np.int64) for j, (s, c) in enumerate(plan) if s != d and c]
            rows += mine
            ptr.append(ptr[-1] + sum(r.size for r in mine))
        rows = np.concatenate(rows) if rows else np.zeros(0, dtype=np.int64)
        src_x = torch.cat([x_own, gx])
        src_y = torch.cat([y_own, gy])
        n = rows.size
        x = torch.empty((n, self.F), dtype=x_own.dtype, device=dev)
        y = torch.empty(n, dtype=torch.int64, device=dev)
        if n:
            d_rows = self.inner._upload([rows])[0]
            self.ops.gather_batch(src_x, None, src_y, d_rows, x, y)
        return x, y, np.asarray(ptr, dtype=np.int64)
