"""Numpy restatement of the streaming sampler and injection (TEST INFRASTRUCTURE ONLY).

Follows /root/reference/pkg/src/streamsgd/streams.py, datagen.py and the sampler section of
engine.py (run_iteration lines 213-242 and _materialize 201-204).
"""

from __future__ import annotations

import hashlib
import math
from collections import deque

import numpy as np

FLOOR_EPS = 1e-9  # streams.py:19


def derive_seed(master: int, label: str) -> int:
    """config.py:235-238 — first 8 bytes (little endian) of sha256('master:label')."""
    return int.from_bytes(hashlib.sha256(f"{master}:{label}".encode()).digest()[:8], "little")


def sample_rates(kind: str, mean: float, std: float, n: int, seed: int) -> list[int]:
    """streams.py:58-69 — uniform with the given mean/std (support mean +- std*sqrt 3) or
    normal; rounded to nearest and clamped >= 1."""
    rng = np.random.default_rng(seed)
    if kind == "uniform":
        h = std * math.sqrt(3.0)
        raw = rng.uniform(mean - h, mean + h, n)
    else:
        raw = rng.normal(mean, std, n)
    return [int(r) for r in np.maximum(1, np.rint(raw).astype(int))]


def batch_size(mode: str, rate: int, b_min: int, b_max: int, fixed: int) -> int:
    """engine.py:93-99."""
    return fixed if mode == "fixed_batch" else min(max(rate, b_min), b_max)


def streaming_wait(buffer_len: int, b: int, rate: int) -> float:
    """streams.py:130-134."""
    return max(0.0, (b - buffer_len) / rate)


class DequeBuffer:
    """streams.py:72-127 with an explicit deque of ids (the reference representation)."""

    def __init__(self, rate: int, policy: str = "persistence"):
        self.rate, self.policy = rate, policy
        self.pending: deque = deque()
        self.credit = 0.0
        self.next_id = 0

    def __len__(self):
        return len(self.pending)

    def enqueue(self, elapsed: float) -> int:
        exact = self.rate * elapsed + self.credit
        added = int(math.floor(exact + FLOOR_EPS))
        self.credit = min(max(exact - added, 0.0), math.nextafter(1.0, 0.0))
        self.pending.extend(range(self.next_id, self.next_id + added))
        self.next_id += added
        return added

    def draw(self, b: int) -> list[int]:
        if len(self.pending) < b:
            raise RuntimeError("would block")
        return [self.pending.popleft() for _ in range(b)]

    def retain(self) -> int:
        if self.policy == "persistence":
            return 0
        drop = max(0, len(self.pending) - self.rate)
        for _ in range(drop):
            self.pending.popleft()
        return drop


def partition_iid(n_train: int, n: int, seed: int) -> list[np.ndarray]:
    """datagen.py:121-123 — uniform random disjoint split."""
    rng = np.random.default_rng(seed)
    perm = rng.permutation(n_train)
    return [np.sort(p) for p in np.array_split(perm, n)]


def partition_noniid(train_y: np.ndarray, n: int, lpd: int, seed: int) -> list[np.ndarray]:
    """datagen.py:125-144 — label groups of size lpd, devices join groups round-robin."""
    rng = np.random.default_rng(seed)
    labels = np.unique(train_y)
    groups = len(labels) // lpd
    perm = rng.permutation(labels)
    members: list[list[int]] = [[] for _ in range(groups)]
    for d in range(n):
        members[d % groups].append(d)
    pools = [None] * n
    for gi in range(groups):
        idx = rng.permutation(np.flatnonzero(np.isin(train_y, perm[gi * lpd:(gi + 1) * lpd])))
        for d, part in zip(members[gi], np.array_split(idx, len(members[gi]))):
            pools[d] = np.sort(part)
    return pools


def injection_plan(n: int, alpha: float, beta: float, batch_sizes, seed: int):
    """datagen.py:162-179 — ceil(alpha*n) senders (sorted choice), ceil(beta*b_i) shares."""
    k = math.ceil(alpha * n)
    if k == 0:
        return []
    rng = np.random.default_rng(seed)
    senders = np.sort(rng.choice(n, size=k, replace=False))
    return [(int(s), math.ceil(beta * batch_sizes[s])) for s in senders]


def inject(batches, plan, sample_bytes: int, rng):
    """datagen.py:182-210 — picks without replacement from each sender's pre-injection batch,
    appended to every other batch in plan order; bytes counts every copy."""
    n = len(batches)
    out = [list(b) for b in batches]
    moved = 0
    for s, cnt in plan:
        if cnt == 0:
            continue
        picks = rng.choice(len(batches[s]), size=cnt, replace=False)
        shared = [batches[s][p] for p in picks]
        for d in range(n):
            if d != s:
                out[d].extend(shared)
        moved += cnt * (n - 1) * sample_bytes
    return out, moved


def materialize(train_x, augment, train_y, rows):
    """engine.py:201-204 — x = train_x[idx] + augment[idx]."""
    idx = np.asarray(rows, dtype=np.int64)
    return train_x[idx] + augment[idx], train_y[idx]
