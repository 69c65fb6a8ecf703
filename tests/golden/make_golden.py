"""Generate the golden fixtures by running the REFERENCE implementation (build container only).

    python tests/golden/make_golden.py [--ref /root/reference/pkg/src]

Imports ``streamsgd`` read-only from the reference tree (no bytecode written there) and
records inputs and outputs of the hot-path functions, including the reference's own
known-answer tests (pkg/tests/test_comm.py, test_acceptance.py, test_nn.py, test_engine.py).
The fixtures are committed; nothing on the GPU box reads the reference.
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import math
import sys
import types
from pathlib import Path

sys.dont_write_bytecode = True
import numpy as np  # noqa: E402

OUT = Path(__file__).resolve().parent


def load_reference(path: str):
    sys.path.insert(0, path)
    import streamsgd  # noqa: F401
    from streamsgd import cli, comm, config, datagen, engine, nn, streams

    return types.SimpleNamespace(cli=cli, comm=comm, config=config, datagen=datagen, engine=engine, nn=nn, streams=streams)


def topk_cases(R):
    rng = np.random.default_rng(20260101)
    cases = []
    # reference known answers (test_comm.py:91-104) and survey probes (SURVEY §0 trap 2, §8(c))
    nan, inf = float("nan"), float("inf")
    fixed = [
        ([3.0, -4.0, 1.0, 0.5], 0.5),
        ([1.0, -1.0, 1.0, 1.0], 0.5),
        ([0.0, -1.0, 2.0, 0.0], 1.0),
        ([nan, 1.0, 2.0, 0.5], 0.5),
        ([nan, 1.0, nan, 2.0], 0.75),
        ([nan, nan, nan, nan, nan, 0.0], 0.5),
        ([-0.0, 0.0, 1e-300, 0.0], 0.5),
        ([1.0, inf, -inf, nan, 2.0], 0.6),
        ([0.0] * 16, 0.25),
        ([-0.0] * 7 + [0.0] * 9, 0.5),
        ([5.0], 0.1),
        ([2.0, -2.0], 0.5),
    ]
    for g, cr in fixed:
        cases.append((np.array(g, dtype=np.float64), cr, "fixed"))
    ratios = [0.001, 0.01, 0.1, 0.25, 0.3, 0.5, 0.9, 1.0]
    # hypothesis-style (test_comm.py:114-130): dim <= 2000, forced ties
    for i in range(48):
        dim = int(rng.integers(1, 2001))
        g = rng.normal(size=dim)
        if dim > 3:
            g[dim // 2] = g[0]
            g[dim // 3] = -g[0]
        cases.append((g, ratios[i % len(ratios)], "hypo"))
    # acceptance-style (test_acceptance.py:140-154): dim <= 1e4, ties at D/2, D/3, D-1
    for i in range(36):
        dim = int(rng.integers(1, 10001))
        g = rng.normal(size=dim)
        if i % 3 == 0 and dim >= 6:
            g[dim // 2] = g[0]
            g[dim // 3] = -g[0]
            g[dim - 1] = abs(g[0])
        cases.append((g, ratios[i % len(ratios)], "accept"))
    # float32-representable values (the fp32 throughput path's inputs), incl. tie stress
    for i in range(24):
        dim = int(rng.integers(1000, 16001))
        z = rng.normal(size=dim)
        fam = i % 3
        if fam == 0:
            g = z
        elif fam == 1:
            g = np.sign(z) * np.exp(1.5 * rng.normal(size=dim))
        else:
            g = np.round(z * 8) / 8
            g[dim // 2] = g[0]
            g[dim // 3] = -g[0]
            g[dim - 1] = abs(g[0])
        g = g.astype(np.float32).astype(np.float64)
        cases.append((g, ratios[i % len(ratios)], "f32"))
    out = {}
    meta = []
    for i, (g, cr, tag) in enumerate(cases):
        sp = R.comm.topk_sparsify(g, cr)
        out[f"g{i}"] = g
        out[f"idx{i}"] = sp.indices.astype(np.int64)
        out[f"val{i}"] = sp.values
        meta.append({"cr": cr, "tag": tag, "m": R.comm.topk_count(len(g), cr)})
    out["meta"] = np.array(json.dumps(meta))
    np.savez_compressed(OUT / "topk.npz", **out)


def gate_cases(R):
    out = {}
    streams_meta = []

    def record(name, stream, cr, delta, f=0.9, raw=False):
        st = R.comm.CompressionState(cr=cr, delta=delta, ewma_factor=f, raw_gate=raw)
        dec, rho, ef, et = [], [], [], []
        for g in stream:
            d = R.comm.compression_gate(g, st)
            dec.append(d.compressed)
            rho.append(d.ratio)
            ef.append(st.ewma_full)
            et.append(st.ewma_topk)
        out[f"{name}_stream"] = np.array(stream, dtype=np.float64)
        out[f"{name}_dec"] = np.array(dec, dtype=bool)
        out[f"{name}_rho"] = np.array(rho)
        out[f"{name}_ewma_full"] = np.array(ef)
        out[f"{name}_ewma_topk"] = np.array(et)
        streams_meta.append({"name": name, "cr": cr, "delta": delta, "ewma_factor": f, "raw_gate": raw,
                             "n_compressed": st.n_compressed, "n_uncompressed": st.n_uncompressed})

    # test_comm.py:136-162 single-shot known answers
    record("capture", [np.array([3.0, 4.0, 0.0, 0.0])], 0.5, 0.0)
    record("flat", [np.array([1.0, 1.0, 1.0, 1.0])], 0.25, 0.3)
    record("zero", [np.zeros(8)], 0.5, 0.0)
    # test_comm.py:174-183 replay stream
    rng = np.random.default_rng(5)
    s = [rng.normal(size=30) for _ in range(100)]
    for i in (0, 7, 20):
        v = np.zeros(30)
        v[:3] = rng.normal(size=3)
        s[i] = v
    record("replay", s, 0.1, 0.25)
    # test_comm.py:186-198 raw vs smoothed
    dense = np.ones(10)
    sv = np.zeros(10)
    sv[0] = 5.0
    record("smoothed", [dense, sv], 0.1, 0.05)
    record("raw", [dense, sv], 0.1, 0.05, raw=True)
    # test_acceptance.py:157-190 frozen stream, CNC monotone in delta
    rng = np.random.default_rng(66)
    fs = []
    for i in range(500):
        if i < 120:
            v = np.zeros(64)
            spots = rng.choice(64, size=7, replace=False)
            v[spots] = rng.integers(1, 4, size=7).astype(float)
        else:
            v = rng.integers(-3, 4, size=64).astype(float)
            if not np.any(v):
                v[0] = 1.0
        fs.append(v)
    for dl in (0.0, 0.1, 0.2, 0.3, 0.4, 1.0):
        record(f"frozen_{dl}", fs, 0.1, dl)
    # heavy-tailed float32-representable stream: mixed decisions at cr .01
    rng = np.random.default_rng(77)
    hs = [(np.sign(z) * np.exp(1.5 * rng.normal(size=z.size)) * (1 + 0.5 * np.sin(t))).astype(np.float32).astype(np.float64)
          for t, z in enumerate(rng.normal(size=(30, 4000)))]
    record("heavy", hs, 0.01, 0.3)
    out["meta"] = np.array(json.dumps(streams_meta))
    np.savez_compressed(OUT / "gate.npz", **out)


def aggregate_cases(R):
    out = {}
    meta = []
    rng = np.random.default_rng(88)

    def rec(name, payloads, weights):
        agg = R.comm.weighted_aggregate(payloads, weights)
        kinds = []
        for j, p in enumerate(payloads):
            if isinstance(p, R.comm.SparseGradient):
                out[f"{name}_p{j}_idx"] = p.indices
                out[f"{name}_p{j}_val"] = p.values
                kinds.append("sparse")
            else:
                out[f"{name}_p{j}"] = np.asarray(p, dtype=np.float64)
                kinds.append("dense")
        out[f"{name}_w"] = np.asarray(weights, dtype=np.float64)
        out[f"{name}_agg"] = agg
        meta.append({"name": name, "kinds": kinds, "dim": int(len(agg))})

    g5 = [rng.normal(size=32) for _ in range(5)]
    rec("uniform", g5, np.full(5, 0.2))
    rec("degenerate", [np.arange(4.0), np.ones(4)], [1.0, 0.0])
    rec("mixed", [rng.normal(size=50), R.comm.topk_sparsify(rng.normal(size=50), 0.2)], [0.6, 0.4])
    rec("rates4", [rng.normal(size=64) for _ in range(4)], R.comm.weights_from_rates([64, 40, 88, 64]))
    # 8 workers at the S1 rates (SURVEY §0 trap 1), mixed dense/sparse, signed zeros
    rates = R.streams.sample_rates(R.streams.RateDistribution("uniform", 38, 24), 8, R.config.derive_seed(0, "rates"))
    out["s1_rates"] = np.array(rates)
    ps = []
    for j in range(8):
        g = (rng.normal(size=3000) * (1 + 0.1 * j)).astype(np.float32).astype(np.float64)
        g[::97] = -0.0
        ps.append(R.comm.topk_sparsify(g, 0.01) if j % 3 else g)
    rec("s1_mixed", ps, R.comm.weights_from_rates(rates))
    ps = [R.comm.topk_sparsify(rng.normal(size=5000).astype(np.float32).astype(np.float64), 0.1) for _ in range(8)]
    rec("s1_sparse", ps, R.comm.weights_from_rates(rates))
    out["meta"] = np.array(json.dumps(meta))
    np.savez_compressed(OUT / "aggregate.npz", **out)


def sgd_cases(R):
    out = {}
    # test_nn.py:118-148 known answers, plus a multi-step random trajectory
    rng = np.random.default_rng(99)
    cases = [
        ("plain", np.array([1.0, -2.0]), [np.array([0.5, 0.25])], 0.0, 0.0, 0.1),
        ("fixed", np.array([3.0, 4.0]), [np.zeros(2)], 0.9, 0.0, 0.5),
        ("unrolled", np.array([1.0, -1.0, 0.5]), [np.array([0.3, 0.1, -0.2]), np.array([-0.1, 0.2, 0.4])], 0.9, 0.01, 0.2),
        ("random", rng.normal(size=4099), [rng.normal(size=4099) for _ in range(4)], 0.9, 1e-4, 0.037),
        ("signed_zero", np.array([0.0, -0.0, 1.0, -1.0]), [np.array([-0.0, -0.0, 0.0, -0.0])], 0.9, 0.0, 0.1),
    ]
    meta = []
    for name, p0, gs, mu, wd, lr in cases:
        st = R.nn.OptimizerState(momentum=mu, weight_decay=wd)
        p = p0.copy()
        out[f"{name}_p0"] = p0
        for t, g in enumerate(gs):
            R.nn.sgd_momentum_step(st, p, g, lr)
            out[f"{name}_g{t}"] = g
            out[f"{name}_p{t + 1}"] = p.copy()
            out[f"{name}_b{t + 1}"] = st.momentum_buffer.copy()
        meta.append({"name": name, "steps": len(gs), "momentum": mu, "weight_decay": wd, "lr": lr})
    out["meta"] = np.array(json.dumps(meta))
    np.savez_compressed(OUT / "sgd.npz", **out)


CONFIG1 = dict(
    n_devices=4,
    rate_dist=dict(kind="uniform", mean=38, std=24),
    dataset=dict(n_classes=10, feature_dim=16, samples_per_class=100, cluster_spread=0.5, seed=101),
    seed=1,
    mode="rate_matched",
    fixed_batch=64,
    retention="persistence",
    partition=dict(mode="iid", labels_per_device=1),
    model=dict(hidden=[32], augment_std=0.05),
    optimizer=dict(base_lr=0.2, momentum=0.9),
    compression=dict(enabled=True, cr=0.1, delta=0.5),
    injection=dict(enabled=False),
    cost=dict(c0=1.0, c1=0.001, link_latency=0.005, link_bandwidth=625e6),
    max_epochs=8,
)


def engine_cases(R):
    """Config-1 run of the reference loop (4 devices, heterogeneous rates, cr .1, delta .5):
    record every gate input/output, aggregate and post-step parameters, and metrics.csv."""
    cfg = R.config.parse_config(json.dumps(CONFIG1))
    (OUT / "config1.json").write_text(json.dumps(CONFIG1, indent=2) + "\n")
    sim = R.engine.Simulation(cfg)
    real = R.comm
    log = {"g": [], "dec": [], "rho": [], "agg": [], "w": [], "params": [], "lr": []}

    class Spy(types.ModuleType):
        def __getattr__(self, name):
            return getattr(real, name)

    spy = Spy("spy")

    def gate(g, state):
        d = real.compression_gate(g, state)
        log["g"].append(np.array(g, dtype=np.float64))
        log["dec"].append(d.compressed)
        log["rho"].append(d.ratio)
        return d

    def agg(payloads, weights):
        a = real.weighted_aggregate(payloads, weights)
        log["agg"].append(a.copy())
        log["w"].append(np.asarray(weights, dtype=np.float64))
        return a

    spy.compression_gate = gate
    spy.weighted_aggregate = agg
    R.engine.comm = spy
    try:
        rows = []
        for _ in range(12):
            row = sim.run_iteration()
            rows.append(row)
            log["params"].append(sim.replicas[0].flat.copy())
            log["lr"].append(row.lr_used)
    finally:
        R.engine.comm = real
    p0 = R.nn.init_model((16, 32, 10), R.config.derive_seed(1, "model_init")).flat
    np.savez_compressed(
        OUT / "engine_replay.npz",
        p0=p0,
        g=np.array(log["g"]).reshape(12, 4, -1),
        dec=np.array(log["dec"]).reshape(12, 4),
        rho=np.array(log["rho"]).reshape(12, 4),
        agg=np.array(log["agg"]),
        w=np.array(log["w"]),
        params=np.array(log["params"]),
        lr=np.array(log["lr"]),
        momentum=np.array(0.9),
        weight_decay=np.array(0.0),
    )
    # full-run metrics.csv (the byte-identity artefact of the drop-in)
    result = R.engine.run_experiment(R.config.parse_config(json.dumps(CONFIG1)))
    buf = io.StringIO()
    w = csv.writer(buf, lineterminator="\n")
    w.writerow(R.cli.metrics_columns(cfg.n_devices))
    for row in result.metrics:
        w.writerow(R.cli.metrics_row(row))
    (OUT / "config1_metrics.csv").write_text(buf.getvalue())


def sampler_cases(R):
    out = {}
    S = R.streams
    D = R.datagen
    # stream buffers: enqueue/draw/retain traces for both policies
    traces = []
    for policy in ("persistence", "truncation"):
        rng = np.random.default_rng(5 if policy == "persistence" else 6)
        for rate in (1, 7, 43, 300):
            buf = S.StreamBuffer(rate=rate, policy=policy)
            ops = []
            for _ in range(60):
                op = int(rng.integers(0, 3))
                if op == 0:
                    el = float(rng.choice([0.0, 1 / 3, 0.25, 0.1, 1.7, rng.uniform(0, 3)]))
                    ops.append(["enqueue", el, buf.enqueue_arrivals(el), len(buf)])
                elif op == 1:
                    b = int(rng.integers(1, 2 * rate + 2))
                    if len(buf) >= b:
                        ids = buf.draw_batch(b)
                        ops.append(["draw", b, ids[0], ids[-1], len(buf)])
                else:
                    ops.append(["retain", buf.apply_retention(), len(buf)])
            traces.append({"policy": policy, "rate": rate, "ops": ops})
    (OUT / "stream_traces.json").write_text(json.dumps(traces) + "\n")
    # injection plans and augmented batches
    inj = []
    for it, (alpha, beta) in enumerate([(0.5, 0.5), (0.25, 0.25), (0.1, 0.1), (0.05, 0.05), (1.0, 1.0)]):
        n = 8
        bs = [31, 30, 8, 30, 42, 66, 22, 14]
        cfg = D.InjectionConfig(alpha, beta, 3072)
        plan = D.injection_plan(n, cfg, bs, R.config.derive_seed(0, f"inject-plan:{it}"))
        batches = [list(range(100 * d, 100 * d + bs[d])) for d in range(n)]
        rng = np.random.default_rng(R.config.derive_seed(0, f"inject-draw:{it}"))
        aug, nbytes = D.inject(batches, plan, 3072, rng)
        inj.append({"alpha": alpha, "beta": beta, "it": it, "plan": plan, "batches": aug, "bytes": nbytes})
    (OUT / "injection.json").write_text(json.dumps(inj) + "\n")
    # partition pools and materialised batches on a CIFAR-like (small) dataset
    spec = D.DatasetSpec(n_classes=20, feature_dim=48, samples_per_class=50, cluster_spread=0.5, seed=3)
    ds = D.generate_dataset(spec)
    pools = D.partition(ds, D.PartitionPlan("noniid", 8, 5), R.config.derive_seed(0, "partition"))
    out["train_x"] = ds.train_x
    out["train_y"] = ds.train_y
    for d, p in enumerate(pools):
        out[f"pool{d}"] = p
    pools_iid = D.partition(ds, D.PartitionPlan("iid", 8, 1), R.config.derive_seed(0, "partition"))
    for d, p in enumerate(pools_iid):
        out[f"iidpool{d}"] = p
    augment = np.random.default_rng(R.config.derive_seed(0, "augment:0")).normal(0.0, 0.05, ds.train_x.shape)
    out["augment"] = augment
    rows = [int(pools[d][a % len(pools[d])]) for d in range(8) for a in range(57, 57 + 20)]
    out["rows"] = np.array(rows)
    out["x"] = ds.train_x[np.array(rows)] + augment[np.array(rows)]
    np.savez_compressed(OUT / "sampler.npz", **out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg/src")
    args = ap.parse_args()
    R = load_reference(args.ref)
    topk_cases(R)
    gate_cases(R)
    aggregate_cases(R)
    sgd_cases(R)
    engine_cases(R)
    sampler_cases(R)
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
