"""CPU: pin the oracle (oracle/) against golden vectors produced by the reference itself.

tests/golden/make_golden.py ran streamsgd (the reference) to produce these fixtures; the
oracle is trusted as the GPU tests' checker only because these pass bit-for-bit.
"""

import json

import numpy as np
import pytest

from conftest import GOLDEN, load_npz
from oracle import comm_ref, streams_ref


def test_topk_lexsort_and_threshold_match_reference():
    z, meta = load_npz("topk")
    assert len(meta) >= 100
    for i, mt in enumerate(meta):
        g = z[f"g{i}"]
        want = z[f"idx{i}"]
        assert comm_ref.topk_count(len(g), mt["cr"]) == mt["m"]
        idx, vals = comm_ref.topk(g, mt["cr"], "lexsort")
        assert np.array_equal(idx, want), (i, mt)
        assert np.array_equal(vals.view(np.uint64), z[f"val{i}"].view(np.uint64))
        idx2, _ = comm_ref.topk(g, mt["cr"], "threshold")
        assert np.array_equal(idx2, want), (i, mt)


def test_threshold_method_matches_lexsort_random():
    """The O(D) oracle used at large D equals the lexsort form (SURVEY §8(c) validation)."""
    rng = np.random.default_rng(123)
    for t in range(300):
        D = int(rng.integers(1, 5000))
        kind = t % 5
        g = rng.normal(size=D)
        if kind == 1:
            g = np.round(g * 4) / 4
        elif kind == 2:
            g[rng.integers(0, D, max(1, D // 10))] = np.nan
        elif kind == 3:
            g[rng.integers(0, D, max(1, D // 10))] = rng.choice([np.inf, -np.inf, 0.0, -0.0])
        elif kind == 4:
            g = g.astype(np.float32).astype(np.float64)
        cr = float(rng.choice([0.001, 0.01, 0.1, 0.3, 0.5, 1.0]))
        m = comm_ref.topk_count(D, cr)
        assert np.array_equal(comm_ref.topk_indices_threshold(g, m), comm_ref.topk_indices_lexsort(g, m))


def test_topk_count_matches_exact_decimal():
    """comm.py:81-87 against the reference test oracle's exact-fraction count."""
    from fractions import Fraction
    import math

    for cr in ("0.001", "0.01", "0.1", "0.25", "0.3", "0.5", "0.9", "1.0"):
        for D in list(range(1, 3000)) + [60_192_808, 143_667_240, 10**9]:
            assert comm_ref.topk_count(D, float(cr)) == max(1, math.ceil(Fraction(cr) * D))


def test_gate_streams_match_reference_bitwise():
    z, meta = load_npz("gate")
    for mt in meta:
        name = mt["name"]
        st = comm_ref.GateState(mt["cr"], mt["delta"], mt["ewma_factor"], mt["raw_gate"])
        for t, g in enumerate(z[f"{name}_stream"]):
            c, _, rho, _, _ = comm_ref.gate(g, st)
            assert c == bool(z[f"{name}_dec"][t]), (name, t)
            assert rho == float(z[f"{name}_rho"][t]), (name, t)
            assert st.ewma_full == float(z[f"{name}_ewma_full"][t])
        assert (st.n_compressed, st.n_uncompressed) == (mt["n_compressed"], mt["n_uncompressed"])


def test_aggregate_matches_reference_bitwise():
    z, meta = load_npz("aggregate")
    for mt in meta:
        name = mt["name"]
        ps = []
        for j, kind in enumerate(mt["kinds"]):
            if kind == "sparse":
                ps.append((mt["dim"], z[f"{name}_p{j}_idx"], z[f"{name}_p{j}_val"]))
            else:
                ps.append(z[f"{name}_p{j}"])
        got = comm_ref.aggregate(ps, z[f"{name}_w"])
        assert np.array_equal(got.view(np.uint64), z[f"{name}_agg"].view(np.uint64)), name


def test_rate_weights_reference_examples():
    assert np.allclose(comm_ref.rate_weights([64, 40, 88, 64]), [0.25, 0.15625, 0.34375, 0.25], atol=1e-15)
    z, _ = load_npz("aggregate")
    assert z["s1_rates"].tolist() == [31, 30, 1, 30, 42, 66, 22, 14]
    with pytest.raises(ValueError):
        comm_ref.rate_weights([])


def test_sgd_matches_reference_bitwise():
    z, meta = load_npz("sgd")
    for mt in meta:
        name = mt["name"]
        p, b = z[f"{name}_p0"].copy(), None
        for t in range(mt["steps"]):
            p, b = comm_ref.sgd_momentum(p, b, z[f"{name}_g{t}"], mt["lr"], mt["momentum"], mt["weight_decay"])
            assert np.array_equal(p.view(np.uint64), z[f"{name}_p{t + 1}"].view(np.uint64)), (name, t)
            assert np.array_equal(b.view(np.uint64), z[f"{name}_b{t + 1}"].view(np.uint64))


def test_engine_replay_matches_reference():
    """Config-1 loop (4 devices, cr .1, delta .5): replaying the recorded gradients through the
    oracle reproduces the reference's decisions, aggregates and parameters bit-for-bit."""
    z = np.load(GOLDEN / "engine_replay.npz")
    cfg = json.loads((GOLDEN / "config1.json").read_text())
    cr, delta = cfg["compression"]["cr"], cfg["compression"]["delta"]
    states = [comm_ref.GateState(cr, delta) for _ in range(4)]
    p, b = z["p0"].copy(), None
    for it in range(z["g"].shape[0]):
        p, b, agg, dec = comm_ref.step_reference(list(z["g"][it]), states, z["w"][it], p, b, float(z["lr"][it]),
                                                 float(z["momentum"]), float(z["weight_decay"]))
        assert dec == z["dec"][it].tolist(), it
        assert np.array_equal(agg.view(np.uint64), z["agg"][it].view(np.uint64)), it
        assert np.array_equal(p.view(np.uint64), z["params"][it].view(np.uint64)), it


def test_stream_buffer_traces():
    traces = json.loads((GOLDEN / "stream_traces.json").read_text())
    for tr in traces:
        buf = streams_ref.DequeBuffer(tr["rate"], tr["policy"])
        for op in tr["ops"]:
            if op[0] == "enqueue":
                assert buf.enqueue(op[1]) == op[2]
                assert len(buf) == op[3]
            elif op[0] == "draw":
                ids = buf.draw(op[1])
                assert (ids[0], ids[-1], len(buf)) == (op[2], op[3], op[4])
            else:
                assert buf.retain() == op[1]
                assert len(buf) == op[2]


def test_injection_and_partition_match_reference():
    inj = json.loads((GOLDEN / "injection.json").read_text())
    for case in inj:
        bs = [31, 30, 8, 30, 42, 66, 22, 14]
        plan = streams_ref.injection_plan(8, case["alpha"], case["beta"], bs,
                                          streams_ref.derive_seed(0, f"inject-plan:{case['it']}"))
        assert [list(p) for p in plan] == case["plan"]
        batches = [list(range(100 * d, 100 * d + bs[d])) for d in range(8)]
        rng = np.random.default_rng(streams_ref.derive_seed(0, f"inject-draw:{case['it']}"))
        out, nbytes = streams_ref.inject(batches, plan, 3072, rng)
        assert out == case["batches"] and nbytes == case["bytes"]
    z = np.load(GOLDEN / "sampler.npz")
    pools = streams_ref.partition_noniid(z["train_y"], 8, 5, streams_ref.derive_seed(0, "partition"))
    for d in range(8):
        assert np.array_equal(pools[d], z[f"pool{d}"])
    pools = streams_ref.partition_iid(len(z["train_y"]), 8, streams_ref.derive_seed(0, "partition"))
    for d in range(8):
        assert np.array_equal(pools[d], z[f"iidpool{d}"])
    x, _ = streams_ref.materialize(z["train_x"], z["augment"], z["train_y"], z["rows"])
    assert np.array_equal(x.view(np.uint64), z["x"].view(np.uint64))


def test_sample_rates_s1():
    r = streams_ref.sample_rates("uniform", 38, 24, 8, streams_ref.derive_seed(0, "rates"))
    assert r == [31, 30, 1, 30, 42, 66, 22, 14]
    assert [streams_ref.batch_size("rate_matched", x, 8, 1024, 64) for x in r] == [31, 30, 8, 30, 42, 66, 22, 14]
