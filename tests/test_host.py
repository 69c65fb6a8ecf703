"""CPU: host-side logic of the product package (no kernels): accounting, weights, link cost,
the contiguous-range StreamBuffer, rate sampling, injection planning and partitioning,
checked against the oracle and the reference golden traces."""

import json

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from conftest import GOLDEN
from oracle import comm_ref, streams_ref
from paper_2301_08897_b200 import comm, streams


@given(st.lists(st.integers(1, 10_000), min_size=1, max_size=64))
@settings(max_examples=200, deadline=None)
def test_weights_sum_to_one_and_match_oracle(rates):
    w = comm.weights_from_rates(rates)
    assert np.all(w >= 0) and abs(w.sum() - 1.0) <= 1e-12
    assert np.array_equal(w, comm_ref.rate_weights(rates))


def test_weights_use_rates_not_batch_sizes():
    """SURVEY §0 trap 1: device 2 has S=1 but b=8; its weight is 1/236."""
    rates = streams.sample_rates(streams.RateDistribution("uniform", 38, 24), 8, streams.derive_seed(0, "rates"))
    assert rates == [31, 30, 1, 30, 42, 66, 22, 14]
    w = comm.weights_from_rates(rates)
    assert w[2] == 1 / 236
    b = [streams.compute_batch_size("rate_matched", r, 8, 1024, 64) for r in rates]
    assert b[2] == 8


def test_volume_and_payload_accounting():
    s = comm.account_volume(False, 10**6, 0.1, comm.VolumeStats())
    assert (s.floats_sent, s.bytes_sent) == (10**6, 4 * 10**6)
    s = comm.account_volume(True, 10**6, 0.1, comm.VolumeStats())
    assert (s.floats_sent, s.bytes_sent) == (10**5, 8 * 10**5)
    assert comm.payload_bytes(False, 1000, 0.1) == 4000
    assert comm.payload_bytes(True, 1000, 0.1) == 800
    for c in (True, False):
        for D in (1, 874, 98_666, 60_192_808):
            assert (comm.payload_bytes(c, D, 0.01), comm.account_volume(c, D, 0.01, comm.VolumeStats()).floats_sent) == \
                (comm_ref.volume(c, D, 0.01)[1], comm_ref.volume(c, D, 0.01)[0])


def test_link_model():
    assert comm.comm_time(0, comm.LinkModel(0.01, 1e9), 8) == 0.01
    assert comm.comm_time(1e6, comm.LinkModel(0.0, 1e6), 10_000) == pytest.approx(2.0, rel=1e-3)
    with pytest.raises(ValueError):
        comm.LinkModel(-1, 1)
    with pytest.raises(ValueError):
        comm.comm_time(-1, comm.LinkModel(0, 1), 2)


def test_cnc_ratio():
    s = comm.CompressionState(cr=0.1, delta=0.1)
    s.n_compressed, s.n_uncompressed = 7, 3
    assert comm.cnc_ratio(s) == pytest.approx(0.7)


def test_range_stream_buffer_matches_reference_traces():
    traces = json.loads((GOLDEN / "stream_traces.json").read_text())
    for tr in traces:
        buf = streams.StreamBuffer(tr["rate"], tr["policy"])
        for op in tr["ops"]:
            if op[0] == "enqueue":
                assert buf.enqueue_arrivals(op[1]) == op[2]
                assert len(buf) == op[3]
            elif op[0] == "draw":
                ids = buf.draw_batch(op[1])
                assert (ids[0], ids[-1], len(buf)) == (op[2], op[3], op[4])
            else:
                assert buf.apply_retention() == op[1]
                assert len(buf) == op[2]


@given(st.integers(1, 500), st.lists(st.tuples(st.integers(0, 2), st.floats(0, 3), st.integers(1, 900)), max_size=80),
       st.sampled_from(["persistence", "truncation"]))
@settings(max_examples=200, deadline=None)
def test_range_buffer_equals_deque_buffer(rate, ops, policy):
    """The pending ids are always one contiguous range, so the range form is exact."""
    a, b = streams.StreamBuffer(rate, policy), streams_ref.DequeBuffer(rate, policy)
    for kind, el, n in ops:
        if kind == 0:
            assert a.enqueue_arrivals(el) == b.enqueue(el)
        elif kind == 1:
            if len(b) >= n:
                assert list(a.draw_batch(n)) == b.draw(n)
            else:
                with pytest.raises(streams.WouldBlock):
                    a.draw_batch(n)
        else:
            assert a.apply_retention() == b.retain()
        assert list(a.pending) == list(b.pending)
        assert a.fractional_credit == b.credit


def test_streaming_wait_and_batch_size():
    assert streams.streaming_wait(0, 64, 27) == pytest.approx(64 / 27)
    assert streams.streaming_wait(100, 64, 27) == 0.0
    assert streams.compute_batch_size("fixed_batch", 5, 8, 1024, 64) == 64
    assert streams.compute_batch_size("rate_matched", 5000, 8, 1024, 64) == 1024
    with pytest.raises(ValueError):
        streams.compute_batch_size("bogus", 5, 8, 1024, 64)


def test_injection_plan_and_picks_match_reference():
    inj = json.loads((GOLDEN / "injection.json").read_text())
    bs = [31, 30, 8, 30, 42, 66, 22, 14]
    for case in inj:
        plan = streams.injection_plan(8, case["alpha"], case["beta"], bs,
                                      streams.derive_seed(0, f"inject-plan:{case['it']}"))
        assert [list(p) for p in plan] == case["plan"]
        rng = np.random.default_rng(streams.derive_seed(0, f"inject-draw:{case['it']}"))
        picks = streams.injection_picks(plan, bs, rng)
        batches = [list(range(100 * d, 100 * d + bs[d])) for d in range(8)]
        # rebuild the augmented batches from the picks exactly as the device kernel does
        out = [list(b) for b in batches]
        for (s, c), pk in zip(plan, picks):
            for d in range(8):
                if d != s:
                    out[d].extend(batches[s][p] for p in pk)
        assert out == case["batches"]
        assert streams.injection_bytes(plan, 8, 3072) == case["bytes"]


def test_partition_matches_reference():
    z = np.load(GOLDEN / "sampler.npz")
    pools = streams.partition(z["train_y"], 8, "noniid", 5, streams.derive_seed(0, "partition"))
    for d in range(8):
        assert np.array_equal(pools[d], z[f"pool{d}"])
    pools = streams.partition(z["train_y"], 8, "iid", 1, streams.derive_seed(0, "partition"))
    for d in range(8):
        assert np.array_equal(pools[d], z[f"iidpool{d}"])
    with pytest.raises(ValueError):
        streams.partition(z["train_y"], 8, "noniid", 3, 0)


# -- a14: lr_at_epoch / scale_lr (reference nn.py:175-190; known answers from test_nn.py:160-183) ----


def test_scale_lr_known_answers_and_errors():
    from paper_2301_08897_b200 import nn

    assert nn.scale_lr(0.1, 1024, 1024) == 0.1
    assert nn.scale_lr(0.1, 2048, 1024) == pytest.approx(0.2)
    assert nn.scale_lr(0.01, 16 * 38, 1024) == pytest.approx(0.0059375)
    # the engine's rate_matched lr (engine.py:277-281): base 0.1, S1 rates, B = n*64
    assert nn.scale_lr(0.1, 236, 8 * 64) == 0.1 * 236 / 512
    with pytest.raises(ValueError, match="base global batch must be >= 1"):
        nn.scale_lr(0.1, 10, 0)
    with pytest.raises(ValueError, match="sum of rates must be >= 1"):
        nn.scale_lr(0.1, 0.5, 64)


def test_lr_at_epoch_step_decay_compounds():
    from paper_2301_08897_b200 import nn

    schedule = [(75, 0.2), (150, 0.2), (225, 0.2)]
    assert nn.lr_at_epoch(0.1, schedule, 10) == 0.1
    assert nn.lr_at_epoch(0.1, schedule, 75) == pytest.approx(0.02)
    assert nn.lr_at_epoch(0.1, schedule, 200) == pytest.approx(0.004)
    assert nn.lr_at_epoch(0.1, schedule, 300) == pytest.approx(0.0008)
    assert nn.lr_at_epoch(0.5, [], 1000) == 0.5


@pytest.mark.parametrize("epoch", [0, 1, 2, 3, 74, 75, 149, 150, 224, 225, 1000])
def test_lr_rules_bit_identical_to_reference(epoch):
    """Same floating-point operation order as the reference (the lr feeds metrics.csv's
    lr_used column, which must match byte for byte)."""
    ref = _reference_nn()
    from paper_2301_08897_b200 import nn

    for sched in ([], [(1, 0.5)], [(75, 0.2), (150, 0.2), (225, 0.2)], [(2, 0.1), (3, 0.3)]):
        for base in (0.1, 0.05, 0.3):
            assert nn.lr_at_epoch(base, sched, epoch).hex() == ref.lr_at_epoch(base, sched, epoch).hex()
            for s, b in ((204, 256), (236, 512), (1, 1), (9999, 64)):
                assert nn.scale_lr(base, s, b).hex() == ref.scale_lr(base, s, b).hex()


def _reference_nn():
    import sys

    from conftest import ROOT

    ref = ROOT / "baseline" / "_ref"
    if not (ref / "streamsgd" / "nn.py").exists():
        pytest.skip("reference not installed in baseline/_ref (tools/install_ref.py)")
    if str(ref) not in sys.path:
        sys.path.insert(0, str(ref))
    import streamsgd.nn as ref_nn

    return ref_nn
