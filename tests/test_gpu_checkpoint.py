"""OCTS checkpoints of the device-resident stream: the
reference's checkpoint tests (test_streaming.cpp:188-247) on the device path
-- byte-identical save/load/save, resumed ingest == straight-through ingest
(byte-identical checkpoints), corruption detection, run-to-run determinism
(the schedule-independence contract) -- and container compatibility with the
oracle's restatement of checkpoint.cpp in both directions."""
import numpy as np
import pytest

from oracle import octen_oracle as O
from oracle import rng

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ob():
    import torch
    assert torch.cuda.is_available()
    import paper_1807_01350_b200 as m
    return m


def _full(seed=71, dims=(9, 8, 10), rank=2):
    s = rng.Substream(seed)
    truth = O.KruskalModel([s.fill_uniform(d, rank) for d in dims], np.ones(rank))
    return O.reconstruct_fast(truth)


def _cfg(ob):
    return ob.StreamConfig(rank=2, p=3, q=6, shared=2, seed=53, als=ob.AlsConfig(rank=2, max_iters=100))


def test_save_load_save_byte_identical(ob):
    full = _full()
    st = ob.init_stream(O.slice_mode(full, 2, 0, 5), _cfg(ob))
    b = st.checkpoint_save()
    assert ob.checkpoint_load(b).checkpoint_save() == b


def test_resumed_equals_straight_through(ob):
    full = _full()
    st = ob.init_stream(O.slice_mode(full, 2, 0, 5), _cfg(ob))
    resumed = ob.checkpoint_load(st.checkpoint_save())
    ob.ingest_batch(st, O.slice_mode(full, 2, 5, 5))
    ob.ingest_batch(resumed, O.slice_mode(full, 2, 5, 5))
    assert st.checkpoint_save() == resumed.checkpoint_save()


def test_runs_are_deterministic(ob):
    # test_streaming.cpp:188-203: byte-identical checkpoints of two runs
    full = _full(61, (12, 11, 12), 3)
    cfg = ob.StreamConfig(rank=3, p=5, q=8, shared=3, seed=43, als=ob.AlsConfig(rank=3, max_iters=100))
    a = ob.init_stream(O.slice_mode(full, 2, 0, 6), cfg)
    b = ob.init_stream(O.slice_mode(full, 2, 0, 6), cfg)
    ob.ingest_batch(a, O.slice_mode(full, 2, 6, 6))
    b.ingest_async(O.slice_mode(full, 2, 6, 6))
    assert a.checkpoint_save() == b.checkpoint_save()


def test_corruption_detected(ob):
    full = _full()
    b = ob.init_stream(O.slice_mode(full, 2, 0, 5), _cfg(ob)).checkpoint_save()
    with pytest.raises(ob.IoError, match="payload length mismatch"):
        ob.checkpoint_load(b[:-7])
    flipped = bytearray(b)
    flipped[len(b) // 2] ^= 0x40
    with pytest.raises(ob.IoError, match="checksum mismatch"):
        ob.checkpoint_load(bytes(flipped))
    wrong = bytearray(b)
    wrong[4] = 0x7F
    with pytest.raises(ob.IoError, match="unsupported format version 127"):
        ob.checkpoint_load(bytes(wrong))
    bad = bytearray(b)
    bad[0] = ord("X")
    with pytest.raises(ob.IoError, match="bad magic"):
        ob.checkpoint_load(bytes(bad))


def test_container_compatible_with_the_reference_layout(ob):
    # the oracle (restating checkpoint.cpp) parses the device's container and
    # re-serializes it to the same bytes; the device loads the oracle's
    # container of the oracle's own stream and continues it like the oracle
    full = _full(81, (14, 13, 16), 2)
    st = ob.init_stream(O.slice_mode(full, 2, 0, 8), _cfg(ob))
    ob.ingest_batch(st, O.slice_mode(full, 2, 8, 4))
    b = st.checkpoint_save()
    parsed = O.checkpoint_load(b)
    assert O.checkpoint_save(parsed) == b
    assert parsed.slices_seen == 12 and parsed.summaries.batches_seen == 2 and len(parsed.log) == 2
    m = st.model
    for f, g in zip(m.factors, parsed.model.factors):
        assert np.array_equal(f, g)

    ocfg = O.StreamConfig(rank=2, p=3, q=6, shared=2, seed=53, als=O.AlsConfig(2, 100, 1e-8, 3, 0))
    ref = O.init_stream(O.slice_mode(full, 2, 0, 8), ocfg)
    O.ingest_batch(ref, O.slice_mode(full, 2, 8, 4))
    dev = ob.checkpoint_load(O.checkpoint_save(ref))
    O.ingest_batch(ref, O.slice_mode(full, 2, 12, 4))
    ob.ingest_batch(dev, O.slice_mode(full, 2, 12, 4))
    md = dev.model
    assert min(O.congruence(O.KruskalModel(md.factors, md.lambda_), ref.model)) > 1 - 1e-8
    assert dev.slices_seen == 16 and dev.batches_seen == 3
