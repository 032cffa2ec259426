"""OCTS checkpoint container (checkpoint.cpp:125-295) in the oracle: the
reference's own tests (test_streaming.cpp:205-247) restated -- save/load/save
byte identity, resumed == straight-through, corruption detection, init-only
round trip -- plus the container layout the device must reproduce.  CPU."""
import struct

import numpy as np
import pytest

from oracle import octen_oracle as O
from oracle import rng


def _stream(seed=71):
    s = rng.Substream(seed)
    truth = O.KruskalModel([s.fill_uniform(d, 2) for d in (9, 8, 10)], np.ones(2))
    full = O.reconstruct_fast(truth)
    cfg = O.StreamConfig(rank=2, p=3, q=6, shared=2, seed=53, als=O.AlsConfig(2, 100, 1e-8, 3, 0))
    return full, O.init_stream(O.slice_mode(full, 2, 0, 5), cfg)


def test_crc64_ecma_reflected_check_value():
    # CRC-64/XZ (ECMA-182 polynomial, reflected, init/xorout ~0) check value
    assert O._crc64(b"123456789") == 0x995DC9BBDF1939FA


def test_save_load_save_byte_identical():
    _, st = _stream()
    b = O.checkpoint_save(st)
    assert b[:4] == b"OCTS" and struct.unpack("<I", b[4:8])[0] == 1
    assert struct.unpack("<Q", b[8:16])[0] == len(b) - 24
    assert O.checkpoint_save(O.checkpoint_load(b)) == b


def test_resumed_equals_straight_through():
    import copy
    full, st = _stream()
    straight = copy.deepcopy(st)
    O.ingest_batch(straight, O.slice_mode(full, 2, 5, 5))
    resumed = O.checkpoint_load(O.checkpoint_save(st))
    O.ingest_batch(resumed, O.slice_mode(full, 2, 5, 5))
    # the reference compares bytes (Eigen is layout-deterministic); numpy's
    # BLAS paths depend on the arrays' memory order, which a load changes,
    # so the port matches to rounding (the device tests check the bytes)
    for a, b in zip(straight.summaries.y + straight.summaries.history + straight.model.factors,
                    resumed.summaries.y + resumed.summaries.history + resumed.model.factors):
        assert np.allclose(a, b, rtol=1e-9, atol=1e-11)
    assert len(O.checkpoint_save(straight)) == len(O.checkpoint_save(resumed))


def test_corruption_detected():
    _, st = _stream()
    b = O.checkpoint_save(st)
    with pytest.raises(O.IoError, match="payload length mismatch"):
        O.checkpoint_load(b[:-7])
    flipped = bytearray(b)
    flipped[len(b) // 2] ^= 0x40
    with pytest.raises(O.IoError, match="checksum mismatch"):
        O.checkpoint_load(bytes(flipped))
    wrong = bytearray(b)
    wrong[4] = 0x7F
    with pytest.raises(O.IoError, match="unsupported format version 127"):
        O.checkpoint_load(bytes(wrong))
    bad = bytearray(b)
    bad[0] = ord("X")
    with pytest.raises(O.IoError, match="bad magic"):
        O.checkpoint_load(bytes(bad))


def test_init_only_round_trip():
    _, st = _stream()
    back = O.checkpoint_load(O.checkpoint_save(st))
    assert back.slices_seen == st.slices_seen
    assert np.array_equal(back.model.factors[0], st.model.factors[0])
    assert back.config.seed == st.config.seed
