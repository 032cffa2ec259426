"""read_tensor_coo (io.cpp:49-84) through the C-ABI (octen_read_coo): the
format and every error message of the reference's reader.  CPU only (host
parsing; the device COO compression of the result is in test_gpu_coo.py)."""
import re

import numpy as np
import pytest

import paper_1807_01350_b200 as ob


def _write(tmp_path, text, name="t.coo"):
    p = tmp_path / name
    p.write_text(text)
    return str(p)


def test_read_round_trip(tmp_path):
    # write_tensor_coo's format (io.cpp:37-47): 1-based indices, %.17g values
    entries = [((0, 0, 0), 1.5), ((2, 1, 3), -0.25), ((4, 2, 1), 1e-300)]
    text = "3 5 3 4\n" + "".join("%d %d %d %.17g\n" % (i + 1, j + 1, k + 1, v) for (i, j, k), v in entries)
    sp = ob.SparseTensor.read(_write(tmp_path, text + "\n"))  # blank lines are skipped
    assert sp.shape == (5, 3, 4) and sp.nnz == 3
    assert sp.i.tolist() == [0, 2, 4] and sp.j.tolist() == [0, 1, 2] and sp.k.tolist() == [0, 3, 1]
    assert np.array_equal(sp.values, np.array([v for _, v in entries], dtype=np.float32))


@pytest.mark.parametrize("text,msg", [
    ("", "empty file"),
    ("1 5\n", "bad header"),
    ("x\n", "bad header"),
    ("3 5 3\n", "header lists fewer extents than the order"),
    ("3 5 3 4\n1 1 x 2.0\n", "malformed entry at line 2"),
    ("3 5 3 4\n1 1 1 1.0\n2 2 2\n", "missing value at line 3"),
    ("3 5 3 4\n6 1 1 1.0\n", "SparseTensor: index out of bounds"),
    ("3 5 3 4\n0 1 1 1.0\n", "SparseTensor: index out of bounds"),
    # std::istream does not parse "nan": the reference reports a missing value
    ("3 5 3 4\n1 1 1 nan\n", "missing value at line 2"),
])
def test_read_errors(tmp_path, text, msg):
    p = _write(tmp_path, text)
    with pytest.raises(ob.IoError, match=msg):
        ob.SparseTensor.read(p)
    if "SparseTensor" in msg or "line" in msg:
        with pytest.raises(ob.IoError, match="^'" + re.escape(p) + "': "):
            ob.SparseTensor.read(p)


def test_missing_file(tmp_path):
    with pytest.raises(ob.IoError, match="cannot open"):
        ob.SparseTensor.read(str(tmp_path / "nope.coo"))
