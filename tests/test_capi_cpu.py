"""The C-ABI library builds, loads on a CPU-only machine and exports every
symbol include/octen_b200.h declares (no compute calls: no GPU here)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "octen_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(octen_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib_path():
    from paper_1807_01350_b200 import build
    return build.build(verbose=False)


def test_header_declares_the_boundary():
    fns = declared_functions()
    for f in ("octen_stream_init", "octen_stream_ingest", "octen_compress", "octen_cp_als_batched",
              "octen_align_replicas", "octen_recover_nontemporal", "octen_temporal_stack_from_summaries",
              "octen_recover_temporal_append", "octen_last_error"):
        assert f in fns


def test_library_exports_every_declared_symbol(lib_path):
    out = subprocess.run(["nm", "-D", "--defined-only", lib_path], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (octen_[a-z_0-9]+)$", out, flags=re.M))
    missing = [f for f in declared_functions() if f not in exported]
    assert not missing, missing


def test_library_loads_and_binds_on_cpu(lib_path):
    from paper_1807_01350_b200 import _capi
    assert set(_capi.SIGNATURES) == set(declared_functions())
    lib = _capi.load(lib_path)
    assert b"sm_100a" in lib.octen_version()
    assert lib.octen_last_error() == b""


def test_kernels_are_sm100a_cubins(lib_path):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib_path], capture_output=True, text=True,
                         check=True).stdout
    assert "sm_100a" in out


def test_python_api_surface():
    import paper_1807_01350_b200 as ob
    for name in ("init_stream", "ingest_batch", "compress", "cp_als_batched", "align_replicas",
                 "recover_nontemporal", "temporal_stack_from_summaries", "recover_temporal_append",
                 "StreamConfig", "AlsConfig", "ConfigError", "NumericError"):
        assert hasattr(ob, name)
    cfg = ob.StreamConfig(rank=4, p=6, q=15, shared=3, seed=17)
    c = cfg._c()
    assert (c.rank, c.p, c.q, c.shared, c.temporal_mode) == (4, 6, 15, 3, -1)
