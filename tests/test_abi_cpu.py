"""CPU-side checks of the C ABI (no kernel launches): the library loads, exports every
symbol include/szx_b200.h declares, and its host-side container parsing rejects malformed
streams with the reference's error taxonomy before any device work."""
import ctypes
import struct

import numpy as np
import pytest

import oracle
from conftest import golden_cases
from paper_2201_13020_b200 import _abi


@pytest.fixture(scope="module")
def L():
    return _abi.lib()


def test_exports_every_declared_symbol(L):
    names = _abi.declared_symbols()
    assert len(names) >= 18
    for name in names:
        assert hasattr(L, name), name
    assert set(names) <= set(_abi._SIGS), set(names) - set(_abi._SIGS)


def test_built_for_sm100a():
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _abi.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version(L):
    assert b"sm_100a" in L.szx_version()


def test_bound_exponent_matches_oracle(L):
    rng = np.random.default_rng(1)
    for e in np.concatenate([10.0 ** rng.uniform(-300, 300, 500), [1.0, 0.5, 2.0 ** -1074]]):
        assert L.szx_bound_exponent(float(e)) == oracle.bound_exponent(float(e))


def test_sizes(L):
    assert L.szx_num_blocks(300, 128) == 3
    assert L.szx_map_bytes(1, 128) == 4
    assert L.szx_codes_capacity(1) >= 1
    g = golden_cases()
    for k in range(len(g)):
        m, x, blob, _ = g.case(k)
        bound = L.szx_compress_bound(x.size, len(m["dims"]), m["block_size"])
        assert len(blob) <= bound


def _info(L, blob):
    n = ctypes.c_uint64()
    nd = ctypes.c_uint32()
    dims = (ctypes.c_uint64 * 8)()
    bs = ctypes.c_uint32()
    e = ctypes.c_double()
    buf = ctypes.create_string_buffer(blob, len(blob))
    rc = L.szx_stream_info(buf, len(blob), ctypes.byref(n), ctypes.byref(nd), dims, 8,
                           ctypes.byref(bs), ctypes.byref(e))
    return rc, n.value, list(dims)[: nd.value], bs.value, e.value


def test_stream_info_on_golden(L):
    g = golden_cases()
    for k in range(0, len(g), 7):
        m, x, blob, _ = g.case(k)
        rc, n, dims, bs, e = _info(L, blob)
        assert rc == 0
        assert n == x.size and dims == m["dims"] and bs == m["block_size"]
        assert e == struct.unpack_from("<d", blob, 8)[0]


def _dec(L, blob):
    out = np.empty(max(1, 1 << 16), np.float32)
    buf = ctypes.create_string_buffer(bytes(blob), len(blob))
    return L.szx_decompress_host(buf, len(blob), out.ctypes.data_as(ctypes.c_void_p), out.size)


@pytest.fixture
def blob():
    # a reference stream with every pool non-empty (reference test_container.py:108-113)
    g = golden_cases()
    for k in range(len(g)):
        m, x, b, _ = g.case(k)
        p = oracle.parse(b)
        if p["n_nc"] and len(p["mid"]) and 1000 < x.size < 5000 and p["m"] % 4:
            return b
    raise AssertionError("no suitable golden stream")


def test_header_errors_map_to_reference_classes(L, blob):
    assert _dec(L, b"VFZX" + blob[4:]) == _abi.ERR_MAGIC
    assert _dec(L, blob[:4] + b"\x02" + blob[5:]) == _abi.ERR_VERSION
    assert _dec(L, blob[:5] + b"\x01" + blob[6:]) == _abi.ERR_DTYPE
    assert _dec(L, blob[:5] + b"\x07" + blob[6:]) == _abi.ERR_DTYPE
    assert _dec(L, blob[:6] + struct.pack("<H", 3) + blob[8:]) == _abi.ERR_INCONSISTENT
    assert _dec(L, blob[:8] + struct.pack("<d", -1.0) + blob[16:]) == _abi.ERR_INCONSISTENT
    assert _dec(L, blob[:17] + struct.pack("<Q", 0) + blob[25:]) == _abi.ERR_INCONSISTENT
    assert _dec(L, blob[:16] + b"\x00" + blob[17:]) == _abi.ERR_INCONSISTENT


def test_truncation_before_mid_pool(L, blob):
    p = oracle.parse(blob)
    o_mid = len(blob) - len(p["mid"])
    for cut in range(o_mid):
        assert _dec(L, blob[:cut]) == _abi.ERR_TRUNCATED, cut


def test_padding_and_req_checks(L, blob):
    p = oracle.parse(blob)
    hdr = 17 + 8 * len(p["dims"])
    o_req = hdr + (p["nb"] + 7) // 8 + 4 * p["nb"]
    bad = bytearray(blob)
    bad[o_req] = 0
    assert _dec(L, bytes(bad)) == _abi.ERR_INCONSISTENT
    bad[o_req] = 40
    assert _dec(L, bytes(bad)) == _abi.ERR_INCONSISTENT
    o_mid = len(blob) - len(p["mid"])
    bad = bytearray(blob)
    bad[o_mid - 1] |= 0xC0  # m % 4 != 0: top code bits are padding
    assert _dec(L, bytes(bad)) == _abi.ERR_INCONSISTENT
    if p["nb"] % 8:
        bad = bytearray(blob)
        bad[hdr + (p["nb"] + 7) // 8 - 1] |= 0x80
        assert _dec(L, bytes(bad)) == _abi.ERR_INCONSISTENT


def test_no_cpu_path(L, blob):
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    assert _dec(L, blob) == _abi.ERR_NO_DEVICE
    x = np.ones(16, np.float32)
    dims = (ctypes.c_uint64 * 1)(16)
    out = np.empty(1024, np.uint8)
    olen = ctypes.c_uint64()
    rc = L.szx_compress_host(x.ctypes.data_as(ctypes.c_void_p), dims, 1, 128, 0, 0.1,
                             out.ctypes.data_as(ctypes.c_void_p), out.size, ctypes.byref(olen))
    assert rc == _abi.ERR_NO_DEVICE


def test_compress_host_argument_errors(L):
    x = np.ones(16, np.float32)
    out = np.empty(1024, np.uint8)
    olen = ctypes.c_uint64()
    P = lambda a: a.ctypes.data_as(ctypes.c_void_p)
    dims = (ctypes.c_uint64 * 1)(16)
    assert L.szx_compress_host(P(x), dims, 1, 7, 0, 0.1, P(out), 1024, ctypes.byref(olen)) == 1
    assert L.szx_compress_host(P(x), dims, 1, 65536, 0, 0.1, P(out), 1024, ctypes.byref(olen)) == 1
    assert L.szx_compress_host(P(x), dims, 1, 128, 0, 0.0, P(out), 1024, ctypes.byref(olen)) == 1
    assert L.szx_compress_host(P(x), dims, 1, 128, 2, 0.1, P(out), 1024, ctypes.byref(olen)) == 1
    zero = (ctypes.c_uint64 * 1)(0)
    assert L.szx_compress_host(P(x), zero, 1, 128, 0, 0.1, P(out), 1024, ctypes.byref(olen)) == 1


def test_host_pipeline_setting(L):
    """szx_set_host_pipeline: parts 1..32 set the decompress chunking (returns the previous
    value), anything else only queries it; no device is touched."""
    old = L.szx_set_host_pipeline(0, 0)
    try:
        assert 1 <= old <= 32
        assert L.szx_set_host_pipeline(16, 0) == old
        assert L.szx_set_host_pipeline(0, 0) == 16
        assert L.szx_set_host_pipeline(33, 0) == 16
        assert L.szx_set_host_pipeline(-1, 0) == 16
        assert L.szx_set_host_pipeline(1, 0) == 16
    finally:
        L.szx_set_host_pipeline(old, 0)
    assert L.szx_set_host_pipeline(0, 0) == old


def test_bench_host_launch_count(L):
    """bench.py's gpu_launches claim for one host round trip on the NYX field: K0, one K1,
    K3 over the first chunk, K3, the plan kernel and one K2 per decode chunk."""
    import importlib.util
    import os

    spec = importlib.util.spec_from_file_location(
        "bench", os.path.join(os.path.dirname(__file__), "..", "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    old = L.szx_set_host_pipeline(8, 0)
    try:
        assert bench.host_launches(L, 512 ** 3, 128) == 1 + 1 + 1 + 1 + 1 + 8
        assert bench.host_launches(L, 8192, 128) == 1 + 1 + 0 + 1 + 1 + 1  # one tile: no prefix
    finally:
        L.szx_set_host_pipeline(old, 0)
