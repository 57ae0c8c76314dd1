"""deserialize() error taxonomy through the Python facade, mirroring the reference's
``pkg/tests/test_container.py:107-203`` (TestDeserializeErrors).

Every check below fires in the host-side header / pool-length parse, before any device work
(container.py:349-416 order), so these run without a GPU.  Streams come from the oracle
(the reference algorithm restated in C, pinned to the reference's own outputs)."""
import struct

import numpy as np
import pytest

import fields
import oracle
import paper_2201_13020_b200 as szx


@pytest.fixture
def blob():
    # the reference fixture: 3000 random-walk values, bs 64, rel 1e-4, non-empty pools
    x = fields.random_walk(np.random.default_rng(0xC0FFEE), 3000, step=0.5)
    b = oracle.compress(x, (3000,), 64, "rel", 1e-4)
    assert len(oracle.parse(b)["mid"]) > 0
    return b


def test_truncated_inside_every_host_checked_region(blob):
    # every prefix that ends before the mid pool is rejected on the host
    p = oracle.parse(blob)
    mid_start = len(blob) - len(p["mid"])
    for cut in range(mid_start):
        with pytest.raises(szx.TruncatedStreamError):
            szx.deserialize(blob[:cut])


def test_magic_flip(blob):
    with pytest.raises(szx.MalformedMagicError):
        szx.deserialize(b"VFZX" + blob[4:])


def test_version_mismatch(blob):
    with pytest.raises(szx.VersionMismatchError):
        szx.deserialize(blob[:4] + b"\x02" + blob[5:])


def test_f64_dtype_rejected(blob):
    with pytest.raises(szx.UnsupportedDtypeError):
        szx.deserialize(blob[:5] + b"\x01" + blob[6:])


def test_unknown_dtype_rejected(blob):
    with pytest.raises(szx.UnsupportedDtypeError):
        szx.deserialize(blob[:5] + b"\x07" + blob[6:])


def test_bad_block_size(blob):
    with pytest.raises(szx.InconsistentLengthError):
        szx.deserialize(blob[:6] + struct.pack("<H", 3) + blob[8:])


def test_bad_bound(blob):
    with pytest.raises(szx.InconsistentLengthError):
        szx.deserialize(blob[:8] + struct.pack("<d", -1.0) + blob[16:])
    with pytest.raises(szx.InconsistentLengthError):
        szx.deserialize(blob[:8] + struct.pack("<d", float("inf")) + blob[16:])


def test_zero_dim(blob):
    with pytest.raises(szx.InconsistentLengthError):
        szx.deserialize(blob[:17] + struct.pack("<Q", 0) + blob[25:])


def test_zero_ndims(blob):
    with pytest.raises(szx.InconsistentLengthError):
        szx.deserialize(blob[:16] + b"\x00" + blob[17:])


def test_req_len_out_of_range():
    x = fields.random_walk(np.random.default_rng(3), 256, step=1.0)
    b = bytearray(oracle.compress(x, (256,), 64, "rel", 1e-5))
    p = oracle.parse(bytes(b))
    assert len(p["req"]) > 0
    nb = p["nb"]
    off = 17 + 8 + -(-nb // 8) + 4 * nb
    for v in (0, 40):
        b[off] = v
        with pytest.raises(szx.InconsistentLengthError):
            szx.deserialize(bytes(b))


def test_nonzero_map_padding_rejected():
    # one constant block of 16: the map byte may only use bit 0
    b = bytearray(oracle.compress(np.full(16, 2.0, np.float32), (16,), 16, "abs", 1.0))
    b[17 + 8] |= 0x02
    with pytest.raises(szx.InconsistentLengthError):
        szx.deserialize(bytes(b))


def test_nonzero_code_padding_rejected():
    # three NC values at bs 8: 6 code bits used, 2 padding bits
    b = bytearray(oracle.compress(np.array([0.0, 1.0, 0.5], np.float32), (3,), 8, "abs", 1e-3))
    p = oracle.parse(bytes(b))
    assert p["m"] == 3
    b[len(b) - len(p["mid"]) - 1] |= 0xC0
    with pytest.raises(szx.InconsistentLengthError):
        szx.deserialize(bytes(b))


def test_errors_are_format_errors(blob):
    for bad in (b"VFZX" + blob[4:], blob[:4] + b"\x02" + blob[5:], blob[:10]):
        with pytest.raises(szx.FormatError):
            szx.deserialize(bad)
    assert issubclass(szx.FormatError, ValueError)
    assert issubclass(szx.PoolUnderrunError, szx.FormatError)
