"""Full-coverage stream parity against the oracle for fields too large for one oracle call.

Blocks are independent once the absolute bound e is fixed (``prev`` restarts at every block,
``pipeline.py:108-111``), so the UFZX stream of a field is the
per-pool concatenation of the streams of its block-aligned windows.  ``check_stream`` walks
the WHOLE field in windows of a multiple of 8 blocks, compresses each window with the oracle
(multithreaded C restatement, test infrastructure), and compares every byte of every pool of
the device stream at the window's offsets -- offsets accumulated from the ORACLE's window
sizes, so a wrong device offset cannot cancel out.  Together with the header this is
byte equality of ``serialize(stream)`` with the oracle's stream, without ever holding the
whole oracle stream in host memory.  The reconstruction is compared window by window too.
"""
from __future__ import annotations

import hashlib
import os

import numpy as np

import oracle


def _threads() -> int:
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except Exception:
        return os.cpu_count() or 1


def check_stream(stream, x_dev, out_dev=None, window_blocks: int = 1 << 19, digest=False):
    """Assert byte equality of every pool of `stream` (device CompressedStream of the device
    float32 vector `x_dev`) with the oracle, and of `out_dev` (its reconstruction, optional)
    with the oracle's decode.  Returns stats (windows, max mid offset checked, sha256 of the
    oracle stream if `digest`)."""
    import torch

    bs = stream.block_size
    assert bs % 4 == 0 and window_blocks % 8 == 0
    e = stream.error_bound
    n, nb = stream.n_values, stream.n_blocks
    x = x_dev.reshape(-1)
    assert x.numel() == n
    pools = stream.device_pools
    head = oracle.header(stream.dims, bs, e)
    h = hashlib.sha256(head) if digest else None
    parts = {k: [] for k in ("map", "mu", "req", "codes", "mid")} if digest else None
    nc0 = m0 = mid0 = 0
    th = _threads()
    windows = 0
    max_mid_off = 0
    for b0 in range(0, nb, window_blocks):
        b1 = min(nb, b0 + window_blocks)
        v0, v1 = b0 * bs, min(n, b1 * bs)
        xw = x[v0:v1].cpu().numpy()
        p = oracle.compress_pools(xw, bs, e, nthreads=th)
        assert not p["bad_req"]
        got_map = pools["constant_map"][b0 // 8: (b1 + 7) // 8].cpu().numpy()
        assert np.array_equal(got_map, p["map"]), ("map", b0)
        got_mu = pools["mu"][b0:b1].view(torch.int32).cpu().numpy()
        assert np.array_equal(got_mu, p["mu"].view(np.int32)), ("mu", b0)
        assert m0 % 4 == 0
        got_req = pools["req"][nc0: nc0 + p["n_nc"]].cpu().numpy()
        assert np.array_equal(got_req, p["req"]), ("req", b0)
        got_codes = pools["codes"][m0 // 4: m0 // 4 + p["codes"].size].cpu().numpy()
        assert np.array_equal(got_codes, p["codes"]), ("codes", b0)
        got_mid = pools["mid"][mid0: mid0 + p["mid_len"]].cpu().numpy()
        assert got_mid.size == p["mid_len"] and np.array_equal(got_mid, p["mid"]), ("mid", b0, mid0)
        if out_dev is not None:
            blob = oracle.serialize((v1 - v0,), bs, e, p)
            ref = oracle.decompress(blob, nthreads=th)
            got = out_dev.reshape(-1)[v0:v1].view(torch.int32).cpu().numpy()
            assert np.array_equal(got, ref.view(np.int32)), ("recon", b0)
        if digest:
            for k in parts:
                parts[k].append(p[k].tobytes() if k != "mu" else p["mu"].astype("<f4").tobytes())
        max_mid_off = max(max_mid_off, mid0 + p["mid_len"])
        nc0 += p["n_nc"]
        m0 += p["m"]
        mid0 += p["mid_len"]
        windows += 1
    assert (nc0, m0, mid0) == (stream.n_nonconstant_blocks, stream.n_nonconstant_elements,
                               stream.mid_len)
    sha = None
    if digest:
        for k in ("map", "mu", "req", "codes", "mid"):
            for b in parts[k]:
                h.update(b)
        sha = h.hexdigest()
    return {"windows": windows, "mid_end": max_mid_off, "oracle_sha256": sha}
