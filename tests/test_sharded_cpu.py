"""Host logic of the multi-GPU path on CPU: shard plans, single-stream offsets, and a
world-size-2 gloo run of the size all-gather + range all-reduce + pool assembly.

Per-shard pools come from the oracle (test infrastructure) compressing each block-aligned shard
with the global absolute bound -- by block independence they are byte ranges of the
single-stream pools; the assembled file must equal the reference's stream."""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch.multiprocessing as mp

import fields
import oracle
from paper_2201_13020_b200 import sharded


def test_shard_plan_alignment_and_coverage():
    for n, bs, world in [(1, 128, 2), (1000, 128, 2), (25_000_000, 128, 8), (280_953_867, 128, 8),
                         (4096 * 8 + 17, 17, 3), (12345, 8, 4)]:
        plan = sharded.shard_plan(n, bs, world)
        assert len(plan) == world
        assert plan[0][0] == 0 and plan[-1][1] == n
        for (a0, a1), (b0, _) in zip(plan, plan[1:]):
            assert a1 == b0
        for v0, v1 in plan[:-1]:
            if v1 > v0 and v1 < n:
                assert (v1 - v0) % (8 * bs) == 0


def _pools_for(values, bs, e):
    p = oracle.compress_pools(values, bs, e)
    return p, sharded.ShardSizes(int(p["nb"]), int(p["n_nc"]), int(p["m"]), int(p["mid_len"]))


def test_offsets_reassemble_stream_serially():
    rng = np.random.default_rng(4)
    x = fields.smooth_ridges(rng, 8 * 128 * 37 + 11)
    e = oracle.resolve_bound(x, "rel", 1e-3)
    blob = oracle.compress(x, None, 128, "abs", e)
    for world in (1, 2, 3, 5):
        plan = sharded.shard_plan(x.size, 128, world)
        parts = [_pools_for(x[v0:v1], 128, e) if v1 > v0 else (None, sharded.ShardSizes(0, 0, 0, 0))
                 for v0, v1 in plan]
        sizes = [s for _, s in parts]
        out = bytearray(sharded.shard_offsets(sizes, 0, 1).total_len)
        head = sharded.header_bytes((x.size,), 128, e)
        out[: len(head)] = head
        for r, (p, _) in enumerate(parts):
            if p is None:
                continue
            off = sharded.shard_offsets(sizes, r, 1)
            for key, pos in (("map", off.map_off), ("mu", off.mu_off), ("req", off.req_off),
                             ("codes", off.codes_off), ("mid", off.mid_off)):
                b = np.ascontiguousarray(p[key]).view(np.uint8).tobytes()
                out[pos: pos + len(b)] = b
        assert bytes(out) == blob, world


def test_offsets_reject_misaligned_code_pools():
    sizes = [sharded.ShardSizes(8, 8, 17 * 8 - 3, 10), sharded.ShardSizes(8, 8, 17 * 8, 10)]
    with pytest.raises(ValueError):
        sharded.shard_offsets(sizes, 1, 1)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, path, x, bs, rel, result_q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        v0, v1 = sharded.shard_plan(x.size, bs, world)[rank]
        local = x[v0:v1]
        lo, hi = (float(local.min()), float(local.max())) if local.size else (np.inf, -np.inf)
        gmin, gmax, bad = sharded.global_range(lo, hi, False)
        e = rel * (gmax - gmin)
        if local.size:
            p, size = _pools_for(local, bs, e)
        else:
            p, size = ({k: np.zeros(0, np.uint8) for k in ("map", "mu", "req", "codes", "mid")},
                       sharded.ShardSizes(0, 0, 0, 0))
        sizes = sharded.gather_sizes(size)
        off = sharded.shard_offsets(sizes, rank, 1)
        pools = {"constant_map": p["map"], "mu": p["mu"], "req": p["req"], "codes": p["codes"],
                 "mid": p["mid"]}
        sharded.write_pools(path, off, sharded.header_bytes((x.size,), bs, e), pools, rank)
        dist.barrier()
        if rank == 0:
            result_q.put((e, off.total_len))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_two_ranks_assemble_one_stream(world):
    rng = np.random.default_rng(9)
    x = fields.random_walk(rng, 128 * 8 * 50 + 77, step=0.05)
    bs, rel = 128, 1e-3
    blob = oracle.compress(x, None, bs, "rel", rel)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "stream.ufzx")
        mp.start_processes(_worker, args=(world, port, path, x, bs, rel, q), nprocs=world,
                           join=True, start_method="spawn")
        e, total = q.get(timeout=30)
        with open(path, "rb") as f:
            got = f.read()
    assert total == len(blob)
    assert got == blob


# ---- sharded decompression: shard pool location + the mid-total all-gather ----------------
def _decode_shard_with_oracle(blob, rank, world, group_mid):
    """One rank's decode of its shard of `blob`: pools located by read_shard, the shard's mid
    total from the oracle's restatement of expected_mid_bytes (the device does this with K3),
    its mid offset from `group_mid` (the all-gather), the decode by the oracle."""
    import ctypes

    sp = sharded.read_shard(blob, rank, world)
    n_local = sp.v1 - sp.v0
    req = np.frombuffer(blob[sp.req_range[0]: sum(sp.req_range)], np.uint8).copy()
    codes = np.frombuffer(blob[sp.codes_range[0]: sum(sp.codes_range)], np.uint8).copy()
    mu = np.frombuffer(blob[sp.mu_range[0]: sum(sp.mu_range)], "<f4").astype(np.float32)
    cmap = sp.map_bytes.copy()
    P = lambda a: a.ctypes.data_as(ctypes.c_void_p)
    local_mid = int(oracle.lib().szxo_expected_mid(P(cmap), P(req), P(codes), n_local,
                                                   sp.block_size)) if n_local else 0
    before, total = group_mid(local_mid)
    sharded.check_mid_total(sp, total)
    mid = np.frombuffer(blob[sp.mid0 + before: sp.mid0 + before + local_mid], np.uint8).copy()
    if not n_local:
        return sp, np.zeros(0, np.float32)
    pools = {"map": cmap, "mu": mu, "req": req, "codes": codes, "mid": mid}
    shard_blob = oracle.serialize((n_local,), sp.block_size, sp.error_bound, pools)
    return sp, oracle.decompress(shard_blob)


def test_read_shard_ranges_serially():
    """Every rank's pool ranges, mid total and decode, with the all-gather done by hand."""
    import ctypes

    rng = np.random.default_rng(12)
    x = fields.smooth_ridges(rng, 128 * 8 * 41 + 5)
    P = lambda a: a.ctypes.data_as(ctypes.c_void_p)
    for bs in (128, 64, 32):
        blob = oracle.compress(x, None, bs, "rel", 1e-4)
        ref = oracle.decompress(blob)
        for world in (1, 2, 3, 7):
            totals = []
            for r in range(world):  # what each rank contributes to the all-gather
                sp = sharded.read_shard(blob, r, world)
                n_local = sp.v1 - sp.v0
                req = np.frombuffer(blob[sp.req_range[0]: sum(sp.req_range)], np.uint8).copy()
                codes = np.frombuffer(blob[sp.codes_range[0]: sum(sp.codes_range)], np.uint8).copy()
                cmap = sp.map_bytes.copy()
                totals.append(int(oracle.lib().szxo_expected_mid(P(cmap), P(req), P(codes),
                                                                n_local, bs)) if n_local else 0)
            outs = []
            for r in range(world):
                before, total = sum(totals[:r]), sum(totals)
                sp, out = _decode_shard_with_oracle(blob, r, world, lambda _l: (before, total))
                assert np.array_equal(out.view(np.uint32), ref[sp.v0: sp.v1].view(np.uint32)), \
                    (bs, world, r)
                outs.append(out)
            assert np.array_equal(np.concatenate(outs).view(np.uint32), ref.view(np.uint32))


def test_read_shard_rejects_like_deserialize():
    from paper_2201_13020_b200 import errors

    x = fields.random_walk(np.random.default_rng(3), 5000, step=0.5)
    blob = oracle.compress(x, None, 128, "rel", 1e-4)
    with pytest.raises(errors.MalformedMagicError):
        sharded.read_shard(b"VFZX" + blob[4:], 0, 2)
    with pytest.raises(errors.TruncatedStreamError):
        sharded.read_shard(blob[:30], 0, 2)
    sp = sharded.read_shard(blob, 0, 2)
    with pytest.raises(errors.TruncatedStreamError):
        sharded.check_mid_total(sp, sp.total_len - sp.mid0 + 1)
    with pytest.raises(errors.InconsistentLengthError):
        sharded.check_mid_total(sp, sp.total_len - sp.mid0 - 1)


def _dec_worker(rank, world, port, blob, result_q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sp, out = _decode_shard_with_oracle(blob, rank, world,
                                            lambda local: sharded.mid_offsets(local))
        result_q.put((rank, sp.v0, sp.v1, out.tobytes()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_two_ranks_decode_one_stream(world):
    rng = np.random.default_rng(17)
    x = fields.smooth_ridges(rng, 128 * 8 * 60 + 33)
    blob = oracle.compress(x, None, 128, "rel", 1e-3)
    ref = oracle.decompress(blob)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    pc = mp.start_processes(_dec_worker, args=(world, _free_port(), blob, q), nprocs=world,
                            join=False, start_method="spawn")
    # drain the queue before joining: a child cannot exit while its queued bytes are unread
    got = sorted(q.get(timeout=60) for _ in range(world))
    while not pc.join():
        pass
    out = np.concatenate([np.frombuffer(b, np.float32) for _, _, _, b in got])
    assert [g[1] for g in got] == [sharded.shard_plan(x.size, 128, world)[r][0] for r in range(world)]
    assert np.array_equal(out.view(np.uint32), ref.view(np.uint32))
