"""GPU: sharded compression assembles the single-stream bytes (one GPU, 1-2 ranks).

NCCL needs one GPU per rank, so the 2-rank case shares cuda:0 through gloo collectives; the
1-rank case runs the NCCL path.  Both must write exactly the stream `serialize(compress(...))`
produces for the whole field."""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch.multiprocessing as mp

import fields

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, backend, port, path, x, dims, rel):
    import torch
    import torch.distributed as dist

    import paper_2201_13020_b200 as szx
    from paper_2201_13020_b200 import sharded

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    kw = {"device_id": torch.device("cuda", 0)} if backend == "nccl" else {}
    dist.init_process_group(backend, rank=rank, world_size=world, **kw)
    try:
        v0, v1 = sharded.shard_plan(x.size, 128, world)[rank]
        local = torch.from_numpy(x[v0:v1].copy()).cuda()
        cfg = szx.CompressorConfig(szx.ErrorBound("rel", rel))
        res = sharded.compress_sharded(local, dims, cfg, v0)
        sharded.write_sharded(res, path)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,backend", [(1, "nccl"), (2, "gloo"), (3, "gloo")])
def test_sharded_stream_equals_single_stream(cuda, world, backend):
    import paper_2201_13020_b200 as szx

    rng = np.random.default_rng(21)
    x = fields.smooth_ridges(rng, 128 * 8 * 300 + 45)
    dims = (x.size,)
    rel = 1e-3
    want = szx.serialize(szx.compress(szx.DataField(x, dims),
                                      szx.CompressorConfig(szx.ErrorBound("rel", rel))))
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "s.ufzx")
        mp.start_processes(_worker, args=(world, backend, _free_port(), path, x, dims, rel),
                           nprocs=world, join=True, start_method="spawn")
        with open(path, "rb") as f:
            got = f.read()
    assert got == want


def _dec_worker(rank, world, backend, port, path, outdir):
    import torch
    import torch.distributed as dist

    from paper_2201_13020_b200 import sharded

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    kw = {"device_id": torch.device("cuda", 0)} if backend == "nccl" else {}
    dist.init_process_group(backend, rank=rank, world_size=world, **kw)
    try:
        fd = os.open(path, os.O_RDONLY)
        try:
            vals, v0, v1 = sharded.decompress_sharded(fd)
        finally:
            os.close(fd)
        np.save(os.path.join(outdir, f"r{rank}.npy"),
                np.array([v0, v1], np.int64))
        np.save(os.path.join(outdir, f"v{rank}.npy"), vals.cpu().numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,backend,bs", [(1, "nccl", 128), (2, "gloo", 128), (3, "gloo", 128),
                                              (2, "gloo", 64)])
def test_sharded_decompress_equals_single_decode(cuda, world, backend, bs):
    """Every rank decodes its shard of ONE stream (K3 per shard, all-gather of the shard mid
    totals, K2); the shards concatenate to the single-stream reconstruction bit for bit."""
    import oracle

    rng = np.random.default_rng(23)
    x = fields.smooth_ridges(rng, 128 * 8 * 300 + 45)
    blob = oracle.compress(x, None, bs, "rel", 1e-4)
    ref = oracle.decompress(blob)
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "s.ufzx")
        with open(path, "wb") as f:
            f.write(blob)
        mp.start_processes(_dec_worker, args=(world, backend, _free_port(), path, d),
                           nprocs=world, join=True, start_method="spawn")
        parts = []
        for r in range(world):
            v0, v1 = np.load(os.path.join(d, f"r{r}.npy"))
            vals = np.load(os.path.join(d, f"v{r}.npy"))
            assert vals.size == v1 - v0
            parts.append(vals)
    out = np.concatenate(parts)
    assert np.array_equal(out.view(np.uint32), ref.view(np.uint32))
