import sys, time, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import torch, oracle, fields
import paper_2201_13020_b200 as szx
for n in (1, 5, 128, 129, 4096, 4097, 100_000, 1_000_003):
    x = fields.smooth_ridges(np.random.default_rng(n), n) if n > 300 else np.random.default_rng(n).normal(size=n).astype(np.float32)
    for rel in (1e-3,):
        t = time.time()
        s = szx.compress(szx.DataField(x, (n,)), szx.CompressorConfig(szx.ErrorBound("rel" if n > 1 else "abs", rel)))
        torch.cuda.synchronize()
        blob = szx.serialize(s)
        ref = oracle.compress(x, (n,), 128, "rel" if n > 1 else "abs", rel)
        ok1 = blob == ref
        out = szx.decompress(s).values
        ok2 = np.array_equal(out.view(np.uint32), oracle.decompress(ref).view(np.uint32))
        out2 = szx.decompress(szx.deserialize(ref)).values
        ok3 = np.array_equal(out2.view(np.uint32), oracle.decompress(ref).view(np.uint32))
        print(n, rel, ok1, ok2, ok3, f"{time.time()-t:.2f}s", flush=True)
