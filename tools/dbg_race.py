import sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np
import oracle
import paper_2201_13020_b200 as szx
from test_gpu_parity import TestWarpPaths
tail = 100
rng = np.random.default_rng(1000 + tail)
e = 1e-3
nblocks = 64 * 5 + 7
x = TestWarpPaths._mixed_q_field(rng, nblocks, e)
x = x[: x.size - 128 + tail]
P = oracle.compress_pools(x, 128, e)
cmap = np.unpackbits(P["map"], bitorder="little")[:P["nb"]].astype(bool)
codes = np.stack([(P["codes"] >> (2 * j)) & 3 for j in range(4)], axis=1).reshape(-1)
boff = np.zeros(P["nb"] + 1, np.int64); r = 0; ci = 0; qs = []
for b in range(P["nb"]):
    if cmap[b]:
        boff[b + 1] = boff[b]; qs.append(0); continue
    req = int(P["req"][r]); s_ = (8 - req % 8) % 8; q = (req + s_) // 8; qs.append(q)
    cnt = min(128, x.size - 128 * b)
    c = codes[ci:ci + cnt]; ci += cnt; r += 1
    boff[b + 1] = boff[b] + int(np.sum(q - np.minimum(c, q)))
fails = 0
for rep in range(200):
    s = szx.compress(szx.DataField(x, (x.size,)), szx.CompressorConfig(szx.ErrorBound("abs", e)))
    m = s.mid_bytes
    d = np.nonzero(P["mid"] != m)[0]
    if len(d):
        fails += 1
        blocks = np.unique(np.searchsorted(boff, d, side="right") - 1)
        print(f"rep {rep}: {len(d)} diffs at {d[0]}..{d[-1]}; blocks {blocks[:8]} tiles {np.unique(blocks // 64)}"
              f" warps {np.unique((blocks % 64) // 4)}; tile mid starts {[int(boff[64*t]) for t in np.unique(blocks//64)]}"
              f" q {[qs[b] for b in blocks[:8]]}")
        if fails > 6:
            break
print("fails", fails)
