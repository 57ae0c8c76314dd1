"""Generate golden fixtures by importing the Python reference (build container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes, next to this script:
  cases.npz      -- small seeded fields, their reference streams (serialize() bytes) and
                    reference reconstructions (decompress() bit patterns);
  digests.json   -- sha256 of input / stream / reconstruction for 1M-value seeded fields
                    (the SURVEY.md Appendix C set, plus the block sizes the reference tests).
The reference cannot travel to the GPU box, so these files are what the -m gpu parity tests
compare against.  Mixed-sign all-zero blocks are excluded (trap 3).
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import ufzx  # noqa: E402
from ufzx import synth  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def ref_random_values(rng, n, kind):
    # same families as the reference's conftest.random_field_values
    kind %= 3
    if kind == 0:
        lo, hi = sorted(rng.normal(0.0, 50.0, 2))
        return synth.white_noise(rng, n, width=max((hi - lo) / 2, 1e-6), offset=(lo + hi) / 2)
    if kind == 1:
        return synth.random_walk(rng, n, step=float(10.0 ** rng.uniform(-4, 1)),
                                 start=float(rng.normal(0, 50)))
    return synth.plateaus(rng, n, n_levels=int(rng.integers(2, 8)))


def has_mixed_zero_block(vals, bs):
    n = len(vals)
    for s in range(0, n, bs):
        b = vals[s:s + bs]
        if np.all(b == 0) and np.signbit(b).any() and (~np.signbit(b)).any():
            return True
    return False


def run(vals, dims, bound, bs):
    field = ufzx.DataField(vals, dims)
    stream = ufzx.compress(field, ufzx.CompressorConfig(bound, bs))
    blob = ufzx.serialize(stream)
    out = ufzx.decompress(ufzx.deserialize(blob))
    return blob, out.values.view(np.uint32).copy()


def cases():
    out = []
    rng = np.random.default_rng(20260117)
    sizes = [1, 2, 3, 7, 8, 9, 31, 127, 128, 129, 255, 256, 300, 1000, 4096, 4097]
    bss = [8, 16, 17, 32, 33, 64, 128, 256]
    i = 0
    for n in sizes:
        for bs in bss:
            kind = i % 3
            i += 1
            vals = ref_random_values(rng, n, kind)
            if has_mixed_zero_block(vals, bs):
                continue
            if float(vals.max()) == float(vals.min()):
                bound = ufzx.ErrorBound("abs", 1e-3)
                mode, mag = "abs", 1e-3
            else:
                mag = float(10.0 ** rng.uniform(-6, -1))
                bound = ufzx.ErrorBound("rel", mag)
                mode = "rel"
            out.append(("rand", vals, (n,), mode, mag, bs))
    # larger seeded fields at several bounds (the headline block size and a few others)
    for j, (gen, n) in enumerate([("ridges", 20_000), ("walk", 16_000), ("noise", 8_000),
                                  ("plateaus", 8_000)]):
        r = np.random.default_rng(100 + j)
        if gen == "ridges":
            vals = synth.smooth_ridges(r, n)
        elif gen == "walk":
            vals = synth.random_walk(r, n, step=0.01)
        elif gen == "noise":
            vals = synth.white_noise(r, n)
        else:
            vals = synth.plateaus(r, n, n_levels=8)
        for rel in (1e-2, 1e-3, 1e-4, 1e-6):
            for bs in (128, 64, 17):
                out.append((gen, vals, (n,), "rel", rel, bs))
    # edge cases mirrored from the reference tests
    out.append(("const1", np.array([1.0], np.float32), (1,), "abs", 0.01, 128))
    out.append(("const128", np.full(128, 3.14, np.float32), (128,), "abs", 0.01, 128))
    out.append(("const512sq", np.full(512 * 512, 3.14, np.float32), (512, 512), "abs", 1e-2, 128))
    out.append(("kat4", np.array([0.1234, 0.1235, 0.1211, -0.1235], np.float32), (4,),
                "abs", 5e-4, 8))
    out.append(("kat4b", np.array([0.1234, 0.1235, 0.1211, -0.1235], np.float32), (4,),
                "abs", 1e-4, 8))
    r = np.random.default_rng(7)
    walk = (1.5 + np.clip(np.cumsum(r.normal(0, 1e-4, 20_000)), -0.45, 0.45)).astype(np.float32)
    out.append(("lossless", walk, (20_000,), "abs", 1e-12, 128))
    chains = np.tile(np.concatenate([[0.0], np.full(127, 1.0)]), 4).astype(np.float32)
    out.append(("chains", chains, (512,), "abs", 1e-6, 128))
    sub = (r.uniform(-1, 1, 4096) * 2.0 ** -140).astype(np.float32)
    sub[sub == 0] = np.float32(2.0 ** -149)
    out.append(("subnormal", sub, (4096,), "rel", 1e-2, 16))
    out.append(("subnormal128", sub, (4096,), "rel", 1e-3, 128))
    ulp = np.float32(2.0 ** -23)
    ce = np.concatenate([np.full(64, 1.0), np.full(64, 1.0 + 3 * float(ulp))]).astype(np.float32)
    out.append(("range2e", ce, (128,), "abs", 1.5 * float(ulp), 128))
    near = (r.normal(0, 1, 4096) + 1000.0).astype(np.float32)
    out.append(("near_radius", near, (16, 16, 16), "rel", 0.4999, 32))
    out.append(("dims3", ref_random_values(r, 24 * 9 * 5, 1), (24, 9, 5), "abs", 1e-3, 128))
    big = (r.normal(0, 1, 3000) * 1e30).astype(np.float32)
    out.append(("huge", big, (3000,), "rel", 1e-5, 128))
    tiny_e = ref_random_values(r, 2000, 1)
    out.append(("tiny_e", tiny_e, (2000,), "abs", 1e-40, 128))
    return out


def main():
    arrays = {}
    meta = []
    inputs = {}
    for k, (name, vals, dims, mode, mag, bs) in enumerate(cases()):
        key = id(vals)
        vals = np.ascontiguousarray(vals, np.float32)
        if key not in inputs:
            inputs[key] = len(inputs)
            arrays[f"x{inputs[key]}"] = vals
        bound = ufzx.ErrorBound(mode, mag)
        blob, recon = run(vals, dims, bound, bs)
        arrays[f"blob{k}"] = np.frombuffer(blob, np.uint8)
        arrays[f"recon{k}"] = recon
        meta.append({"name": name, "input": inputs[key], "dims": list(dims), "mode": mode,
                     "magnitude": mag, "block_size": bs})
    arrays["meta"] = np.frombuffer(json.dumps(meta).encode(), np.uint8)
    np.savez_compressed(os.path.join(HERE, "cases.npz"), **arrays)

    digests = []
    sha = lambda b: hashlib.sha256(b).hexdigest()
    gens = [("smooth_ridges", lambda: synth.smooth_ridges(np.random.default_rng(0), 1_000_000)),
            ("random_walk", lambda: synth.random_walk(np.random.default_rng(0), 1_000_000,
                                                      step=0.01)),
            ("white_noise", lambda: synth.white_noise(np.random.default_rng(0), 1_000_000))]
    for gname, gen in gens:
        vals = gen()
        for rel, bs in ((1e-3, 128), (1e-2, 128), (1e-4, 128), (1e-3, 17), (1e-3, 8),
                        (1e-3, 256)):
            blob, recon = run(vals, (vals.size,), ufzx.ErrorBound("rel", rel), bs)
            digests.append({"generator": gname, "n": int(vals.size), "seed": 0, "rel": rel,
                            "block_size": bs, "input": sha(vals.tobytes()),
                            "stream_len": len(blob), "stream": sha(blob),
                            "recon": sha(recon.tobytes()),
                            "e": ufzx.deserialize(blob).error_bound})
    with open(os.path.join(HERE, "digests.json"), "w") as f:
        json.dump(digests, f, indent=1)
    print(f"{len(meta)} cases, {len(digests)} digests")


if __name__ == "__main__":
    main()
