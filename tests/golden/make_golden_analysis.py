"""Reference outputs of the measurement / simulation API (build container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_analysis.py

For every case of cases.npz (make_golden.py) it records, from the Python reference:
  * compress_with_accounting -> ShiftAccounting (pipeline.py:186-190, metrics.py:21-27),
  * mse / max_abs_error / psnr of (input, reference reconstruction) (metrics.py:78-103),
  * block_range_cdf at the case's block size (metrics.py:128-146);
plus prefix_scan vectors (parallel.py:21-44) and propagate_indices / propagate_round
outputs (parallel.py:74-101).  Writes analysis.json and analysis.npz next to this script.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import ufzx  # noqa: E402
from ufzx import metrics, parallel  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
THRESHOLDS = (0.0, 1e-4, 1e-3, 2e-3, 1e-2, 1e-1, 0.5, 1.0)


def main():
    z = np.load(os.path.join(HERE, "cases.npz"))
    meta = json.loads(bytes(z["meta"]).decode())
    out = []
    for k, m in enumerate(meta):
        x = z[f"x{m['input']}"]
        recon = z[f"recon{k}"].view(np.float32)
        field = ufzx.DataField(x, tuple(m["dims"]))
        cfg = ufzx.CompressorConfig(ufzx.ErrorBound(m["mode"], m["magnitude"]), m["block_size"])
        _, acct = ufzx.compress_with_accounting(field, cfg)
        rec = {"case": k, "bits_shifted": int(acct.bits_shifted_scheme),
               "bits_unshifted": int(acct.bits_unshifted_scheme),
               "compressed_size_bytes": int(acct.compressed_size_bytes),
               "shift_overhead": metrics.shift_overhead(acct),
               "mse": metrics.mse(x, recon), "max_abs_error": metrics.max_abs_error(x, recon)}
        try:
            p = metrics.psnr(x, recon)
            rec["psnr"] = "inf" if p == float("inf") else p
        except metrics.DegenerateRangeError:
            rec["psnr"] = "degenerate"
        try:
            rec["cdf"] = metrics.block_range_cdf(x, m["block_size"], THRESHOLDS)
        except metrics.DegenerateRangeError:
            rec["cdf"] = "degenerate"
        out.append(rec)

    arrays = {}
    rng = np.random.default_rng(424242)
    scans = []
    for j, n in enumerate([0, 1, 2, 31, 32, 33, 1000, 2047, 2048, 2049, 70_001]):
        x = rng.integers(0, 5000, n).astype(np.int64)
        if j % 3 == 2:
            x[rng.random(n) < 0.5] = 0
        arrays[f"scan_in{j}"] = x
        arrays[f"scan_out{j}"] = parallel.prefix_scan(x)
        scans.append(j)
    props = []
    for j, (n, q) in enumerate([(1, 1), (2, 4), (5, 2), (6, 3), (17, 4), (128, 2), (128, 3),
                                (129, 4), (1000, 4), (4099, 3), (65535, 4)]):
        codes = rng.integers(0, 4, n).astype(np.uint8)
        if j % 2:
            codes[rng.random(n) < 0.7] = 3  # long reuse chains
        lay = parallel.BlockByteLayout(codes, q, n)
        rp = parallel.propagate_indices(lay)
        arrays[f"prop_codes{j}"] = codes
        arrays[f"prop_pos{j}"] = rp.positions
        props.append({"n": n, "q": q, "rounds": rp.rounds})
    base = rng.integers(0, 100, (40, 3)).astype(np.int64)
    for s in (1, 2, 7, 39, 40, 64):
        arrays[f"round_out{s}"] = parallel.propagate_round(base, s)
    arrays["round_in"] = base
    np.savez_compressed(os.path.join(HERE, "analysis.npz"), **arrays)
    with open(os.path.join(HERE, "analysis.json"), "w") as f:
        json.dump({"thresholds": THRESHOLDS, "cases": out, "scans": scans, "props": props,
                   "round_strides": [1, 2, 7, 39, 40, 64]}, f)
    print(f"{len(out)} cases, {len(scans)} scans, {len(props)} propagations")


if __name__ == "__main__":
    main()
