"""GPU parity of the measurement / simulation API (csrc/analysis.cu) against the
reference's own outputs (tests/golden/analysis.*) and, at BASELINE sizes, the pinned oracle:
compress_with_accounting / shift_overhead, max_abs_error / mse / psnr, block_range_cdf,
prefix_scan, propagate_indices / propagate_round.

Bars: integer outputs (bit totals, CDF counts, scans, positions) and max_abs_error are
exact; mse / psnr are float64 sums whose order differs from NumPy's pairwise sum, so they
are compared with a relative tolerance of 1e-12 (stated here).
"""
import math

import numpy as np
import pytest

import oracle
from analysis_golden import analysis_golden
from conftest import golden_cases
import paper_2201_13020_b200 as szx
from paper_2201_13020_b200 import metrics

pytestmark = pytest.mark.gpu
G = analysis_golden()
REL = 1e-12


def _case(k):
    m, x, blob, recon = golden_cases().case(k)
    return m, x, blob, recon.view(np.float32)


class TestAccounting:
    def test_golden(self, cuda):
        for k, g in enumerate(G.cases):
            m, x, blob, _ = _case(k)
            field = szx.DataField(x, m["dims"])
            cfg = szx.CompressorConfig(szx.ErrorBound(m["mode"], m["magnitude"]), m["block_size"])
            s, a = szx.compress_with_accounting(field, cfg)
            assert szx.serialize(s) == blob, k
            assert (a.bits_shifted_scheme, a.bits_unshifted_scheme,
                    a.compressed_size_bytes) == (g["bits_shifted"], g["bits_unshifted"],
                                                 g["compressed_size_bytes"]), (k, m)
            assert szx.shift_overhead(a) == g["shift_overhead"]

    def test_disabled(self):
        with pytest.raises(metrics.AccountingDisabledError):
            szx.shift_overhead(None)

    @pytest.mark.parametrize("kind,n,bs", [("smooth_ridges", 512 ** 3, 128),
                                           ("white_noise", 25_000_000, 128),
                                           ("smooth_ridges", 3_000_001, 17)])
    def test_full_size_vs_oracle(self, cuda, kind, n, bs):
        from paper_2201_13020_b200 import synth

        xd = synth.field(kind, n, seed=3)
        field = szx.DataField(xd, (n,))
        s, a = szx.compress_with_accounting(field, szx.CompressorConfig(szx.ErrorBound("rel", 1e-3), bs))
        sh, un = oracle.accounting(xd.cpu().numpy(), bs, s.error_bound)
        assert (a.bits_shifted_scheme, a.bits_unshifted_scheme) == (sh, un)
        assert a.bits_shifted_scheme == 8 * s.mid_len


class TestQuality:
    def test_golden(self, cuda):
        for k, g in enumerate(G.cases):
            m, x, _, recon = _case(k)
            assert szx.max_abs_error(x, recon) == g["max_abs_error"], k
            assert szx.mse(x, recon) == pytest.approx(g["mse"], rel=REL, abs=0), k
            if g["psnr"] == "degenerate":
                with pytest.raises(metrics.DegenerateRangeError):
                    szx.psnr(x, recon)
            elif g["psnr"] == "inf":
                assert szx.psnr(x, recon) == math.inf
            else:
                assert szx.psnr(x, recon) == pytest.approx(g["psnr"], rel=REL), k

    def test_datafields_and_tensors(self, cuda):
        rng = np.random.default_rng(5)
        x = rng.normal(size=100_003).astype(np.float32)
        y = (x + rng.normal(scale=1e-3, size=x.size)).astype(np.float32)
        mx, ms, _ = oracle.quality(x, y)
        fa, fb = szx.DataField(x, (x.size,)), szx.DataField(y, (y.size,))
        assert szx.max_abs_error(fa, fb) == mx
        assert szx.max_abs_error(cuda.from_numpy(x).cuda(), cuda.from_numpy(y).cuda()) == mx
        assert szx.mse(fa, y[None, :]) == pytest.approx(ms, rel=REL)
        # unaligned device views take the scalar path
        assert szx.max_abs_error(cuda.from_numpy(x).cuda()[1:], cuda.from_numpy(y).cuda()[1:]) == \
            oracle.quality(x[1:], y[1:])[0]
        with pytest.raises(ValueError, match="length mismatch"):
            szx.mse(x, y[:-1])

    def test_nan_propagates(self, cuda):
        x = np.array([1.0, np.inf, 3.0], np.float32)
        assert math.isnan(szx.max_abs_error(x, x)) and math.isnan(szx.mse(x, x))

    def test_full_size_round_trip(self, cuda):
        from paper_2201_13020_b200 import synth

        n = 512 ** 3
        xd = synth.field("smooth_ridges", n, seed=1)
        field = szx.DataField(xd, (512, 512, 512))
        s = szx.compress(field, szx.CompressorConfig(szx.ErrorBound("rel", 1e-3)))
        out = szx.decompress(s)
        q = metrics.quality(field, out)
        xh, yh = xd.cpu().numpy(), out.device_values.cpu().numpy()
        mx, ms, rng = oracle.quality(xh, yh)
        assert q["max_abs_error"] == mx <= s.error_bound
        assert q["sum_sq"] / n == pytest.approx(ms, rel=1e-11)
        assert q["max"] - q["min"] == rng


class TestBlockRangeCdf:
    def test_golden(self, cuda):
        for k, g in enumerate(G.cases):
            m, x, _, _ = _case(k)
            if g["cdf"] == "degenerate":
                with pytest.raises(metrics.DegenerateRangeError):
                    szx.block_range_cdf(x, m["block_size"], G.thresholds)
            else:
                got = szx.block_range_cdf(x, m["block_size"], G.thresholds)
                assert got == [tuple(p) for p in g["cdf"]], k

    def test_field_and_defaults(self, cuda):
        from paper_2201_13020_b200 import synth

        n = 25_000_000
        xd = synth.field("smooth_ridges", n, seed=2)
        field = szx.DataField(xd, (100, 500, 500))
        got = szx.block_range_cdf(field, 128)
        assert got == oracle.block_range_cdf(xd.cpu().numpy(), 128, metrics.DEFAULT_CDF_THRESHOLDS)
        many = [i / 100 for i in range(101)]  # > 64 thresholds: two launches
        assert szx.block_range_cdf(field, 100, many) == oracle.block_range_cdf(
            xd.cpu().numpy(), 100, many)

    def test_errors(self, cuda):
        with pytest.raises(ValueError, match="empty"):
            szx.block_range_cdf(np.zeros(0, np.float32), 128)
        with pytest.raises(metrics.DegenerateRangeError):
            szx.block_range_cdf(np.full(300, 2.0, np.float32), 128)


class TestScanAndPropagation:
    def test_prefix_scan_golden(self, cuda):
        for j in G.meta["scans"]:
            got = szx.prefix_scan(G.z[f"scan_in{j}"])
            assert got.dtype == np.int64 and np.array_equal(got, G.z[f"scan_out{j}"])

    def test_prefix_scan_large_and_tensor(self, cuda):
        rng = np.random.default_rng(9)
        x = rng.integers(-2 ** 40, 2 ** 40, 5_000_001).astype(np.int64)
        assert np.array_equal(szx.prefix_scan(x), oracle.prefix_scan(x))
        t = szx.prefix_scan(cuda.from_numpy(x[:1000]).cuda())
        assert t.is_cuda and np.array_equal(t.cpu().numpy(), oracle.prefix_scan(x[:1000]))
        assert szx.prefix_scan([3, 0, 2, 5]).tolist() == [0, 3, 3, 5]  # test_parallel.py:49-50

    def test_propagate_indices_golden(self, cuda):
        from paper_2201_13020_b200.parallel import BlockByteLayout

        for j, p in enumerate(G.meta["props"]):
            rp = szx.propagate_indices(BlockByteLayout(G.z[f"prop_codes{j}"], p["q"], p["n"]))
            assert rp.rounds == p["rounds"]
            assert np.array_equal(rp.positions, G.z[f"prop_pos{j}"]), j

    def test_propagate_round_golden(self, cuda):
        base = G.z["round_in"]
        for s in G.meta["round_strides"]:
            assert np.array_equal(szx.propagate_round(base, s), G.z[f"round_out{s}"]), s
        with pytest.raises(ValueError):
            szx.propagate_round(base, 0)
