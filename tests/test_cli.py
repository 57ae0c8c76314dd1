"""CLI front end (ufzx/cli.py contract): exit codes and byte-identical containers."""
import numpy as np
import pytest

import fields
import oracle
from paper_2201_13020_b200 import cli


def test_usage_errors_exit_1(tmp_path, capsys):
    assert cli.main(["compress", "a", "b", "--dims", "0,3", "--rel", "1e-3"]) == cli.EXIT_USAGE
    assert cli.main(["compress", "a", "b", "--dims", "3"]) == cli.EXIT_USAGE
    assert cli.main(["compress", "a", "b", "--dims", "3", "--abs", "1", "--rel", "1"]) == 1
    assert cli.main(["compress", "a", "b", "--dims", "3", "--rel", "x"]) == cli.EXIT_USAGE
    assert cli.main(["compress", "a", "b", "--dims", "3", "--rel", "-1"]) == cli.EXIT_USAGE
    assert cli.main(["nope"]) == cli.EXIT_USAGE


@pytest.mark.gpu
def test_round_trip_files(cuda, tmp_path, capsys):
    rng = np.random.default_rng(2)
    x = fields.smooth_ridges(rng, 100 * 77)
    raw = tmp_path / "f.f32"
    x.astype("<f4").tofile(raw)
    out = tmp_path / "f.ufzx"
    assert cli.main(["compress", str(raw), str(out), "--dims", "100,77", "--rel", "1e-3"]) == 0
    assert out.read_bytes() == oracle.compress(x, (100, 77), 128, "rel", 1e-3)
    back = tmp_path / "back.f32"
    assert cli.main(["decompress", str(out), str(back), "--original", str(raw)]) == 0
    got = np.fromfile(back, "<f4")
    assert np.array_equal(got.view(np.uint32),
                          oracle.decompress(out.read_bytes()).view(np.uint32))
    assert "max_abs_error=" in capsys.readouterr().out


@pytest.mark.gpu
def test_exit_codes(cuda, tmp_path):
    x = np.linspace(0, 1, 1000, dtype=np.float32)
    raw = tmp_path / "x.f32"
    x.tofile(raw)
    # I/O: missing input, size / dims mismatch
    assert cli.main(["compress", str(tmp_path / "missing.f32"), str(tmp_path / "o"),
                     "--dims", "1000", "--abs", "0.01"]) == cli.EXIT_IO
    assert cli.main(["compress", str(raw), str(tmp_path / "o"), "--dims", "999",
                     "--abs", "0.01"]) == cli.EXIT_IO
    # format: a truncated container
    good = tmp_path / "g.ufzx"
    assert cli.main(["compress", str(raw), str(good), "--dims", "1000", "--abs", "0.01"]) == 0
    bad = tmp_path / "b.ufzx"
    bad.write_bytes(good.read_bytes()[:-3])
    assert cli.main(["decompress", str(bad), str(tmp_path / "r.f32")]) == cli.EXIT_FORMAT
    # bound violation: verify against a different original
    other = tmp_path / "other.f32"
    (x + 1).astype("<f4").tofile(other)
    assert cli.main(["decompress", str(good), str(tmp_path / "r.f32"), "--original",
                     str(other)]) == cli.EXIT_BOUND
    # zero-range relative bound -> usage (cli.py:322-324)
    flat = tmp_path / "flat.f32"
    np.full(1000, 3.0, np.float32).tofile(flat)
    assert cli.main(["compress", str(flat), str(tmp_path / "o2"), "--dims", "1000",
                     "--rel", "1e-3"]) == cli.EXIT_USAGE


@pytest.mark.gpu
def test_bench_directory(cuda, tmp_path, capsys):
    for i in range(2):
        fields.smooth_ridges(np.random.default_rng(i), 4096).astype("<f4").tofile(
            tmp_path / f"f{i}.f32")
    assert cli.main(["bench", str(tmp_path), "--dims", "64,64", "--rel", "1e-3,1e-4"]) == 0
    out = capsys.readouterr().out
    assert "aggregate rel:0.001" in out and "aggregate rel:0.0001" in out
