"""Seeded synthetic float32 fields for parity tests.

Restates the reference generators (``pkg/src/ufzx/synth.py:9-58``) and the test helper
``random_field_values`` (``pkg/tests/conftest.py:20-33``) so that the same seed gives the same
array as the reference; ``tests/test_oracle.py`` pins that via the input digests of
SURVEY.md Appendix C.
"""
from __future__ import annotations

import numpy as np


def white_noise(rng, n, width=1.0, offset=0.0):
    # synth.py:9-10
    return (rng.uniform(-width, width, n) + offset).astype(np.float32)


def random_walk(rng, n, step=1.0, start=0.0):
    # synth.py:13-14
    steps = rng.normal(0.0, step, n)
    return (start + np.cumsum(steps)).astype(np.float32)


def plateaus(rng, n, n_levels=6, spread=10.0):
    # synth.py:17-22: random level values, sorted distinct cut points, repeated levels
    levels = rng.normal(0.0, spread, n_levels)
    cuts = rng.choice(np.arange(1, n), size=min(n_levels - 1, n - 1), replace=False)
    bounds = np.concatenate(([0], np.sort(cuts), [n]))
    runs = np.diff(bounds)
    return np.repeat(levels[: runs.size], runs).astype(np.float32)


def smooth_ridges(rng, n, spacing=(100, 300), texture=4.0, texture_scale=16):
    # synth.py:25-53: piecewise-linear vertices + gaussian-smoothed texture + offset
    verts = [0]
    while verts[-1] < n:
        verts.append(verts[-1] + int(rng.integers(spacing[0], spacing[1])))
    verts = np.asarray(verts)
    verts[-1] = max(verts[-1], n)
    heights = rng.uniform(-1.0, 1.0, verts.size)
    base = np.interp(np.arange(n), verts, heights)
    mean_step = 2.0 * np.abs(np.diff(heights)).mean() / ((spacing[0] + spacing[1]) / 2)
    half = 3 * texture_scale
    taps = np.exp(-0.5 * (np.arange(-half, half + 1) / texture_scale) ** 2)
    taps /= taps.sum()
    tex = np.convolve(rng.normal(0.0, 1.0, n), taps, mode="same")
    sd = tex.std()
    if sd > 0:
        tex *= texture * mean_step / sd
    return (base + tex + rng.normal(0.0, 3.0)).astype(np.float32)


def random_field_values(rng, n, kind):
    # conftest.py:20-33 -- the three families used by the reference round-trip tests
    kind %= 3
    if kind == 0:
        lo, hi = sorted(rng.normal(0.0, 50.0, 2))
        return white_noise(rng, n, width=max((hi - lo) / 2, 1e-6), offset=(lo + hi) / 2)
    if kind == 1:
        return random_walk(rng, n, step=float(10.0 ** rng.uniform(-4, 1)),
                           start=float(rng.normal(0, 50)))
    return plateaus(rng, n, n_levels=int(rng.integers(2, 8)))
