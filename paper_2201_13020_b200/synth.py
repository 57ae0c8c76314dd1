"""Device-side synthetic fields of the paper's dataset shapes (benchmark inputs).

Same families as the reference generators (``ufzx/synth.py:9-58``), generated directly in
HBM with torch so multi-GB inputs cost milliseconds instead of minutes of NumPy.  They are
statistically equivalent to the reference's, not bit-identical (different RNG stream);
bit-exact parity uses the host generators in ``tests/fields.py``.
"""
from __future__ import annotations

import math


def _torch():
    import torch

    return torch


def smooth_ridges(n: int, seed: int = 0, spacing=(100, 300), texture: float = 4.0,
                  texture_scale: int = 16, device="cuda"):
    """Piecewise-linear ridges + gaussian-smoothed texture + offset (synth.py:25-53)."""
    torch = _torch()
    g = torch.Generator(device=device).manual_seed(seed)
    nseg = n // spacing[0] + 2
    steps = torch.randint(spacing[0], spacing[1], (nseg,), generator=g, device=device)
    pts = torch.cat([torch.zeros(1, dtype=torch.int64, device=device), torch.cumsum(steps, 0)])
    k = int(torch.searchsorted(pts, torch.tensor([n], device=device)).item()) + 1
    pts = pts[: k + 1].clone()
    pts[-1] = torch.clamp(pts[-1], min=n)
    levels = torch.rand(pts.numel(), generator=g, device=device, dtype=torch.float64) * 2 - 1
    out = torch.empty(n, dtype=torch.float32, device=device)
    mean_step = 2.0 * float(levels.diff().abs().mean()) / ((spacing[0] + spacing[1]) / 2)
    half = 3 * texture_scale
    taps = torch.exp(-0.5 * (torch.arange(-half, half + 1, device=device, dtype=torch.float32)
                             / texture_scale) ** 2)
    taps = (taps / taps.sum()).view(1, 1, -1)
    offset = float(torch.randn(1, generator=g, device=device, dtype=torch.float64)) * 3.0
    chunk = 1 << 26
    noise_scale = None
    for c0 in range(0, n, chunk):
        c1 = min(n, c0 + chunk)
        idx = torch.arange(c0, c1, device=device, dtype=torch.int64)
        seg = torch.searchsorted(pts, idx, right=True) - 1
        x0, x1 = pts[seg], pts[seg + 1]
        t = (idx - x0).to(torch.float64) / (x1 - x0).to(torch.float64)
        y = levels[seg] + t * (levels[seg + 1] - levels[seg])
        noise = torch.randn(c1 - c0 + 2 * half, generator=g, device=device, dtype=torch.float32)
        tex = torch.nn.functional.conv1d(noise.view(1, 1, -1), taps).view(-1)
        if noise_scale is None:
            sd = float(tex.std())
            noise_scale = texture * mean_step / sd if sd > 0 else 0.0
        out[c0:c1] = (y + tex.to(torch.float64) * noise_scale + offset).to(torch.float32)
    return out


def random_walk(n: int, seed: int = 0, step: float = 0.01, start: float = 0.0, device="cuda"):
    """Cumulative Gaussian steps (synth.py:13-14), float64 accumulation per chunk."""
    torch = _torch()
    g = torch.Generator(device=device).manual_seed(seed)
    out = torch.empty(n, dtype=torch.float32, device=device)
    carry = float(start)
    chunk = 1 << 26
    for c0 in range(0, n, chunk):
        c1 = min(n, c0 + chunk)
        s = torch.randn(c1 - c0, generator=g, device=device, dtype=torch.float64) * step
        cs = torch.cumsum(s, 0) + carry
        carry = float(cs[-1])
        out[c0:c1] = cs.to(torch.float32)
    return out


def white_noise(n: int, seed: int = 0, width: float = 1.0, offset: float = 0.0, device="cuda"):
    """Uniform noise in [offset-width, offset+width) (synth.py:9-10)."""
    torch = _torch()
    g = torch.Generator(device=device).manual_seed(seed)
    out = torch.rand(n, generator=g, device=device)  # in place: no multi-GB temporaries
    return out.mul_(2 * width).sub_(width).add_(offset)


GENERATORS = {"smooth_ridges": smooth_ridges, "random_walk": random_walk,
              "white_noise": white_noise}


def field(kind: str, n: int, seed: int = 0, device="cuda"):
    return GENERATORS[kind](n, seed=seed, device=device)


def dataset_shape(name: str):
    """The BASELINE.json config shapes."""
    shapes = {
        "hurricane": (100, 500, 500),
        "nyx": (512, 512, 512),
        "cesm": (1800, 3600),
        "hacc": (280_953_867,),
    }
    return shapes[name]


def numel(dims) -> int:
    return math.prod(dims)
