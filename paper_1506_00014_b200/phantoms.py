"""Synthetic inputs generated on the device (so the device-resident bench
inputs need no host copy): the modified Shepp-Logan head phantom
(point-sampled, as the reference's phantom_image, oracle.cpp:95-163) and
smooth random discs in the style of the reference's test helper
smooth_disc_image (helpers.hpp:55-112)."""
from __future__ import annotations

import math

import torch

# Toft's modified Shepp-Logan table on [-1, 1]^2: amplitude, centre, semi-axes, rotation (deg).
SHEPP_LOGAN = [
    (1.0, 0.0, 0.0, 0.69, 0.92, 0.0),
    (-0.8, 0.0, -0.0184, 0.6624, 0.874, 0.0),
    (-0.2, 0.22, 0.0, 0.11, 0.31, -18.0),
    (-0.2, -0.22, 0.0, 0.16, 0.41, 18.0),
    (0.1, 0.0, 0.35, 0.21, 0.25, 0.0),
    (0.1, 0.0, 0.1, 0.046, 0.046, 0.0),
    (0.1, 0.0, -0.1, 0.046, 0.046, 0.0),
    (0.1, -0.08, -0.605, 0.046, 0.023, 0.0),
    (0.1, 0.0, -0.605, 0.023, 0.023, 0.0),
    (0.1, 0.06, -0.605, 0.023, 0.046, 0.0),
]


def shepp_logan(N: int, device="cuda") -> torch.Tensor:
    c = torch.arange(N, device=device, dtype=torch.float64) / N - 0.5
    y, x = torch.meshgrid(c, c, indexing="ij")
    v = torch.zeros(N, N, dtype=torch.float64, device=device)
    for A, x0, y0, a, b, deg in SHEPP_LOGAN:
        t = math.radians(deg)
        dx, dy = x - 0.5 * x0, y - 0.5 * y0
        u = (math.cos(t) * dx + math.sin(t) * dy) / (0.5 * a)
        w = (-math.sin(t) * dx + math.cos(t) * dy) / (0.5 * b)
        v += A * (u * u + w * w <= 1.0)
    return (torch.round(v * 10) / 10).float()


def random_disc(N: int, seed: int, support_radius: float = 0.9, sigma: float = 3.0, device="cuda") -> torch.Tensor:
    gen = torch.Generator(device=device)
    gen.manual_seed(int(seed))
    img = torch.randn(1, 1, N, N, device=device, generator=gen)
    half = int(math.ceil(3 * sigma))
    t = torch.arange(-half, half + 1, device=device, dtype=torch.float32)
    k = torch.exp(-0.5 * t * t / sigma ** 2)
    k = k / k.sum()
    img = torch.nn.functional.conv2d(img, k.view(1, 1, 1, -1), padding=(0, half))
    img = torch.nn.functional.conv2d(img, k.view(1, 1, -1, 1), padding=(half, 0))[0, 0]
    c = (torch.arange(N, device=device, dtype=torch.float32) - N // 2) / N
    rad = torch.hypot(c[None, :], c[:, None])
    r = support_radius / 2
    edge = 0.85 * r
    w = torch.where(rad < edge, torch.ones_like(rad),
                    torch.where(rad < r, 0.5 * (1 + torch.cos(math.pi * (rad - edge) / (r - edge))),
                                torch.zeros_like(rad)))
    img = img * w
    return (img / img.abs().max()).contiguous()


def stack(N: int, count: int, seed0: int = 0x5EED, device="cuda") -> torch.Tensor:
    """Alternating Shepp-Logan and random-disc slices (the two synthetic families)."""
    sl = shepp_logan(N, device)
    out = torch.empty(count, N, N, device=device)
    for i in range(count):
        out[i] = sl if i % 2 == 0 else random_disc(N, seed0 + i, device=device)
    return out
