"""Synthetic workloads of BASELINE.json (the paper's SIFT/GIST/Deep corpora
are not available offline; seeded mixtures with their shapes and value
ranges stand in for them).

  * d=128 "SIFT-like": 256-component isotropic Gaussian mixture, centres
    U[0, 100), sigma 10, clipped at 0 (configs 0, 1, 2, 4);
  * d=960 "GIST-like": 512 components, centres U[0, 1), sigma 0.05,
    clipped at 0 (config 3).

Streams: 0 = centres, 1 = learn, 2 = base, 3 = queries. The NumPy
generator (PCG64 seeded with [seed, stream, chunk]) is used for test-size
data; `mixture_torch` draws the same distribution on the GPU (Philox) for
bench-size bases that never need to leave the device.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

STREAM_CENTRES, STREAM_LEARN, STREAM_BASE, STREAM_QUERY = 0, 1, 2, 3
CHUNK = 1 << 20


@dataclass(frozen=True)
class Mixture:
    d: int
    components: int
    centre_high: float
    sigma: float

    def centres(self, seed: int) -> np.ndarray:
        rng = np.random.default_rng([seed, STREAM_CENTRES])
        return rng.uniform(0.0, self.centre_high, (self.components, self.d)).astype(np.float32)


SIFT_LIKE = Mixture(d=128, components=256, centre_high=100.0, sigma=10.0)
GIST_LIKE = Mixture(d=960, components=512, centre_high=1.0, sigma=0.05)


def mixture_numpy(mix: Mixture, n: int, seed: int, stream: int,
                  centre_seed: int | None = None) -> np.ndarray:
    """n vectors (float32) drawn chunk by chunk, reproducible per chunk.
    `centre_seed` (default: seed) picks the mixture's centres, so learn,
    base and query splits of one corpus share them."""
    cen = mix.centres(seed if centre_seed is None else centre_seed)
    out = np.empty((n, mix.d), dtype=np.float32)
    for c0 in range(0, n, CHUNK):
        k = min(CHUNK, n - c0)
        rng = np.random.default_rng([seed, stream, c0 // CHUNK])
        comp = rng.integers(0, mix.components, k)
        x = cen[comp] + mix.sigma * rng.standard_normal((k, mix.d)).astype(np.float32)
        np.maximum(x, 0.0, out=x)
        out[c0:c0 + k] = x
    return out


def mixture_torch(mix: Mixture, n: int, seed: int, stream: int, device="cuda",
                  centre_seed: int | None = None):
    """Same distribution drawn on the GPU (torch Philox), chunk-seeded."""
    import torch

    cen = torch.from_numpy(mix.centres(seed if centre_seed is None else centre_seed)).to(device)
    out = torch.empty((n, mix.d), dtype=torch.float32, device=device)
    g = torch.Generator(device=device)
    for c0 in range(0, n, CHUNK):
        k = min(CHUNK, n - c0)
        g.manual_seed((seed * 1_000_003 + stream) * 1_000_003 + c0 // CHUNK)
        comp = torch.randint(0, mix.components, (k,), generator=g, device=device)
        x = torch.randn((k, mix.d), generator=g, device=device, dtype=torch.float32)
        x.mul_(mix.sigma).add_(cen[comp]).clamp_(min=0.0)
        out[c0:c0 + k] = x
    return out
