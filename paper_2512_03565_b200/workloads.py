"""Seeded synthetic workloads of BASELINE.json's configurations.

No dataset is involved; every configuration is generated from its stated
shape, density and seed.  Random gases use random sequential addition (RSA)
with a minimum-image distance of 0.9 sigma, done in parallel batches on a
fine periodic grid (one point per grid cell at most); within a batch a
candidate conflicting with an earlier-index candidate is dropped, so the
result is deterministic for a seed and device.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from .particles import lattice_positions


@dataclass
class Workload:
    name: str
    positions: np.ndarray | torch.Tensor   # (N, 3) float64
    box_length: float
    cutoff: float
    skin: float
    velocities: np.ndarray | torch.Tensor | None = None
    note: str = ""

    @property
    def n(self) -> int:
        return int(self.positions.shape[0])


def maxwell_boltzmann(n: int, temperature: float, seed: int, mass: float = 1.0,
                      device="cpu") -> torch.Tensor:
    """N(0, sqrt(T/m)) per component (numpy default_rng(seed)), centre-of-mass
    velocity removed -- the construction of SURVEY.md §8(d)."""
    rng = np.random.default_rng(int(seed))
    v = rng.normal(0.0, math.sqrt(temperature / mass), (n, 3))
    v -= v.mean(axis=0)
    return torch.from_numpy(v).to(device)


def rsa_positions(n: int, length: float, dmin: float, seed: int, device="cpu",
                  region=None, batch: int | None = None, existing=None) -> torch.Tensor:
    """Uniform random positions in a periodic cube with pairwise minimum-image
    distance >= dmin.  ``region(points) -> bool mask`` restricts candidates
    (e.g. a droplet); ``existing`` points are kept and respected."""
    dev = torch.device(device)
    g = torch.Generator(device="cpu").manual_seed(int(seed))
    h = dmin / math.sqrt(3.0) * 0.999
    m = max(1, int(length / h))
    h = length / m
    grid = torch.full((m * m * m,), -1, dtype=torch.int64, device=dev)
    pts = torch.empty((0, 3), dtype=torch.float64, device=dev)
    if existing is not None and len(existing):
        pts = torch.as_tensor(existing, dtype=torch.float64, device=dev).reshape(-1, 3)
        c = _cells(pts, h, m)
        grid[c] = torch.arange(pts.shape[0], device=dev)
    target = pts.shape[0] + n
    r = int(math.ceil(dmin / h))
    offs = torch.stack(torch.meshgrid(*[torch.arange(-r, r + 1, device=dev)] * 3,
                                      indexing="ij"), dim=-1).reshape(-1, 3)
    batch = batch or max(4096, min(1 << 18, n // 4 + 1))
    d2min = dmin * dmin
    stall = 0
    while pts.shape[0] < target:
        cand = torch.rand((batch, 3), generator=g, dtype=torch.float64).to(dev) * length
        if region is not None:
            cand = cand[region(cand)]
            if cand.shape[0] == 0:
                continue
        cc = _cells(cand, h, m)
        # one candidate per grid cell, earliest index wins, and only empty cells
        k = torch.arange(cand.shape[0], device=dev)
        uniq, inv = torch.unique(cc, return_inverse=True)
        first = torch.full((uniq.shape[0],), cand.shape[0], dtype=torch.int64, device=dev)
        first.scatter_reduce_(0, inv, k, reduce="amin")
        keep = (first[inv] == k) & (grid[cc] < 0)
        cand, cc = cand[keep], cc[keep]
        if cand.shape[0] == 0:
            stall += 1
            if stall > 200:
                raise RuntimeError("RSA stalled: density too close to jamming")
            continue
        # tentatively place the batch, then reject conflicts with existing points
        # or with earlier-index batch members
        base = pts.shape[0]
        me = base + torch.arange(cand.shape[0], device=dev)
        grid[cc] = me
        allpts = torch.cat([pts, cand])
        ci = torch.stack([cc % m, (cc // m) % m, cc // (m * m)], dim=1)
        ok = torch.ones(cand.shape[0], dtype=torch.bool, device=dev)
        for o in offs:
            if int(o.abs().sum()) == 0:
                continue
            nb = (ci + o) % m
            lin = nb[:, 0] + m * (nb[:, 1] + m * nb[:, 2])
            other = grid[lin]
            relevant = (other >= 0) & (other < me)
            if not bool(relevant.any()):
                continue
            q = allpts[other.clamp(min=0)]
            d = cand - q
            d -= length * torch.round(d / length)
            close = (d * d).sum(dim=1) < d2min
            ok &= ~(relevant & close)
        grid[cc[~ok]] = -1
        cand, cc = cand[ok], cc[ok]
        room = target - pts.shape[0]
        if cand.shape[0] > room:
            grid[cc[room:]] = -1
            cand, cc = cand[:room], cc[:room]
        # accepted candidates are renumbered densely after the existing points
        grid[cc] = pts.shape[0] + torch.arange(cand.shape[0], device=dev)
        pts = torch.cat([pts, cand])
        stall = 0
    return pts


def _cells(p: torch.Tensor, h: float, m: int) -> torch.Tensor:
    c = torch.clamp((p / h).floor().to(torch.int64), 0, m - 1)
    return c[:, 0] + m * (c[:, 1] + m * c[:, 2])


def config1() -> Workload:
    """20^3 SC lattice, spacing 1.1, L = 22, rc = 2.5, skin 0 (LC, Newton3)."""
    pos = lattice_positions((0.0, 0.0, 0.0), (20, 20, 20), 1.1)
    v = maxwell_boltzmann(8000, 1.0, 42).numpy()
    return Workload("c1-lattice-8000", pos, 22.0, 2.5, 0.0, v, "seed 42")


def config2(rho: float = 0.8, n: int = 1_000_000, seed: int = 42, device="cpu",
            skin: float = 0.3) -> Workload:
    """Uniform random gas at density rho, RSA min distance 0.9, rc 2.5."""
    L = (n / rho) ** (1.0 / 3.0)
    pos = rsa_positions(n, L, 0.9, seed, device=device)
    return Workload(f"c2-uniform-rho{rho}-{n}", pos, L, 2.5, skin,
                    maxwell_boltzmann(n, 1.0, seed + 1, device=device),
                    f"RSA dmin 0.9, seed {seed}")


def config3(n: int = 2_000_000, seed: int = 42, device="cpu") -> Workload:
    """Droplet (rho 0.8, radius 0.3 L) in vapour (rho 0.05), rc 3.0."""
    vol_frac = 4.0 / 3.0 * math.pi * 0.3 ** 3
    rho_mean = 0.8 * vol_frac + 0.05 * (1 - vol_frac)
    L = (n / rho_mean) ** (1.0 / 3.0)
    n_drop = int(round(0.8 * vol_frac * L ** 3))
    c = L / 2
    R = 0.3 * L
    inside = lambda p: ((p - c) ** 2).sum(dim=1) < R * R  # noqa: E731
    outside = lambda p: ((p - c) ** 2).sum(dim=1) >= R * R  # noqa: E731
    drop = rsa_positions(n_drop, L, 0.9, seed, device=device, region=inside)
    pos = rsa_positions(n - n_drop, L, 0.9, seed + 7, device=device, region=outside,
                        existing=drop)
    return Workload(f"c3-droplet-{n}", pos, L, 3.0, 0.3,
                    maxwell_boltzmann(n, 1.2, seed + 1, device=device),
                    "droplet rho 0.8 r=0.3L + vapour rho 0.05; RSA dmin 0.9 (builder's choice)")


def config4(side: int = 256, seed: int = 42, device="cpu") -> Workload:
    """side^3 SC lattice at rho 0.8 + N(0, 0.05^2) per component, rc 2.5, skin 0.3."""
    a = (1.0 / 0.8) ** (1.0 / 3.0)
    L = side * a
    pos = torch.as_tensor(lattice_positions((0.0, 0.0, 0.0), (side,) * 3, a), device=device)
    g = torch.Generator(device="cpu").manual_seed(seed)
    pos = pos + (torch.randn(pos.shape, generator=g, dtype=torch.float64) * 0.05).to(device)
    pos = torch.remainder(pos, L)
    return Workload(f"c4-lattice-{side ** 3}", pos, L, 2.5, 0.3,
                    maxwell_boltzmann(side ** 3, 1.0, seed + 1, device=device))


def config5(n: int = 8_388_608, seed: int = 42, device="cpu") -> Workload:
    """Uniform gas at rho 0.3 (per GPU brick), RSA min distance 0.9, rc 2.5, T 0.7."""
    L = (n / 0.3) ** (1.0 / 3.0)
    pos = rsa_positions(n, L, 0.9, seed, device=device)
    return Workload(f"c5-gas-rho0.3-{n}", pos, L, 2.5, 0.3,
                    maxwell_boltzmann(n, 0.7, seed + 1, device=device), "RSA dmin 0.9")
