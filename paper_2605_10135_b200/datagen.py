"""Seeded synthetic inputs shared by the CUDA path, the oracle tests and bench.py.

This module holds NO arithmetic of the method (no distances, no partition rule,
no graph logic): it only draws numbers.  Both sides (the CUDA path through
``paper_2605_10135_b200.api`` and the CPU ``oracle/``) are fed the arrays it
returns, so parity compares the two implementations on identical inputs.

Workload shapes follow the paper's datasets (PAPER.md Table ``tab:dataset``,
lines 391-416: Sift 128-d uint8, Deep 96-d float, Laion 768-d float) and the
recipe of SURVEY.md §8(d) "Generator parameters":

* Gaussian mixture with ``K_MIX = 1024`` components of uniform weight, centres
  ``mu_c ~ N(0, I)``; a point is ``mu_c + 1.5 * sqrt(lambda) * z`` with
  ``lambda_i = i^-beta`` normalised to mean 1 (beta 0.3 SIFT-like, 0.7
  DEEP-like, 1.0 text-like).
* SIFT-shaped (C1 float, C4 uint8): ``clip(round(30 * max(0, x + 0.4)), 0, 255)``
  which gives ~41% zeros and mean norm ~512, integer valued.  The spread 1.5 (not the
  0.35 SURVEY §8(d) proposed) makes neighbouring components overlap as real descriptors do:
  at 0.35 the ~1000 points per component of a 1M dataset form disjoint exact-kNN graphs
  (one strong component per mixture component, recall@10 ~ 0.06 even for the oracle-built
  graph); at 1.5 the graph is connected and the oracle-built graph reaches recall ~0.99.
* DEEP/text-shaped: rows L2-normalised.
* C0: iid N(0, 1).

Generation is chunked by 2**20 rows, chunk ``c`` seeded ``seed + 7919*c``, so
the result does not depend on the device or on how many rows are asked for
beyond the chunk boundary; the mixture centres come from their own seed so that
queries (``seed + 1000``) share the dataset's centres.
"""
from __future__ import annotations

import dataclasses

import torch

K_MIX = 1024
SPREAD = 1.5
SIFT_SCALE = 30.0
SIFT_OFFSET = 0.4
CHUNK = 1 << 20
DATA_SEED = 0x5CA1E
QUERY_SEED_OFFSET = 1000
CENTRE_SEED = 0xC3E7


def _spectrum(d: int, beta: float) -> torch.Tensor:
    lam = torch.arange(1, d + 1, dtype=torch.float64) ** (-beta)
    lam = lam / lam.mean()
    return lam.sqrt().to(torch.float32)


def _centres(d: int) -> torch.Tensor:
    g = torch.Generator(device="cpu").manual_seed(CENTRE_SEED + d)
    return torch.randn(K_MIX, d, generator=g, dtype=torch.float32)


def _mixture_chunk(rows: int, d: int, beta: float, seed: int, device) -> torch.Tensor:
    g = torch.Generator(device=device).manual_seed(seed)
    comp = torch.randint(0, K_MIX, (rows,), generator=g, device=device)
    z = torch.randn(rows, d, generator=g, device=device, dtype=torch.float32)
    mu = _centres(d).to(device)
    return mu[comp] + SPREAD * _spectrum(d, beta).to(device) * z


def gaussian(n: int, d: int, seed: int = DATA_SEED, device="cpu") -> torch.Tensor:
    """C0: n x d float32, iid N(0,1)."""
    out = torch.empty(n, d, dtype=torch.float32, device=device)
    for c, r0 in enumerate(range(0, n, CHUNK)):
        r1 = min(n, r0 + CHUNK)
        g = torch.Generator(device=device).manual_seed(seed + 7919 * c)
        out[r0:r1] = torch.randn(r1 - r0, d, generator=g, device=device, dtype=torch.float32)
    return out


def mixture(n: int, d: int, beta: float, seed: int = DATA_SEED, normalise: bool = False,
            device="cpu") -> torch.Tensor:
    out = torch.empty(n, d, dtype=torch.float32, device=device)
    for c, r0 in enumerate(range(0, n, CHUNK)):
        r1 = min(n, r0 + CHUNK)
        x = _mixture_chunk(r1 - r0, d, beta, seed + 7919 * c, device)
        if normalise:
            x = x / x.norm(dim=1, keepdim=True).clamp_min(1e-12)
        out[r0:r1] = x
    return out


def sift_like(n: int, d: int = 128, seed: int = DATA_SEED, as_u8: bool = False,
              device="cpu") -> torch.Tensor:
    """SIFT/BIGANN-shaped integer data in [0, 255] (float32 holding integers, or uint8)."""
    out = torch.empty(n, d, dtype=torch.uint8 if as_u8 else torch.float32, device=device)
    for c, r0 in enumerate(range(0, n, CHUNK)):
        r1 = min(n, r0 + CHUNK)
        x = _mixture_chunk(r1 - r0, d, 0.3, seed + 7919 * c, device)
        y = torch.clamp(torch.round(SIFT_SCALE * torch.clamp_min(x + SIFT_OFFSET, 0.0)), 0, 255)
        out[r0:r1] = y.to(out.dtype)
    return out


@dataclasses.dataclass(frozen=True)
class Workload:
    """One synthetic workload (BASELINE.json ``configs``)."""
    name: str
    n: int
    d: int
    kind: str           # "gauss" | "sift" | "sift_u8" | "deep" | "text"
    k: int              # shards (= k-means clusters)
    omega: int = 2      # max homes per vector ("replication 2")
    L: int = 128        # intermediate kNN degree
    R: int = 64         # final out-degree
    nq: int = 1000

    def data(self, device="cpu", seed: int = DATA_SEED) -> torch.Tensor:
        return _make(self.kind, self.n, self.d, seed, device)

    def queries(self, device="cpu", seed: int = DATA_SEED) -> torch.Tensor:
        return _make(self.kind, self.nq, self.d, seed + QUERY_SEED_OFFSET, device)


def _make(kind: str, n: int, d: int, seed: int, device) -> torch.Tensor:
    if kind == "gauss":
        return gaussian(n, d, seed, device)
    if kind == "sift":
        return sift_like(n, d, seed, False, device)
    if kind == "sift_u8":
        return sift_like(n, d, seed, True, device)
    if kind == "deep":
        return mixture(n, d, 0.7, seed, True, device)
    if kind == "text":
        return mixture(n, d, 1.0, seed, True, device)
    raise ValueError(kind)


C0 = Workload("C0-gauss-10Kx128-f32", 10_000, 128, "gauss", k=2, omega=2, L=64, R=32, nq=1000)
C1 = Workload("C1-sift1M-1Mx128-f32", 1_000_000, 128, "sift", k=4, omega=2, L=128, R=64, nq=10_000)
C2 = Workload("C2-deep10M-10Mx96-f32", 10_000_000, 96, "deep", k=8, omega=2, L=128, R=64, nq=10_000)
C3 = Workload("C3-text5M-5Mx768-f32", 5_000_000, 768, "text", k=8, omega=2, L=128, R=64, nq=10_000)
C4 = Workload("C4-bigann100M-100Mx128-u8", 100_000_000, 128, "sift_u8", k=8, omega=2, L=128, R=64,
              nq=10_000)
CONFIGS = {"C0": C0, "C1": C1, "C2": C2, "C3": C3, "C4": C4}
