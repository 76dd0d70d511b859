"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds NO arithmetic of the method (no contraction, no MTTKRP,
no solve). It only fixes *inputs*:

* the five BASELINE.json configurations (shape, rank R, noise, seeds),
* factor matrices drawn on the host with NumPy ``Generator(PCG64(seed))``
  (true factors, initial factors), including the collinearity construction
  of PAPER.md §V "Tensor 1",
* the *specification* of the counter-based element generator used for the
  tensor noise / the uniform C3 entries: SplitMix64 keyed by
  (seed, global linear index).  Both sides implement it independently: the
  CUDA kernel ``cpd_gen_tensor`` in ``libcpd.so`` and the NumPy version
  below (used by the oracle to build T).  The hash is defined here once, in
  words and in NumPy, so a reader can compare the CUDA code against it.

Readings: "N(0, x)" noise in BASELINE.json is read
as variance x; initial factors are N(0,1) per BASELINE (Q11);
collinearity is fixed at C=0.5 for C4 (Q13).
"""
from __future__ import annotations

import dataclasses
import numpy as np

MASK64 = np.uint64(0xFFFFFFFFFFFFFFFF)
GOLDEN = np.uint64(0x9E3779B97F4A7C15)


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    N: int
    s: int
    R: int
    kind: str            # "kruskal" (exact rank + Gaussian noise) | "uniform" (i.i.d. U(0,1))
    true_rank: int
    noise_var: float     # variance of the additive Gaussian noise (Q12)
    collinearity: float  # C for the collinear factor construction; None/-1 -> plain N(0,1) factors
    seed_true: int
    seed_noise: int
    seed_init: int
    dims: tuple = None   # non-equidimensional shape (s_1..s_N); None -> (s,) * N

    @property
    def shape(self):
        return tuple(self.dims) if self.dims else (self.s,) * self.N

    @property
    def numel(self):
        n = 1
        for d in self.shape:
            n *= d
        return n


def config(c: int) -> Config:
    """BASELINE.json configs[c-1] (c = 1..5), seeds per SURVEY §8(d)."""
    table = {
        1: dict(N=3, s=64, R=8, kind="kruskal", true_rank=8, noise_var=1e-6, collinearity=-1.0),
        2: dict(N=3, s=1024, R=64, kind="kruskal", true_rank=64, noise_var=1e-4, collinearity=-1.0),
        3: dict(N=4, s=200, R=100, kind="uniform", true_rank=0, noise_var=0.0, collinearity=-1.0),
        4: dict(N=5, s=64, R=32, kind="kruskal", true_rank=32, noise_var=1e-3, collinearity=0.5),
        5: dict(N=3, s=2048, R=200, kind="kruskal", true_rank=200, noise_var=1e-4, collinearity=-1.0),
    }[c]
    return Config(name=f"C{c}", seed_true=1000 + c, seed_noise=2000 + c, seed_init=3000 + c, **table)


def custom(N, s, R, kind="kruskal", true_rank=None, noise_var=1e-6, collinearity=-1.0, seed=7, dims=None):
    """A small ad-hoc configuration for tests (same recipe as the BASELINE configs); `dims`
    gives a non-equidimensional shape (then N = len(dims) and s is unused)."""
    if dims is not None:
        dims = tuple(int(d) for d in dims)
        N = len(dims)
    name = f"N{N}s{s}R{R}" if dims is None else "x".join(map(str, dims)) + f"R{R}"
    return Config(name=name, N=N, s=s, R=R, kind=kind,
                  true_rank=R if true_rank is None else true_rank, noise_var=noise_var,
                  collinearity=collinearity, seed_true=1000 + seed, seed_noise=2000 + seed,
                  seed_init=3000 + seed, dims=dims)


def gaussian_factors(shape, R, seed):
    """N factor matrices s_n x R, i.i.d. N(0,1), row-major float64 (BASELINE.json configs)."""
    g = np.random.Generator(np.random.PCG64(seed))
    return [np.ascontiguousarray(g.standard_normal((s, R))) for s in shape]


def collinear_factors(shape, R, C, seed):
    """Factor matrices whose columns have pairwise cosine exactly C.

    Construction: an orthonormal set {u, v_1..v_R}
    from the QR of a seeded s x (R+1) Gaussian; a_r = sqrt(C) u + sqrt(1-C) v_r,
    then scaled to ||a_r|| = sqrt(s) (unit-RMS entries).  Needs s >= R+1.
    """
    g = np.random.Generator(np.random.PCG64(seed))
    out = []
    for s in shape:
        if s < R + 1:
            raise ValueError("collinear construction needs s >= R+1")
        q, _ = np.linalg.qr(g.standard_normal((s, R + 1)))
        u, V = q[:, :1], q[:, 1:]
        A = np.sqrt(C) * u + np.sqrt(1.0 - C) * V
        out.append(np.ascontiguousarray(A * np.sqrt(s)))
    return out


def true_factors(cfg: Config):
    if cfg.kind != "kruskal":
        return None
    if cfg.collinearity is not None and cfg.collinearity >= 0:
        return collinear_factors(cfg.shape, cfg.true_rank, cfg.collinearity, cfg.seed_true)
    return gaussian_factors(cfg.shape, cfg.true_rank, cfg.seed_true)


def init_factors(cfg: Config):
    """Initial ALS factors: i.i.d. N(0,1) from seed_init (BASELINE)."""
    return gaussian_factors(cfg.shape, cfg.R, cfg.seed_init)


# ---------------------------------------------------------------------------
# Counter-based element generator (specification + NumPy implementation).
#
#   splitmix64(x):  z = x + 0x9E3779B97F4A7C15
#                   z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9
#                   z = (z ^ (z >> 27)) * 0x94D049BB133111EB
#                   return z ^ (z >> 31)                      (all mod 2^64)
#   key            = splitmix64(seed)
#   u(i, lane)     = (splitmix64(key ^ (2*i + lane)) >> 11) * 2^-53    in [0,1)
#   uniform(i)     = u(i, 0)
#   normal(i)      = sqrt(-2 ln(1 - u(i,0))) * cos(2*pi*u(i,1))         (Box-Muller)
# i is the GLOBAL row-major linear index of the tensor element, so every rank
# generates only its slab and the tensor does not depend on the GPU count.
# ---------------------------------------------------------------------------

def _splitmix64(x):
    with np.errstate(over="ignore"):
        z = (x + GOLDEN) & MASK64
        z = ((z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)) & MASK64
        z = ((z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)) & MASK64
        return z ^ (z >> np.uint64(31))


def _key(seed):
    return _splitmix64(np.uint64(seed))


def hash_uniform(seed, idx, lane=0):
    """u(idx, lane) in [0, 1) for an array of uint64 global indices."""
    idx = np.asarray(idx, dtype=np.uint64)
    h = _splitmix64(_key(seed) ^ (np.uint64(2) * idx + np.uint64(lane)))
    return (h >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def hash_normal(seed, idx):
    u1 = hash_uniform(seed, idx, 0)
    u2 = hash_uniform(seed, idx, 1)
    return np.sqrt(-2.0 * np.log1p(-u1)) * np.cos(2.0 * np.pi * u2)


def element_noise(cfg: Config, idx):
    """The additive term of T at global linear indices idx (before adding the Kruskal part).

    kruskal: sqrt(noise_var) * normal(idx);  uniform: uniform(idx) (the whole entry).
    """
    if cfg.kind == "uniform":
        return hash_uniform(cfg.seed_noise, idx, 0)
    if cfg.noise_var == 0.0:
        return np.zeros(np.shape(idx))
    return np.sqrt(cfg.noise_var) * hash_normal(cfg.seed_noise, idx)


def slab_range(s_last, rank, world):
    """1-D block partition of the last mode (Alg. 3 grid 1x..x1xP).

    Returns [lo, hi) of the rows of mode N owned by `rank`. s_last must divide
    evenly (all configs do)."""
    if s_last % world != 0:
        raise ValueError("s_N must be divisible by the number of ranks")
    b = s_last // world
    return rank * b, (rank + 1) * b
