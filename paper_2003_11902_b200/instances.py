"""Seeded synthetic TSP instances shaped like the paper's TSPLIB set.

This module is the ONE piece shared by the CUDA path and the oracle: it only
draws integer city coordinates (and names the five workload configurations).
It holds none of the method's arithmetic -- no distances, weights, random keys
or pheromone -- so it cannot make the two sides agree by construction.

The paper runs on TSPLIB instances (Sec. 5); those files
are not available here, so each configuration gets a synthetic EUC_2D instance
with the size and point distribution of its TSPLIB namesake (DESIGN.md "Input
recipe"): uniform squares sized so that the BHH estimate 0.7124*sqrt(n*A)
matches the TSPLIB optimum for the pr*/d18512 shapes, Gaussian clusters for
the drilling (d198) and fl3795 shapes.  Coordinates are integers (exact
distances on both sides), and exact duplicates are redrawn.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

_MASK64 = (1 << 64) - 1


class SplitMix64:
    """Steele/Lea/Flood SplitMix64 (public-domain reference constants)."""

    def __init__(self, seed: int):
        self.state = seed & _MASK64

    def next_u64(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & _MASK64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK64
        return z ^ (z >> 31)

    def uniform(self) -> float:
        """Double in [0, 1) from the top 53 bits."""
        return (self.next_u64() >> 11) * (1.0 / 9007199254740992.0)

    def below(self, k: int) -> int:
        return int(self.uniform() * k)

    def gauss(self) -> float:
        """Standard normal by Box-Muller (one value per call; the pair's twin is dropped)."""
        u1 = 1.0 - self.uniform()
        u2 = self.uniform()
        return math.sqrt(-2.0 * math.log(u1)) * math.cos(2.0 * math.pi * u2)


def _unique_points(n: int, draw) -> np.ndarray:
    seen = set()
    pts = []
    while len(pts) < n:
        p = draw()
        if p in seen:
            continue
        seen.add(p)
        pts.append(p)
    return np.asarray(pts, dtype=np.float64).reshape(n, 2)


def uniform_square(n: int, side: int, seed: int) -> np.ndarray:
    g = SplitMix64(seed)
    return _unique_points(n, lambda: (g.below(side), g.below(side)))


def clustered(n: int, side: int, clusters: int, sigma: float, seed: int, frac_uniform: float = 0.0) -> np.ndarray:
    g = SplitMix64(seed)
    centres = [(g.uniform() * side, g.uniform() * side) for _ in range(clusters)]
    n_uni = int(round(frac_uniform * n))
    state = {"k": 0}

    def draw():
        k = state["k"]
        state["k"] = k + 1
        if k < n_uni:
            return (g.below(side), g.below(side))
        cx, cy = centres[g.below(clusters)]
        x = int(round(cx + sigma * g.gauss()))
        y = int(round(cy + sigma * g.gauss()))
        return (min(max(x, 0), side - 1), min(max(y, 0), side - 1))

    return _unique_points(n, draw)


@dataclass(frozen=True)
class Workload:
    """One BASELINE.json configuration."""

    name: str
    n: int
    n_ants: int
    cand_len: int
    iterations: int
    rho: float
    local_search: int
    shape: str
    seed: int
    alpha: float = 1.0
    beta: float = 2.0
    mmas_seed: int = 42
    tabu: int = 0         # full-row tabu: 0 = bitmask (BT), 1 = compact (CT, R27)
    selection: int = 0    # node selection: 0 = WRS (Alg. 3), 1 = parallel roulette wheel (R28)
    colonies: int = 1     # concurrent independent colonies, colony c seeded mmas_seed + c (R29)
    pheromone: int = 0    # 0 = dense n x n matrices, 1 = memory-lean (R30, same results)

    def coords(self) -> np.ndarray:
        return make_coords(self.shape, self.n, self.seed)


def make_coords(shape: str, n: int, seed: int) -> np.ndarray:
    if shape == "d198":
        return clustered(n, 1600, 6, 40.0, seed, frac_uniform=0.6)
    if shape == "pr1002":
        return uniform_square(n, 11500, seed)
    if shape == "fl3795":
        return clustered(n, 4000, 50, 15.0, seed)
    if shape == "pr2392":
        return uniform_square(n, 10850, seed)
    if shape == "d18512":
        return uniform_square(n, 6660, seed)
    if shape == "uniform":
        side = max(4, int(math.sqrt(n) * 100))
        return uniform_square(n, side, seed)
    raise ValueError(f"unknown shape {shape!r}")


CONFIGS = {
    "C1": Workload("d198-shaped", 198, 198, 16, 50, 0.5, 0, "d198", 198),
    "C2": Workload("pr1002-shaped", 1002, 1002, 32, 1000, 0.5, 0, "pr1002", 1002),
    "C3": Workload("fl3795-shaped", 3795, 3795, 32, 100, 0.5, 0, "fl3795", 3795),
    "C4": Workload("pr2392-shaped", 2392, 2392, 0, 100, 0.5, 0, "pr2392", 2392),
    # C4 over the compact tabu (MMAS-WRS-CT, the paper's choice without candidate lists)
    "C4CT": Workload("pr2392-shaped, compact tabu", 2392, 2392, 0, 100, 0.5, 0, "pr2392", 2392, tabu=1),
    # the paper's comparison (T3-T6): the same workloads with the parallel roulette wheel
    "C2RWM": Workload("pr1002-shaped, roulette wheel", 1002, 1002, 32, 1000, 0.5, 0, "pr1002", 1002, selection=1),
    "C4RWM": Workload("pr2392-shaped, roulette wheel", 2392, 2392, 0, 100, 0.5, 0, "pr2392", 2392, selection=1),
    "C4RWMCT": Workload("pr2392-shaped, roulette wheel, compact tabu", 2392, 2392, 0, 100, 0.5, 0, "pr2392", 2392,
                        tabu=1, selection=1),
    "C5": Workload("d18512-shaped", 18512, 800, 32, 20, 0.7, 1, "d18512", 18512),
    # 8 concurrent independent pr1002-shaped colonies (the paper's repeated-run
    # protocol P:1143-1145) in one context, every launch running all eight
    # the memory-lean pheromone (R30) on the d18512 workload (~20 MB of pheromone
    # state instead of 3 x 1.37 GB) and on the largest u16 instance (n = 65535)
    "C5L": Workload("d18512-shaped, lean pheromone", 18512, 800, 32, 20, 0.7, 1, "d18512", 18512, pheromone=1),
    "C65KL": Workload("65535-city uniform, lean pheromone", 65535, 800, 32, 10, 0.7, 0, "uniform", 65535,
                      pheromone=1),
    "C2x8": Workload("pr1002-shaped, 8 concurrent colonies", 1002, 1002, 32, 1000, 0.5, 0, "pr1002", 1002,
                     colonies=8),
}
