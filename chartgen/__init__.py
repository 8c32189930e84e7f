"""Seeded synthetic chart-set generator shared by the oracle tests and the CUDA path.

This module holds NONE of the packing method's arithmetic: it only draws
polygons. Both sides (``oracle/`` and ``paper_2602_07782_b200``) consume its
output; neither imports the other.

Workload shapes follow SURVEY.md §8(d) (which restates the paper's workload
structure, "Results", 1021 "Experimental Setup"):

* ``mixed``    -- C1a: 16 charts of every family, sides U[16, 64], 256^2 atlas.
* ``rectl``    -- C1b: 16 rectangles / L-shapes, sides U[60, 76] (forces downscale).
* ``uv``       -- C2: UV-unwrap-like, side ~ logN(ln 64, 0.9), aspect logU[1, 3],
                  60 % concave (L / U / star), fill ratio rho = 1.1, 1024^2.
* ``tss``      -- C3/C5: texture-space-shading-like, side ~ logN(ln 16, 1.2)
                  clipped to [3, 0.25 W], random rotation, convex/star heavy.
* ``lightmap`` -- C4: 80 % axis-aligned rectangles + 20 % L / trapezoid quads,
                  sides U[4, 48], rho = 0.8, 8192^2.

All charts are then scaled by ONE common factor so that the total polygon
area is rho * W * H (P:1021 packs at sizes "where downscaling may often be
unavoidable"), charts whose longest side exceeds the config's side limit are
shrunk to it once, and every coordinate is snapped to the 1/256-texel grid so
float32 holds it exactly.

Randomness is SplitMix64 (Steele et al. 2014) so that any consumer can
re-derive the same stream.
"""
from __future__ import annotations

import hashlib
import math
from dataclasses import dataclass, field

import numpy as np

MASK64 = (1 << 64) - 1


class SplitMix64:
    """SplitMix64 counter-based PRNG (public-domain reference algorithm)."""

    def __init__(self, seed: int):
        self.state = seed & MASK64

    def next_u64(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & MASK64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
        return z ^ (z >> 31)

    def uniform(self, lo: float = 0.0, hi: float = 1.0) -> float:
        return lo + (hi - lo) * ((self.next_u64() >> 11) * (1.0 / (1 << 53)))

    def randint(self, lo: int, hi: int) -> int:
        """Uniform integer in [lo, hi] inclusive."""
        return lo + self.next_u64() % (hi - lo + 1)

    def normal(self) -> float:
        u1 = max(self.uniform(), 1e-300)
        u2 = self.uniform()
        return math.sqrt(-2.0 * math.log(u1)) * math.cos(2.0 * math.pi * u2)


def splitmix64_hash(i: int) -> int:
    """One SplitMix64 output for counter i (used for per-atlas sizes in C5)."""
    return SplitMix64(i).next_u64()


@dataclass
class ChartSet:
    """Charts as polygon outlines in texel units (y grows downward)."""

    name: str
    xy: np.ndarray          # float32 [2V]: x0, y0, x1, y1, ...
    start: np.ndarray       # int32 [N+1]: chart c = vertices [start[c], start[c+1])
    atlas_w: int
    atlas_h: int
    gutter: int = 1
    scale_count: int = 64
    local_aabb_count: int = 10
    t_opt_bp: int = 0
    res: float = 1.0
    meta: dict = field(default_factory=dict)

    @property
    def n_charts(self) -> int:
        return int(self.start.shape[0] - 1)

    @property
    def n_vertices(self) -> int:
        return int(self.start[-1])

    def polygon(self, c: int) -> np.ndarray:
        a, b = int(self.start[c]), int(self.start[c + 1])
        return self.xy[2 * a:2 * b].reshape(-1, 2)

    def sha256(self) -> str:
        h = hashlib.sha256()
        h.update(np.ascontiguousarray(self.start, dtype="<i4").tobytes())
        h.update(np.ascontiguousarray(self.xy, dtype="<f4").tobytes())
        return h.hexdigest()


# ----------------------------------------------------------------------------
# Shape families (unit-free outlines; later scaled and translated)
# ----------------------------------------------------------------------------

def _rect(a, b, rng):
    return [(0.0, 0.0), (a, 0.0), (a, b), (0.0, b)]


def _tri(a, b, rng):
    corner = rng.randint(0, 3)
    pts = [[(0.0, 0.0), (a, 0.0), (0.0, b)],
           [(0.0, 0.0), (a, 0.0), (a, b)],
           [(a, 0.0), (a, b), (0.0, b)],
           [(0.0, 0.0), (a, b), (0.0, b)]][corner]
    return pts


def _lshape(a, b, rng):
    t = rng.uniform(0.25, 0.75)
    u = rng.uniform(0.25, 0.75)
    pts = [(0.0, 0.0), (a * u, 0.0), (a * u, b * t), (a, b * t), (a, b), (0.0, b)]
    if rng.randint(0, 1):  # mirror half of them so every orientation occurs
        pts = [(a - x, y) for (x, y) in reversed(pts)]
    if rng.randint(0, 1):
        pts = [(x, b - y) for (x, y) in reversed(pts)]
    return pts


def _ushape(a, b, rng):
    u1 = rng.uniform(0.2, 0.4)
    u2 = rng.uniform(0.6, 0.8)
    t = rng.uniform(0.3, 0.8)
    pts = [(0.0, 0.0), (a * u1, 0.0), (a * u1, b * t), (a * u2, b * t), (a * u2, 0.0),
           (a, 0.0), (a, b), (0.0, b)]
    if rng.randint(0, 1):
        pts = [(x, b - y) for (x, y) in reversed(pts)]
    return pts


def _trapezoid(a, b, rng):
    d1 = rng.uniform(0.0, 0.4) * a
    d2 = rng.uniform(0.0, 0.4) * a
    return [(d1, 0.0), (a - d2, 0.0), (a, b), (0.0, b)]


def _convex(a, b, rng):
    n = rng.randint(5, 12)
    pts = []
    for i in range(n):
        th = 2.0 * math.pi * (i + rng.uniform(-0.3, 0.3)) / n
        pts.append((0.5 * a * (1.0 + math.cos(th)), 0.5 * b * (1.0 + math.sin(th))))
    return pts


def _star(a, b, rng):
    n = rng.randint(8, 24)
    pts = []
    for i in range(n):
        th = 2.0 * math.pi * (i + rng.uniform(-0.3, 0.3)) / n
        r = rng.uniform(0.45, 1.0)
        pts.append((0.5 * a * (1.0 + r * math.cos(th)), 0.5 * b * (1.0 + r * math.sin(th))))
    return pts


FAMILIES = {
    "rect": _rect, "tri": _tri, "L": _lshape, "U": _ushape,
    "trap": _trapezoid, "convex": _convex, "star": _star,
}


def _rotate(pts, th):
    c, s = math.cos(th), math.sin(th)
    return [(x * c - y * s, x * s + y * c) for (x, y) in pts]


def _area(pts):
    s = 0.0
    for i in range(len(pts)):
        x0, y0 = pts[i]
        x1, y1 = pts[(i + 1) % len(pts)]
        s += x0 * y1 - x1 * y0
    return abs(s) * 0.5


def _extent(pts):
    xs = [p[0] for p in pts]
    ys = [p[1] for p in pts]
    return max(xs) - min(xs), max(ys) - min(ys)


def _pick(rng, table):
    u = rng.uniform()
    acc = 0.0
    for name, p in table:
        acc += p
        if u < acc:
            return name
    return table[-1][0]


def _draw_chart(family: str, rng: SplitMix64, atlas_w: int):
    """Return an outline (list of (x, y)) for one chart of the given workload family."""
    if family == "mixed":
        a, b = rng.uniform(16, 64), rng.uniform(16, 64)
        kind = _pick(rng, [("rect", 1 / 7), ("tri", 1 / 7), ("L", 1 / 7), ("U", 1 / 7),
                           ("convex", 1 / 7), ("star", 1 / 7), ("rrect", 1 / 7)])
        if kind == "rrect":
            return _rotate(_rect(a, b, rng), rng.uniform(0, 2 * math.pi))
        return FAMILIES[kind](a, b, rng)
    if family == "rectl":
        a, b = rng.uniform(60, 76), rng.uniform(60, 76)
        return FAMILIES["rect" if rng.randint(0, 1) else "L"](a, b, rng)
    if family == "uv":
        side = math.exp(math.log(64.0) + 0.9 * rng.normal())
        aspect = math.exp(rng.uniform(0.0, math.log(3.0)))
        a, b = side * math.sqrt(aspect), side / math.sqrt(aspect)
        if rng.randint(0, 1):
            a, b = b, a
        kind = _pick(rng, [("L", 0.2), ("U", 0.2), ("star", 0.2),
                           ("convex", 0.15), ("rect", 0.15), ("tri", 0.1)])
        return FAMILIES[kind](a, b, rng)
    if family == "tss":
        side = math.exp(math.log(16.0) + 1.2 * rng.normal())
        side = min(max(side, 3.0), 0.25 * atlas_w)
        aspect = math.exp(rng.uniform(0.0, math.log(2.0)))
        a, b = side * math.sqrt(aspect), side / math.sqrt(aspect)
        kind = _pick(rng, [("convex", 0.45), ("star", 0.35), ("tri", 0.1), ("rect", 0.1)])
        return _rotate(FAMILIES[kind](a, b, rng), rng.uniform(0, 2 * math.pi))
    if family == "lightmap":
        a, b = rng.uniform(4, 48), rng.uniform(4, 48)
        if rng.uniform() < 0.8:
            return _rect(a, b, rng)
        return FAMILIES["L" if rng.randint(0, 1) else "trap"](a, b, rng)
    raise ValueError(f"unknown family {family!r}")


def generate(family: str, n: int, atlas_w: int, atlas_h: int, seed: int, rho: float | None,
             side_limit: float | None = None, min_side: float = 1.0, name: str | None = None,
             **spec) -> ChartSet:
    """Generate ``n`` charts of ``family``.

    rho: target fill ratio (sum of polygon areas / (W*H)); None keeps raw sizes.
    side_limit: longest-side cap applied once after the common rescale.
    """
    if n < 1:
        raise ValueError("n must be >= 1")
    rng = SplitMix64(seed * 0x100000001B3 + 0x5EED)
    charts = [_draw_chart(family, rng, atlas_w) for _ in range(n)]
    if rho is not None:
        total = sum(_area(p) for p in charts)
        f = math.sqrt(rho * atlas_w * atlas_h / total)
        charts = [[(x * f, y * f) for (x, y) in p] for p in charts]
    out_xy = []
    start = [0]
    for p in charts:
        ex, ey = _extent(p)
        big = max(ex, ey)
        g = 1.0
        if side_limit is not None and big > side_limit:
            g = side_limit / big
        elif big * g < min_side:
            g = min_side / big
        ox = rng.uniform(0, atlas_w)
        oy = rng.uniform(0, atlas_h)
        mx = min(q[0] for q in p)
        my = min(q[1] for q in p)
        for (x, y) in p:
            X = round(((x - mx) * g + ox) * 256.0) / 256.0
            Y = round(((y - my) * g + oy) * 256.0) / 256.0
            out_xy.extend((X, Y))
        start.append(start[-1] + len(p))
    return ChartSet(name=name or f"{family}-n{n}-s{seed}",
                    xy=np.asarray(out_xy, dtype=np.float32),
                    start=np.asarray(start, dtype=np.int32),
                    atlas_w=atlas_w, atlas_h=atlas_h,
                    meta={"family": family, "seed": seed, "rho": rho}, **spec)


# ----------------------------------------------------------------------------
# The five workloads of BASELINE.json "configs"
# ----------------------------------------------------------------------------

def config1a(seed: int = 0) -> ChartSet:
    return generate("mixed", 16, 256, 256, seed, rho=None, name=f"C1a-s{seed}")


def config1b(seed: int = 0) -> ChartSet:
    return generate("rectl", 16, 256, 256, seed, rho=None, name=f"C1b-s{seed}")


def config2(seed: int = 0) -> ChartSet:
    return generate("uv", 214, 1024, 1024, seed, rho=1.1, side_limit=1024, name=f"C2-s{seed}")


def config3(seed: int = 0, rho: float = 0.5, k: int = 10, t_opt_bp: int = 0) -> ChartSet:
    return generate("tss", 1572, 4096, 4096, seed, rho=rho, side_limit=1024,
                    name=f"C3-rho{rho}-s{seed}", local_aabb_count=k, t_opt_bp=t_opt_bp)


def config4(seed: int = 0, t_opt_bp: int = -1) -> ChartSet:
    return generate("lightmap", 20000, 8192, 8192, seed, rho=0.8, side_limit=2048,
                    name=f"C4-s{seed}", t_opt_bp=t_opt_bp)


def config5_sizes(n_atlases: int = 512):
    return [200 + splitmix64_hash(i) % 1801 for i in range(n_atlases)]


def config5(i: int) -> ChartSet:
    n = config5_sizes(i + 1)[i]
    rng = SplitMix64(0xC5C5 + i)
    rho = rng.uniform(0.3, 1.5)
    return generate("tss", n, 2048, 2048, 1000 + i, rho=rho, side_limit=512, name=f"C5-{i}")


def small_case(seed: int = 0, n: int = 40, side: int = 256, family: str = "tss",
               rho: float = 0.6, **spec) -> ChartSet:
    """A case the oracle finishes in well under a second (several rows, ragged tail)."""
    return generate(family, n, side, side, seed, rho=rho, side_limit=side / 2,
                    name=f"small-{family}-n{n}-s{seed}", **spec)


def from_polygons(polys, atlas_w, atlas_h, name="custom", **spec) -> ChartSet:
    """Build a ChartSet from explicit outlines (used by golden fixtures)."""
    xy, start = [], [0]
    for p in polys:
        for (x, y) in p:
            xy.extend((float(x), float(y)))
        start.append(start[-1] + len(p))
    return ChartSet(name=name, xy=np.asarray(xy, dtype=np.float32),
                    start=np.asarray(start, dtype=np.int32), atlas_w=atlas_w,
                    atlas_h=atlas_h, **spec)
