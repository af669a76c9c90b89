"""The five BASELINE.json configurations, as (geometry, p, spans, forms, M)."""
from __future__ import annotations

from dataclasses import dataclass

from .geometry import quarter_annulus, sin_map_standin, twisted_cube_standin


@dataclass(frozen=True)
class Config:
    idx: int
    name: str
    geometry: str
    p: int
    spans: tuple
    forms: tuple
    M: int
    q: int = 3

    def geom(self):
        return {"annulus": lambda: quarter_annulus(1.0, 2.0), "twisted": twisted_cube_standin,
                "sinmap": sin_map_standin}[self.geometry]()


CONFIGS = {
    1: Config(1, "annulus32_p2_poisson", "annulus", 2, (32, 32), ("poisson",), 8),
    2: Config(2, "annulus512_p3_poisson_mass", "annulus", 3, (512, 512), ("poisson", "mass"), 16),
    3: Config(3, "twisted64_p2_poisson", "twisted", 2, (64, 64, 64), ("poisson",), 8),
    4: Config(4, "sinmap1024_p3_biharmonic", "sinmap", 3, (1024, 1024), ("biharmonic",), 32),
    5: Config(5, "twisted128_p3_poisson_mass", "twisted", 3, (128, 128, 128), ("poisson", "mass"), 16),
}
