"""The five BASELINE.json workloads (synthetic, seeded).

Generator (not in the reference): per plane, K Voronoi
regions with levels U[0,1] + a linear ramp of amplitude 0.2
(0.2 * ((x/(W-1) + y/(H-1))/2 - 0.5)) + N(0, 0.03^2) noise, plus 5%
salt-and-pepper for c3, clipped to [0,1].  RGB channels use independent
seeds; the joint config's grayscale guide uses its own seed:
seed = 1000*cfg + 10*image + channel, guide seed = 1000*cfg + 500 + image.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Config:
    name: str
    index: int          # 1-based position in BASELINE.json "configs"
    height: int
    width: int
    channels: int
    batch: int
    radius: int
    sigma_s: float
    sigma_r: float
    lam: float
    iters: int
    n_sites: int = 12
    p_salt_pepper: float = 0.0
    guide: bool = False  # joint BLF with a separate grayscale guide

    def seeds(self, image: int) -> list[int]:
        return [1000 * self.index + 10 * image + c for c in range(self.channels)]

    def guide_seed(self, image: int) -> int:
        return 1000 * self.index + 500 + image

    @property
    def megapixels(self) -> float:
        return self.height * self.width * self.batch / 1e6


CONFIGS = {
    "c1": Config("c1", 1, 512, 512, 1, 1, 5, 5.0, 0.05, 1000.0, 1),
    "c2": Config("c2", 2, 1024, 1024, 3, 1, 7, 7.0, 0.1, 1000.0, 3),
    "c3": Config("c3", 3, 1080, 1920, 3, 1, 5, 5.0, 0.05, 500.0, 3, p_salt_pepper=0.05),
    "c4": Config("c4", 4, 4096, 4096, 1, 1, 15, 12.0, 0.08, 2000.0, 2, n_sites=64),
    "c5": Config("c5", 5, 2048, 2048, 3, 64, 7, 7.0, 0.1, 1000.0, 3, guide=True),
}
