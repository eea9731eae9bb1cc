"""Seeded synthetic inputs for the BASELINE.json configurations.

No public dataset is involved; these stand in for the paper's 256x256 test
image and the reference's missing astronaut_256.pgm. Generator (numpy PCG64):

  base      G(x, y) = 32 (x/(W-1) + y/(H-1))                       (0..64)
  rects     K axis-aligned rectangles painted (overwrite) into R:
            x0 ~ U[0,W), y0 ~ U[0,H), w ~ U[W/64, W/4], h ~ U[H/64, H/4],
            value ~ U[0, 255)
  image     f = clip(G + R + N(0, noise^2), 0, 255), stored as fp32
  checker   f = clip(255 (((x>>6) + (y>>6)) & 1) + N(0, noise^2), 0, 255)

Seeds: rectangles use config_id*1000 + channel, noise uses
config_id*1000 + frame*3 + channel + 500 (C4 rectangles drift +4 px per frame).
Frame k > 0 of a still-image config (C1/C2/C3 batches) uses seed
config_id*1000 + channel + 17k for both; frame 0 is the canonical image.
"""
from __future__ import annotations

import dataclasses

import numpy as np


@dataclasses.dataclass(frozen=True)
class Config:
    cid: int
    name: str
    width: int
    height: int
    rects: int
    noise: float
    sigma_s: tuple
    sigma_r: float
    degree: int = 20
    frames: int = 1
    channels: int = 1
    kind: str = "rects"

    @property
    def pixels(self) -> int:
        return self.width * self.height * self.frames * self.channels


CONFIGS = {
    1: Config(1, "C1 512x512 rects16 n10 ss3 sr30", 512, 512, 16, 10.0, (3.0,), 30.0),
    2: Config(2, "C2 2048x2048 rects64 n15 ss5 sr20", 2048, 2048, 64, 15.0, (5.0,), 20.0),
    3: Config(3, "C3 8192x8192 rects1024 n10 sr30 ss{2,5,10,20,50}", 8192, 8192, 1024, 10.0,
              (2.0, 5.0, 10.0, 20.0, 50.0), 30.0),
    4: Config(4, "C4 64x3x3840x2160 drift4 n8 ss8 sr25", 3840, 2160, 0, 8.0, (8.0,), 25.0,
              frames=64, channels=3, kind="video"),
    5: Config(5, "C5 4096x4096 checker64 n5 ss6 sr10", 4096, 4096, 0, 5.0, (6.0,), 10.0,
              kind="checker"),
}


def _rect_layer(rng: np.random.Generator, w: int, h: int, k: int, dx: int = 0) -> np.ndarray:
    R = np.zeros((h, w), np.float64)
    lo_w, hi_w = max(1, w // 64), max(1, w // 4)
    lo_h, hi_h = max(1, h // 64), max(1, h // 4)
    for _ in range(k):
        x0 = int(rng.integers(0, w)) + dx
        y0 = int(rng.integers(0, h))
        rw = int(rng.integers(lo_w, hi_w + 1))
        rh = int(rng.integers(lo_h, hi_h + 1))
        v = float(rng.uniform(0.0, 255.0))
        xa, xb = max(0, x0), min(w, x0 + rw)
        if xa < xb:
            R[y0:y0 + rh, xa:xb] = v
    return R


def rects_image(w: int, h: int, rects: int, noise: float, seed: int, noise_seed: int | None = None,
                dx: int = 0) -> np.ndarray:
    """Gradient + painted rectangles + Gaussian noise, clipped to [0,255], fp32."""
    rng = np.random.default_rng(seed)
    x = np.arange(w, dtype=np.float64) / max(1, w - 1)
    y = np.arange(h, dtype=np.float64) / max(1, h - 1)
    img = 32.0 * (x[None, :] + y[:, None])
    img += _rect_layer(rng, w, h, rects, dx)
    nrng = np.random.default_rng(seed + 500 if noise_seed is None else noise_seed)
    img += nrng.normal(0.0, noise, size=(h, w))
    np.clip(img, 0.0, 255.0, out=img)
    return img.astype(np.float32)


def checker_image(w: int, h: int, noise: float, seed: int, cell_log2: int = 6) -> np.ndarray:
    rng = np.random.default_rng(seed)
    x = np.arange(w)[None, :] >> cell_log2
    y = np.arange(h)[:, None] >> cell_log2
    img = 255.0 * ((x + y) & 1) + rng.normal(0.0, noise, size=(h, w))
    np.clip(img, 0.0, 255.0, out=img)
    return img.astype(np.float32)


def make(cfg: Config, frame: int = 0, channel: int = 0) -> np.ndarray:
    """One fp32 grayscale frame of configuration `cfg`."""
    base = cfg.cid * 1000
    if cfg.kind == "checker":
        return checker_image(cfg.width, cfg.height, cfg.noise, base + 500)
    if cfg.kind == "video":
        return rects_image(cfg.width, cfg.height, 48, cfg.noise, base + channel,
                           noise_seed=base + frame * 3 + channel + 500, dx=4 * frame)
    # further frames of a still-image config (a frame batch: C3's per-sigma_s
    # frames, the frames each rank shards) draw fresh rectangles and noise
    return rects_image(cfg.width, cfg.height, cfg.rects, cfg.noise, base + channel + 17 * frame)


def scaled(cfg: Config, width: int, height: int) -> Config:
    """Same generator family at another size (rect count scaled by area)."""
    k = max(1, int(round(cfg.rects * (width * height) / (cfg.width * cfg.height)))) if cfg.rects else 0
    return dataclasses.replace(cfg, width=width, height=height, rects=k, frames=1, channels=1)
