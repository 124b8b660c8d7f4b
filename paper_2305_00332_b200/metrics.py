"""Pixel metrics between a reference and a downsampled rendering, on the device
(reference ``tsdown/metrics.py:69-132``).

``conv_mask`` and ``pem`` are exact; the SSIM map is exact (its 8x8 window
sums of integer images are exact in fp64), and the ``dssim`` / ``mse`` masked
means are summed in a fixed order that differs from numpy's pairwise sum
(agreement to ~1e-13 relative; tests assert 1e-12).
"""
from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _native as N
from .errors import DimensionMismatch
from .raster import RasterImage

__all__ = ["ConvMask", "conv_mask", "pem", "dssim", "mse", "metrics"]


@dataclass(frozen=True, eq=False)
class ConvMask:
    """Boolean pixel mask restricting metric computation (metrics.py:38-45)."""

    pixels: torch.Tensor  # uint8 0/1 on the device

    @property
    def size(self) -> int:
        return int(torch.count_nonzero(self.pixels).item())


def _pair(ref: RasterImage, cand: RasterImage):
    if (ref.height, ref.width) != (cand.height, cand.width):
        raise DimensionMismatch(f"image shapes differ: {(ref.height, ref.width)} vs {(cand.height, cand.width)}")
    a = ref.device_pixels()
    return a, cand.device_pixels(a.device)


def conv_mask(ref: RasterImage, cand: RasterImage, kernel: int = 3) -> ConvMask:
    """Dilated union of both images' ink pixels (metrics.py:69-82)."""
    a, b = _pair(ref, cand)
    if kernel < 1 or kernel % 2 == 0:
        raise ValueError(f"kernel must be a positive odd integer, got {kernel}")
    m = torch.empty_like(a)
    with torch.cuda.device(a.device):
        N.check(N.lib().mmlttb_conv_mask(a.data_ptr(), b.data_ptr(), a.shape[0], a.shape[1], kernel, m.data_ptr(),
                                         N.stream_ptr(a.device)), "conv_mask")
    return ConvMask(m)


def metrics(ref: RasterImage, cand: RasterImage, mask: ConvMask, margin: int = 20) -> tuple[float, float, float]:
    """(pem, dssim, mse) in one device pass (metrics.py:85-132)."""
    a, b = _pair(ref, cand)
    if not 0 <= margin <= 255:
        raise ValueError(f"margin must be in [0, 255], got {margin}")
    out = torch.empty(4, dtype=torch.float64, device=a.device)
    h, w = a.shape
    wsb = 5 * h * w * 8 + ((h * w + 255) // 256) * 16 + 1024
    ws = N.workspace(wsb, a.device)
    with torch.cuda.device(a.device):
        N.check(N.lib().mmlttb_pixel_metrics(a.data_ptr(), b.data_ptr(), mask.pixels.data_ptr(), h, w, margin,
                                             out.data_ptr(), ws.data_ptr(), wsb, N.stream_ptr(a.device)), "metrics")
    p, d, e, _ = out.tolist()
    return p, d, e


def pem(ref: RasterImage, cand: RasterImage, mask: ConvMask, margin: int = 20) -> float:
    """Share of mask pixels differing by more than ``margin`` levels (metrics.py:85-95)."""
    return metrics(ref, cand, mask, margin)[0]


def dssim(ref: RasterImage, cand: RasterImage, mask: ConvMask) -> float:
    """Mean (1 - SSIM) / 2 over the mask, 8x8 uniform window (metrics.py:98-123)."""
    return metrics(ref, cand, mask)[1]


def mse(ref: RasterImage, cand: RasterImage, mask: ConvMask) -> float:
    """Mean squared error over the mask, intensities scaled to [0, 1] (metrics.py:126-132)."""
    return metrics(ref, cand, mask)[2]
