"""Orthonormal 2D Haar transform with the reference's flat subband layout.

Mirrors src/wavelet.py: the layout/index types are host metadata; ``dwt`` and
``idwt`` run the sm_100a strip kernels (vdamp_dwt / vdamp_idwt).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from ._lib import DimensionError

ORIENTATIONS = ("approx", "horizontal", "vertical", "diagonal")


@dataclass(frozen=True)
class Subband:
    scale: int
    orientation: str
    offset: int
    length: int
    shape: tuple


def _is_pow2(v: int) -> bool:
    return v > 0 and (v & (v - 1)) == 0


@dataclass(frozen=True)
class SubbandLayout:
    """approx_s, then (horizontal, vertical, diagonal) per scale s..1 (src/wavelet.py:34-74)."""

    image_height: int
    image_width: int
    scales: int
    subbands: tuple = field(default=())

    @staticmethod
    def create(image_height: int, image_width: int, scales: int) -> "SubbandLayout":
        if scales < 1:
            raise ValueError(f"scales must be >= 1, got {scales}")
        div = 2 ** scales
        if image_height % div or image_width % div:
            raise DimensionError(
                f"image shape ({image_height}, {image_width}) not divisible by 2^{scales}")
        if not (_is_pow2(image_height) and _is_pow2(image_width)) or max(image_height, image_width) > 2048:
            # documented scope cut of the GPU build (SURVEY §7 hard part 6)
            raise ValueError("the B200 build supports power-of-two image sizes up to 2048 only")
        hs, ws = image_height // div, image_width // div
        bands = [Subband(scales, "approx", 0, hs * ws, (hs, ws))]
        pos = hs * ws
        for lev in range(scales, 0, -1):
            h, w = image_height >> lev, image_width >> lev
            for o in ORIENTATIONS[1:]:
                bands.append(Subband(lev, o, pos, h * w, (h, w)))
                pos += h * w
        return SubbandLayout(image_height, image_width, scales, tuple(bands))

    @property
    def n_subbands(self) -> int:
        return len(self.subbands)

    @property
    def size(self) -> int:
        return self.image_height * self.image_width

    def subband_lengths(self) -> np.ndarray:
        return np.array([b.length for b in self.subbands])


@dataclass
class WaveletCoeffs:
    """Flat complex coefficient vector plus its layout (src/wavelet.py:77-97)."""

    values: np.ndarray
    layout: SubbandLayout

    def __post_init__(self):
        self.values = np.asarray(self.values)
        if self.values.shape != (self.layout.size,):
            raise ValueError(f"coefficient vector of length {self.values.shape} does not match "
                             f"layout size {self.layout.size}")

    def subband(self, j: int) -> np.ndarray:
        return subband_view(self, j)

    def copy(self) -> "WaveletCoeffs":
        return WaveletCoeffs(self.values.copy(), self.layout)


def subband_view(coeffs: WaveletCoeffs, j: int) -> np.ndarray:
    if not 0 <= j < coeffs.layout.n_subbands:
        raise IndexError(f"subband index {j} out of range [0, {coeffs.layout.n_subbands})")
    b = coeffs.layout.subbands[j]
    return coeffs.values[b.offset:b.offset + b.length]


def dwt(image, scales: int, *, precision="fp64", device=None) -> WaveletCoeffs:
    """Forward orthonormal Haar transform on the GPU (src/wavelet.py:132-148)."""
    from .plan import get_plan
    image = np.asarray(image)
    if image.ndim != 2:
        raise DimensionError(f"expected a 2D image, got shape {image.shape}")
    layout = SubbandLayout.create(image.shape[0], image.shape[1], scales)
    plan = get_plan(image.shape[0], image.shape[1], scales, 1, precision, device)
    x = plan.to_device(image, plan.cdtype).reshape(1, *image.shape).contiguous()
    out = plan.empty_coeffs()
    plan.dwt(x, out)
    return WaveletCoeffs(out[0].cpu().numpy(), layout)


def idwt(coeffs: WaveletCoeffs, *, precision="fp64", device=None) -> np.ndarray:
    """Inverse transform on the GPU (src/wavelet.py:169-181)."""
    from .plan import get_plan
    lay = coeffs.layout
    plan = get_plan(lay.image_height, lay.image_width, lay.scales, 1, precision, device)
    c = plan.to_device(coeffs.values, plan.cdtype).reshape(1, -1).contiguous()
    out = plan.empty_images()
    plan.idwt(c, out)
    return out[0].cpu().numpy()
