"""Spectral conventions of the half-plane grid (reference: fdl/spectra.py:1-101).

Unnormalised forward DFT, inverse scaled by 1/(W*H) ("ufwd-inv1/WH");
frequencies in cycles per pixel; floor(W/2)+1 stored columns, the even-W
Nyquist column labelled -0.5; omega_y = fftfreq(H).  The CUDA kernels
recompute these labels bit-identically (csrc/common.cuh: omega_x_label,
omega_y_label).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

DFT_CONVENTION = "ufwd-inv1/WH"

__all__ = ["DFT_CONVENTION", "FrequencyGrid"]


@dataclass(frozen=True)
class FrequencyGrid:
    """Frequency bookkeeping of a W x H real image (spectra.py:41-101)."""

    width: int
    height: int
    omega_x: np.ndarray = field(init=False, repr=False, compare=False)
    omega_y: np.ndarray = field(init=False, repr=False, compare=False)

    def __post_init__(self):
        if self.width < 1 or self.height < 1:
            raise ValueError(f"invalid grid dimensions {self.width}x{self.height}")
        cols = np.arange(self.width // 2 + 1, dtype=np.float64) / self.width
        if self.width % 2 == 0:
            cols[-1] = -0.5
        rows = np.fft.fftfreq(self.height)
        cols.setflags(write=False)
        rows.setflags(write=False)
        object.__setattr__(self, "omega_x", cols)
        object.__setattr__(self, "omega_y", rows)

    @property
    def half_width(self) -> int:
        return self.width // 2 + 1

    @property
    def num_entries(self) -> int:
        return self.half_width * self.height

    def entries(self):
        """(index, omega_x, omega_y) for every stored bin, row-major in (ky, kx)."""
        for ky in range(self.height):
            for kx in range(self.half_width):
                yield ky * self.half_width + kx, self.omega_x[kx], self.omega_y[ky]

    def self_conjugate_x(self) -> list[int]:
        return [0, self.width // 2] if self.width % 2 == 0 else [0]

    def self_conjugate_y(self) -> list[int]:
        return [0, self.height // 2] if self.height % 2 == 0 else [0]

    def pair_weights(self) -> np.ndarray:
        w = np.full(self.half_width, 2.0)
        w[self.self_conjugate_x()] = 1.0
        return w

    def mirror_rows(self) -> np.ndarray:
        """Row index of the conjugate partner of every row: (H - ky) % H."""
        return (self.height - np.arange(self.height)) % self.height
