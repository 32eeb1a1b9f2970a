"""Radio materials (host descriptors of what the interaction kernels evaluate).

Same public types and validation as emtrace/materials.py:43-146.  The
Fresnel / ITU-R P.2040 slab / diffuse operators themselves run on the GPU
(csrc/sbr_physics.cuh); this module only freezes a material at one
frequency into an `SbrMaterial` row.
"""

import dataclasses
import math

import numpy as np

from . import _abi
from .em import SPEED_OF_LIGHT, VACUUM_PERMITTIVITY

EPS_FRAME = 1e-9
EPS_EDGE_GRAZE = 1e-9
EPS_COT_POLE = 1e-6

_SCAT_KINDS = {
    "lambertian": _abi.SBR_SCAT_LAMBERTIAN,
    "directive": _abi.SBR_SCAT_DIRECTIVE,
    "backscattering": _abi.SBR_SCAT_BACKSCATTERING,
}


@dataclasses.dataclass(frozen=True)
class ScatteringPattern:
    """Angular density of diffusely scattered power (materials.py:43-73)."""

    kind: str = "lambertian"
    alpha_r: int = 1
    alpha_i: int = 1
    lambda_mix: float = 1.0

    def __post_init__(self):
        if self.kind not in _SCAT_KINDS:
            raise ValueError(f"unknown scattering pattern kind: {self.kind!r}")
        if self.alpha_r < 1 or self.alpha_r != int(self.alpha_r):
            raise ValueError("alpha_r must be a positive integer")
        if self.alpha_i < 1 or self.alpha_i != int(self.alpha_i):
            raise ValueError("alpha_i must be a positive integer")
        if not 0.0 <= self.lambda_mix <= 1.0:
            raise ValueError("lambda_mix must lie in [0, 1]")


@dataclasses.dataclass(frozen=True)
class RadioMaterial:
    """Electromagnetic description of a surface (materials.py:76-127)."""

    name: str = "custom"
    eps_r: float = 1.0
    sigma: float = 0.0
    thickness: float = 0.0
    scattering: float = 0.0
    xpd_kx: float = 0.0
    pattern: ScatteringPattern = dataclasses.field(default_factory=ScatteringPattern)
    random_phases: bool = False

    def __post_init__(self):
        if self.eps_r < 1.0:
            raise ValueError("eps_r must be >= 1")
        if self.sigma < 0.0:
            raise ValueError("sigma must be >= 0")
        if self.thickness < 0.0:
            raise ValueError("thickness must be >= 0")
        if not 0.0 <= self.scattering <= 1.0:
            raise ValueError("scattering must lie in [0, 1]")
        if not 0.0 <= self.xpd_kx <= 1.0:
            raise ValueError("xpd_kx must lie in [0, 1]")

    @property
    def specular_factor(self) -> float:
        return math.sqrt(max(0.0, 1.0 - self.scattering ** 2))

    def complex_permittivity(self, frequency: float) -> complex:
        return complex_permittivity(self.eps_r, self.sigma, frequency)

    def to_abi(self, frequency):
        """Freeze at `frequency` into one SbrMaterial row.

        eta, sqrt(eta) and 2*pi*d/lambda are evaluated here with the same
        Python/numpy expressions as the reference (materials.py:130-134,
        195, 232) so the device sees bit-identical constants.
        """
        wavelength = SPEED_OF_LIGHT / frequency
        eta = self.complex_permittivity(frequency)
        root = complex(np.sqrt(np.asarray(eta, dtype=np.complex128)))
        m = _abi.SbrMaterial()
        m.eta_re, m.eta_im = eta.real, eta.imag
        m.sqrt_eta_re, m.sqrt_eta_im = root.real, root.imag
        m.kd = 2.0 * np.pi * self.thickness / wavelength
        m.thickness = float(self.thickness)
        m.scattering = float(self.scattering)
        m.spec_amp = self.specular_factor
        m.xpd_kx = float(self.xpd_kx)
        m.lambda_mix = float(self.pattern.lambda_mix)
        m.pattern_kind = _SCAT_KINDS[self.pattern.kind]
        m.alpha_r = int(self.pattern.alpha_r)
        m.alpha_i = int(self.pattern.alpha_i)
        m.random_phases = int(bool(self.random_phases))
        return m


def complex_permittivity(eps_r: float, sigma: float, frequency: float) -> complex:
    """eta = eps_r - j sigma / (eps0 * 2 pi f)  (materials.py:130-134)."""
    if frequency <= 0.0:
        raise ValueError("frequency must be positive")
    return eps_r - 1j * sigma / (VACUUM_PERMITTIVITY * 2.0 * math.pi * frequency)


def material_presets() -> dict:
    """Fixed presets (materials.py:137-146)."""
    return {
        "vacuum": RadioMaterial(name="vacuum"),
        "concrete": RadioMaterial(name="concrete", eps_r=5.24, sigma=0.0462,
                                  thickness=0.1),
        "glass": RadioMaterial(name="glass", eps_r=6.31, sigma=0.0236,
                               thickness=0.003),
        "metal": RadioMaterial(name="metal", eps_r=1.0, sigma=1e7, thickness=0.1),
    }


def pack_materials(materials, frequency):
    """ctypes array of SbrMaterial rows in the given order."""
    arr = (_abi.SbrMaterial * max(1, len(materials)))()
    for i, m in enumerate(materials):
        arr[i] = m.to_abi(frequency)
    return arr
