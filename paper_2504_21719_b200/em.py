"""Antenna patterns, arrays and physical constants (host side).

Mirrors the parts of emtrace/em.py that parametrise the device kernels:
the built-in patterns ('isotropic', 'tr38901', em.py:258-308) are evaluated
on the GPU from a compact descriptor (`SbrAntenna`), so a pattern here is a
name + orientation + normalisation scale rather than a Python callable.
Arbitrary Python evaluators cannot run inside the sm_100a kernels and are
rejected with NotImplementedError.
"""

import math
from dataclasses import dataclass

import numpy as np

from . import _abi

# scipy.constants values used by the reference (em.py:11-13, scipy 1.18)
SPEED_OF_LIGHT = 299792458.0
VACUUM_PERMITTIVITY = 8.8541878188e-12
MU_0 = 1.25663706127e-06
VACUUM_IMPEDANCE = float(np.sqrt(MU_0 / VACUUM_PERMITTIVITY))

QUAD_THETA_NODES = 128
QUAD_PHI_NODES = 256


def rotation_ypr(alpha, beta, gamma):
    """World rotation from yaw (z), pitch (y), roll (x) applied z.y.x (em.py:51-59)."""
    ca, sa = np.cos(alpha), np.sin(alpha)
    cb, sb = np.cos(beta), np.sin(beta)
    cg, sg = np.cos(gamma), np.sin(gamma)
    rz = np.array([[ca, -sa, 0.0], [sa, ca, 0.0], [0.0, 0.0, 1.0]])
    ry = np.array([[cb, 0.0, sb], [0.0, 1.0, 0.0], [-sb, 0.0, cb]])
    rx = np.array([[1.0, 0.0, 0.0], [0.0, cg, -sg], [0.0, sg, cg]])
    return rz @ ry @ rx


def angles_of(direction):
    """Zenith and azimuth of unit vectors, last axis xyz (em.py:37-42)."""
    d = np.asarray(direction, dtype=np.float64)
    return np.arccos(np.clip(d[..., 2], -1.0, 1.0)), np.arctan2(d[..., 1], d[..., 0])


def spherical_basis(theta, phi):
    """(r_hat, theta_hat, phi_hat) stacked on the last axis (em.py:22-36)."""
    theta = np.asarray(theta, dtype=np.float64)
    phi = np.asarray(phi, dtype=np.float64)
    st, ct = np.sin(theta), np.cos(theta)
    sp, cp = np.sin(phi), np.cos(phi)
    r_hat = np.stack([st * cp, st * sp, ct], axis=-1)
    theta_hat = np.stack([ct * cp, ct * sp, -st], axis=-1)
    phi_hat = np.stack([-sp, cp, np.zeros_like(sp)], axis=-1)
    return r_hat, theta_hat, phi_hat


def _tr38901_gain_db(theta, phi):
    theta_deg = np.rad2deg(np.asarray(theta, dtype=np.float64))
    phi_deg = np.rad2deg(np.arctan2(np.sin(phi), np.cos(phi)))
    a_v = -np.minimum(12.0 * ((theta_deg - 90.0) / 65.0) ** 2, 30.0)
    a_h = -np.minimum(12.0 * (phi_deg / 65.0) ** 2, 30.0)
    return -np.minimum(-(a_v + a_h), 30.0) + 8.0


def _gauss_legendre(n):
    try:
        from scipy.special import roots_legendre
        return roots_legendre(n)
    except ImportError:  # pragma: no cover - scipy is in the image
        return np.polynomial.legendre.leggauss(n)


def _sphere_integral(evaluate):
    """Gauss-Legendre in theta x trapezoid in phi (em.py:222-237)."""
    x, w = _gauss_legendre(QUAD_THETA_NODES)
    theta = (x + 1.0) * (np.pi / 2.0)
    w_theta = w * (np.pi / 2.0)
    phi = np.linspace(0.0, 2.0 * np.pi, QUAD_PHI_NODES + 1)
    tg, pg = np.meshgrid(theta, phi, indexing="ij")
    gain = evaluate(tg, pg)
    inner = np.trapezoid(gain, phi, axis=1)
    return float(np.sum(inner * np.sin(theta) * w_theta))


_TR38901_SCALE = None


def tr38901_scale():
    """Amplitude scale making the TR 38.901 element radiate unit power (em.py:275-282)."""
    global _TR38901_SCALE
    if _TR38901_SCALE is None:
        integral = _sphere_integral(
            lambda t, p: np.abs(10.0 ** (_tr38901_gain_db(t, p) / 20.0)) ** 2)
        _TR38901_SCALE = float(np.sqrt(4.0 * np.pi / integral))
    return _TR38901_SCALE


@dataclass(frozen=True)
class AntennaPattern:
    """Built-in directional pattern with orientation (em.py:150-172)."""

    name: str = "isotropic"
    orientation: tuple = (0.0, 0.0, 0.0)
    gain: float = 1.0
    eta_rad: float = 1.0

    def rotation(self):
        return rotation_ypr(*self.orientation)

    def with_orientation(self, orientation):
        return AntennaPattern(self.name, tuple(orientation), self.gain, self.eta_rad)

    def evaluator(self, theta, phi):
        """Host evaluation of (c_theta, c_phi) in the antenna frame."""
        theta = np.asarray(theta, dtype=np.float64)
        if self.name == "isotropic":
            one = np.ones_like(theta)
            return one.astype(np.complex128), np.zeros_like(one, dtype=np.complex128)
        if self.name == "tr38901":
            amp = tr38901_scale() * 10.0 ** (_tr38901_gain_db(theta, phi) / 20.0)
            amp = np.asarray(amp, dtype=np.complex128)
            return amp, np.zeros_like(amp)
        raise NotImplementedError(f"pattern {self.name!r} has no device kernel")

    def to_abi(self):
        """Pack into the SbrAntenna descriptor the kernels evaluate."""
        a = _abi.SbrAntenna()
        if self.name == "isotropic":
            a.kind = _abi.SBR_PATTERN_ISOTROPIC
            a.scale = 1.0
        elif self.name == "tr38901":
            a.kind = _abi.SBR_PATTERN_TR38901
            a.scale = tr38901_scale()
        else:
            raise NotImplementedError(
                f"pattern {self.name!r}: only the built-in 'isotropic' and "
                "'tr38901' patterns run on the device")
        rot = self.rotation()
        a.identity = int(np.array_equal(rot, np.eye(3)))
        for k in range(9):
            a.rot[k] = float(rot.reshape(-1)[k])
        return a


def make_pattern(name, orientation=(0.0, 0.0, 0.0)):
    """Factory for the built-in patterns: 'isotropic' ('iso'), 'tr38901' (em.py:294-308)."""
    key = name.lower()
    if key in ("iso", "isotropic"):
        return AntennaPattern("isotropic", tuple(orientation), gain=1.0)
    if key == "tr38901":
        gain = float(tr38901_scale() * 10.0 ** (8.0 / 20.0)) ** 2
        return AntennaPattern("tr38901", tuple(orientation), gain=gain)
    raise ValueError(f"unknown pattern {name!r}")


@dataclass(frozen=True)
class ArrayGeometry:
    """Element offsets (m) relative to the array centre (em.py:175-195)."""

    offsets: np.ndarray
    pattern_names: tuple = ("isotropic",)

    def __post_init__(self):
        off = np.atleast_2d(np.asarray(self.offsets, dtype=np.float64))
        if not np.all(np.isfinite(off)):
            raise ValueError("element offsets must be finite")
        object.__setattr__(self, "offsets", off)

    @property
    def num_elements(self):
        return len(self.offsets)

    def max_radius(self):
        if self.num_elements == 0:
            return 0.0
        return float(np.max(np.linalg.norm(self.offsets, axis=1)))


def planar_array(rows, cols, spacing_v, spacing_h):
    """Rectangular panel in the y-z plane centred at the origin (sceneio 'array r c dv dh')."""
    ys = (np.arange(cols) - (cols - 1) / 2.0) * spacing_h
    zs = (np.arange(rows) - (rows - 1) / 2.0) * spacing_v
    off = np.array([[0.0, y, z] for z in zs for y in ys])
    return ArrayGeometry(off)


def array_response(geometry, direction, wavelength, incoming):
    """Per-element steering phases exp(j 2pi/lambda (+-k).d) (em.py:240-251)."""
    if wavelength <= 0:
        raise ValueError("wavelength must be positive")
    k_hat = np.asarray(direction, dtype=np.float64)
    sign = -1.0 if incoming else 1.0
    phase = (2.0 * np.pi / wavelength) * (geometry.offsets @ (sign * k_hat))
    return np.exp(1j * phase)


def wavelength_of(frequency):
    return SPEED_OF_LIGHT / frequency


__all__ = [
    "SPEED_OF_LIGHT", "VACUUM_PERMITTIVITY", "MU_0", "VACUUM_IMPEDANCE",
    "AntennaPattern", "ArrayGeometry", "array_response", "make_pattern",
    "planar_array", "rotation_ypr", "spherical_basis", "tr38901_scale",
    "math",
]
