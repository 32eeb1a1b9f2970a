"""Interaction kinds and the counter-based RNG stream identities.

The draws themselves happen on the GPU (csrc/sbr_common.cuh: stateless
Philox4x64-10 keyed exactly like emtrace's RngStream, sampling.py:49-78), so
this module only names the streams.  `fibonacci_directions` and
`rng_uniform` expose the device generators for API parity and tests.
"""

import enum

_MASK64 = 0xFFFFFFFFFFFFFFFF
_FNV_OFFSET = 0xCBF29CE484222325
_FNV_PRIME = 0x100000001B3

GOLDEN_RATIO = (1.0 + 5.0 ** 0.5) / 2.0


class Interaction(enum.Enum):
    """Surface interaction kinds, in the fixed sampling order (sampling.py:25-39)."""

    REFLECTION = "R"
    SCATTERING = "S"
    TRANSMISSION = "T"
    DIFFRACTION = "D"


INTERACTION_ORDER = (
    Interaction.REFLECTION,
    Interaction.SCATTERING,
    Interaction.TRANSMISSION,
    Interaction.DIFFRACTION,
)


def tag_hash(text):
    """FNV-1a of the purpose tag (sampling.py:42-46)."""
    h = _FNV_OFFSET
    for byte in text.encode("utf-8"):
        h = ((h ^ byte) * _FNV_PRIME) & _MASK64
    return h


def allow_mask(enabled):
    """Bit mask R=1, S=2, T=4, D=8 of an enabled-kinds set."""
    mask = 0
    for bit, kind in enumerate(INTERACTION_ORDER):
        if kind in enabled:
            mask |= 1 << bit
    return mask


def fibonacci_directions(n_samples, begin=0, end=None, device=None):
    """fibonacci_directions(N)[begin:end] evaluated on the GPU (sampling.py:81-95).

    Returns a (end-begin, 3) float64 torch tensor on the device.
    """
    from . import _native
    return _native.fibonacci(int(n_samples), begin, end, device)


def rng_uniform(seed, sample, depth, purpose, count, first=0, device=None):
    """RngStream(seed, sample, depth, purpose).generator().random(...)[first:first+count]."""
    from . import _native
    return _native.philox_uniform(seed, sample, depth, tag_hash(purpose), first,
                                  count, device)
