"""ctypes mirror of the structs and constants in include/sbr.h.

Pure data description (no library loading), shared by the product host code
and the test-only oracle wrapper so both pack parameters identically.
"""

import ctypes

SBR_OK = 0
SBR_ERR_INVALID = 1
SBR_ERR_EMPTY_SCENE = 2
SBR_ERR_STACK = 3
SBR_ERR_CUDA = 4
SBR_ERR_UNSUPPORTED = 5
SBR_ERR_NOMEM = 6

SBR_CHUNK_LOG2 = 19

SBR_SCAT_LAMBERTIAN = 0
SBR_SCAT_DIRECTIVE = 1
SBR_SCAT_BACKSCATTERING = 2

SBR_PATTERN_ISOTROPIC = 0
SBR_PATTERN_TR38901 = 1

# radio-map counters, same order as the SBR_MC_* enum
MAP_COUNTERS = (
    "deposits",
    "escaped",
    "terminated",
    "respawns",
    "threshold_killed",
    "roulette_killed",
    "ray_bounces",
    "direct_visible",
    "stack_overflow",
)
SBR_MC_COUNT = len(MAP_COUNTERS)


class SbrMaterial(ctypes.Structure):
    _fields_ = [
        ("eta_re", ctypes.c_double),
        ("eta_im", ctypes.c_double),
        ("sqrt_eta_re", ctypes.c_double),
        ("sqrt_eta_im", ctypes.c_double),
        ("kd", ctypes.c_double),
        ("thickness", ctypes.c_double),
        ("scattering", ctypes.c_double),
        ("spec_amp", ctypes.c_double),
        ("xpd_kx", ctypes.c_double),
        ("lambda_mix", ctypes.c_double),
        ("pattern_kind", ctypes.c_int32),
        ("alpha_r", ctypes.c_int32),
        ("alpha_i", ctypes.c_int32),
        ("random_phases", ctypes.c_int32),
    ]


class SbrAntenna(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int32),
        ("identity", ctypes.c_int32),
        ("scale", ctypes.c_double),
        ("rot", ctypes.c_double * 9),
    ]


class SbrMapParams(ctypes.Structure):
    _fields_ = [
        ("source", ctypes.c_double * 3),
        ("corner", ctypes.c_double * 3),
        ("u_hat", ctypes.c_double * 3),
        ("v_hat", ctypes.c_double * 3),
        ("normal", ctypes.c_double * 3),
        ("plane_off", ctypes.c_double),
        ("cell_w", ctypes.c_double),
        ("cell_h", ctypes.c_double),
        ("scale", ctypes.c_double),
        ("wavelength", ctypes.c_double),
        ("omega0", ctypes.c_double),
        ("rr_max", ctypes.c_double),
        ("gain_threshold", ctypes.c_double),
        ("num_samples", ctypes.c_uint64),
        ("seed", ctypes.c_uint64),
        ("nx", ctypes.c_int32),
        ("ny", ctypes.c_int32),
        ("max_depth", ctypes.c_int32),
        ("allow_mask", ctypes.c_int32),
        ("rr_depth", ctypes.c_int32),
        ("cull_from", ctypes.c_int32),
        ("any_random_phase", ctypes.c_int32),
        ("n_elements", ctypes.c_int32),
        ("pattern", SbrAntenna),
        ("elem_offsets_dev", ctypes.c_void_p),
        ("precoder_dev", ctypes.c_void_p),
    ]


def vec3(values):
    arr = (ctypes.c_double * 3)()
    for k in range(3):
        arr[k] = float(values[k])
    return arr
