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
SBR_ERR_INTERNAL = 7

SBR_CHUNK_LOG2 = 19
SBR_CIR_SHARD_LOG2 = 12   # id chunks of the chunk-cyclic CIR shards (sbr_cir_sweep_sharded)

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
    "cone_samples",
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


# ---- path solver (CIR) ------------------------------------------------------
CIR_COUNTERS = (
    "samples_escaped",
    "samples_terminated",
    "ray_bounces",
    "vertices",
    "visibility_rays",
    "rows",
    "duplicates",
    "chunk_truncated",
    "buffer_overflow",
    "candidates",
    "hash_registered",
    "hash_slots",
    "rej_coplanar_miss",
    "rej_occluded",
    "rej_degenerate",
    "stack_overflow",
    "vertex_overflow",
    "row_overflow",
    "rej_off_edge",
)
SBR_CC_COUNT = len(CIR_COUNTERS)
CC = {name: i for i, name in enumerate(CIR_COUNTERS)}

SBR_REFINE_OK = 0
SBR_REFINE_COPLANAR_MISS = 1
SBR_REFINE_OCCLUDED = 2
SBR_REFINE_DEGENERATE = 3
SBR_REFINE_OFF_EDGE = 4
REJECTION_NAMES = {SBR_REFINE_COPLANAR_MISS: "coplanar-miss", SBR_REFINE_OCCLUDED: "occluded",
                   SBR_REFINE_DEGENERATE: "degenerate", SBR_REFINE_OFF_EDGE: "off-edge"}
REJECTION_COUNTERS = {SBR_REFINE_COPLANAR_MISS: "rej_coplanar_miss",
                      SBR_REFINE_OCCLUDED: "rej_occluded", SBR_REFINE_DEGENERATE: "rej_degenerate",
                      SBR_REFINE_OFF_EDGE: "rej_off_edge"}


class SbrCirParams(ctypes.Structure):
    _fields_ = [
        ("source", ctypes.c_double * 3),
        ("q_diffraction", ctypes.c_double),
        ("num_samples", ctypes.c_uint64),
        ("seed", ctypes.c_uint64),
        ("max_depth", ctypes.c_int32),
        ("allow_mask", ctypes.c_int32),
        ("n_targets", ctypes.c_int32),
        ("pad_", ctypes.c_int32),
        ("targets_dev", ctypes.c_void_p),
    ]


class SbrVertexBuf(ctypes.Structure):
    _fields_ = [(name, ctypes.c_void_p) for name in (
        "point", "normal", "run_prob", "sample", "hash_r", "hash_f", "parent", "tri",
        "code", "depth", "suffix_start", "wedge")] + [("capacity", ctypes.c_int64)]


class SbrRecordBuf(ctypes.Structure):
    _fields_ = [(name, ctypes.c_void_p) for name in (
        "target", "sample", "depth", "suffix_start", "diffuse", "chain_hash", "prefix_prob",
        "anchor", "kind", "tri", "vertex", "normal")] + [
        ("max_depth", ctypes.c_int32), ("pad_", ctypes.c_int32), ("wedge", ctypes.c_void_p)]


class SbrWedgeTable(ctypes.Structure):
    _fields_ = [("n_wedges", ctypes.c_int64)] + [(name, ctypes.c_void_p) for name in (
        "origin", "e_hat", "t0_hat", "n0_hat", "nn_hat", "length", "n_open", "hash_r",
        "hash_f", "mat0", "matn", "slot_offsets", "slot_ids")]


class SbrFieldParams(ctypes.Structure):
    _fields_ = [
        ("wavelength", ctypes.c_double),
        ("q_diffraction", ctypes.c_double),
        ("tx_velocity", ctypes.c_double * 3),
        ("num_samples", ctypes.c_uint64),
        ("seed", ctypes.c_uint64),
        ("allow_mask", ctypes.c_int32),
        ("n_objects", ctypes.c_int32),
        ("tx_pattern", SbrAntenna),
        ("rx_pattern_dev", ctypes.c_void_p),
        ("rx_velocity_dev", ctypes.c_void_p),
        ("obj_velocity_dev", ctypes.c_void_p),
    ]
