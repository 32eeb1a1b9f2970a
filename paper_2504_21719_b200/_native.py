"""Loader and thin typed wrappers for the sm_100a C-ABI library (libsbr.so).

There is deliberately no CPU fallback: if the library is missing or no CUDA
device is available every entry point raises `NativeUnavailable`.  Device
buffers are torch tensors; raw pointers, sizes and the current CUDA stream
are handed to the C ABI (include/sbr.h).
"""

import ctypes
import os

from . import _abi
from .errors import EmptyScene, NativeUnavailable

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SBR_LIB_PATH") or os.path.join(_HERE, "_lib", "libsbr.so")

_lib = None

c_dbl_p = ctypes.c_void_p  # device pointers travel as void*


def _declare(lib):
    vp, i64, i32, u64, dbl = (ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32,
                              ctypes.c_uint64, ctypes.c_double)
    sig = {
        "sbr_scene_create": (ctypes.c_int, [vp, vp, vp, i64, i32, vp,
                                            ctypes.POINTER(vp)]),
        "sbr_scene_destroy": (None, [vp]),
        "sbr_set_bvh_builder": (ctypes.c_int, [i32]),
        "sbr_scene_num_triangles": (i64, [vp]),
        "sbr_scene_num_nodes": (i64, [vp]),
        "sbr_scene_permutation": (ctypes.c_int, [vp, vp]),
        "sbr_scene_copy_nodes": (ctypes.c_int, [vp, vp]),
        "sbr_scene_set_attributes": (ctypes.c_int, [vp, vp, vp, vp, vp, vp]),
        "sbr_scene_set_materials": (ctypes.c_int, [vp, vp, i32]),
        "sbr_scene_set_wedges": (ctypes.c_int, [vp, vp]),
        "sbr_scene_check": (ctypes.c_int, [vp, vp]),
        "sbr_release_scratch": (ctypes.c_int, [i32]),
        "sbr_scene_copy_tables": (ctypes.c_int, [vp, vp, vp, vp]),
        "sbr_wedges_extract": (ctypes.c_int, [vp, vp, vp, vp, vp, i64, dbl, i32, vp,
                                              ctypes.POINTER(vp)]),
        "sbr_wedges_count": (ctypes.c_int, [vp, ctypes.POINTER(i64), ctypes.POINTER(i64),
                                            ctypes.POINTER(i64)]),
        "sbr_wedges_copy": (ctypes.c_int, [vp] * 14),
        "sbr_wedges_free": (None, [vp]),
        "sbr_trace_closest": (ctypes.c_int, [vp, vp, vp, dbl, vp, i64, vp, vp,
                                             vp, vp, vp]),
        "sbr_trace_any": (ctypes.c_int, [vp, vp, vp, dbl, vp, i64, vp, vp]),
        "sbr_occluded": (ctypes.c_int, [vp, vp, vp, dbl, i64, vp, vp]),
        "sbr_fibonacci": (ctypes.c_int, [u64, u64, u64, vp, vp]),
        "sbr_philox_uniform": (ctypes.c_int, [u64, u64, u64, u64, u64, u64, vp,
                                              vp]),
        "sbr_radiomap_bounce": (ctypes.c_int, [vp, vp, u64, u64, vp, vp, vp]),
        "sbr_radiomap_bounce_sharded": (ctypes.c_int, [vp, vp, i32, i32, vp, vp, vp]),
        "sbr_radiomap_direct": (ctypes.c_int, [vp, vp, vp, vp, vp]),
        "sbr_set_wave_streams": (ctypes.c_int, [i32]),
        "sbr_set_exact_maps": (ctypes.c_int, [i32]),
        "sbr_radiomap_wedges": (ctypes.c_int, [vp, vp, vp, i32, u64, vp, vp, vp]),
        "sbr_cir_sweep": (ctypes.c_int, [vp, vp, u64, u64, vp, vp, vp]),
        "sbr_cir_sweep_sharded": (ctypes.c_int, [vp, vp, i32, i32, vp, vp, vp]),
        "sbr_cir_vertex_order": (ctypes.c_int, [vp, vp, i64, vp, vp]),
        "sbr_cir_visibility": (ctypes.c_int, [vp, vp, vp, i64, i64, vp, vp, vp, i64, vp, vp]),
        "sbr_cir_row_pairs": (ctypes.c_int, [vp, vp, vp, i64, vp, vp, vp, vp]),
        "sbr_cir_select": (ctypes.c_int, [vp, vp, vp, vp, vp, i64, vp, u64, i64, vp,
                                          ctypes.POINTER(i64), vp, vp]),
        "sbr_cir_local_dedup": (ctypes.c_int, [vp, vp, vp, vp, vp, i64, vp, ctypes.POINTER(i64),
                                               ctypes.POINTER(u64), vp]),
        "sbr_cir_resolve_records": (ctypes.c_int, [vp, i64, vp, vp, vp, vp, vp]),
        "sbr_cir_records": (ctypes.c_int, [vp, vp, vp, vp, i64, vp, vp]),
        "sbr_cir_refine": (ctypes.c_int, [vp, vp, vp, i64, vp, vp, vp, vp]),
        "sbr_cir_fields": (ctypes.c_int, [vp, vp, vp, vp, vp, i64, vp, vp, vp, vp, vp, vp]),
        "sbr_cfr": (ctypes.c_int, [vp, vp, vp, vp, vp, vp, i64, vp, i32, vp, i32, vp, i32,
                                   dbl, i32, vp, vp]),
        "sbr_set_cfr_dmma_min_paths": (ctypes.c_int, [i64]),
        "sbr_obj_parse": (ctypes.c_int, [ctypes.c_char_p, i64, ctypes.POINTER(vp),
                                         ctypes.POINTER(i64), ctypes.POINTER(i32),
                                         ctypes.c_char_p, i64]),
        "sbr_obj_sizes": (ctypes.c_int, [vp, ctypes.POINTER(i64), ctypes.POINTER(i64)]),
        "sbr_obj_copy": (ctypes.c_int, [vp, vp, vp]),
        "sbr_obj_free": (None, [vp]),
        "sbr_last_error": (ctypes.c_char_p, []),
        "sbr_version": (ctypes.c_int, []),
        "sbr_build_flags": (ctypes.c_int, []),
        "sbr_kernel_launches": (u64, []),
        "sbr_profile_enable": (ctypes.c_int, [i32]),
        "sbr_profile_kernel_ms": (dbl, [ctypes.c_char_p, ctypes.POINTER(u64)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


def exported_symbols():
    """Names every build of libsbr.so must export (checked by the CPU tests)."""
    return [
        "sbr_scene_create", "sbr_scene_destroy", "sbr_set_bvh_builder", "sbr_scene_num_triangles",
        "sbr_scene_num_nodes", "sbr_scene_permutation", "sbr_scene_copy_nodes",
        "sbr_scene_set_attributes", "sbr_scene_set_materials", "sbr_scene_set_wedges",
        "sbr_scene_check", "sbr_release_scratch", "sbr_scene_copy_tables", "sbr_wedges_extract", "sbr_wedges_count",
        "sbr_wedges_copy", "sbr_wedges_free", "sbr_trace_closest", "sbr_trace_any",
        "sbr_occluded", "sbr_fibonacci", "sbr_philox_uniform",
        "sbr_radiomap_bounce", "sbr_radiomap_bounce_sharded", "sbr_radiomap_direct",
        "sbr_set_wave_streams", "sbr_set_exact_maps",
        "sbr_radiomap_wedges", "sbr_cir_sweep", "sbr_cir_sweep_sharded",
        "sbr_cir_vertex_order",
        "sbr_cir_visibility", "sbr_cir_row_pairs", "sbr_cir_select", "sbr_cir_local_dedup",
        "sbr_cir_resolve_records", "sbr_cir_records", "sbr_cir_refine",
        "sbr_cir_fields", "sbr_cfr", "sbr_set_cfr_dmma_min_paths",
        "sbr_obj_parse", "sbr_obj_sizes", "sbr_obj_copy", "sbr_obj_free", "sbr_last_error",
        "sbr_version", "sbr_build_flags", "sbr_kernel_launches", "sbr_profile_enable", "sbr_profile_kernel_ms",
    ]


def load_library():
    """dlopen libsbr.so (no device needed).  Raises NativeUnavailable."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise NativeUnavailable(
                f"{LIB_PATH} is missing; run __graft_entry__.build() "
                "(this package has no CPU fallback)")
        _lib = _declare(ctypes.CDLL(LIB_PATH))
        builder = os.environ.get("SBR_BVH_BUILDER")  # "lbvh" / "ploc" (default)
        if builder:
            check(_lib.sbr_set_bvh_builder({"lbvh": 0, "ploc": 1}[builder.lower()]))
    return _lib


def lib():
    """The library, after checking that a CUDA device is usable."""
    import torch
    if not torch.cuda.is_available():
        raise NativeUnavailable("no CUDA device: the SBR core runs only on sm_100a")
    return load_library()


def check(status):
    if status == _abi.SBR_OK:
        return
    msg = (_lib.sbr_last_error() or b"").decode(errors="replace")
    if status == _abi.SBR_ERR_EMPTY_SCENE:
        raise EmptyScene(msg or "no triangles")
    if status == _abi.SBR_ERR_INVALID:
        raise ValueError(msg)
    if status == _abi.SBR_ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    if status == _abi.SBR_ERR_NOMEM:
        raise MemoryError(msg)
    raise RuntimeError(msg or f"sbr status {status}")


def stream_ptr(device=None):
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def device_of(device):
    import torch
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device(device)


def kernel_launches():
    return int(load_library().sbr_kernel_launches())


def release_scratch(device):
    """Return libsbr's cached scratch memory on `device` to the driver."""
    check(load_library().sbr_release_scratch(int(device_of(device).index or 0)))


def profile_enable(on=True):
    """Start (reset) or stop per-kernel CUDA-event timing inside libsbr."""
    check(load_library().sbr_profile_enable(1 if on else 0))


def profile_kernel_ms(name):
    """(summed ms, launches) of one library kernel since profile_enable()."""
    n = ctypes.c_uint64(0)
    ms = load_library().sbr_profile_kernel_ms(name.encode(), ctypes.byref(n))
    return float(ms), int(n.value)


def fibonacci(n_samples, begin, end, device):
    import torch
    L = lib()
    dev = device_of(device)
    end = n_samples if end is None else int(end)
    if n_samples < 1:
        raise ValueError("need at least one direction")
    out = torch.empty((max(end - begin, 0), 3), dtype=torch.float64, device=dev)
    with torch.cuda.device(dev):
        check(L.sbr_fibonacci(n_samples, begin, end, ptr(out), stream_ptr(dev)))
    return out


def philox_uniform(seed, sample, depth, tag, first, count, device):
    import torch
    L = lib()
    dev = device_of(device)
    out = torch.empty(int(count), dtype=torch.float64, device=dev)
    with torch.cuda.device(dev):
        check(L.sbr_philox_uniform(seed & (2**64 - 1), sample & (2**64 - 1),
                                   depth & (2**64 - 1), tag, first, count,
                                   ptr(out), stream_ptr(dev)))
    return out
