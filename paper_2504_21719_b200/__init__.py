"""B200-native SBR core of Sionna RT (arXiv 2504.21719), drop-in for emtrace's hot path.

Public names follow emtrace/__init__.py:11-70 for the solver entry points.
Every compute call runs hand-written sm_100a CUDA kernels through the C ABI
in include/sbr.h (library: paper_2504_21719_b200/_lib/libsbr.so).  There is
no CPU fallback: without the library or a CUDA device the entry points raise
`errors.NativeUnavailable`.  Importing the package does not touch the GPU.
"""

__version__ = "0.1.0"

from .em import ArrayGeometry, AntennaPattern, make_pattern, planar_array  # noqa: E402
from .geometry import Mesh, Ray, build_scene_accel, intersect_closest, is_occluded  # noqa: E402
from .materials import RadioMaterial, ScatteringPattern, material_presets  # noqa: E402
from .paths import PathConfig, RadioDevice, SceneModel  # noqa: E402
from .cir import (  # noqa: E402
    CandidateRecord,
    GenerationResult,
    PathSet,
    PathTensors,
    ValidPath,
    baseband_gains,
    compute_paths,
    frequency_response,
    generate_candidates,
    refine_candidate,
)
from .radiomap import (  # noqa: E402
    MeasurementGrid,
    RadioMapConfig,
    RadioMapResult,
    compute_radio_map,
    compute_radio_map_diffraction,
    compute_radio_map_sbr,
    exact_maps,
)
from .sampling import Interaction  # noqa: E402
from .sceneio import (  # noqa: E402
    LoadedScene,
    SceneDescription,
    load_mesh_obj,
    load_scene,
    read_paths_csv,
    read_radio_map_csv,
    write_mesh_obj,
    write_paths,
    write_radio_map,
    write_scene,
)

__all__ = [
    "ArrayGeometry", "AntennaPattern", "make_pattern", "planar_array",
    "Mesh", "Ray", "build_scene_accel", "intersect_closest", "is_occluded",
    "RadioMaterial", "ScatteringPattern", "material_presets",
    "PathConfig", "RadioDevice", "SceneModel", "CandidateRecord", "GenerationResult",
    "PathSet", "PathTensors", "ValidPath", "baseband_gains", "compute_paths",
    "frequency_response", "generate_candidates", "refine_candidate",
    "MeasurementGrid", "RadioMapConfig", "RadioMapResult",
    "compute_radio_map", "compute_radio_map_diffraction", "compute_radio_map_sbr", "exact_maps",
    "Interaction", "LoadedScene", "SceneDescription", "load_mesh_obj", "load_scene",
    "read_paths_csv", "read_radio_map_csv", "write_mesh_obj", "write_paths",
    "write_radio_map", "write_scene", "__version__",
]
