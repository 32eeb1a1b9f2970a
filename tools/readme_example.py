import sys; sys.path.insert(0, '.')
from paper_2504_21719_b200 import (SceneModel, RadioDevice, PathConfig, RadioMapConfig,
                                   MeasurementGrid, compute_paths, compute_radio_map,
                                   frequency_response, load_scene, scenes)

meshes = scenes.street_canyon()
scene = SceneModel(meshes, scenes.uniform_materials(meshes, scenes.concrete(scattering=0.3)))
grid = MeasurementGrid((0, 0, 1.5), (1, 0, 0), (0, 1, 0), (1.0, 1.0), (200, 200))
maps = compute_radio_map(scene, [(0.0, 5.0, 20.0)], grid, RadioMapConfig(num_samples=10_000_000))
paths = compute_paths(scene, [RadioDevice(position=(0, 5, 20))],
                      [RadioDevice(position=(30, 2, 1.5))], PathConfig(num_samples=1_000_000))
print(maps.values.shape, len(paths.paths))
