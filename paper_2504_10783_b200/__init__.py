"""B200-native EI-ZO hot path with the reference ``corridor`` package's API.

Public names mirror ``corridor/__init__.py:10-22`` for the hot-path subset
(SURVEY.md §8b).  Host data types (models, polytopes, grids) are plain
Python; checking, hit-and-run, inflation, voxelisation and the DRM prune run
as hand-written sm_100a kernels behind the C ABI of ``include/corridor_b200.h``.
"""

from .checker import CollisionChecker, segment_samples
from .eizo import (InflationParams, InflationReport, Segment, bisection_update, compute_step_back,
                   default_bisection_steps, dist_gradient, dist_to_segment, inflate_edge, project_batch,
                   project_to_segment, required_batch_size, unadaptive_test)
from .errors import (CorridorError, DimensionMismatch, EmptyChord, GradientUndefined, GridMismatch,
                     NativeError, SeedOutside, SeedOutsideDomain, SegmentInCollision)
from .model import (BOX, FIXED, PRISMATIC, REVOLUTE, SPHERE, Geometry, Joint, Link, RigidTransform,
                    RobotModel, fk_batch, forward_kinematics, pose_vector, rotation_about_axis)
from .polytope import HPolytope, SampleBatch, hit_and_run_device, hit_and_run_sample
from .roadmap import (CollisionSet, DeviceRoadmap, Drm, Grid, PwlPath, build_collision_map, build_drm, collision_set,
                      load_drm, pose_rows, sample_free_configurations, sample_free_nodes, save_drm)
from .rng import child_seed
from .scene import (VoxelMap, World, load_point_cloud, load_scene, save_point_cloud, save_scene,
                    voxelize_point_cloud)

__version__ = "0.1.0"
