"""B200-native AdR-Gaussian forward rasterizer (arXiv 2409.08669).

Drop-in for the reference package's render API (splatbench 0.1.0,
sb/__init__.py:10-48): the same stage functions, containers, constants and
exceptions, backed by hand-written sm_100a kernels in libadrsplat.so
(include/adr_splat.h).  Arrays are CUDA tensors; each container has
``to_numpy()`` for the reference's numpy layout.
"""

from .errors import CapacityError, InternalError, SceneFormatError, SceneValidationError
from .footprint import (CullExtent, EllipseCoefficients, ProjectedGaussian, aabb_extents,
                        bounding_box_halfwidths, bounding_circle_radius, build_covariance3d,
                        composite_pixels, eigen_extents, ellipse_coefficients, evaluate_sh,
                        project_gaussian, quaternion_to_rotation, radius_adaptive, radius_baseline)
from .metrics import (DEFAULT_WEIGHTS, PSNR_IDENTICAL_SENTINEL, BalanceStepResult, LoadStats,
                      LossWeights, l1_loss, load_loss, psnr, replace_opacity, ssim, toy_balance_step,
                      total_loss)
from .pipeline import (MAX_BATCH_VIEWS, STAGE_NAMES, PipelineResult, Rasterizer, RenderStats,
                       preprocess_views, render_views_batched, run_pipeline)
from .projection import (ALPHA_LOW, BASE_RADIUS_MULTIPLIER, COV_DILATION, FOV_CLAMP_FACTOR,
                         CullingMode, Projection, preprocess)
from .refrender import render_reference
from .render import ALPHA_CLAMP, TERMINATION_THRESHOLD, Image, LoadMap, render
from .scene import (Camera, DeviceScene, Gaussian3D, Scene, SceneArrays, SyntheticSpec,
                    generate_synthetic, synthetic_arrays)
from .scene_io import (SceneDiagnostic, load_json, load_ply, load_ply_arrays, load_ply_device, load_scene,
                       load_scene_arrays, normalize_quaternion, save_json, save_ply, save_scene,
                       validate_scene)
from .tiling import (TILE_SIZE, TileGrid, TilePairList, TileRect, build_pairs,
                     duplicate_with_keys, identify_tile_ranges, inclusive_sum, sort_pairs,
                     tiles_touched, touched_counts)

__version__ = "0.1.0"

__all__ = [
    "ALPHA_CLAMP", "ALPHA_LOW", "BASE_RADIUS_MULTIPLIER", "COV_DILATION", "FOV_CLAMP_FACTOR",
    "PSNR_IDENTICAL_SENTINEL", "STAGE_NAMES", "TERMINATION_THRESHOLD", "TILE_SIZE", "Camera",
    "CapacityError", "CullingMode", "DeviceScene", "Gaussian3D", "Image", "InternalError",
    "LoadMap", "LoadStats", "PipelineResult", "Projection", "Rasterizer", "RenderStats", "Scene",
    "SceneArrays", "SceneFormatError", "SceneValidationError", "SyntheticSpec", "TileGrid",
    "TilePairList", "TileRect", "build_pairs", "SceneDiagnostic", "load_json", "load_ply",
    "load_ply_arrays", "load_ply_device", "load_scene", "load_scene_arrays", "normalize_quaternion", "save_json",
    "save_ply", "save_scene", "validate_scene", "DEFAULT_WEIGHTS", "BalanceStepResult", "LossWeights",
    "l1_loss", "render_reference", "CullExtent", "EllipseCoefficients", "ProjectedGaussian",
    "aabb_extents", "bounding_box_halfwidths", "bounding_circle_radius", "build_covariance3d",
    "composite_pixels", "eigen_extents", "ellipse_coefficients", "evaluate_sh", "project_gaussian",
    "quaternion_to_rotation", "radius_adaptive", "radius_baseline", "replace_opacity", "ssim", "toy_balance_step", "total_loss", "duplicate_with_keys", "generate_synthetic",
    "identify_tile_ranges", "inclusive_sum", "load_loss", "preprocess", "psnr", "render",
    "run_pipeline", "sort_pairs", "MAX_BATCH_VIEWS", "preprocess_views", "render_views_batched", "synthetic_arrays", "tiles_touched", "touched_counts",
]
