"""meshlayers on B200: the GPU layer-editing hot path of arXiv 2501.14807, rebuilt for sm_100a.

Drop-in surface
  * ``_native``  -- kernel backend with the reference's ``_kernels_numpy`` signatures
                    (``coverage_fill``, ``raster_depth``, ``raster_tea``), backed by
                    ``libmeshlayers_b200.so`` (C ABI: ``include/meshlayers_b200.h``).
  * SPEC operation names: ``pool_acquire``, ``rasterize``, ``create_layer``, ``uv_coverage``, ``render_depth``,
    ``compute_tool_projection``, ``project_fragment``, ``apply_stroke``, ``build_outline_mask``,
    ``apply_padding``, ``mesh_surface_area``.
Extensions named by the north star (not in the reference): ``build_surface_map``,
``select_sphere``, ``select_sphere_batch``, ``select_threshold``, ``layer_union`` /
``layer_intersection`` / ``layer_difference`` / ``layer_mask`` / ``layer_chain``, ``layer_area`` /
``layers_area`` / ``label_area`` / ``layer_stats``, and row sharding in ``sharding``.

Importing the package never touches CUDA; every operation raises ``BackendUnavailable`` when the
library or a device is missing (no CPU fallback).
"""
from . import errors
from .errors import *  # noqa: F401,F403
from .mesh_core import (Camera, DepthMap, SurfaceMap, TriangleMesh, build_surface_map,
                        mesh_surface_area, render_depth, uv_coverage)
from .raster_device import TexturePool, default_pool, pool_acquire, rasterize
from .layer_core import (InformationLayer, create_layer, label_area, layer_area, layer_chain,
                         layer_difference, layer_intersection, layer_mask, layer_precision,
                         layer_stats, layer_union, layers_area)
from .editing import (EditingTool, EditProjection, EditResult, StrokeContext, apply_padding,
                      apply_stroke, build_outline_mask, compute_tool_projection, project_fragment,
                      select_sphere, select_sphere_batch, select_threshold, stroke, stroke_gesture)
from .display import Palette, map_value_to_color, resolve_display
from .layer_io import decode_layer, encode_layer, load_layer, save_layer
from .octree import (OctreeLayer, SurfaceOctree, build_octree, create_octree_layer, octree_edit,
                     octree_precision, octree_upload_size)

__version__ = "0.1.0"
