"""BlitzGS (arXiv 2605.13794) per-view distributed splatting step on B200 (sm_100a).

The product is libbgs.so (include/bgs.h); this package is its thin binding.  See DESIGN.md.
"""
from .bgs import (BGS_IMPORTANCE, BGS_NO_COLOR, BgsError, Context, GaussianPlanes, GradPlanes, bgs_importance,
                  bgs_project, bgs_project_bwd, bgs_raster_bwd, bgs_raster_fwd, bgs_route, bgs_route_reverse,
                  bgs_sort_tiles, bgs_view_step, bgs_view_step_host, camera, importance_out, lod_gate, unique_id)

__all__ = ["BGS_IMPORTANCE", "BGS_NO_COLOR", "BgsError", "Context", "GaussianPlanes", "GradPlanes", "bgs_importance",
           "bgs_project", "bgs_project_bwd", "bgs_raster_bwd", "bgs_raster_fwd", "bgs_route", "bgs_route_reverse",
           "bgs_sort_tiles", "bgs_view_step", "bgs_view_step_host", "camera", "importance_out", "lod_gate",
           "unique_id"]
