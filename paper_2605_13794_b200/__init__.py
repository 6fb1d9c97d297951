"""BlitzGS (arXiv 2605.13794) per-view distributed splatting step on B200 (sm_100a).

The product is libbgs.so (include/bgs.h); `paper_2605_13794_b200.bgs` is its thin binding.
The binding is imported lazily so that `paper_2605_13794_b200.build` can (re)build the library
without loading a stale one.  See DESIGN.md.
"""
import importlib

_BINDING = ("BGS_IMPORTANCE", "BGS_NO_COLOR", "BgsError", "Context", "GaussianPlanes", "GradPlanes", "bgs_importance",
            "bgs_project", "bgs_project_bwd", "bgs_raster_bwd", "bgs_raster_fwd", "bgs_route", "bgs_route_reverse",
            "bgs_sort_tiles", "bgs_view_step", "bgs_view_step_host", "bgs_spatial_order", "spatial_order", "camera",
            "importance_out", "lod_gate", "unique_id")

__all__ = list(_BINDING)


def __getattr__(name):
    if name in _BINDING:
        return getattr(importlib.import_module(".bgs", __name__), name)
    raise AttributeError(name)
