"""B200-native (sm_100a) reconstruction path of arXiv 2305.02064.

Public API: :class:`Plan` (``sar_plan_create`` / ``sar_reconstruct`` /
``sar_plan_destroy`` of ``include/sar_b200.h``).  All compute runs in the
in-tree CUDA library ``libsar_b200.so``; PyTorch provides device memory and
streams only.  There is no CPU fallback.
"""
from .sar import (Plan, SlabPlan, SarError, bpa, bpa_scene, describe, describe_scene, describe_stolt_ranges,  # noqa: F401
                  describe_stolt_ranges_scene, describe_nearest, describe_nearest_scene, load_library, LIB_PATH,
                  SAR_NO_COMPENSATION, SAR_OUTPUT_COMPLEX, SAR_PROFILE_STAGES, SAR_IMAGE_2D, SAR_GRID_NUFFT,
                  SAR_GRID_NEAREST, SAR_STOLT_NUFFT, SAR_REPORT_PEAK, SAR_FORCE_PLAIN, SAR_CUDA_GRAPH, STAGE_NAMES)

__all__ = ["Plan", "SlabPlan", "SarError", "bpa", "bpa_scene", "describe", "describe_scene", "describe_stolt_ranges",
           "describe_stolt_ranges_scene", "describe_nearest", "describe_nearest_scene", "load_library", "LIB_PATH", "SAR_NO_COMPENSATION", "SAR_OUTPUT_COMPLEX",
           "SAR_PROFILE_STAGES", "SAR_IMAGE_2D", "SAR_GRID_NUFFT", "SAR_GRID_NEAREST", "SAR_STOLT_NUFFT", "SAR_REPORT_PEAK", "SAR_FORCE_PLAIN", "SAR_CUDA_GRAPH",
           "STAGE_NAMES"]
