"""paper_2412_02244_b200 -- B200-native exact Lloyd step (the hot path of Dask-means,
arXiv 2412.02244) behind the C ABI of include/km.h.

The product is libkm.so (csrc/, sm_100a).  This package only binds it (km.py).
"""
from .km import (KM_MODE_AUTO, KM_MODE_BRUTE, KM_MODE_TILES, KM_MODE_BOUNDS, km_read_stats, km_set_mode, KM_E_CUDA, KM_E_INVALID, KM_E_NOMEM, KM_E_STATE, KM_E_UNSUPPORTED, KM_OK, Context, KmError,
                 LIB_PATH, km_assign, km_create, km_destroy, km_launch_count, km_max_k, km_read_traces, km_run,
                 km_run_ctx, km_set_stream, km_timing_enable, km_timing_read, km_update)

__all__ = ["Context", "KmError", "LIB_PATH", "km_assign", "km_create", "km_destroy", "km_launch_count", "km_max_k",
           "km_read_traces", "km_run", "km_run_ctx", "km_set_stream", "km_timing_enable", "km_timing_read",
           "km_update", "km_set_mode", "km_read_stats", "KM_MODE_AUTO", "KM_MODE_BRUTE", "KM_MODE_TILES", "KM_MODE_BOUNDS", "KM_OK", "KM_E_INVALID", "KM_E_UNSUPPORTED", "KM_E_NOMEM", "KM_E_CUDA", "KM_E_STATE"]
