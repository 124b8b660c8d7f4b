"""B200-native MinMaxLTTB: a drop-in for the reference ``tsdown`` downsampling path.

Same public names as ``tsdown`` (``/root/reference/pkg/src/tsdown/__init__.py:
8-33``) for the MinMaxLTTB path; the compute runs in hand-written sm_100a
kernels (``libmmlttb.so``, C ABI in ``include/mmlttb.h``).  Multi-GPU
sharding lives in :mod:`paper_2305_00332_b200.sharding`.
"""
from . import errors
from .core import Algorithm, BucketPartition, DownsampleConfig, TimeSeries, partition, validate
from . import metrics, raster
from .metrics import ConvMask, conv_mask, dssim, mse, pem
from .plan import MinMaxLTTBPlan
from .raster import Canvas, RasterImage, fit_canvas, rasterize, read_pgm, write_pgm
from .seriesio import read_series, write_series
from .downsamplers import (
    Batch,
    check_deferred,
    downsample,
    every_nth,
    lttb,
    m4,
    minmax,
    minmax_preselect,
    minmaxlttb,
    run_parallel,
)

__version__ = "0.1.0"

__all__ = [
    "Algorithm",
    "Batch",
    "Canvas",
    "check_deferred",
    "ConvMask",
    "RasterImage",
    "conv_mask",
    "dssim",
    "fit_canvas",
    "mse",
    "pem",
    "rasterize",
    "read_pgm",
    "write_pgm",
    "MinMaxLTTBPlan",
    "BucketPartition",
    "DownsampleConfig",
    "TimeSeries",
    "downsample",
    "errors",
    "every_nth",
    "lttb",
    "m4",
    "minmax",
    "minmax_preselect",
    "minmaxlttb",
    "partition",
    "read_series",
    "run_parallel",
    "validate",
    "write_series",
]
