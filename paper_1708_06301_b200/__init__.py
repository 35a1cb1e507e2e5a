"""B200-native hot path of the temporal stereo method of arXiv 1708.06301.

Drop-in for the reference package ``egostereo``: the same public names and
signatures (see the reference ``__init__.py:20-81``), with every per-pixel
stage running as hand-written sm_100a CUDA behind the C ABI in
``include/egostereo_b200.h``.  The CUDA library is loaded on first use;
there is no CPU fallback.

Modules: core (boundary types), geometry (4x4 homographies, device warp),
prediction, sgm, fusion (drop-in stage functions), pipeline
(DisparityPipeline / BatchedPipeline on device-resident state), metrics
(device bad-pixel evaluation), install (drop-in rebinding of the reference
package ``egostereo``: its own sequence runner, KITTI I/O and CLI then run on
top of the device stages), scenes (seeded benchmark inputs), build (nvcc
build of libegostereo_b200.so).
"""

from .core import (DisparityMap, FilterState, GrayImage, StereoRig, VarianceMap,
                   make_empty_state, make_invalid_map, make_motion)
from .errors import (BehindCameraError, DeviceUnavailableError, DeviceUnsupportedError,
                     PointAtInfinityError)
from .fusion import FusionParams, fuse_maps
from .geometry import disparity_homography, euclidean_warp_oracle, warp_point
from .metrics import BadPixelResult, bad_pixel_rate, search_space_fraction
from .pipeline import BatchedPipeline, DisparityPipeline, FrameResult, PipelineParams
from .prediction import PredictionParams, predict_maps
from .sgm import IntervalMap, SgmParams, full_range_intervals, search_intervals

__version__ = "0.1.0"

__all__ = [
    "BadPixelResult", "BatchedPipeline", "BehindCameraError", "DeviceUnavailableError", "DeviceUnsupportedError",
    "DisparityMap", "DisparityPipeline", "FilterState", "FrameResult", "FusionParams",
    "GrayImage", "IntervalMap", "PipelineParams", "PointAtInfinityError", "PredictionParams",
    "SgmParams", "StereoRig", "VarianceMap", "disparity_homography",
    "euclidean_warp_oracle", "full_range_intervals", "fuse_maps", "make_empty_state",
    "make_invalid_map", "make_motion", "predict_maps", "search_intervals",
    "bad_pixel_rate",
    "search_space_fraction", "warp_point", "__version__",
]
