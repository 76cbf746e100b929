"""B200-native unified HDR LPA operator (arXiv 1308.4908 re-built for sm_100a).

Host layer mirroring the reference package ``hdrfuse``'s reconstruction API
(``frames_to_samples`` -> ``reconstruct_frame``) over hand-written CUDA
kernels behind a C ABI (include/hdr_lpa.h, libhdrlpa.so).  See DESIGN.md.
"""

__version__ = "0.1.0"

from .bayer import BayerPattern, ColorChannel, channel_at, channel_map, channel_masks
from .images import CFAImage, FloatFrame, HDRImage
from .lpa import (
    SUPPORT_SIGMAS,
    ReconstructionParams,
    basis_row,
    grid_coordinates,
    reconstruct_channel,
    reconstruct_frame,
)
from .radiometry import (
    ConfigurationError,
    NoiseCalibration,
    RawFrameSet,
    SensorConfig,
    estimate_radiance,
    estimate_variance,
    frame_to_samples,
    frames_to_samples,
    saturation_mask,
)
from .validation import ShapeMismatchError

from .samples import (  # noqa: E402
    LocalPolynomialRegressor,
    RadianceSample,
    RadianceSamples,
    SampleIndex,
)
from .steering import (  # noqa: E402
    AdaptiveParams,
    SteeringField,
    calpa_reconstruct,
    compute_steering_field,
    gradient_field,
)

from .pipeline import FramePipeline  # noqa: E402  (streaming: pinned H2D, graphs, D2H)

__all__ = [
    "BayerPattern", "CFAImage", "ColorChannel", "ConfigurationError", "FloatFrame", "HDRImage",
    "NoiseCalibration", "RawFrameSet", "ReconstructionParams", "SUPPORT_SIGMAS", "SensorConfig",
    "ShapeMismatchError", "basis_row", "channel_at", "channel_map", "channel_masks",
    "estimate_radiance", "estimate_variance", "frame_to_samples", "frames_to_samples",
    "grid_coordinates", "reconstruct_channel", "reconstruct_frame", "saturation_mask",
    "AdaptiveParams", "SteeringField", "calpa_reconstruct", "compute_steering_field",
    "gradient_field", "LocalPolynomialRegressor", "RadianceSample", "RadianceSamples",
    "SampleIndex", "FramePipeline",
]
