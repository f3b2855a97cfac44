"""B200-native (sm_100a) Splat-LOAM hot path: spherical 2D-Gaussian tile
rasterizer (forward + backward) and photometric Gauss-Newton registration.

Drop-in names follow the reference package ``splatscan`` (see DESIGN.md and
INTEGRATION.md); arithmetic runs only in libsplatb200.so (no CPU fallback).
"""
from .errors import DegenerateRayError, GeometryError, NoIntersectionError, RegistrationError, SplatScanError
from .geometry import SE3Pose, SphericalCamera, se3_exp, so3_exp
from .rasterizer import (BlendRecords, PixelGradients, RasterConfig, RenderOutput, SplatGradients,
                         rasterize_backward, rasterize_forward)
from .splats import SplatModel
from .keyframe import (NormalImage, RangeImage, build_range_image, estimate_camera, make_keyframe, range_image_normals,
                       smooth_range_image)

__all__ = ["SplatScanError", "GeometryError", "DegenerateRayError", "NoIntersectionError", "RegistrationError",
           "SE3Pose", "SphericalCamera", "se3_exp", "so3_exp", "SplatModel", "RasterConfig", "RenderOutput",
           "PixelGradients", "SplatGradients", "BlendRecords", "rasterize_forward", "rasterize_backward",
           "RangeImage", "NormalImage", "build_range_image", "smooth_range_image", "range_image_normals",
           "estimate_camera", "make_keyframe"]
__version__ = "0.1.0"
