"""Exception types of the drop-in API.

Same class names and hierarchy as the reference (pkg/src/splatscan/errors.py:4-33)
so callers written against the reference catch the same exceptions.  When the
reference package is importable, its classes are reused so that
``except splatscan.errors.GeometryError`` also catches ours.
"""
try:  # pragma: no cover - depends on the environment
    from splatscan.errors import (DegenerateRayError, GeometryError, NoIntersectionError,  # type: ignore
                                  RegistrationError, SplatScanError)
except Exception:  # the reference is not installed (e.g. on the GPU box)

    class SplatScanError(Exception):
        """Base class (errors.py:4)."""

    class GeometryError(SplatScanError, ValueError):
        """Invalid geometric input (errors.py:8)."""

    class DegenerateRayError(GeometryError):
        """Pixel ray too close to a pole (errors.py:12)."""

    class NoIntersectionError(SplatScanError):
        """Ray/splat pair has no usable intersection (errors.py:16)."""

    class RegistrationError(SplatScanError, RuntimeError):
        """Scan-to-map alignment failed (errors.py:24)."""

__all__ = ["SplatScanError", "GeometryError", "DegenerateRayError", "NoIntersectionError", "RegistrationError"]
