"""Route an unchanged ``splatscan`` (the reference package) through the B200 path.

The reference's consumers import the hot-path functions BY NAME, so replacing
``splatscan.rasterizer.rasterize_forward`` alone would not reach them.  The
bound names (SURVEY 8(b) "Callers to patch"):

  splatscan/mapping.py:38-44        rasterize_forward, rasterize_backward
                                    (+ make_keyframe :106, refine :455 defined there)
  splatscan/registration.py:27      rasterize_forward (+ register :387, build_leaf_tree :98)
  splatscan/pipeline.py:30-32       rasterize_forward, register, refine, make_keyframe
  splatscan/cli.py:45               rasterize_forward

``install()`` re-points every one of them at the B200 implementations and
returns a handle whose ``uninstall()`` restores the originals.  The patched
functions accept the reference's own objects (``SphericalCamera``,
``SE3Pose``, ``SplatModel``, ``RasterConfig``, ``RegistrationConfig``,
``LocalMap``) and return objects with the reference's field names; where a
caller relies on the reference's concrete classes (``Keyframe``,
``RangeImage``, ``NormalImage``, ``RegistrationResult``, ``SE3Pose``) the
adapter builds those classes from the B200 results.
"""
from __future__ import annotations

import importlib
from dataclasses import dataclass, field

__all__ = ["install", "Installed", "PATCH_TABLE"]

# module -> names the adapter replaces in it (reference file:line of the binding)
PATCH_TABLE = {
    "rasterizer": ("rasterize_forward", "rasterize_backward"),          # rasterizer.py:455, :534
    "mapping": ("rasterize_forward", "rasterize_backward",              # mapping.py:38-44
                "make_keyframe", "refine"),                             # mapping.py:106, :455
    "registration": ("rasterize_forward", "register", "build_leaf_tree"),  # registration.py:27, :387, :98
    "pipeline": ("rasterize_forward", "register", "refine", "make_keyframe"),  # pipeline.py:21-32
    "cli": ("rasterize_forward",),                                       # cli.py:45
}


@dataclass
class Installed:
    package: str
    originals: dict = field(default_factory=dict)  # (module, name) -> original object

    def uninstall(self) -> None:
        for (mod, name), obj in self.originals.items():
            setattr(importlib.import_module(f"{self.package}.{mod}"), name, obj)
        self.originals.clear()

    @property
    def patched(self) -> list:
        return sorted(self.originals)


def _replacements(pkg: str) -> dict:
    from . import keyframe as KF
    from . import mapping as MP
    from . import rasterizer as RZ
    from . import registration as REG

    ref_geo = importlib.import_module(f"{pkg}.geometry")
    ref_map = importlib.import_module(f"{pkg}.mapping")
    ref_reg = importlib.import_module(f"{pkg}.registration")

    def make_keyframe(index, cloud, pose, width, height):
        """mapping.py:106-114: the reference's camera estimate, B200 range image and normals,
        returned as the reference's Keyframe / RangeImage / NormalImage."""
        import numpy as np
        cloud = np.asarray(cloud, dtype=float)
        cam = ref_geo.estimate_camera(cloud, width, height)
        im = KF.keyframe_images(cam, cloud)
        rimg = ref_geo.RangeImage(im["range"].cpu().numpy(), im["valid"].cpu().numpy().astype(bool))
        nimg = ref_geo.NormalImage(im["normal"].cpu().numpy(), im["nvalid"].cpu().numpy().astype(bool))
        return ref_map.Keyframe(index, cloud, pose.copy(), cam, rimg, nimg)

    def register(model, scan, cam, initial, cfg=None, raster=None, rng=None):
        """registration.py:387-524 on the device; the result is the reference's
        RegistrationResult holding a pose of the caller's SE3Pose class."""
        res = REG.register(model, scan, cam, initial, cfg, raster, rng)
        pose = type(initial)(res.pose.rotation, res.pose.translation)
        return ref_reg.RegistrationResult(pose, res.converged, res.iterations, res.geo_rms, res.photo_rms,
                                          res.n_geo, res.n_photo, res.mode, res.used_fallback, res.message)

    return {"rasterize_forward": RZ.rasterize_forward, "rasterize_backward": RZ.rasterize_backward,
            "make_keyframe": make_keyframe, "refine": MP.refine, "register": register,
            "build_leaf_tree": REG.build_leaf_tree}


def install(package: str = "splatscan") -> Installed:
    """Patch every bound hot-path name of ``package`` (the reference) in place."""
    importlib.import_module(package)
    repl = _replacements(package)
    inst = Installed(package)
    for mod, names in PATCH_TABLE.items():
        m = importlib.import_module(f"{package}.{mod}")
        for name in names:
            if not hasattr(m, name):
                inst.uninstall()
                raise AttributeError(f"{package}.{mod} has no attribute {name!r}: not the expected reference")
            inst.originals[(mod, name)] = getattr(m, name)
            setattr(m, name, repl[name])
    return inst
