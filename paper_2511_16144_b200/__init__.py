"""B200-native (sm_100a) differentiable tile rasterizer for the LEGO-SLAM hot path.

Renders RGB, depth and a d-dim (16-D) language feature per pixel from a 3D Gaussian map and
back-propagates to every Gaussian attribute and the camera pose, behind a C ABI (include/lgs.h,
liblgs.so) that mirrors the reference's lego::render / lego::render_backward
(proj/include/legoslam/renderer.hpp).
"""
from . import scenes  # noqa: F401  (numpy only)

__all__ = ["scenes", "renderer", "multiview"]


def __getattr__(name):
    if name in ("renderer", "multiview", "_lib"):
        import importlib
        return importlib.import_module(f".{name}", __name__)
    raise AttributeError(name)
