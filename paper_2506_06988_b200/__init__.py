"""B200-native hybrid Gaussian-splat + textured-mesh renderer (arXiv 2506.06988).

Drop-in device implementation of the gsmesh render/loss operator API; every
compute step runs in hand-written sm_100a kernels in libhgs.so (C ABI:
include/hgs.h).  There is no CPU fallback.
"""

from .scene import Camera, GaussianSet, RenderOutputs, SceneError, TexturedMesh  # noqa: F401
from .splat import (ALPHA_CLAMP, COV_FLOOR, EARLY_STOP_T, SH_C0, SH_C1, SIGMA_SKIP, SUPPORT_MAHAL2, TILE_PX,  # noqa: F401
                    GaussianGrads, MeshLayer, ProjectedGaussians, RenderCtx, TileBins, build_tiles, project,
                    rasterize_backward, rasterize_forward, render, render_depth)

__version__ = "0.1.0"
