"""B200-native (sm_100a) motion-blur rasterizer with the fast barycentric solver of arxiv 2602.07860.

Layers: include/blurrast.h (C ABI) -> csrc/*.cu (libblurrast.so: K1..K7 CUDA kernels + host plan)
-> _lib.py (ctypes binding, same names as the C entry points) -> renderer.py (BlurRenderer,
blur_render autograd op) -> dist.py (image / sub-frame sharding over torch.distributed + NCCL).
"""
from . import _lib  # noqa: F401
from ._lib import BlurError  # noqa: F401
from .renderer import BlurRenderer, blur_render  # noqa: F401
from .recover import Recovery  # noqa: F401

__all__ = ["BlurRenderer", "blur_render", "BlurError", "Recovery"]
