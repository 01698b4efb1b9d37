"""B200-native LiGen dock-and-score hot path (arXiv 2303.06150).

The product is libvsdock.so (include/vsdock.h): CUDA kernels for sm_100a plus a
C++ host runtime.  ``vsdock`` is its ctypes binding; ``parallel`` the
multi-GPU shard / gather / merge over torch.distributed (NCCL).
"""
from .vsdock import Engine, VsError, load_library, SO_PATH  # noqa: F401
