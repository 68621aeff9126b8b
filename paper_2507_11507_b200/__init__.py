"""B200-native MIRAGE decode-step hot path (arXiv 2507.11507).

``paper_2507_11507_b200._lib`` binds libmirage.so (include/mirage.h). The
package never imports ``oracle/``; it fails loudly when the CUDA library is
missing.
"""
from . import _lib  # noqa: F401  (raises ImportError if libmirage.so is absent)
from ._lib import Context, MirageError, model_sizes, model_arena_bytes, plan  # noqa: F401
