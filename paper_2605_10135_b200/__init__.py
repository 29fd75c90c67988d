"""B200-native (sm_100a) hot path of ScaleGANN's divide-and-merge graph-index build
(arxiv 2605.10135): partition -> per-shard exact kNN (tcgen05) -> detour prune + reverse
edges -> cross-shard merge, behind the C ABI of include/scalegann.h."""
from . import datagen  # noqa: F401  (no method arithmetic; safe without a GPU)

__all__ = ["datagen", "api", "pipeline"]
