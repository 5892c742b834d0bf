"""B200 (sm_100a) query path of the Product Quantization Tree (arXiv 1702.05911).

The hot path (traverse → bin selection → gather → line-quantized re-rank → top-k) runs as
hand-written CUDA kernels in libpqtg.so behind the C-ABI in include/pqtg.h; this package is
the host-side mirror of the reference's query API (proj/include/pqt/search.hpp).
"""
from .index import FormatError, HostIndex, PqtConfig  # noqa: F401
from .search import (DeviceIndex, QueryResult, QueryStats, brute_force_knn, knn_query,  # noqa: F401
                     knn_query_batch, load_index, merge_topk_host, shard_range)
