"""B200-native k-hop knowledge-graph retrieval (LogosKG hot path).

Drop-in for the retriever API of the reference ``triplehop`` package
(``/root/reference/pkg/src/triplehop/__init__.py:13-91``, hot-path subset):
``build_incidence``, ``k_hop``, ``one_hop``, ``reconstruct_paths`` and the
types they return, plus the batched ``retrieve(seeds, k, relation_filter)``.
Every hop runs in hand-written sm_100a kernels (``csrc/``) behind the C ABI
of ``include/th_b200.h``; there is no CPU fallback.
"""

__version__ = "0.1.0"

from .core_types import (
    DEFAULT_MAX_PATHS,
    EntityVector,
    HopSemantics,
    HopStep,
    HopTrace,
    PathResult,
    Triple,
    TripleVector,
    jaccard,
)
from .batch import BatchQuery, BatchResult, QueryBatch, plan_batch, run_batch, signature
from .archive import graph_from_bytes, graph_to_bytes, load_graph, save_graph
from .cache import CacheCounters, SubgraphCache, simulate_lru
from .device_graph import IncidenceGraph, build_incidence
from .errors import DataError, IntegrityError, TripleHopError, UsageError
from .partition import (
    UNASSIGNED,
    DistExchange,
    LoopbackExchange,
    PartitionedGraph,
    PartitionPlan,
    RouteResult,
    ShardPlan,
    cross_graph_k_hop,
    cross_graph_paths,
    plan_partitions,
    plan_sharding,
    route,
)
from .retriever import RetrievalResult, Retriever, k_hop, one_hop, reconstruct_paths, retrieve
from .pipeline import HostBatch, RetrievalPipeline
from .store import (
    DirectoryStore,
    InMemoryStore,
    PartitionManifest,
    StorePartitionedGraph,
    Subgraph,
    load_partition_plan,
    materialize_subgraphs,
    open_partitioned,
    save_partition_dir,
)
from .service import Labels as Dictionary, LookupResult, lookup_entities
from .targets import GpuTarget, PartitionedGpuTarget

__all__ = [
    "HostBatch",
    "RetrievalPipeline",
    "Dictionary",
    "LookupResult",
    "lookup_entities",
    "simulate_lru",
    "BatchQuery",
    "BatchResult",
    "QueryBatch",
    "plan_batch",
    "run_batch",
    "signature",
    "DirectoryStore",
    "InMemoryStore",
    "PartitionManifest",
    "StorePartitionedGraph",
    "Subgraph",
    "load_partition_plan",
    "materialize_subgraphs",
    "open_partitioned",
    "save_partition_dir",
    "CacheCounters",
    "SubgraphCache",
    "GpuTarget",
    "PartitionedGpuTarget",
    "graph_from_bytes",
    "graph_to_bytes",
    "load_graph",
    "save_graph",
    "UNASSIGNED",
    "DataError",
    "DistExchange",
    "IntegrityError",
    "LoopbackExchange",
    "PartitionPlan",
    "PartitionedGraph",
    "RouteResult",
    "ShardPlan",
    "TripleHopError",
    "UsageError",
    "cross_graph_k_hop",
    "cross_graph_paths",
    "plan_partitions",
    "plan_sharding",
    "route",
    "DEFAULT_MAX_PATHS",
    "EntityVector",
    "HopSemantics",
    "HopStep",
    "HopTrace",
    "IncidenceGraph",
    "PathResult",
    "RetrievalResult",
    "Retriever",
    "Triple",
    "TripleVector",
    "build_incidence",
    "jaccard",
    "k_hop",
    "one_hop",
    "reconstruct_paths",
    "retrieve",
]
