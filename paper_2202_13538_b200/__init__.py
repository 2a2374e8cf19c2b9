"""B200-native walk -> RPE -> join hot path of SUREL (reference package ``walkjoin``).

Drop-in for the reference's hot-path API (/root/reference/pkg/src/walkjoin):
``preprocess``, ``sample_walks``, ``compute_rpe``, ``get_rpe_id``,
``join_batch_arrays``, ``join_query``, ``join_batch``, ``gather_rpe`` and the
``_dense_batch`` call site (``dense_batch``), backed by hand-written sm_100a
kernels behind the C ABI in include/walkjoin_b200.h.  There is no CPU
fallback: every call needs the in-tree CUDA library and a CUDA device.
"""

from .graph import DeviceGraph, Graph, GraphFormatError, Query, load_edge_list, project_hyperedges
from .sampler import (RawRpeMap, TypedCSR, WalkRng, WalkSet, compute_rpe, edge_types_from_node_types, preprocess,
                      preprocess_typed, sample_walks, sample_walks_typed, typed_csr)
from .store import (NodeEntry, RpeTable, StoreFormatError, SubgraphStore, dedup_and_reindex, dict_capacities,
                    get_rpe_id, intern_vectors, load_store, save_store)
from .joiner import JoinedQuery, dense_batch, gather_rpe, join_batch, join_batch_arrays, join_query
from .encoder import AdamState, ModelParams, adam_step, backward, bce_loss, forward, init_params
from .pipeline import (BatchPlanner, QueryOverlapIndex, QuerySplit, TrainConfig, TrainStep, infer, sample_minibatch,
                       sample_negatives, score_array, train, validation_metric)
from .metrics import RankedQueryResult, hits_at_k, mrr, rank_of_positive, roc_auc
from .seeds import derive_seed

_dense_batch = dense_batch  # reference call-site name (pipeline.py:169)

__version__ = "0.1.0"

__all__ = [
    "Graph", "DeviceGraph", "GraphFormatError", "Query", "load_edge_list", "project_hyperedges",
    "WalkSet", "RawRpeMap", "WalkRng", "sample_walks", "compute_rpe", "preprocess",
    "TypedCSR", "typed_csr", "sample_walks_typed", "preprocess_typed", "edge_types_from_node_types",
    "RpeTable", "NodeEntry", "SubgraphStore", "StoreFormatError", "dict_capacities", "get_rpe_id",
    "intern_vectors", "dedup_and_reindex",
    "save_store", "load_store",
    "JoinedQuery", "join_query", "join_batch", "join_batch_arrays", "gather_rpe", "dense_batch",
    "ModelParams", "AdamState", "init_params", "forward", "backward", "bce_loss", "adam_step",
    "TrainConfig", "TrainStep", "BatchPlanner", "QuerySplit", "QueryOverlapIndex", "sample_minibatch",
    "sample_negatives", "train", "infer", "score_array", "validation_metric",
    "RankedQueryResult", "rank_of_positive", "mrr", "hits_at_k", "roc_auc", "derive_seed",
]
