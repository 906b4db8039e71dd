"""B200-native Euler-tour graph pipeline (arXiv 2103.15217): LCA and bridges.

Public surface mirrors the reference's ``ett`` namespace; see ``ett.py`` and
include/ettg.h for the C-ABI underneath.
"""
from . import _lib
from .ett import *  # noqa: F401,F403
from .ett import (AdjacencyIndex, BridgeMask, EdgeList, InlabelIndex, NaiveIndex, NodeStats,
                  RmqLcaIndex, RootedTree, SpanningTree, answer_batch, bfs_tree, build_adjacency,
                  ck_bridges, hybrid_bridges, inlabel_build, inlabel_lca, naive_build, naive_lca,
                  node_stats, rmq_lca, rmq_lca_build, tv_bridges)
from ._lib import InvalidArgument, OutOfRange, ParseError, lib

__all__ = [
    "AdjacencyIndex", "BridgeMask", "EdgeList", "InlabelIndex", "NaiveIndex", "NodeStats",
    "RmqLcaIndex", "RootedTree", "SpanningTree", "answer_batch", "bfs_tree", "build_adjacency",
    "ck_bridges", "hybrid_bridges", "inlabel_build", "inlabel_lca", "naive_build", "naive_lca",
    "node_stats", "rmq_lca", "rmq_lca_build", "tv_bridges", "InvalidArgument", "OutOfRange", "ParseError", "lib",
]
