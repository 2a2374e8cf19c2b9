"""Ranking and classification metrics (reference metrics.py:1-59).

Same definitions and tie convention as the reference: a positive tied with t
negatives sits half-way between its optimistic and pessimistic rank
(metrics.py:24-31), and ROC AUC is the rank-sum form with average ranks for
ties (metrics.py:50-59, ``scipy.stats.rankdata(method="average")``).

Host inputs (lists / numpy) are scored in float64 numpy exactly as the
reference does.  CUDA tensors are scored on the device without leaving HBM:
validation at the paper's protocol (1,000 negatives per positive,
PAPER.md:284) produces millions of scores per epoch, and moving them to the
host to rank would cost more than computing them.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

import numpy as np
import torch


@dataclass
class RankedQueryResult:
    """One positive score against its paired negative scores (metrics.py:16-21)."""

    pos_score: float
    neg_scores: Sequence[float]


def rank_of_positive(result: RankedQueryResult) -> float:
    """Mid-rank of the positive among its negatives, 1 = best (metrics.py:24-31)."""
    neg = np.asarray(result.neg_scores, dtype=np.float64)
    if neg.size == 0:
        raise ValueError("ranking needs at least one negative score")
    greater = int(np.count_nonzero(neg > result.pos_score))
    ties = int(np.count_nonzero(neg == result.pos_score))
    return 1.0 + greater + 0.5 * ties


def mrr(results: Sequence[RankedQueryResult]) -> float:
    """Mean reciprocal rank (metrics.py:34-38)."""
    if not results:
        raise ValueError("mrr needs at least one result")
    return float(np.mean([1.0 / rank_of_positive(r) for r in results]))


def hits_at_k(results: Sequence[RankedQueryResult], k: int) -> float:
    """Fraction of positives ranked within the top k (metrics.py:41-47)."""
    if k < 1:
        raise ValueError("k must be >= 1")
    if not results:
        raise ValueError("hits_at_k needs at least one result")
    return float(np.mean([1.0 if rank_of_positive(r) <= k else 0.0 for r in results]))


def _average_ranks(x: np.ndarray) -> np.ndarray:
    """1-based average ranks with ties sharing their mean rank
    (= scipy.stats.rankdata(x, method="average"))."""
    order = np.argsort(x, kind="mergesort")
    xs = x[order]
    n = xs.shape[0]
    starts = np.flatnonzero(np.concatenate([[True], xs[1:] != xs[:-1]]))
    ends = np.concatenate([starts[1:], [n]])
    avg = (starts + ends + 1) / 2.0  # mean of ranks starts+1 .. ends
    ranks = np.empty(n, dtype=np.float64)
    ranks[order] = np.repeat(avg, ends - starts)
    return ranks


def roc_auc(pos_scores, neg_scores) -> float:
    """P(random positive outscores random negative), ties count one half
    (metrics.py:50-59).  CUDA tensors are ranked on the device."""
    if isinstance(pos_scores, torch.Tensor) and pos_scores.is_cuda:
        return roc_auc_device(pos_scores, neg_scores)
    pos = np.asarray(pos_scores, dtype=np.float64)
    neg = np.asarray(neg_scores, dtype=np.float64)
    if pos.size == 0 or neg.size == 0:
        raise ValueError("roc_auc needs scores on both sides")
    ranks = _average_ranks(np.concatenate([pos, neg]))
    pos_rank_sum = ranks[: pos.size].sum()
    return float((pos_rank_sum - pos.size * (pos.size + 1) / 2.0) / (pos.size * neg.size))


# ----------------------------------------------------------------- device --

def roc_auc_device(pos: torch.Tensor, neg: torch.Tensor) -> float:
    """Rank-sum AUC on the device: one sort, tie groups from
    ``unique_consecutive``, float64 rank sums (exact for < 2^53 scores)."""
    pos = pos.reshape(-1).double()
    neg = neg.reshape(-1).double()
    p, q = pos.numel(), neg.numel()
    if p == 0 or q == 0:
        raise ValueError("roc_auc needs scores on both sides")
    allv = torch.cat([pos, neg])
    xs, order = torch.sort(allv, stable=True)
    _, counts = torch.unique_consecutive(xs, return_counts=True)
    ends = torch.cumsum(counts, 0)
    starts = ends - counts
    avg = (starts + ends + 1).double() / 2.0
    ranks_sorted = torch.repeat_interleave(avg, counts)
    is_pos = (order < p).double()
    pos_rank_sum = float((ranks_sorted * is_pos).sum())
    return (pos_rank_sum - p * (p + 1) / 2.0) / (p * q)


def positive_ranks_device(pos: torch.Tensor, neg: torch.Tensor, group_sizes) -> torch.Tensor:
    """Mid-rank of every positive among its own negatives (metrics.py:24-31).

    ``neg`` is the flat concatenation of the groups; ``group_sizes`` their
    lengths (an int for equal groups)."""
    pos = pos.reshape(-1).double()
    neg = neg.reshape(-1).double()
    P = pos.numel()
    if isinstance(group_sizes, int):
        if group_sizes < 1:
            raise ValueError("ranking needs at least one negative score")
        sizes = torch.full((P,), group_sizes, dtype=torch.int64, device=pos.device)
    else:
        sizes = torch.as_tensor(np.asarray(group_sizes, dtype=np.int64), device=pos.device)
        if bool((sizes < 1).any()):
            raise ValueError("ranking needs at least one negative score")
    owner = torch.repeat_interleave(torch.arange(P, device=pos.device), sizes)
    pv = pos[owner]
    greater = torch.zeros(P, dtype=torch.float64, device=pos.device).index_add_(0, owner, (neg > pv).double())
    ties = torch.zeros(P, dtype=torch.float64, device=pos.device).index_add_(0, owner, (neg == pv).double())
    return 1.0 + greater + 0.5 * ties


def mrr_device(pos: torch.Tensor, neg: torch.Tensor, group_sizes) -> float:
    if pos.numel() == 0:
        raise ValueError("mrr needs at least one result")
    return float((1.0 / positive_ranks_device(pos, neg, group_sizes)).mean())


def hits_at_k_device(pos: torch.Tensor, neg: torch.Tensor, group_sizes, k: int) -> float:
    if k < 1:
        raise ValueError("k must be >= 1")
    if pos.numel() == 0:
        raise ValueError("hits_at_k needs at least one result")
    return float((positive_ranks_device(pos, neg, group_sizes) <= k).double().mean())
