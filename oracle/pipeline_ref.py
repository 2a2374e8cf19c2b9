"""Restatement of the reference training-loop body (TEST INFRASTRUCTURE ONLY).

/root/reference/pkg/src/walkjoin/pipeline.py: QueryOverlapIndex (:54-69),
sample_minibatch (:77-129), sample_negatives (:132-166) and one iteration of
the train loop (:293-310).  Used by bench.py's cpu_baseline / --impl
reference legs to time the reference CPU path.
"""

from __future__ import annotations

from collections import deque

import numpy as np

from . import core, encoder_ref


class QueryOverlapIndex:
    """pipeline.py:54-69 (queries are tuples of node ids)."""

    def __init__(self, queries):
        index: dict[int, list[int]] = {}
        for qid, q in enumerate(queries):
            for u in q:
                index.setdefault(int(u), []).append(qid)
        self._index = index
        self.nodes = np.array(sorted(index), dtype=np.int64)

    def queries_of(self, u):
        return self._index.get(u, [])

    def __len__(self):
        return len(self._index)


def canonical_nodes(nodes):
    return tuple(sorted(int(v) for v in nodes))


def sample_minibatch(index, queries, batch_capacity, batch_size, rng, n_seeds=None):
    """pipeline.py:77-129."""
    if n_seeds is None:
        n_seeds = min(16, batch_capacity)
    n_seeds = min(n_seeds, len(index.nodes))
    seeds = rng.choice(index.nodes, size=n_seeds, replace=False)
    seed_list, in_seed, batch, in_batch, queue = [], set(), [], set(), deque()
    for s in seeds:
        s = int(s)
        if s not in in_seed:
            in_seed.add(s)
            seed_list.append(s)
            queue.append(s)
    full = False
    while queue and not full:
        u = queue.popleft()
        for qid in index.queries_of(u):
            if qid in in_batch:
                continue
            if len(batch) >= batch_size:
                full = True
                break
            in_batch.add(qid)
            batch.append(qid)
            for w in queries[qid]:
                if w not in in_seed:
                    if len(seed_list) >= batch_capacity:
                        full = True
                        break
                    in_seed.add(w)
                    seed_list.append(w)
                    queue.append(w)
            if full:
                break
    return seed_list, batch


def sample_negatives(seed_set, arity, count, positive_filter, rng):
    """pipeline.py:132-166."""
    nodes = np.asarray(list(seed_set), dtype=np.int64)
    if nodes.shape[0] < arity:
        raise ValueError(f"seed set of {nodes.shape[0]} nodes cannot host arity-{arity} negatives")
    out = []
    budget = 1000 * count
    while len(out) < count:
        chunk = min(max(2 * (count - len(out)), 64), budget)
        if chunk <= 0:
            break
        draws = rng.integers(0, nodes.shape[0], size=(chunk, arity))
        budget -= chunk
        for row in draws:
            if len(out) >= count:
                break
            picked = nodes[row]
            if len(set(picked.tolist())) != arity:
                continue
            if canonical_nodes(picked) in positive_filter:
                continue
            out.append(tuple(int(v) for v in picked))
        if budget <= 0 and len(out) < count:
            raise ValueError("negative sampling budget exhausted")
    return out


def make_batch(index, positives, pos_filter, rng, batch_capacity=1500, batch_size=32, k_neg=50):
    """pipeline.py:293-304: one mini-batch of queries + labels."""
    seed_list, batch_ids = sample_minibatch(index, positives, batch_capacity, batch_size, rng)
    pos_batch = [positives[i] for i in batch_ids]
    arity = len(positives[0])
    negs = sample_negatives(seed_list, arity, k_neg * len(pos_batch), pos_filter, rng)
    nodes = np.array(list(pos_batch) + negs, dtype=np.int64)
    labels = np.concatenate([np.ones(len(pos_batch)), np.zeros(len(negs))])
    return nodes, labels


def train_step(store, params, adam, batch_nodes, labels, walk_steps, dropout, drop_rng, threads=None):
    """pipeline.py:305-309: _dense_batch -> forward -> bce -> backward -> adam."""
    dense = core.dense_batch(store, batch_nodes, threads)
    logits, cache = encoder_ref.forward(params, dense, walk_steps, dropout=dropout, training=True,
                                        dropout_rng=drop_rng)
    loss = encoder_ref.bce_loss(logits, labels)
    grads = encoder_ref.backward(params, cache, labels)
    adam.update(params, grads)
    return loss
