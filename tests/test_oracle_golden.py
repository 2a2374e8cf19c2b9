"""The CPU oracle reproduces the reference's own outputs (fixtures made by
tests/golden/make_golden.py from the real reference)."""

import os

import numpy as np
import pytest

from conftest import golden_cases, load_golden
from oracle import core, encoder_ref, pipeline_ref

GOLDEN_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.mark.parametrize("name", golden_cases())
def test_preprocess_matches_reference(name):
    g = load_golden(name)
    for threads in (1, 3):
        s = core.preprocess(g["idxptr"], g["indices"], int(g["M"]), int(g["L"]), int(g["seed"]), threads=threads)
        np.testing.assert_array_equal(s.walks, g["walks"])
        np.testing.assert_array_equal(s.table, g["table"])
        np.testing.assert_array_equal(s.dict_offsets, g["dict_offsets"])
        np.testing.assert_array_equal(s.dict_keys, g["dict_keys"])
        np.testing.assert_array_equal(s.dict_vals, g["dict_vals"])


@pytest.mark.parametrize("name", [c for c in golden_cases() if "queries" in load_golden(c)])
def test_join_and_dense_match_reference(name):
    g = load_golden(name)
    s = core.preprocess(g["idxptr"], g["indices"], int(g["M"]), int(g["L"]), int(g["seed"]), threads=2)
    wn, ri = core.join_batch_arrays(s, g["queries"], threads=2)
    np.testing.assert_array_equal(wn, g["walk_nodes"])
    np.testing.assert_array_equal(ri, g["rpe_ids"])
    dense = core.dense_batch(s, g["queries"], threads=2)
    np.testing.assert_array_equal(dense, g["dense"])
    for b in range(ri.shape[0]):
        np.testing.assert_array_equal(core.gather_rpe(s.table, ri[b]), g["dense"][b])


@pytest.mark.parametrize("name", [c for c in golden_cases() if "logits" in load_golden(c)])
def test_encoder_matches_reference(name):
    g = load_golden(name)
    p = {k: g["p_" + k].copy() for k in encoder_ref.TENSOR_ORDER}
    logits, cache = encoder_ref.forward(p, g["dense"], int(g["L"]))
    np.testing.assert_array_equal(logits, g["logits"])
    assert encoder_ref.bce_loss(logits, g["labels"]) == float(g["loss"])
    grads = encoder_ref.backward(p, cache, g["labels"])
    for k in encoder_ref.TENSOR_ORDER:
        np.testing.assert_array_equal(grads[k], g["g_" + k])
    adam = encoder_ref.Adam(p)
    adam.update(p, grads)
    for k in encoder_ref.TENSOR_ORDER:
        np.testing.assert_array_equal(p[k], g["p2_" + k])


def test_spec_vectors(golden_meta):
    # SPEC.md:155-157 triangle / seed 42, SURVEY Appendix B
    assert core.node_stream_state(42, 0) == golden_meta["triangle_state_42_0"] == 0xBDD732262FEB6E95
    g = load_golden("triangle")
    w, end = core.sample_walks(g["idxptr"], g["indices"], 0, 4, 3, core.node_stream_state(42, 0))
    assert w.tolist() == golden_meta["triangle_walks_u0"] == [[0, 1, 2, 0], [0, 1, 2, 0], [0, 1, 2, 0], [0, 2, 1, 0]]
    assert end == golden_meta["triangle_end_state"]
    raw = core.compute_rpe(w)
    assert {str(k): v.tolist() for k, v in raw.items()} == golden_meta["triangle_rpe_u0"]
    table, dicts = core.dedup_and_reindex([{0: [2, 0, 2], 1: [0, 2, 0]}, {1: [2, 0, 2], 0: [0, 2, 0]}])
    assert table.tolist() == golden_meta["dedup_path_table"] == [[0, 0, 0], [2, 0, 2], [0, 2, 0]]
    assert [{str(k): v for k, v in d.items()} for d in dicts] == golden_meta["dedup_path_dicts"]
    p = load_golden("path")
    assert p["walks"].tolist() == [[[0, 1, 0], [0, 1, 0]], [[1, 0, 1], [1, 0, 1]]]
    assert p["dict_keys"].tolist() == [0, 1, -1, -1, 0, 1, -1, -1]
    assert p["dict_vals"].tolist() == [1, 2, 0, 0, 2, 1, 0, 0]
    s = core.preprocess(p["idxptr"], p["indices"], 2, 2, 5)
    assert core.get_rpe_id(s, 0, 1) == 2 and core.get_rpe_id(s, 0, 99) == 0
    with pytest.raises(ValueError):
        core.get_rpe_id(s, 2, 0)
    iso = load_golden("isolated")
    assert iso["table"].tolist() == [[0, 0], [1, 1]] and iso["walks"].tolist() == [[[0, 0]]]


def test_minibatcher_matches_reference(golden_meta):
    mb = golden_meta["minibatch"]
    pos = [tuple(q) for q in mb["train_pos"]]
    index = pipeline_ref.QueryOverlapIndex(pos)
    pos_filter = {pipeline_ref.canonical_nodes(q) for q in pos}
    pos_filter.update(pipeline_ref.canonical_nodes(q) for q in mb["pos_filter_extra"])
    rng = np.random.default_rng(mb["rng_seed"])
    for want in mb["batches"]:
        seeds, ids = pipeline_ref.sample_minibatch(index, pos, mb["batch_capacity"], mb["batch_size"], rng)
        negs = pipeline_ref.sample_negatives(seeds, 2, mb["k_neg"] * len(ids), pos_filter, rng)
        assert seeds == want["seeds"] and ids == want["ids"]
        assert [list(q) for q in negs] == want["negs"]


@pytest.mark.parametrize("name", ["er200", "idmap120"])
def test_oracle_surl_writer_matches_reference_file(name):
    """The oracle's restatement of store._write_store reproduces the bytes
    the reference save_store wrote (tests/golden/make_surl_golden.py)."""
    from oracle import core

    d = np.load(os.path.join(GOLDEN_DIR, f"surl_{name}.npz"))
    ref = open(os.path.join(GOLDEN_DIR, f"surl_{name}.surl"), "rb").read()
    s = core.preprocess(d["idxptr"], d["indices"], int(d["M"]), int(d["L"]), int(d["seed"]))
    id_map = {int(k): int(v) for k, v in zip(d["id_keys"], d["id_vals"])} if len(d["id_keys"]) else None
    assert core.write_surl(s, id_map) == ref
