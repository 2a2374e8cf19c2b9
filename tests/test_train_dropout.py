"""Training quality WITH dropout (north_star: "final MRR/AUC must agree within
0.5 points") on BASELINE.json configs[0] (C1: 10K-node / 100K-edge ER graph,
M=50, L=3, one epoch, dropout 0.1).

The fixtures were written by the REAL reference ``train`` + ``infer``
(pipeline.py:241-355) for five training seeds (tests/golden/
make_train_dropout_golden.py).  The reference draws its dropout masks from
numpy PCG64 (encoder.py:154-158); the fused kernel draws equal-in-
distribution masks from its own counter-based stream, so runs agree per seed
only up to dropout noise.  With ``exact_batches=True`` the mini-batches, the
negatives and the initial parameters are the reference's for the same seed,
so the dropout realisation is the only difference.  The test compares the
mean over the five seeds of the test AUC and MRR (1,000-style ranking against
each positive's 10 negatives, the fixture's protocol) with the reference's
mean, and reports the per-seed spread it measured."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

DIR = os.path.join(GOLDEN, "train_dropout")
SEEDS = sorted(int(f[len("c1_seed"):-4]) for f in os.listdir(DIR) if f.startswith("c1_seed"))


def _load(name):
    with np.load(os.path.join(DIR, name + ".npz")) as z:
        return {k: z[k] for k in z.files}


def test_fixture_set_complete():
    """Five reference seeds, each with the test metrics and scores."""
    assert len(SEEDS) >= 5
    for s in SEEDS:
        d = _load(f"c1_seed{s}")
        assert {"test_auc", "test_mrr", "train_loss", "test_pos_scores"} <= set(d)


@pytest.mark.gpu
def test_train_with_dropout_matches_reference_mean():
    import torch

    import paper_2202_13538_b200 as wj
    from paper_2202_13538_b200 import metrics as M

    c = _load("c1")
    g = wj.Graph(int(c["n"]), c["idxptr"], c["indices"])
    store = wj.preprocess(g, int(c["M"]), int(c["L"]), 3)
    split = wj.QuerySplit(train_pos=c["train_pos"], valid_pos=c["valid_pos"], test_pos=c["test_pos"],
                          valid_neg=list(c["valid_neg"]), test_neg=list(c["test_neg"]))
    k = c["test_neg"].shape[1]
    ours, ref = [], []
    for s in SEEDS:
        r = _load(f"c1_seed{s}")
        cfg = wj.TrainConfig(k_neg=50, max_epochs=1, seed=s, metric="auc", patience=1, dropout=0.1)
        params, hist = wj.train(store, split, cfg, exact_batches=True)
        pos = wj.score_array(store, params, c["test_pos"])
        neg = wj.score_array(store, params, c["test_neg"].reshape(-1, 2))
        ours.append((M.roc_auc_device(pos, neg), M.mrr_device(pos, neg, k), float(hist[0]["train_loss"])))
        ref.append((float(r["test_auc"]), float(r["test_mrr"]), float(r["train_loss"])))
    torch.cuda.synchronize()
    ours, ref = np.array(ours), np.array(ref)
    diff = ours.mean(0) - ref.mean(0)
    report = {"seeds": SEEDS, "ours": ours.tolist(), "ref": ref.tolist(), "mean_diff": diff.tolist(),
              "ref_seed_std": ref.std(0, ddof=1).tolist(), "ours_seed_std": ours.std(0, ddof=1).tolist()}
    print(json.dumps(report))
    out = os.environ.get("WJ_TRAIN_DROPOUT_REPORT")
    if out:
        with open(out, "w") as fh:
            json.dump(report, fh, indent=1)
    # mean training loss of the epoch: dropout noise averages out over ~155 batches
    assert abs(diff[2]) < 0.02 * ref[:, 2].mean(), report
    # final test AUC / MRR: the five-seed means within 0.5 points (the north
    # star's criterion); single seeds differ by their dropout realisation
    # alone (same batches and initial parameters), which moves this model's
    # test AUC by up to ~1 point (B200: 0.22 / 0.05 points on the means, at
    # most 1.08 points on one seed; profiles/r02/train_dropout_c1_5seeds.json)
    assert abs(diff[0]) < 0.005 and abs(diff[1]) < 0.005, report
    assert np.max(np.abs(ours[:, :2] - ref[:, :2])) < 0.02, report
