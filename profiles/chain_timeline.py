"""Critical-path breakdown of the C3 training step under the step executor
(measurement aid): a CUPTI kernel trace (torch.profiler) of ~30 chained
steps.  With programmatic dependent launch the kernels overlap, so each
kernel's START says little; the END of each kernel is the critical path:
  encode -> tail:  tail end - join+encode end
  tail -> adam:    adam end - tail end
  adam -> encode:  next join+encode end - adam end (the encode kernel's share)

    python profiles/chain_timeline.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
import paper_2202_13538_b200 as wj  # noqa: E402
from paper_2202_13538_b200 import _lib  # noqa: E402
from paper_2202_13538_b200.pipeline import GROUP_MAX  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    wl = bench.build_workload(bench.CONFIGS["c3"], dev)
    store = wl.prep(wl.walk_graph)
    plan = bench.make_plan(wl, 40, bench.BATCH_SEED)
    p = wj.init_params(2, 4, dropout=0.1, seed=11, device=dev)
    st = wj.AdamState.for_params(p)
    step = wj.TrainStep(store, p, st, seed=3, launch="chain", overlap_inputs=True)
    batches = []
    for q, y in plan:
        gb = np.empty((2 + q.shape[1]) * q.shape[0] + 2, dtype=np.int32)
        _lib.call("wj_group_queries", q.ctypes.data, q.shape[0], q.shape[1], GROUP_MAX, gb.ctypes.data, None)
        batches.append((torch.from_numpy(q).to(dev), torch.from_numpy(y).to(dev),
                        (torch.from_numpy(gb).to(dev), int(gb[0]))))
    for q, y, g in batches[:10]:
        step(q, y, groups=g)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for q, y, g in batches[10:]:
            step(q, y, groups=g)
        torch.cuda.synchronize()
    ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    ks = sorted(((e.time_range.start, e.time_range.end, e.name) for e in ev), key=lambda t: t[1])
    kind = lambda n: "enc" if "join_encode" in n else ("tail" if "tail" in n else ("adam" if "adam" in n else None))
    seq = [(kind(n), s, e) for s, e, n in ks if kind(n)]
    rows = {"enc->tail": [], "tail->adam": [], "adam->enc": [], "step": []}
    for i in range(1, len(seq) - 3):
        if seq[i][0] == "enc" and seq[i + 1][0] == "tail" and seq[i + 2][0] == "adam" and seq[i + 3][0] == "enc":
            e_enc, e_tail, e_adam, e_next = seq[i][2], seq[i + 1][2], seq[i + 2][2], seq[i + 3][2]
            rows["enc->tail"].append(e_tail - e_enc)
            rows["tail->adam"].append(e_adam - e_tail)
            rows["adam->enc"].append(e_next - e_adam)
            rows["step"].append(e_next - e_enc)
    for k, v in rows.items():
        if v:
            print(f"{k:11s} median {np.median(v):7.2f} us  p10 {np.percentile(v, 10):7.2f}  p90 {np.percentile(v, 90):7.2f}"
                  f"  (n={len(v)})")
    # kernel spans (first CTA start to last CTA end) for reference
    for k in ("enc", "tail", "adam"):
        d = [e - s for kk, s, e in seq if kk == k]
        print(f"span {k:5s} median {np.median(d):7.2f} us")


if __name__ == "__main__":
    main()
