import sys; sys.path.insert(0, "/root/repo")
import numpy as np, paper_2202_13538_b200 as wj
from oracle import core
rng = np.random.default_rng(3)
for (n, m, M, L) in [(500, 3000, 20, 1), (300, 2000, 7, 2), (400, 2500, 33, 5), (200, 1500, 300, 3)]:
    g = wj.Graph.from_edges(rng.integers(0, n, size=(m, 2)), n)
    s = wj.preprocess(g, M, L, 5)
    r = core.preprocess(g.idxptr, g.indices, M, L, 5)
    ok = np.array_equal(s.table.vectors, r.table) and np.array_equal(s.dict_keys, r.dict_keys) and np.array_equal(s.dict_vals, r.dict_vals)
    print(n, M, L, "store == oracle:", ok)
    assert ok
