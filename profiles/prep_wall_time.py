import sys, time, torch
sys.path.insert(0, "/root/repo")
import bench
import paper_2202_13538_b200 as wj
from paper_2202_13538_b200.graph import DeviceGraph
dev = torch.device("cuda", 0)
wl = bench.build_workload(bench.CONFIGS["c3"], dev)
g = wl.walk_graph
host = g.to_host()
for r in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    s = wl.prep(g); torch.cuda.synchronize(); a = time.perf_counter() - t
    del s
    torch.cuda.synchronize(); t = time.perf_counter()
    dg = DeviceGraph.from_graph(host, dev); torch.cuda.synchronize(); b = time.perf_counter() - t
    t = time.perf_counter()
    s = wl.prep(host); torch.cuda.synchronize(); c = time.perf_counter() - t
    del s, dg
    print(f"prep(device g) wall {a*1e3:.1f} ms  upload {b*1e3:.1f} ms  prep(host g) wall {c*1e3:.1f} ms", flush=True)
import cProfile, pstats
pr = cProfile.Profile(); pr.enable(); s = wl.prep(host); torch.cuda.synchronize(); pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
