import os, sys, cProfile, pstats
root = sys.argv[1]
sys.path.insert(0, root)
import torch
import bench
w = dict(bench.WORKLOADS["lru"])
prob = bench.build_problem(w, w["B"], torch.device("cuda", 0))
for _ in range(5):
    ctx = prob["fwd"](); prob["bwd"](ctx)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(50):
    ctx = prob["fwd"](); prob["bwd"](ctx)
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr); st.sort_stats("tottime").print_stats(14)
