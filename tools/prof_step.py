"""One fwd+bwd step of a bench workload, for ncu captures (no timing here).
    python tools/prof_step.py --workload rglru [--batch B] [--steps N]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="rglru")
ap.add_argument("--batch", type=int, default=0)
ap.add_argument("--steps", type=int, default=2)
a = ap.parse_args()
w = dict(bench.WORKLOADS[a.workload])
B = a.batch or w["B"]
prob = bench.build_problem(w, B, torch.device("cuda", 0))
torch.cuda.synchronize()
for _ in range(a.steps):
    prob["bwd"](prob["fwd"]())
torch.cuda.synchronize()
print("ok", a.workload, B)
