"""RG-LRU plan grid at per-rank batch shares: fwd and bwd timed separately
(graph-replayed) for every (PF, STAGES, SEGS) override, in one process (the
plan reads its LRX_RGLRU_* overrides at every launch).
python tools/rg_plan_grid.py 32 16 8"""
import itertools, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from rg_smallb_util import tm  # noqa: E402

w = dict(bench.WORKLOADS["rglru"])
for B in [int(x) for x in sys.argv[1:]] or [32, 16, 8]:
    prob = bench.build_problem(w, B, torch.device("cuda", 0))
    segs = (1, 2, 3, 4) if B <= 8 else (1, 2) if B <= 16 else (1,)
    res = []
    for pf, st, sg in itertools.product((2, 4, 8, 16), (2, 3, 4, 6), segs):
        os.environ.update(LRX_RGLRU_PF=str(pf), LRX_RGLRU_STAGES=str(st), LRX_RGLRU_SEGS=str(sg))
        try:
            ctx = prob["fwd"]()
            f = tm(prob["fwd"])
            b = tm(lambda: prob["bwd"](ctx))
        except Exception as e:  # plan does not fit
            print(f"B={B} pf{pf} st{st} seg{sg}: {type(e).__name__}", flush=True)
            continue
        res.append((f, b, pf, st, sg))
        print(f"B={B} pf{pf:2d} st{st} seg{sg}: fwd {f:.3f} bwd {b:.3f}", flush=True)
    for k in ("LRX_RGLRU_PF", "LRX_RGLRU_STAGES", "LRX_RGLRU_SEGS"):
        os.environ.pop(k, None)
    ctx = prob["fwd"]()
    f0, b0 = tm(prob["fwd"]), tm(lambda: prob["bwd"](ctx))
    bf, bb = min(res), min(res, key=lambda r: r[1])
    print(f"== B={B} default fwd {f0:.3f} bwd {b0:.3f} | best fwd {bf[0]:.3f} (pf{bf[2]} st{bf[3]} seg{bf[4]}) "
          f"best bwd {bb[1]:.3f} (pf{bb[2]} st{bb[3]} seg{bb[4]}) | ideal total {20.26 * B / 64:.3f}", flush=True)
    del prob, ctx
    torch.cuda.empty_cache()
