"""Per-layer kernel time over the seeds {42, 123, 2026} (SURVEY §8d "GPU timing method"):
for each single-layer config, HBM-cold (a CUDA graph cycling R weight replicas, R x layer
bytes >= 4 x L2) and L2-warm (the same graph over one replica) launch times; median over
>= 30 graph replays per seed, and the coefficient of variation (sample std / mean) of the
three seeds' medians.

    python tools/seed_cv.py [--replays 30] [--configs c2,c3a,c3b] > profiles/.../seed_cv.txt
"""
from __future__ import annotations

import argparse
import os
import statistics
import sys
import types

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--replays", type=int, default=30)
    ap.add_argument("--configs", default="c2,c3a,c3b")
    ap.add_argument("--seeds", default="42,123,2026")
    a = ap.parse_args()

    import torch
    import bench
    import ww_inputs as wi

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    s = torch.cuda.Stream(dev)
    specs = {"c2": wi.C2, "c3a": wi.C3A, "c3b": wi.C3B}
    print(torch.cuda.get_device_name(dev))
    print(f"{'config':26s} {'seed':>5s} {'R':>3s} {'HBM-cold us':>12s} {'L2-warm us':>11s}")
    for c in a.configs.split(","):
        spec = specs[c]
        cold_meds, warm_meds = [], []
        for seed in (int(x) for x in a.seeds.split(",")):
            args = types.SimpleNamespace(batch=1, seed=seed, no_pdl=False)
            lay = bench._ReplicaLayer(spec, args, 0, 1, dev, None)
            yv = lay.Y[0].view(1, -1)[:, :lay.nloc]

            def graph_of(replicas):
                with torch.cuda.stream(s):
                    for r in replicas:
                        lay.ww.wl_gemv_batched(lay.L, lay.Wr[r], lay.S, lay.X, yv, stream=s)
                torch.cuda.synchronize(dev)
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=s):
                    for r in replicas:
                        lay.ww.wl_gemv_batched(lay.L, lay.Wr[r], lay.S, lay.X, yv, stream=s)
                return g

            res = []
            for replicas in (list(range(lay.R)), [0] * lay.R):
                g = graph_of(replicas)
                times = []
                with torch.cuda.stream(s):
                    for _ in range(3):
                        g.replay()
                    for _ in range(a.replays):
                        e0 = torch.cuda.Event(enable_timing=True)
                        e1 = torch.cuda.Event(enable_timing=True)
                        e0.record(s)
                        g.replay()
                        e1.record(s)
                        e1.synchronize()
                        times.append(e0.elapsed_time(e1) * 1e3 / len(replicas))
                res.append(statistics.median(times))
            cold_meds.append(res[0])
            warm_meds.append(res[1])
            print(f"{spec.name:26s} {seed:5d} {lay.R:3d} {res[0]:12.3f} {res[1]:11.3f}")
            del lay
            torch.cuda.empty_cache()
        for label, v in (("HBM-cold", cold_meds), ("L2-warm", warm_meds)):
            cv = statistics.stdev(v) / statistics.mean(v)
            print(f"  {spec.name} {label}: mean of seed medians {statistics.mean(v):.3f} us, "
                  f"CV {100 * cv:.2f} %")


if __name__ == "__main__":
    main()
