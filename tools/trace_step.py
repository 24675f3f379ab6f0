"""Trace one bench step with torch.profiler (CUPTI: every kernel, memset, memcpy) and
print GPU activity plus the largest idle gaps on the GPU timeline (dev tool)."""

import json
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench                                                        # noqa: E402
import paper_2203_01877_b200 as T                                   # noqa: E402


def main():
    orders, li = bench.make_data(0, 1, torch.device("cuda", 0), "shuffled")
    hp = bench.HotPath(T, orders, li, 1)
    for _ in range(3):
        hp.step()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        hp.step()
        torch.cuda.synchronize()
    print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=30))
    path = "gpurun_out/trace_step.json"
    prof.export_chrome_trace(path)
    ev = json.load(open(path))["traceEvents"]
    gpu = sorted([e for e in ev if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memset", "gpu_memcpy")],
                 key=lambda e: e["ts"])
    gaps = []
    for a, b in zip(gpu, gpu[1:]):
        g = b["ts"] - (a["ts"] + a["dur"])
        if g > 50:
            gaps.append((g, a["name"][:60], b["name"][:60]))
    gaps.sort(reverse=True)
    tot = sum(g for g, *_ in gaps)
    print(f"GPU span {gpu[-1]['ts'] + gpu[-1]['dur'] - gpu[0]['ts']:.0f} us, busy "
          f"{sum(e['dur'] for e in gpu):.0f} us, gaps>50us total {tot:.0f} us")
    for g in gaps[:25]:
        print(f"gap {g[0]:9.1f} us after {g[1]} before {g[2]}")
    cpu = [e for e in ev if e.get("ph") == "X" and e.get("cat") == "cuda_runtime"]
    agg = {}
    for e in cpu:
        agg.setdefault(e["name"], [0, 0])
        agg[e["name"]][0] += e["dur"]
        agg[e["name"]][1] += 1
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:15]:
        print(f"runtime {k:40s} {v[0]:10.1f} us  x{v[1]}")


if __name__ == "__main__":
    main()
