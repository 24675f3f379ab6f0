import json, sys
d = json.load(open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/q_bench.json"))
print(f"ms/step {d['ms_per_step']:.3f}  value {d['value']/1e9:.3f} G rows/s  e2e {d['e2e']['value']/1e9:.3f}  launches {d['gpu_launches']}  clocks {d['clocks']}")
print("ops", {k: round(v, 3) for k, v in d["operators_ms"].items()})
r = d["roofline"]; print(f"roofline {r['kernel']} {r['achieved']:.0f} GB/s frac {r['frac']:.3f} share {r['share_of_step']:.2f}")
tot = 0
for k, v in d["kernels"].items():
    tot += v["ms_per_step"]
    print(f"  {k:28s} {v['ms_per_step']:8.3f} ms x{v['launches_per_step']:4.1f} {v['algorithmic_GBps'] or 0:8.0f} GB/s")
print("kernel sum", round(tot, 3))
if "cpu_baseline" in d: print("cpu", d["cpu_baseline"])
