import sys, torch, json
sys.path.insert(0, "/root/repo")
import paper_2203_01877_b200 as T
from datagen import zipf_keys, uniform_keys
l = zipf_keys(100_000_000, 100_000_000, seed=42, device="cuda")
r = zipf_keys(100_000_000, 100_000_000, seed=43, device="cuda")
u = uniform_keys(100_000_000, 100_000_000, seed=43, device="cuda")
ctx = T.context()
for name, (a, b) in {"both_zipf": (l, r), "zipf_uniform": (l, u)}.items():
    p = ctx.smj_prepare(a, b); p.release()
    torch.cuda.synchronize()
    ctx.reset_counters(); ctx.set_profiling(True)
    p = ctx.smj_prepare(a, b)
    if name == "zipf_uniform":
        x = p.expand(0, p.size)
    p.release()
    st = ctx.kernel_stats(); ctx.set_profiling(False)
    print(name, json.dumps({k: round(v[0], 3) for k, v in sorted(st.items(), key=lambda kv: -kv[1][0])}))
