"""Where the SF10 step's non-kernel time goes: step time with libtqp's per-launch
profiling events off and on, and the sum of kernel time, on one B200."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench                                   # noqa: E402
import paper_2203_01877_b200 as T              # noqa: E402


def timed(hp, steps, prof):
    hp.ctx.reset_counters()
    hp.ctx.set_profiling(prof)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        hp.step()
    b.record()
    torch.cuda.synchronize()
    st = hp.ctx.kernel_stats()
    hp.ctx.set_profiling(False)
    hp._ev = []
    return a.elapsed_time(b) / steps, sum(v[0] for v in st.values()) / steps


def main():
    torch.cuda.set_device(0)
    orders, li = bench.make_data(0, 1, torch.device("cuda", 0), "shuffled")
    hp = bench.HotPath(T, orders, li, 1)
    for _ in range(3):
        hp.step()
    out = {}
    for rep in range(2):
        out[f"prof_off_{rep}"] = timed(hp, 10, False)[0]
        on, k = timed(hp, 10, True)
        out[f"prof_on_{rep}"] = on
        out[f"kernel_sum_{rep}"] = k
    print(json.dumps(out))


if __name__ == "__main__":
    main()
