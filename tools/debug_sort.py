import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2203_01877_b200 as T
from datagen import random_small_keys
for kind, n, lo, hi in [("u64", 4097, -(1<<63), (1<<63)-1), ("u64", 4096, -(1<<63), (1<<63)-1),
                        ("u32", 9000, 0, (1<<26)), ("u32", 300000, 0, (1<<26))]:
    k = random_small_keys(n, lo, hi, n + 7)
    s, p = T.sort(k.cuda())
    torch.cuda.synchronize()
    ref = np.argsort(k.numpy(), kind="stable")
    got = p.cpu().numpy()
    bad = np.nonzero(got != ref)[0]
    print(kind, n, "mismatches", bad.size, "first", bad[:10], "got", got[bad[:5]], "ref", ref[bad[:5]], flush=True)
