"""Child process of test_pkfk_multipass_probe: TQP_PROBE_SLICE_MB (read once per process)
is set tiny so the multi-pass probe runs at sizes the oracle checks element by element."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle                                  # noqa: E402
import paper_2203_01877_b200 as T              # noqa: E402

CASES = [  # nb, np, span, build dtype, probe dtype, offset
    (5000, 100_001, 20_000, torch.int64, torch.int64, 0),
    (5000, 100_001, 20_000, torch.int32, torch.int32, -7000),
    (300_000, 1_000_003, 1_000_000, torch.int64, torch.int64, 5),
    (2047, 2049, 4096, torch.int64, torch.int64, 1 << 40),
    (1, 10_000, 3, torch.int64, torch.int64, 0),
    (60_000, 250_000, 1 << 29, torch.int64, torch.int64, 0),   # sparse: 1 key per 8,900
]

for nb, n_p, span, bd, pd, off in CASES:
    rng = np.random.default_rng(nb + n_p)
    build = (rng.choice(span, nb, replace=False) + off).astype(np.int64)
    probe = np.concatenate([rng.choice(build, n_p // 2), rng.integers(off - 5, off + span + 5, n_p - n_p // 2)])
    probe = rng.permutation(probe).astype(np.int64)
    lo, ro = T.pkfk_join(torch.as_tensor(build).to(bd).cuda(), torch.as_tensor(probe).to(pd).cuda())
    olo, oro = oracle.pkfk_join(build, probe)
    if not (np.array_equal(lo.cpu().numpy(), olo) and np.array_equal(ro.cpu().numpy(), oro)):
        print("MISMATCH", nb, n_p, span, bd, pd, off, flush=True)
        sys.exit(1)
print("ok", len(CASES))
