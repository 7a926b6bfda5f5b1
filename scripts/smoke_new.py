"""Quick GPU check of one algorithm on small shapes vs the oracle (run under `timeout`)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle  # noqa: E402
import paper_2410_08300_b200 as ai3  # noqa: E402

algo = sys.argv[1]
shapes = [(2, 64, 23, 23, 96, 3, 1, 1, 1), (2, 3, 33, 31, 16, 3, 1, 1, 1), (2, 32, 19, 19, 32, 3, 1, 2, 2),
          (2, 128, 28, 28, 128, 3, 2, 1, 1), (1, 16, 9, 7, 24, 3, 1, 0, 1), (4, 256, 14, 14, 512, 1, 1, 0, 1)]
for dt in (torch.bfloat16, torch.float32):
    for (N, C, H, W, K, R, st, pd, dl) in shapes:
        rng = np.random.default_rng(0)
        x = torch.from_numpy(rng.standard_normal((N, C, H, W)).astype(np.float32)).cuda().to(dt)
        x = x.contiguous(memory_format=torch.channels_last)
        w = torch.from_numpy(rng.uniform(-.2, .2, (K, C, R, R)).astype(np.float32)).cuda().to(dt)
        b = torch.from_numpy(rng.uniform(-.2, .2, K).astype(np.float32)).cuda().to(dt)
        t0 = time.time()
        p = ai3.ConvPlan(w, b, x.shape, st, pd, dl, 1, algo, in_layout=1)
        y = p(x)
        torch.cuda.synchronize()
        ref = oracle.conv2d(x.float().cpu().numpy(), w.float().cpu().numpy(), b.float().cpu().numpy(), st, pd, dl)
        err = oracle.rel_err(y.float().cpu().numpy(), ref)
        print(f"{algo} {dt} {(N, C, H, W, K, R, st, pd, dl)} err={err:.2e} {time.time() - t0:.2f}s", flush=True)
