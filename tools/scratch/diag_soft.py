"""Diagnostic (GPU): soft-coverage forward of a C2 view vs the oracle, error locations."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import scenes  # noqa: E402
from test_gpu_soft import gpu_soft  # noqa: E402

sc = scenes.make_c2().subset([1])
delta = float(sys.argv[1]) if len(sys.argv) > 1 else 1e-4
rng = [[10, 22]]
got = gpu_soft(sc, delta, sub_range=rng)
ref = oracle.render_fwd(sc, eps_amb=1e-6, sub_range=rng, delta=delta)
err = np.abs(got["rgba"] - ref["rgba"])[..., 3]
err[ref["amb_img"]] = 0
print("status", got["status"], "max err", err.max(), "n>1e-4", int((err > 1e-4).sum()))
idx = np.argwhere(err > 1e-4)
for b, j, i in idx[:20]:
    print((j, i), "gpu %.5f ref %.5f" % (got["rgba"][b, j, i, 3], ref["rgba"][b, j, i, 3]), "tile", (i // 16, j // 16),
          "in-tile", (i % 16, j % 16))
