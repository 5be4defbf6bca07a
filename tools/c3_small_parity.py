"""Config-3-shaped parity at n where the CPU oracle finishes: backward error of the GPU
path vs the restated reference on identical inputs."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1212_4560_b200 as rl  # noqa: E402
from oracle.pyoracle import Restated  # noqa: E402

O = Restated()
for n in [int(a) for a in sys.argv[1:]] or [1024]:
    h = n // 2
    rng = np.random.default_rng(n)
    q1, _ = np.linalg.qr(rng.standard_normal((n, n)))
    q2, _ = np.linalg.qr(rng.standard_normal((n, n)))
    A = (q1 * np.logspace(0, -6, n)) @ q2.T
    A[:h, :h] = rng.standard_normal((h, h - 1)) @ rng.standard_normal((h - 1, h))
    xt = rng.standard_normal(n)
    b = A @ xt
    t = time.time()
    xo, ro, eo = O.randomized_genp(A, b, "gaussian", "right", 0, seed=7, sid=11)
    to = time.time() - t
    x, rep = rl.randomized_genp(A, b, rl.MultiplierKind(), rl.MulSide.RIGHT, 0, rl.RngStream(7, 11))
    bw = lambda v: np.linalg.norm(A @ v - b) / (np.linalg.norm(A) * np.linalg.norm(v))
    print(f"n={n}: gpu res {rep.residual:.3e} bwd {bw(x):.3e} att {rep.attempt} raw {rep.raw_residual:.2e} | "
          f"oracle res {ro[0]:.3e} bwd {bw(xo):.3e} att {eo[0]} raw {ro[1]:.2e} ({to:.1f}s) | "
          f"rel dx {np.abs(x - xo).max() / np.abs(xo).max():.2e}", flush=True)
