"""Config-1 spreads with bit-exact multipliers: GPU vs reference golden / C restatement for x,
backward error, and the L/U factors of the preconditioned system A*G (same G bytes)."""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1212_4560_b200 as rl  # noqa: E402
from oracle.pyoracle import Restated  # noqa: E402

O = Restated()
gz = np.load("tests/golden/golden.npz")
A, b = gz["c1/A"], gz["c1/b"]
rel = lambda a, c: float(np.abs(a - c).max() / np.abs(c).max())
bwd = lambda x: float(np.linalg.norm(A @ x - b) / (np.linalg.norm(A) * np.linalg.norm(x)))
out = {}
for kind, refine in [("gaussian", 0), ("gaussian", 1), ("circulant_sign", 0), ("circulant_sign", 1), ("uniform_pm1", 0)]:
    tag = getattr(rl.MultiplierTag, kind.upper())
    x, rep = rl.randomized_genp(A, b, rl.MultiplierKind(tag), rl.MulSide.RIGHT, refine, rl.RngStream(20260825, 11))
    y = gz[f"c1/{kind}/r{refine}/y"]
    out[f"{kind}/r{refine}"] = {"rel_x": rel(x, y), "bwd_ratio": bwd(x) / bwd(y), "attempt": rep.attempt}
sid = 11 ^ 0x5000000000000000
G = rl.gaussian_matrix(256, 256, 0.0, 1.0, rl.RngStream(20260825, sid))
Go = O.gaussian_matrix(256, 256, 20260825, sid)
S = rl.multiply(A, G)
So = O.matmul(A, Go)
f = rl.genp_factor(S)
L, U, piv, w = O.genp_factor(So)
out["G_equal"] = bool(np.array_equal(G, Go))
out["rel_AG"] = rel(S, So)
out["rel_L"] = rel(f.L, L)
out["rel_U"] = rel(f.U, U)
fs = rl.genp_factor(So)  # same system bytes: factor-only spread
out["rel_L_same_system"] = rel(fs.L, L)
out["rel_U_same_system"] = rel(fs.U, U)
print(json.dumps(out, indent=1))
