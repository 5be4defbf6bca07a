"""Full-size parity run, config 5 Householder-pair arm (n = 16384, MulSide::Right): the GPU
path vs the C restatement (row-threaded, bit-identical to its sequential form) on the SAME input
bytes, first right-hand side (the reference API is single-RHS).  The restatement follows
randomized_genp (genp.cpp:207-291) with the NEW orthogonal Householder-pair multiplier (no
reference implementation exists: DESIGN.md §3).  Writes JSON to argv[1]."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1212_4560_b200 as rl  # noqa: E402
from oracle.pyoracle import Restated  # noqa: E402

out_path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/fullsize_c5.json"
dev = torch.device("cuda", 0)
A, B = bench.make_config5_inputs(torch, dev)
n = A.shape[0]
X = torch.empty_like(B)
kind = rl.MultiplierKind(rl.MultiplierTag.HOUSEHOLDER_PAIR)
rep = rl.dev_randomized_genp(A, B, X, kind, rl.MulSide.RIGHT, 0, rl.RngStream(bench.SEED, 55), skip_raw_arm=True)
torch.cuda.synchronize()
Ah = A.cpu().numpy()
b = np.ascontiguousarray(B[:, 0].cpu().numpy())
xg = X[:, 0].cpu().numpy()
del A, B, X
torch.cuda.empty_cache()
O = Restated(threads=os.cpu_count() or 8)
t = time.time()
y, r, e = O.randomized_genp(Ah, b, "householder_pair", "right", 0, seed=bench.SEED, sid=55)
dt = time.time() - t
normA = np.linalg.norm(Ah)
bw = lambda v: float(np.linalg.norm(Ah @ v - b) / (normA * np.linalg.norm(v)))  # noqa: E731
rr = lambda v: float(np.linalg.norm(Ah @ v - b) / np.linalg.norm(b))  # noqa: E731
res = {"n": n, "arm": "householder_pair", "gpu": {"attempt": rep.attempt, "residual_max_over_8_rhs": rep.residual,
                                                   "residual_rhs0": rr(xg), "bwd_rhs0": bw(xg)},
       "oracle": {"attempt": int(e[0]), "residual": float(r[0]), "raw_residual": float(r[1]), "bwd": bw(y),
                  "seconds": dt, "threads": os.cpu_count()},
       "rel_dx": float(np.abs(xg - y).max() / np.abs(y).max())}
with open(out_path, "w") as fh:
    json.dump(res, fh, indent=1)
print(json.dumps(res))
