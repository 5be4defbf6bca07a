"""Full-size parity run (config 3, n = 8192): the GPU path vs the restated reference
(oracle/rl_oracle.c, row-threaded — bit-identical to the sequential reference) on the SAME
input bytes (built once on the GPU, copied to the host), first right-hand side only (the
reference API is single-RHS; 16 columns would be 16 independent calls).  Reports the
accepted attempt, residuals and backward errors on both sides.  Writes JSON to argv[1]."""
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

out_path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/fullsize_c3.json"
cols = int(sys.argv[2]) if len(sys.argv) > 2 else 1
dev = torch.device("cuda", 0)
A, B = bench.make_config3_inputs(torch, dev)
n = A.shape[0]
X = torch.empty_like(B)
os.environ["RL_DEBUG"] = "1"
rep = rl.dev_randomized_genp(A, B, X, rl.MultiplierKind(), rl.MulSide.RIGHT, 0, rl.RngStream(bench.SEED, 11),
                             skip_raw_arm=True)
torch.cuda.synchronize()
Ah = A.cpu().numpy()
Bh = B.cpu().numpy()
Xh = X.cpu().numpy()
res = {"n": n, "gpu": {"attempt": rep.attempt, "residual_max": rep.residual}, "columns": []}
O = Restated(threads=os.cpu_count() or 8)
normA = np.linalg.norm(Ah)
for j in range(cols):
    b = np.ascontiguousarray(Bh[:, j])
    t = time.time()
    y, r, e = O.randomized_genp(Ah, b, "gaussian", "right", 0, seed=bench.SEED, sid=11)
    dt = time.time() - t
    xg = Xh[:, j]
    bw = lambda v: float(np.linalg.norm(Ah @ v - b) / (normA * np.linalg.norm(v)))
    rr = lambda v: float(np.linalg.norm(Ah @ v - b) / np.linalg.norm(b))
    col = {"j": j, "oracle_attempt": int(e[0]), "oracle_residual": float(r[0]), "oracle_bwd": bw(y),
           "gpu_residual": rr(xg), "gpu_bwd": bw(xg), "oracle_seconds": dt, "oracle_threads": os.cpu_count(),
           "rel_dx": float(np.abs(xg - y).max() / np.abs(y).max())}
    res["columns"].append(col)
    print(json.dumps(col), flush=True)
with open(out_path, "w") as fh:
    json.dump(res, fh, indent=1)
print(json.dumps(res))
