import sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_1212_4560_b200 as rl
from oracle.pyoracle import Restated
O = Restated()
n, seed = 256, 20260825
A = O.gaussian_matrix(n, n, seed, 1)
A[:128, :128] = O.matmul(O.gaussian_matrix(128, 127, seed, 2), O.gaussian_matrix(127, 128, seed, 3))
b = O.matvec(A, O.gaussian_matrix(n, 1, seed, 4).ravel())
kind = rl.MultiplierKind()
for _ in range(5):
    rl.randomized_genp(A, b, kind, rl.MulSide.RIGHT, 0, rl.RngStream(seed, 11))
ts = []
for _ in range(50):
    t0 = time.perf_counter()
    x, rep = rl.randomized_genp(A, b, kind, rl.MulSide.RIGHT, 0, rl.RngStream(seed, 11))
    ts.append(time.perf_counter() - t0)
ts = np.array(ts) * 1e6
print(f"median {np.median(ts):.1f} us  min {ts.min():.1f}  p90 {np.percentile(ts, 90):.1f}  raw {rep.raw_residual:.3e}")
