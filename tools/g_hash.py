"""Config-3 multiplier G (8192 x 8192, attempt-0 right multiplier stream of randomized_genp:
(seed, 11 ^ 0x5000000000000000), genp.cpp:243-246) on the GPU vs the C restatement, byte for byte;
prints both SHA-256 digests and the mismatch count."""
import hashlib
import json
import sys

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1212_4560_b200 as rl  # noqa: E402
from oracle.pyoracle import Restated  # noqa: E402

n = 8192
sid = 11 ^ 0x5000000000000000
g = rl.gaussian_matrix(n, n, 0.0, 1.0, rl.RngStream(bench.SEED, sid))
o = Restated().gaussian_matrix(n, n, bench.SEED, sid)
print(json.dumps({"n": n, "stream": [bench.SEED, sid], "gpu_sha256": hashlib.sha256(g.tobytes()).hexdigest(),
                  "oracle_sha256": hashlib.sha256(o.tobytes()).hexdigest(),
                  "mismatches": int(np.sum(g.view(np.uint64) != o.view(np.uint64)))}))
