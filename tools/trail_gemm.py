"""The LU's trailing-update GEMM shapes alone (dev aid): C (rest x rest) -= L21 (rest x K) U12
(K x rest) at K = 512 / 128 on strided views of an n x n matrix, CUDA-event timed."""
import sys
sys.path.insert(0, ".")
import torch  # noqa: E402
import paper_1212_4560_b200 as rl  # noqa: E402
import ctypes as C  # noqa: E402
n = 8192
M = torch.randn(n, n, dtype=torch.float64, device="cuda")
lib = rl.lib()
rl._bind_stream()  # launches on torch's current stream (the events below)
for rest, K in ((7168, 512), (5120, 512), (3072, 512), (2048, 512), (7168, 128), (7168, 1024)):
    o = n - rest - K
    a = M[o + K:, o:o + K]
    b = M[o:o + K, o + K:]
    c = M[o + K:, o + K:]
    f = lambda: lib.rl_dev_gemm(0, 0, rest, rest, K, -1.0, a.data_ptr(), n, b.data_ptr(), n, 1.0, c.data_ptr(), n)  # noqa
    for _ in range(2):
        f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(5):
        f()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"rest {rest} K {K}: {ms:.3f} ms {2 * rest * rest * K / ms / 1e9:.1f} TFLOP/s", flush=True)
