"""CPU: csrc/glibc_math.cuh (the GPU's log / sincos for Box-Muller) evaluated on the host against
the installed libm, bit for bit (tests/cpp/test_glibc_math.cpp). The same header is compiled into
the CUDA generator with __dmul_rn/__dadd_rn/__fma_rn, so a host match pins the operation
sequence; tests/test_gpu_rng.py then checks the GPU's bits against the host libm directly."""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(ROOT, "paper_1212_4560_b200", "csrc")


def test_glibc_math_host_matches_libm(tmp_path):
    exe = os.path.join(ROOT, "paper_1212_4560_b200", "lib", "test_glibc_math")
    if not os.path.exists(exe):
        exe = str(tmp_path / "test_glibc_math")
        subprocess.run(["g++", "-std=c++17", "-O2", "-mfma", "-ffp-contract=off", "-pthread", "-I", CSRC,
                        "-o", exe, os.path.join(HERE, "cpp", "test_glibc_math.cpp"), "-lm"], check=True)
    r = subprocess.run([exe, "21"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count(" 0 mismatches") == 8, r.stdout
