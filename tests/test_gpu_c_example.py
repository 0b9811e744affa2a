"""The C ABI from plain C: examples/dgt_c_example.c (plan, execute_host, window_dual,
execute_inverse, query, destroy) compiled with gcc against libnsdgt.so and run; it
reconstructs config 1's signal from its coefficients through the GPU dual window."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_c_example_round_trip(tmp_path):
    import paper_1307_4569_b200  # noqa: F401  (builds / loads libnsdgt.so)
    libdir = os.path.join(ROOT, "paper_1307_4569_b200")
    exe = str(tmp_path / "dgt_c_example")
    subprocess.check_call(["gcc", "-O2", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
                           os.path.join(ROOT, "examples", "dgt_c_example.c"), "-L", libdir, "-lnsdgt",
                           f"-Wl,-rpath,{libdir}", "-L/usr/local/cuda/lib64", "-lcudart", "-lm", "-o", exe])
    out = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    err = float(out.stdout.strip().splitlines()[-1].split()[-1])
    assert err < 1e-10, out.stdout
