"""The C ABI driven from C: examples/decode_step.c (no Python in the loop) runs a hybrid
decode step through include/hylra.h and checks it against its own float64 evaluation."""
import shutil
import subprocess
from pathlib import Path

import pytest

from conftest import cuda_ok

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")]

ROOT = Path(__file__).resolve().parent.parent


def test_c_host_decode_step(tmp_path):
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    lib_dir = ROOT / "paper_2602_00777_b200"
    exe = tmp_path / "decode_step"
    subprocess.run(["gcc", "-O2", "-std=c11", str(ROOT / "examples" / "decode_step.c"),
                    f"-I{ROOT / 'include'}", "-I/usr/local/cuda/include", f"-L{lib_dir}",
                    "-lhylra", "-L/usr/local/cuda/lib64", "-lcudart", "-lm",
                    f"-Wl,-rpath,{lib_dir}", "-o", str(exe)], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "set mismatches 0" in r.stdout
    assert "single-launch step: 1 launch, bit-identical 1" in r.stdout
