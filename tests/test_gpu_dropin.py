"""The C++17 drop-in (include/rrgpu/rrgpu.hpp) against the reference's own
run_imm / generate_batch / select_seeds, in one C++ program
(tests/cpp/dropin_parity.cpp; built where the reference headers exist)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "build", "dropin_parity")


@pytest.mark.gpu
def test_cpp_dropin_matches_reference(cuda):
    if not os.path.exists(BIN):
        pytest.skip("tests/cpp/build/dropin_parity not built (reference headers absent)")
    out = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(out.stdout[-4000:])
    assert out.returncode == 0, out.stdout[-4000:] + out.stderr[-2000:]
    assert "ALL PASS" in out.stdout


def test_adapter_header_compiles_cpp17(tmp_path):
    """The adapter is C++17-clean (the reference headers are not)."""
    src = tmp_path / "t.cpp"
    src.write_text('#include "rrgpu/rrgpu.hpp"\nint main(){ rrgpu::ImmConfig c; return c.k == 50 ? 0 : 1; }\n')
    r = subprocess.run(["g++", "-std=c++17", "-Wall", "-Wextra", "-Werror", "-fsyntax-only",
                        f"-I{ROOT}/include", str(src)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
