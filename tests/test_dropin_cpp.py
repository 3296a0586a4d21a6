"""The C++ drop-in (include/streamrl/{engine,rl_math,policy,trajectory,rng}.hpp)
compiled as a reference caller would compile it, linked against
libsrl_b200.so, and run over the reference's engine-level and rlmath tests
restated in-process (tests/cpp/dropin_test.cpp; expected values from the
unmodified reference, tests/golden/reference_vectors.json)."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
LIBDIR = ROOT / "paper_2509_19128_b200"
# nlohmann/json 3.11.3 (the reference's JSON library) as vendored in this image's venv;
# only the test program parses the golden file with it
NLOHMANN = Path("/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann")


def build(tmp_path):
    from paper_2509_19128_b200 import _lib

    _lib.lib()  # the library is built
    if not (NLOHMANN / "json.hpp").exists():
        pytest.skip("nlohmann/json.hpp not present in this image")
    exe = tmp_path / "dropin_test"
    r = subprocess.run(["g++", "-std=c++20", "-O1", "-Wall", "-Werror", "-I", str(ROOT / "include"),
                        "-I", str(NLOHMANN), str(ROOT / "tests" / "cpp" / "dropin_test.cpp"),
                        "-L", str(LIBDIR), "-lsrl_b200", f"-Wl,-rpath,{LIBDIR}", "-o", str(exe)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def run(exe):
    return subprocess.run([str(exe), str(ROOT / "tests" / "golden" / "reference_vectors.json")],
                          capture_output=True, text=True, timeout=600)


def test_dropin_headers_compile_and_fail_loudly_without_gpu(tmp_path):
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present: the gpu variant runs the full program")
    r = run(build(tmp_path))
    assert "[ok] crc_and_groups" in r.stdout  # host-only entry points
    assert "[ok] policy_documents" in r.stdout  # document functions + host-side validate()
    assert "[FAIL] demo_scenario" in r.stdout and "no_device" in r.stderr
    assert r.returncode == 1


@pytest.mark.gpu
def test_dropin_reference_tests_pass_on_device(cuda, tmp_path):
    r = run(build(tmp_path))
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout
