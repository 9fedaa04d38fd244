"""The C++ drop-in layer (include/loopdyn_b200) compiles against the C-ABI and
behaves like the reference API (CPU part here; the stepping part on the GPU)."""
import os
import subprocess

import pytest

import oracle_lib

ROOT = oracle_lib.ROOT
JSON_INC = "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann"
BIN = os.path.join(ROOT, "tests", "cpp", "test_cpp_api")


def build():
    lib_dir = os.path.join(ROOT, "paper_2603_16536_b200")
    subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"), "-I", JSON_INC,
                    os.path.join(ROOT, "tests", "cpp", "test_cpp_api.cpp"), "-o", BIN, "-L", lib_dir,
                    "-lkamino_b200", f"-Wl,-rpath,{lib_dir}"], check=True)


SHIM = os.path.join(ROOT, "tests", "cpp", "batch_b200_shim")


def build_shim():
    """INTEGRATION.md §3's reference-side shim, against the test stub of the
    reference declarations it uses (tests/cpp/ref_stub)."""
    lib_dir = os.path.join(ROOT, "paper_2603_16536_b200")
    subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"), "-I",
                    os.path.join(ROOT, "tests", "cpp", "ref_stub"), os.path.join(ROOT, "tests", "cpp",
                    "batch_b200_shim.cpp"), "-o", SHIM, "-L", lib_dir, "-lkamino_b200",
                    f"-Wl,-rpath,{lib_dir}"], check=True)


def test_integration_shim_compiles_and_links():
    build_shim()
    r = subprocess.run([SHIM], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_integration_shim_steps_on_device():
    build_shim()
    r = subprocess.run([SHIM, "--gpu"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr


def test_cpp_api_cpu():
    build()
    r = subprocess.run([BIN, oracle_lib.BUNDLE], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_cpp_api_gpu():
    build()
    r = subprocess.run([BIN, oracle_lib.BUNDLE, "--gpu"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
