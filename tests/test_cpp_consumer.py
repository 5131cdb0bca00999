"""A compiled C++ consumer of include/cad.h (tests/cpp/layer_consumer.cpp):
built with g++ against the header and libcad.so only, as a cadsim maintainer
would. CPU: the golden config-1 plan through cad_schedule;
GPU: one CA layer through the per-layer executor (cad_layer_ctx_create /
export / connect / begin / dispatch / compute / return / finish) against the
whole-batch kernels."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")


@pytest.fixture(scope="module")
def binary(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("cpp") / "layer_consumer")
    libdir = os.path.join(ROOT, "paper_2510_18121_b200", "lib")
    cmd = ["g++", "-std=c++17", "-O2", "-Wall", "-I", os.path.join(ROOT, "include"), "-I",
           os.path.join(CUDA, "include"), os.path.join(ROOT, "tests", "cpp", "layer_consumer.cpp"), "-o", out,
           "-L", libdir, "-lcad", f"-Wl,-rpath,{libdir}", "-L", os.path.join(CUDA, "lib64"), "-lcudart",
           f"-Wl,-rpath,{os.path.join(CUDA, 'lib64')}"]
    subprocess.run(cmd, check=True)
    return out


def test_cpp_consumer_schedules_golden_plan(binary):
    r = subprocess.run([binary, "cpu"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "golden plan ok" in r.stdout


@pytest.mark.gpu
def test_cpp_consumer_runs_a_layer(binary):
    r = subprocess.run([binary, "gpu"], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "layer ok" in r.stdout
