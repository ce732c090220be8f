"""The C++ drop-in headers (include/rgo/*.hpp) compile against the C ABI and
link with librgo_b200.so (CPU); the C++ restatement of the reference's unit
tests passes on the GPU (gpu)."""
import os
import subprocess

import pytest

from conftest import ROOT

BIN = os.path.join(ROOT, "tests", "cpp", "test_rgo")


def build():
    lib_dir = os.path.join(ROOT, "paper_2410_07531_b200")
    subprocess.run(["g++", "-std=c++20", "-O1", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "test_rgo.cpp"), "-o", BIN, "-L", lib_dir, "-lrgo_b200",
                    f"-Wl,-rpath,{lib_dir}"], check=True)


def test_cpp_dropin_builds_and_links():
    build()
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    assert r.returncode in (0, 77), r.stdout + r.stderr


@pytest.mark.gpu
def test_cpp_dropin_reference_tests_on_gpu():
    build()
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
