"""Host ASan + UBSan over libphub's planning code (-m "not gpu").

Builds an instrumented copy of the host core (phub_core.cpp, g++
-fsanitize=address,undefined) linked with the normally compiled kernels
object and runs tests/host_sanitize/fuzz_host.c against it: chunk tables,
owner tables, layouts and phub_init's host planning for 400 random manifests.
Without a GPU phub_init stops at the device query, after all host planning.
"""
import os
import shutil
import subprocess

import pytest

from conftest import ROOT

CUDA = "/usr/local/cuda"
SRC = os.path.join(ROOT, "paper_1805_07891_b200", "csrc")
INC = os.path.join(ROOT, "include")


@pytest.mark.skipif(not shutil.which("g++") or not os.path.exists(os.path.join(CUDA, "bin", "nvcc")),
                    reason="needs g++ and nvcc")
def test_host_planning_under_asan_ubsan(tmp_path):
    nvcc = os.path.join(CUDA, "bin", "nvcc")
    kobj = tmp_path / "kernels.o"
    subprocess.check_call([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-O1", "-std=c++17",
                           "-Xcompiler", "-fPIC", "-I", INC, "-I", SRC, "-c",
                           os.path.join(SRC, "phub_kernels.cu"), "-o", str(kobj)])
    san = ["-fsanitize=address,undefined", "-fno-sanitize-recover=undefined", "-g", "-O1"]
    cobj = tmp_path / "core.o"
    subprocess.check_call(["g++", *san, "-std=c++17", "-fPIC", "-I", INC, "-I", SRC,
                           "-I", os.path.join(CUDA, "include"), "-c",
                           os.path.join(SRC, "phub_core.cpp"), "-o", str(cobj)])
    exe = tmp_path / "fuzz_host"
    subprocess.check_call(["g++", *san, "-I", INC, "-x", "c",
                           os.path.join(ROOT, "tests", "host_sanitize", "fuzz_host.c"), "-x", "none",
                           str(cobj), str(kobj), "-L", os.path.join(CUDA, "lib64"), "-lcudart",
                           f"-Wl,-rpath,{os.path.join(CUDA, 'lib64')}", "-o", str(exe)])
    env = dict(os.environ, ASAN_OPTIONS="detect_leaks=0:abort_on_error=1",
               UBSAN_OPTIONS="print_stacktrace=1:halt_on_error=1")
    r = subprocess.run([str(exe), "400"], capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "host fuzz ok" in r.stdout
    assert "runtime error" not in r.stderr and "AddressSanitizer" not in r.stderr
